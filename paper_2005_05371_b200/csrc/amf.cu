// amf.cu -- adaptive median filter (AMF) for sm_100a.
//
// Semantics: detail::adaptive_median_rows, reference proj/src/adaptive_median.cpp:123-215
// (windows k = 3..smax over the pristine input, edge replication, level A/B, unresolved pixels
// keep their input).  Design:
//
//   * amf_k3_kernel (persistent): 95-99.7 % of pixels finalise at k = 3, so k = 3 runs on every
//     pixel.  128 x 32 tiles plus a 1-pixel halo arrive in shared memory by TMA (mbarrier
//     completion, 4-deep ring); warps claim 4-row strips dynamically, so no CTA-wide barrier
//     sits on the steady-state path, and the last warp done with a buffer refills it.  Pixels
//     are processed as u16x2 row PAIRS (each lane holds v * 257 so lane order = pixel order and
//     one PRMT builds a pair word): a lane owns 2 rows x 8 columns, sorts each 3-tall column
//     once (min / max / xor-median) and reuses it for 3 outputs; level A/B become lane masks
//     through a sign-replicating PRMT.  Every pixel's k = 3 result (or its input when level A
//     fails) is stored; level-A failures are appended to a device-wide work queue
//     (warp-aggregated atomic).
//   * amf_grow_* kernels, one launch per window size k = 5..smax: each walks the compacted
//     queue of pixels still open, gathers their k x k windows from global memory (L1/L2
//     resident: the queue is in raster order) and re-queues survivors for k + 2.  k = 5 and 7
//     put two queued pixels in the u16x2 lanes of one thread and run a generated pruned
//     selection network (min / median / max, networks.cuh); k >= 9 (< 2 % of pixels even at
//     config 4) test level A with SWAR counts of zmin / zmax and take the median by a bitwise
//     radix select only when it is needed.
#include <cuda.h>

#include <algorithm>
#include <cstdint>

#include "hyb_internal.cuh"
#include "networks.cuh"
#include "tma.cuh"

namespace hyb {
namespace {

constexpr int TW = 128;          // tile columns
constexpr int TH = 32;           // tile rows
constexpr int NT = 256;          // threads per CTA
constexpr int NW = NT / 32;      // warps per CTA
constexpr int WR = TH / NW;      // rows per warp strip (4)
constexpr int WPIX = WR * TW;    // pixels per strip (512)
constexpr int CP = 16;           // byte-tile column pad: TMA box x offsets must be 16-byte aligned
constexpr int BS = TW + 2 * CP;  // byte-tile row stride = TMA box width (160)
constexpr int BH = TH + 2;       // byte-tile rows (1-pixel halo)
constexpr int BBYTES = (BS * BH + 127) / 128 * 128;  // ring slot (TMA destinations are 128-byte aligned)
constexpr int NBUF = 4;          // TMA ring depth
constexpr int HDR = 128;         // mbarriers, release counters, tile coordinates
constexpr int WAREA = 2 * WPIX;  // per warp: output strip + finalized_at strip
constexpr size_t SMEM = HDR + NBUF * BBYTES + NW * WAREA + 128;

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) { return __byte_perm(a, b, s); }

// a - b and a + b issued as IMAD (FMA pipe): the k = 3 pass is ALU-pipe bound, the FMA pipe idle.
__device__ __forceinline__ uint32_t fsub(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, 0xFFFFFFFF, %2;" : "=r"(r) : "r"(b), "r"(a));
    return r;
}
__device__ __forceinline__ uint32_t fadd(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, 1, %2;" : "=r"(r) : "r"(b), "r"(a));
    return r;
}

// prmt.b32 with the selector's sign-replicate bit honoured (__byte_perm masks it off): turns
// bit 15 / bit 31 into a full 16-bit lane mask.
__device__ __forceinline__ uint32_t lane_mask(uint32_t x) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(r) : "r"(x));
    return r;
}

// Pair word of byte J of two words: u16x2 lanes = a_J * 257, b_J * 257 (the pixel duplicated into
// both bytes of its lane, so 16-bit lane order is pixel order and no zeroing is needed).
template <int J>
__device__ __forceinline__ uint32_t pairw(uint32_t a, uint32_t b) {
    return __byte_perm(a, b, J | (J << 4) | ((4 + J) << 8) | ((4 + J) << 12));
}
__device__ __forceinline__ uint32_t pairw_rt(uint32_t a, uint32_t b, int j) {
    return __byte_perm(a, b, j | (j << 4) | ((4 + j) << 8) | ((4 + j) << 12));
}

// Number of zero bytes of x among the byte lanes flagged (0x80) in v80.
__device__ __forceinline__ int zero_bytes(uint32_t x, uint32_t v80) {
    const uint32_t t = (x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
    return __popc(~(t | x) & v80);
}

// ------------------------------------------------------------------------------------------
// k = 3 tile kernel
// ------------------------------------------------------------------------------------------

struct K3Args {
    uint8_t* dst;
    size_t dpitch, dslice;
    uint8_t* fin;
    size_t fpitch, fslice;
    int rows, cols;          // source buffer (clamping bounds)
    int row_begin, row_end;  // output rows (source coordinates)
    int n_slices;
    int tiles_x, tiles_y;
    int grow;                // queue level-A failures (smax >= 5)
    uint32_t* queue;         // work queue for k = 5
    int* queue_n;
    int col_bits, row_bits;  // queue id = ((z << row_bits | out_row) << col_bits) | col
};

__device__ __forceinline__ void issue_tile_load(const CUtensorMap* tm, uint8_t* Bbuf, uint64_t* bar, int x0, int y0,
                                                int z) {
    mbar_expect_tx(bar, BS * BH);
    tma_load_3d(Bbuf, tm, bar, x0 - CP, y0 - 1, z);
}

__device__ __forceinline__ void tile_coords(const K3Args& a, int t, int* info) {
    const int per_slice = a.tiles_x * a.tiles_y;
    const int z = t / per_slice, rem = t - z * per_slice;
    const int by = rem / a.tiles_x;
    info[0] = (rem - by * a.tiles_x) * TW;
    info[1] = a.row_begin + by * TH;
    info[2] = z;
}

template <bool FIN>
__global__ void __launch_bounds__(NT, 3)
    amf_k3_kernel(const __grid_constant__ CUtensorMap tm_src, const __grid_constant__ K3Args args) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [NBUF]
    int* done_cnt = reinterpret_cast<int*>(smem + 32);     // [NBUF]
    int* next_strip = reinterpret_cast<int*>(smem + 48);   // dynamic strip counter
    int* tinfo = reinterpret_cast<int*>(smem + 64);        // [NBUF][4]
    uint8_t* bufs = smem + HDR;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint8_t* O = bufs + NBUF * BBYTES + warp * WAREA;
    uint8_t* F = O + WPIX;

    const int rows = args.rows, cols = args.cols;
    const int ntiles = args.tiles_x * args.tiles_y * args.n_slices;
    if ((int)blockIdx.x >= ntiles) return;
    const int my_tiles = (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;

    if (tid == 0) {
        prefetch_tmap(&tm_src);
        for (int s = 0; s < NBUF; ++s) {
            mbar_init(&full[s], 1);
            done_cnt[s] = 0;
        }
        *next_strip = 0;
        fence_mbar_init();
        for (int s = 0; s < NBUF && s < my_tiles; ++s) {
            tile_coords(args, blockIdx.x + s * gridDim.x, tinfo + 4 * s);
            issue_tile_load(&tm_src, bufs + s * BBYTES, &full[s], tinfo[4 * s], tinfo[4 * s + 1], tinfo[4 * s + 2]);
        }
    }
    __syncthreads();

    // Strips (4-row slices of this CTA's tiles, in order) are claimed dynamically by warps.
    for (;;) {
        int claim = 0;
        if (lane == 0) claim = atomicAdd(next_strip, 1);
        claim = __shfl_sync(0xFFFFFFFFu, claim, 0);
        const int ti = claim >> 3, sub = claim & 7;
        if (ti >= my_tiles) break;
        const int s = ti & (NBUF - 1);
        mbar_wait(&full[s], (uint32_t)(ti / NBUF) & 1u);
        const int x0 = tinfo[4 * s], y0 = tinfo[4 * s + 1], z = tinfo[4 * s + 2];
        uint8_t* B = bufs + s * BBYTES;

        // ---- border tiles: edge replication (this strip's rows) in place of TMA's zero fill ----
        const int sx0 = x0 - CP, sy0 = y0 - 1;
        if (sx0 < 0 || sx0 + BS > cols || sy0 < 0 || sy0 + BH > rows) {
            const int c_lo = max(0, -sx0), c_hi = min(BS, cols - sx0);
            const int r_lo = max(0, -sy0), r_hi = min(BH, rows - sy0);
            const int wr0 = sub * WR, wr1 = sub * WR + WR + 2;  // byte-tile rows this strip reads
            if (c_lo > 0 || c_hi < BS) {
                for (int rr = max(wr0, r_lo); rr < min(wr1, r_hi); ++rr) {
                    uint8_t* row = B + rr * BS;
                    const uint8_t lv = row[c_lo], rv = row[c_hi - 1];
                    for (int cc = lane; cc < BS; cc += 32) {
                        if (cc < c_lo) row[cc] = lv;
                        else if (cc >= c_hi) row[cc] = rv;
                    }
                }
                __syncwarp();
            }
            for (int rr = wr0; rr < wr1; ++rr) {
                const int src_r = rr < r_lo ? r_lo : (rr >= r_hi ? r_hi - 1 : rr);
                if (src_r == rr) continue;
                for (int q = lane; q < BS / 4; q += 32)
                    reinterpret_cast<uint32_t*>(B + rr * BS)[q] = reinterpret_cast<const uint32_t*>(B + src_r * BS)[q];
            }
            __syncwarp();
        }

        // ---- k = 3: lane = rows (r0, r0+1) x columns c0..c0+7, u16x2 lanes = the two rows ----
        const int lr = 2 * (lane >> 4);  // local row within the strip
        const int r0 = sub * WR + lr, c0 = 8 * (lane & 15);
        uint32_t failbits = 0;
        {
            uint32_t rw[4][4];  // byte rows r0-1 .. r0+2, columns c0-4 .. c0+11
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t* rp = reinterpret_cast<const uint32_t*>(B + (r0 + i) * BS + c0 + CP - 4);
#pragma unroll
                for (int m = 0; m < 4; ++m) rw[i][m] = rp[m];
            }
            uint32_t lo[10], hi[10], mid[10], gm[10];
#pragma unroll
            for (int p = 0; p < 3; ++p) {
                uint32_t w[10];
                w[0] = pairw<3>(rw[p][0], rw[p + 1][0]);
                w[1] = pairw<0>(rw[p][1], rw[p + 1][1]);
                w[2] = pairw<1>(rw[p][1], rw[p + 1][1]);
                w[3] = pairw<2>(rw[p][1], rw[p + 1][1]);
                w[4] = pairw<3>(rw[p][1], rw[p + 1][1]);
                w[5] = pairw<0>(rw[p][2], rw[p + 1][2]);
                w[6] = pairw<1>(rw[p][2], rw[p + 1][2]);
                w[7] = pairw<2>(rw[p][2], rw[p + 1][2]);
                w[8] = pairw<3>(rw[p][2], rw[p + 1][2]);
                w[9] = pairw<0>(rw[p][3], rw[p + 1][3]);
#pragma unroll
                for (int i = 0; i < 10; ++i) {
                    if (p == 0) {
                        lo[i] = hi[i] = mid[i] = w[i];
                    } else if (p == 1) {
                        gm[i] = w[i];
                        lo[i] = __vminu2(lo[i], w[i]);
                        hi[i] = __vmaxu2(hi[i], w[i]);
                        mid[i] ^= w[i];
                    } else {
                        const uint32_t l = __vminu2(lo[i], w[i]), h = __vmaxu2(hi[i], w[i]);
                        mid[i] = mid[i] ^ w[i] ^ l ^ h;  // median of 3 = a^b^c^min^max
                        lo[i] = l;
                        hi[i] = h;
                    }
                }
            }
            uint32_t o[8], fz[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t zmin = __vimin3_u16x2(lo[j], lo[j + 1], lo[j + 2]);
                const uint32_t zmax = __vimax3_u16x2(hi[j], hi[j + 1], hi[j + 2]);
                const uint32_t a = __vimax3_u16x2(lo[j], lo[j + 1], lo[j + 2]);
                const uint32_t c = __vimin3_u16x2(hi[j], hi[j + 1], hi[j + 2]);
                const uint32_t bl = __vimin3_u16x2(mid[j], mid[j + 1], mid[j + 2]);
                const uint32_t bh = __vimax3_u16x2(mid[j], mid[j + 1], mid[j + 2]);
                const uint32_t b = mid[j] ^ mid[j + 1] ^ mid[j + 2] ^ bl ^ bh;
                const uint32_t ml = __vimin3_u16x2(a, b, c), mh = __vimax3_u16x2(a, b, c);
                const uint32_t zmed = a ^ b ^ c ^ ml ^ mh;  // median of 9 = med3(max lo, med mid, min hi)
                const uint32_t g = gm[j + 1];
                // lane masks (values are v * 257): mA = level A holds, mB = zmin < g < zmax
                const uint32_t mA =
                    lane_mask(fadd(__vimin3_u16x2(fsub(zmed, zmin), fsub(zmax, zmed), 0x01010101u), 0x7FFF7FFFu));
                const uint32_t mB =
                    lane_mask(fadd(__vimin3_u16x2(fsub(g, zmin), fsub(zmax, g), 0x01010101u), 0x7FFF7FFFu));
                const uint32_t sel = mA & ~mB;
                o[j] = (zmed & sel) | (g & ~sel);
                if (FIN) fz[j] = mA & 0x00030003u;     // 3 where finalised at k = 3
                failbits |= (~mA & 0x80008000u) >> j;  // lane 0 -> bit 15 - j, lane 1 -> bit 31 - j
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t t01 = prmt(o[4 * h], o[4 * h + 1], 0x6240);
                const uint32_t t23 = prmt(o[4 * h + 2], o[4 * h + 3], 0x6240);
                *reinterpret_cast<uint32_t*>(O + lr * TW + c0 + 4 * h) = prmt(t01, t23, 0x5410);
                *reinterpret_cast<uint32_t*>(O + (lr + 1) * TW + c0 + 4 * h) = prmt(t01, t23, 0x7632);
                if (FIN) {
                    const uint32_t f01 = prmt(fz[4 * h], fz[4 * h + 1], 0x6240);
                    const uint32_t f23 = prmt(fz[4 * h + 2], fz[4 * h + 3], 0x6240);
                    *reinterpret_cast<uint32_t*>(F + lr * TW + c0 + 4 * h) = prmt(f01, f23, 0x5410);
                    *reinterpret_cast<uint32_t*>(F + (lr + 1) * TW + c0 + 4 * h) = prmt(f01, f23, 0x7632);
                }
            }
        }
        const int orow0 = y0 - args.row_begin + sub * WR;  // output row of strip row 0
        const int row_lim = args.row_end - y0 - sub * WR;  // strip rows < row_lim are in range
        const int col_lim = cols - x0;

        // ---- append level-A failures (inside the output range) to the k = 5 work queue ----
        if (args.grow) {
            const uint32_t rv = __brev(failbits);                     // bit 16+j: row lr; bit j: row lr+1
            uint32_t m = ((rv >> 16) & 0xFFu) | ((rv & 0xFFu) << 8);  // bit j: row lr; bit 8+j: row lr+1
            if (lr >= row_lim) m &= 0xFF00u;
            if (lr + 1 >= row_lim) m &= 0x00FFu;
            if (c0 + 8 > col_lim) {
                const uint32_t cm = col_lim <= c0 ? 0u : ((1u << (col_lim - c0)) - 1u);
                m &= cm | (cm << 8);
            }
            const int nf = __popc(m);
            int incl = nf;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= d) incl += v;
            }
            const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
            int base = 0;
            if (lane == 31 && total) base = atomicAdd(args.queue_n, total);
            base = __shfl_sync(0xFFFFFFFFu, base, 31);
            int pos = base + incl - nf;
            const uint32_t zrow = ((uint32_t)z << args.row_bits) | (uint32_t)(orow0 + lr);
            while (m) {
                const int bit = __ffs(m) - 1;
                m &= m - 1;
                args.queue[pos++] = ((zrow + (uint32_t)(bit >> 3)) << args.col_bits) | (uint32_t)(x0 + c0 + (bit & 7));
            }
        }
        __syncwarp();

        // ---- the strip's 4 output rows (and finalized_at): one 16-byte store per lane ----
        {
            const int sr = lane >> 3, sc = 16 * (lane & 7);
            if (sr < row_lim) {
                uint8_t* drow = args.dst + (size_t)z * args.dslice + (size_t)(orow0 + sr) * args.dpitch + x0 + sc;
                uint8_t* frow =
                    FIN ? args.fin + (size_t)z * args.fslice + (size_t)(orow0 + sr) * args.fpitch + x0 + sc : nullptr;
                if (sc + 16 <= col_lim) {
                    *reinterpret_cast<uint4*>(drow) = *reinterpret_cast<const uint4*>(O + sr * TW + sc);
                    if (FIN) *reinterpret_cast<uint4*>(frow) = *reinterpret_cast<const uint4*>(F + sr * TW + sc);
                } else {
                    for (int c = 0; c < 16 && sc + c < col_lim; ++c) {
                        drow[c] = O[sr * TW + sc + c];
                        if (FIN) frow[c] = F[sr * TW + sc + c];
                    }
                }
            }
        }
        __syncwarp();

        // ---- release the byte buffer; the last warp refills it with this CTA's tile ti + NBUF ----
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(&done_cnt[s], 1) == NW - 1) {
                done_cnt[s] = 0;
                if (ti + NBUF < my_tiles) {
                    tile_coords(args, blockIdx.x + (ti + NBUF) * gridDim.x, tinfo + 4 * s);
                    fence_proxy_async_smem();
                    issue_tile_load(&tm_src, B, &full[s], tinfo[4 * s], tinfo[4 * s + 1], tinfo[4 * s + 2]);
                }
            }
        }
    }
}

// ------------------------------------------------------------------------------------------
// growth kernels (k >= 5) over the device-wide work queue
// ------------------------------------------------------------------------------------------

struct GrowArgs {
    const uint8_t* src;
    size_t spitch, sslice;
    uint8_t* dst;
    size_t dpitch, dslice;
    uint8_t* fin;
    size_t fpitch, fslice;
    int rows, cols, row_begin;
    int col_bits, row_bits;
    const uint32_t* qin;
    const int* nin;
    uint32_t* qout;  // null at the last level
    int* nout;
};

template <int K>
struct Win {
    static constexpr int RK = K / 2;
    static constexpr int AW = (K + 3) / 4;        // aligned words per window row
    static constexpr int NRAW = (K + 2) / 4 + 1;  // raw words read per window row
    static constexpr int TAIL = K % 4;            // valid bytes of the last word (0 = full)
    static constexpr int M = (K * K - 1) / 2;     // median rank
    __device__ static constexpr uint32_t v80(int j) {
        return (j < AW - 1 || TAIL == 0) ? 0x80808080u
                                         : (TAIL == 1 ? 0x00000080u : (TAIL == 2 ? 0x00008080u : 0x00808080u));
    }
};

struct Pix {
    int z, orow, r, c;  // slice, output row, source row, column
};

__device__ __forceinline__ Pix decode(const GrowArgs& a, uint32_t id) {
    Pix p;
    p.c = (int)(id & ((1u << a.col_bits) - 1u));
    const uint32_t zr = id >> a.col_bits;
    p.orow = (int)(zr & ((1u << a.row_bits) - 1u));
    p.z = (int)(zr >> a.row_bits);
    p.r = a.row_begin + p.orow;
    return p;
}

// The K x K window around a pixel as K rows of AW byte-aligned words (edge replication).
template <int K>
__device__ __forceinline__ void load_window(const GrowArgs& a, const Pix& p, uint32_t (&w)[K][Win<K>::AW]) {
    using W = Win<K>;
    const uint8_t* __restrict__ plane = a.src + (size_t)p.z * a.sslice;
    const int start = p.c - W::RK;
    if (p.r - W::RK >= 0 && p.r + W::RK < a.rows && start >= 0 && (start & ~3) + 4 * W::NRAW <= a.cols) {
        const int sh = 8 * (start & 3);
#pragma unroll
        for (int r = 0; r < K; ++r) {
            const uint32_t* rp =
                reinterpret_cast<const uint32_t*>(plane + (size_t)(p.r - W::RK + r) * a.spitch + (start & ~3));
            uint32_t raw[W::NRAW];
#pragma unroll
            for (int j = 0; j < W::NRAW; ++j) raw[j] = __ldg(rp + j);
#pragma unroll
            for (int j = 0; j < W::AW; ++j) w[r][j] = __funnelshift_r(raw[j], (j + 1 < W::NRAW) ? raw[j + 1] : 0u, sh);
        }
    } else {
#pragma unroll
        for (int r = 0; r < K; ++r) {
            const uint8_t* rowp = plane + (size_t)min(max(p.r - W::RK + r, 0), a.rows - 1) * a.spitch;
#pragma unroll
            for (int j = 0; j < W::AW; ++j) {
                uint32_t v = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (4 * j + b < K) v |= (uint32_t)__ldg(rowp + min(max(start + 4 * j + b, 0), a.cols - 1)) << (8 * b);
                w[r][j] = v;
            }
        }
    }
}

template <int K>
__device__ __forceinline__ void select_net(uint32_t (&v)[K * K], uint32_t& a, uint32_t& b, uint32_t& c);
template <>
__device__ __forceinline__ void select_net<5>(uint32_t (&v)[25], uint32_t& a, uint32_t& b, uint32_t& c) {
    select_net5(v, a, b, c);
}
template <>
__device__ __forceinline__ void select_net<7>(uint32_t (&v)[49], uint32_t& a, uint32_t& b, uint32_t& c) {
    select_net7(v, a, b, c);
}

__device__ __forceinline__ void write_result(const GrowArgs& a, const Pix& p, uint32_t v, int k) {
    a.dst[(size_t)p.z * a.dslice + (size_t)p.orow * a.dpitch + p.c] = (uint8_t)v;
    if (a.fin) a.fin[(size_t)p.z * a.fslice + (size_t)p.orow * a.fpitch + p.c] = (uint8_t)k;
}

// Warp-aggregated append of the lanes with keep set to the next level's queue.
__device__ __forceinline__ void requeue(const GrowArgs& a, bool keep, uint32_t id) {
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
    if (!bal || !a.qout) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(bal) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(a.nout, __popc(bal));
    base = __shfl_sync(0xFFFFFFFFu, base, leader);
    if (keep) a.qout[base + __popc(bal & ((1u << lane) - 1u))] = id;
}

// k = 5, 7: two queued pixels per thread in the u16x2 lanes, selection network.
template <int K>
__global__ void __launch_bounds__(256) amf_grow_pair_kernel(const GrowArgs a) {
    using W = Win<K>;
    const int n = *a.nin;
    const int npairs = (n + 1) >> 1;
    const int stride = gridDim.x * blockDim.x;
    for (int base = blockIdx.x * blockDim.x; base < npairs; base += stride) {
        const int i = base + threadIdx.x;
        bool keepA = false, keepB = false;
        uint32_t ida = 0, idb = 0;
        if (i < npairs) {
            ida = a.qin[2 * i];
            const bool hasb = 2 * i + 1 < n;
            idb = hasb ? a.qin[2 * i + 1] : ida;
            const Pix pa = decode(a, ida), pb = decode(a, idb);
            uint32_t wa[K][W::AW], wb[K][W::AW];
            load_window<K>(a, pa, wa);
            load_window<K>(a, pb, wb);
            uint32_t v[K * K];
#pragma unroll
            for (int r = 0; r < K; ++r)
#pragma unroll
                for (int e = 0; e < K; ++e) v[r * K + e] = pairw_rt(wa[r][e >> 2], wb[r][e >> 2], e & 3);
            const uint32_t g = v[W::RK * K + W::RK];
            uint32_t zmin, zmed, zmax;
            select_net<K>(v, zmin, zmed, zmax);
#pragma unroll
            for (int l = 0; l < 2; ++l) {
                const uint32_t zn = (zmin >> (16 * l)) & 0xFFu, zd = (zmed >> (16 * l)) & 0xFFu;
                const uint32_t zx = (zmax >> (16 * l)) & 0xFFu, gl = (g >> (16 * l)) & 0xFFu;
                const bool done = zn < zd && zd < zx;
                if (l == 0) {
                    if (done) write_result(a, pa, (zn < gl && gl < zx) ? gl : zd, K);
                    keepA = !done;
                } else if (hasb) {
                    if (done) write_result(a, pb, (zn < gl && gl < zx) ? gl : zd, K);
                    keepB = !done;
                }
            }
        }
        requeue(a, keepA, ida);
        requeue(a, keepB, idb);
    }
}

// Count of window values equal to v (SWAR over the aligned window words).
template <int K>
__device__ __forceinline__ int count_eq(const uint32_t (&w)[K][Win<K>::AW], uint32_t v) {
    const uint32_t P = v * 0x01010101u;
    int c = 0;
#pragma unroll
    for (int r = 0; r < K; ++r)
#pragma unroll
        for (int j = 0; j < Win<K>::AW; ++j) c += zero_bytes(w[r][j] ^ P, Win<K>::v80(j));
    return c;
}

// Element of rank `rank` (0-based): bitwise radix select.  All values lie in [lo, hi], so the
// bits above the highest bit where lo and hi differ are fixed.
template <int K>
__device__ __forceinline__ uint32_t select_rank(const uint32_t (&w)[K][Win<K>::AW], int rank, uint32_t lo,
                                                uint32_t hi) {
    const int hb = 31 - __clz(lo ^ hi);
    uint32_t prefix = lo & ~((2u << hb) - 1u);
    int below = 0;
    for (int b = hb; b >= 0; --b) {
        const uint32_t M = ((0xFFu << b) & 0xFFu) * 0x01010101u;
        const uint32_t P = prefix * 0x01010101u;
        int c = 0;
#pragma unroll
        for (int r = 0; r < K; ++r)
#pragma unroll
            for (int j = 0; j < Win<K>::AW; ++j) c += zero_bytes((w[r][j] ^ P) & M, Win<K>::v80(j));
        if (below + c <= rank) {
            below += c;
            prefix |= 1u << b;
        }
    }
    return prefix;
}

// k = 9, 11: one pixel per thread; level A from SWAR counts, median by radix select if needed.
template <int K>
__global__ void __launch_bounds__(256) amf_grow_radix_kernel(const GrowArgs a) {
    using W = Win<K>;
    const int n = *a.nin;
    const int stride = gridDim.x * blockDim.x;
    for (int base = blockIdx.x * blockDim.x; base < n; base += stride) {
        const int i = base + threadIdx.x;
        bool keep = false;
        uint32_t id = 0;
        if (i < n) {
            id = a.qin[i];
            const Pix p = decode(a, id);
            uint32_t w[K][W::AW];
            load_window<K>(a, p, w);
            uint32_t mn = 0x00FF00FFu, mx = 0u;
#pragma unroll
            for (int r = 0; r < K; ++r)
#pragma unroll
                for (int j = 0; j < W::AW; ++j) {
                    const uint32_t x = w[r][j];
                    uint32_t lo, hi;
                    if (j < W::AW - 1 || W::TAIL == 0) {
                        lo = prmt(x, 0, 0x4140);
                        hi = prmt(x, 0, 0x4342);
                    } else if (W::TAIL == 1) {
                        lo = hi = prmt(x, 0, 0x4040);
                    } else if (W::TAIL == 2) {
                        lo = hi = prmt(x, 0, 0x4140);
                    } else {
                        lo = prmt(x, 0, 0x4140);
                        hi = prmt(x, 0, 0x4242);
                    }
                    mn = __vimin3_u16x2(mn, lo, hi);
                    mx = __vimax3_u16x2(mx, lo, hi);
                }
            const uint32_t zmin = min(mn & 0xFFFFu, mn >> 16), zmax = max(mx & 0xFFFFu, mx >> 16);
            // level A <=> zmin < zmax, #(v == zmin) <= m and #(v == zmax) <= m
            const bool done = zmin < zmax && count_eq<K>(w, zmin) <= W::M && count_eq<K>(w, zmax) <= W::M;
            if (done) {
                const uint32_t g = (w[W::RK][W::RK >> 2] >> (8 * (W::RK & 3))) & 0xFFu;
                write_result(a, p, (g != zmin && g != zmax) ? g : select_rank<K>(w, W::M, zmin, zmax), K);
            }
            keep = !done;
        }
        requeue(a, keep, id);
    }
}

// k > 11 (windows beyond the compile-time set): same algorithm on clamped byte reads.
__global__ void __launch_bounds__(256) amf_grow_generic_kernel(const GrowArgs a, int k) {
    const int n = *a.nin;
    const int stride = gridDim.x * blockDim.x;
    const int rk = k / 2, m = (k * k - 1) / 2;
    for (int base = blockIdx.x * blockDim.x; base < n; base += stride) {
        const int i = base + threadIdx.x;
        bool keep = false;
        uint32_t id = 0;
        if (i < n) {
            id = a.qin[i];
            const Pix p = decode(a, id);
            const uint8_t* __restrict__ plane = a.src + (size_t)p.z * a.sslice;
            auto at = [&](int dr, int dc) -> uint32_t {
                return __ldg(plane + (size_t)min(max(p.r + dr, 0), a.rows - 1) * a.spitch +
                             min(max(p.c + dc, 0), a.cols - 1));
            };
            uint32_t zmin = 255, zmax = 0;
            for (int dr = -rk; dr <= rk; ++dr)
                for (int dc = -rk; dc <= rk; ++dc) {
                    const uint32_t v = at(dr, dc);
                    zmin = min(zmin, v);
                    zmax = max(zmax, v);
                }
            int cmin = 0, cmax = 0;
            if (zmin < zmax)
                for (int dr = -rk; dr <= rk; ++dr)
                    for (int dc = -rk; dc <= rk; ++dc) {
                        const uint32_t v = at(dr, dc);
                        cmin += v == zmin;
                        cmax += v == zmax;
                    }
            const bool done = zmin < zmax && cmin <= m && cmax <= m;
            if (done) {
                const uint32_t g = at(0, 0);
                uint32_t out = g;
                if (g == zmin || g == zmax) {
                    const int hb = 31 - __clz(zmin ^ zmax);
                    uint32_t prefix = zmin & ~((2u << hb) - 1u);
                    int below = 0;
                    for (int b = hb; b >= 0; --b) {
                        const uint32_t mask = (0xFFu << b) & 0xFFu;
                        int c = 0;
                        for (int dr = -rk; dr <= rk; ++dr)
                            for (int dc = -rk; dc <= rk; ++dc) c += ((at(dr, dc) ^ prefix) & mask) == 0;
                        if (below + c <= m) {
                            below += c;
                            prefix |= 1u << b;
                        }
                    }
                    out = prefix;
                }
                write_result(a, p, out, k);
            }
            keep = !done;
        }
        requeue(a, keep, id);
    }
}

int g_num_sms = 0;

int bits_for(long long n) {
    int b = 0;
    while ((1ll << b) < n) ++b;
    return b;
}

}  // namespace

size_t amf_queue_words(const Plane& p) { return (size_t)(p.row_end - p.row_begin) * p.cols * p.n_slices + 64; }

cudaError_t launch_amf(const Plane& p, int smax, uint8_t* fin, size_t fpitch, size_t fslice, const AmfWork& work,
                       cudaStream_t stream) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e =
            cudaFuncSetAttribute(amf_k3_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(amf_k3_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int out_rows = p.row_end - p.row_begin;
    const int col_bits = bits_for(p.cols), row_bits = bits_for(out_rows), z_bits = bits_for(p.n_slices);
    const bool grow = smax >= 5;
    if (grow && col_bits + row_bits + z_bits > 32) return cudaErrorInvalidValue;  // queue id overflow
    CUtensorMap tm_src;
    cudaError_t e = make_tmap_u8(&tm_src, p.src, p.cols, p.rows, p.n_slices, p.spitch, p.sslice, BS, BH);
    if (e != cudaSuccess) return e;
    const int nlev = grow ? (smax - 3) / 2 : 0;
    if (grow) {
        e = cudaMemsetAsync(work.counts, 0, sizeof(int) * (nlev + 1), stream);
        if (e != cudaSuccess) return e;
    }
    K3Args a;
    a.dst = p.dst;
    a.dpitch = p.dpitch;
    a.dslice = p.dslice;
    a.fin = fin;
    a.fpitch = fpitch;
    a.fslice = fslice;
    a.rows = p.rows;
    a.cols = p.cols;
    a.row_begin = p.row_begin;
    a.row_end = p.row_end;
    a.n_slices = p.n_slices;
    a.tiles_x = (p.cols + TW - 1) / TW;
    a.tiles_y = (out_rows + TH - 1) / TH;
    a.grow = grow;
    a.queue = work.queue[0];
    a.queue_n = work.counts;
    a.col_bits = col_bits;
    a.row_bits = row_bits;
    static int per_sm = 0;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, amf_k3_kernel<false>, NT, SMEM);
        if (per_sm < 1) per_sm = 1;
    }
    const long long ntiles = (long long)a.tiles_x * a.tiles_y * a.n_slices;
    const int grid = (int)std::min<long long>(ntiles, (long long)g_num_sms * per_sm);
    if (fin) amf_k3_kernel<true><<<grid, NT, SMEM, stream>>>(tm_src, a);
    else amf_k3_kernel<false><<<grid, NT, SMEM, stream>>>(tm_src, a);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;

    // growth levels: queue[l & 1] holds the pixels still open at k = 5 + 2 l
    GrowArgs g;
    g.src = p.src;
    g.spitch = p.spitch;
    g.sslice = p.sslice;
    g.dst = p.dst;
    g.dpitch = p.dpitch;
    g.dslice = p.dslice;
    g.fin = fin;
    g.fpitch = fpitch;
    g.fslice = fslice;
    g.rows = p.rows;
    g.cols = p.cols;
    g.row_begin = p.row_begin;
    g.col_bits = col_bits;
    g.row_bits = row_bits;
    const long long npix = (long long)out_rows * p.cols * p.n_slices;
    for (int l = 0; l < nlev; ++l) {
        const int k = 5 + 2 * l;
        g.qin = work.queue[l & 1];
        g.nin = work.counts + l;
        g.qout = (l + 1 < nlev) ? work.queue[(l + 1) & 1] : nullptr;
        g.nout = work.counts + l + 1;
        // grid sized for the worst case of this level, capped at a few waves (grid-stride loops)
        const long long items = (k <= 7) ? (npix + 1) / 2 : npix;
        const int blocks =
            (int)std::max<long long>(1, std::min<long long>((items + 255) / 256, (long long)g_num_sms * 4));
        switch (k) {
            case 5: amf_grow_pair_kernel<5><<<blocks, 256, 0, stream>>>(g); break;
            case 7: amf_grow_pair_kernel<7><<<blocks, 256, 0, stream>>>(g); break;
            case 9: amf_grow_radix_kernel<9><<<blocks, 256, 0, stream>>>(g); break;
            case 11: amf_grow_radix_kernel<11><<<blocks, 256, 0, stream>>>(g); break;
            default: amf_grow_generic_kernel<<<blocks, 256, 0, stream>>>(g, k); break;
        }
        count_launch();
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace hyb
