// amf.cu -- adaptive median filter (AMF) for sm_100a.
//
// Semantics: detail::adaptive_median_rows, reference proj/src/adaptive_median.cpp:123-215
// (windows k = 3..smax over the pristine input, edge replication, level A/B, unresolved pixels
// keep their input).  Design:
//
//   * persistent CTAs walk 128 x 32 output tiles; each tile plus a halo of R = (smax-1)/2 pixels
//     arrives in shared memory by TMA (cp.async.bulk.tensor, mbarrier completion), double
//     buffered so the next tile streams in while this one is filtered; tiles on the image border
//     get their out-of-bounds cells (TMA zero fill) replaced by edge replication in shared
//     memory; the output tile leaves by a TMA store (which clips at the image edge);
//   * k = 3 (95-99.7 % of pixels finalise here) runs on every pixel with u16x2 SIMD: the tile is
//     re-laid out as row PAIRS (word = pixel(r,c) | pixel(r+1,c) << 16) so one VIMNMX.U16x2
//     serves two output rows; each thread owns 2 rows x 8 columns and sorts every 3-tall column
//     once (min / max / xor-median) for its 3 outputs; level A/B become lane masks via a
//     sign-replicating PRMT, with no per-lane branches;
//   * pixels failing level A are compacted (warp scan + one shared atomic per warp) into a
//     per-CTA shared-memory work queue; each growth level k = 5..smax processes only the queue,
//     warp-uniformly, and re-queues its survivors.  k = 5 and 7 gather two queued pixels into
//     the u16x2 lanes of one thread and run a generated pruned selection network (min, median,
//     max; networks.cuh); larger k use a SWAR count test for level A and a bitwise radix select.
#include <cuda.h>

#include <algorithm>
#include <cstdint>

#include "hyb_internal.cuh"
#include "networks.cuh"
#include "tma.cuh"

namespace hyb {
namespace {

constexpr int TW = 128;     // tile columns
constexpr int TH = 32;      // tile rows
constexpr int NT = 256;     // threads per CTA
constexpr int PS = TW + 8;  // pair-tile row stride (words)
constexpr int PO = 4;       // pair-tile column offset: pair word cc' <-> tile column cc' - PO
constexpr int MAX_LEVELS = 128;
constexpr size_t kSmemBudget = 220 * 1024;

struct Geo {
    int R;        // halo radius of the byte tile
    int CP;       // column pad of the byte tile (>= R, multiple of 16: TMA box x offsets must be 16-byte aligned)
    int BH;       // byte-tile rows used
    int BS;       // byte-tile row stride = TMA box width x boxes per row
    int box_w, nbx, box_h, nby;
    int nbuf;     // 1 or 2 byte-tile buffers
    size_t b_bytes;  // bytes per byte-tile buffer (128-aligned)
};

__host__ __device__ inline size_t rup(size_t v, size_t a) { return (v + a - 1) / a * a; }

__host__ __device__ inline size_t fixed_bytes() {
    return 640                                 // mbarriers + level counters
           + rup((size_t)(TH + 2) * PS * 4, 128)  // pair tile (aliased by queue 1)
           + (size_t)TH * TW                   // output tile
           + (size_t)TH * TW                   // finalized_at tile
           + (size_t)TH * TW * 2;              // queue 0
}

__host__ __device__ inline Geo make_geo(int smax) {
    Geo g;
    g.R = (smax - 1) / 2;
    const int cp = 16 * ((g.R + 15) / 16 > 0 ? (g.R + 15) / 16 : 1);
    g.CP = cp;
    g.BH = TH + 2 * g.R;
    const int need = TW + 2 * cp;
    if (need <= 256) {
        g.box_w = need;
        g.nbx = 1;
    } else {
        g.box_w = 128;
        g.nbx = (need + 127) / 128;
    }
    g.BS = g.box_w * g.nbx;
    g.box_h = g.BH <= 256 ? g.BH : 128;
    g.nby = (g.BH + g.box_h - 1) / g.box_h;
    g.b_bytes = rup((size_t)g.BS * g.box_h * g.nby, 128);
    g.nbuf = (2 * g.b_bytes + fixed_bytes() <= kSmemBudget) ? 2 : 1;
    return g;
}

__host__ __device__ inline size_t smem_bytes(const Geo& g) { return g.nbuf * g.b_bytes + fixed_bytes() + 128; }

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) { return __byte_perm(a, b, s); }

// prmt.b32 with the selector's sign-replicate bit honoured (__byte_perm masks it off): 0xBB99
// turns bit 15 / bit 31 into a full 16-bit lane mask.
__device__ __forceinline__ uint32_t lane_mask(uint32_t x) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(r) : "r"(x));
    return r;
}

// Number of zero bytes of x among the byte lanes flagged (0x80) in v80.
__device__ __forceinline__ int zero_bytes(uint32_t x, uint32_t v80) {
    const uint32_t t = (x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
    return __popc(~(t | x) & v80);
}

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

// Loads the K x K window around tile pixel (ty, tx) as K rows of AW byte-aligned words.
template <int K>
__device__ __forceinline__ void load_window(const uint8_t* __restrict__ B, const Geo& geo, int ty, int tx,
                                            uint32_t (&a)[K][Win<K>::AW]) {
    using W = Win<K>;
    const int start = tx + geo.CP - W::RK;
    const int sh = 8 * (start & 3);
    const uint32_t* rowp =
        reinterpret_cast<const uint32_t*>(B + (size_t)(ty + geo.R - W::RK) * geo.BS) + (start >> 2);
#pragma unroll
    for (int r = 0; r < K; ++r) {
        uint32_t raw[W::NRAW];
#pragma unroll
        for (int j = 0; j < W::NRAW; ++j) raw[j] = rowp[r * (geo.BS >> 2) + j];
#pragma unroll
        for (int j = 0; j < W::AW; ++j) a[r][j] = __funnelshift_r(raw[j], (j + 1 < W::NRAW) ? raw[j + 1] : 0u, sh);
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

// Growth level for two queued pixels at once (u16x2 lanes) with a generated selection network.
template <int K>
__device__ __forceinline__ void level_pair(const uint8_t* __restrict__ B, const Geo& geo, int pa, int pb,
                                           uint32_t& done, uint32_t& outw) {
    using W = Win<K>;
    uint32_t A[K][W::AW], Bw[K][W::AW];
    load_window<K>(B, geo, pa / TW, pa % TW, A);
    load_window<K>(B, geo, pb / TW, pb % TW, Bw);
    uint32_t v[K * K];
#pragma unroll
    for (int r = 0; r < K; ++r)
#pragma unroll
        for (int w = 0; w < W::AW; ++w) {
            const uint32_t x = prmt(A[r][w], Bw[r][w], 0x5140);  // A0 B0 A1 B1
            const uint32_t y = prmt(A[r][w], Bw[r][w], 0x7362);  // A2 B2 A3 B3
            const uint32_t e[4] = {prmt(x, 0, 0x4140), prmt(x, 0, 0x4342), prmt(y, 0, 0x4140), prmt(y, 0, 0x4342)};
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (4 * w + j < K) v[r * K + 4 * w + j] = e[j];
        }
    const uint32_t g = v[W::RK * K + W::RK];
    uint32_t zmin, zmed, zmax;
    select_net<K>(v, zmin, zmed, zmax);
    done = 0;
    outw = 0;
#pragma unroll
    for (int l = 0; l < 2; ++l) {
        const uint32_t zn = (zmin >> (16 * l)) & 0xFFu, zd = (zmed >> (16 * l)) & 0xFFu;
        const uint32_t zx = (zmax >> (16 * l)) & 0xFFu, gl = (g >> (16 * l)) & 0xFFu;
        if (zn < zd && zd < zx) {
            done |= 1u << l;
            outw |= ((zn < gl && gl < zx) ? gl : zd) << (8 * l);
        }
    }
}

// Count of window values equal to v (SWAR over the aligned window words).
template <int K>
__device__ __forceinline__ int count_eq(const uint32_t (&a)[K][Win<K>::AW], uint32_t v) {
    const uint32_t P = v * 0x01010101u;
    int c = 0;
#pragma unroll
    for (int r = 0; r < K; ++r)
#pragma unroll
        for (int j = 0; j < Win<K>::AW; ++j) c += zero_bytes(a[r][j] ^ P, Win<K>::v80(j));
    return c;
}

// Element of rank `rank` (0-based): bitwise radix select.  All values lie in [lo, hi], so the
// bits above the highest bit where lo and hi differ are fixed.
template <int K>
__device__ __forceinline__ uint32_t select_rank(const uint32_t (&a)[K][Win<K>::AW], int rank, uint32_t lo,
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
            for (int j = 0; j < Win<K>::AW; ++j) c += zero_bytes((a[r][j] ^ P) & M, Win<K>::v80(j));
        if (below + c <= rank) {
            below += c;
            prefix |= 1u << b;
        }
    }
    return prefix;
}

// One growth level, one pixel, compile-time K (used for K = 9, 11).
template <int K>
__device__ __forceinline__ bool level_fixed(const uint8_t* __restrict__ B, const Geo& geo, int ty, int tx,
                                            uint8_t* out) {
    using W = Win<K>;
    uint32_t a[K][W::AW];
    load_window<K>(B, geo, ty, tx, a);
    uint32_t mn = 0x00FF00FFu, mx = 0u;
#pragma unroll
    for (int r = 0; r < K; ++r)
#pragma unroll
        for (int j = 0; j < W::AW; ++j) {
            const uint32_t w = a[r][j];
            uint32_t lo, hi;
            if (j < W::AW - 1 || W::TAIL == 0) {
                lo = prmt(w, 0, 0x4140);
                hi = prmt(w, 0, 0x4342);
            } else if (W::TAIL == 1) {
                lo = hi = prmt(w, 0, 0x4040);
            } else if (W::TAIL == 2) {
                lo = hi = prmt(w, 0, 0x4140);
            } else {
                lo = prmt(w, 0, 0x4140);
                hi = prmt(w, 0, 0x4242);
            }
            mn = __vimin3_u16x2(mn, lo, hi);
            mx = __vimax3_u16x2(mx, lo, hi);
        }
    const uint32_t zmin = min(mn & 0xFFFFu, mn >> 16);
    const uint32_t zmax = max(mx & 0xFFFFu, mx >> 16);
    if (zmin == zmax) return false;
    // level A <=> #(v == zmin) <= m and #(v == zmax) <= m
    if (count_eq<K>(a, zmin) > W::M || count_eq<K>(a, zmax) > W::M) return false;
    const uint32_t g = B[(size_t)(ty + geo.R) * geo.BS + tx + geo.CP];
    *out = (uint8_t)((g != zmin && g != zmax) ? g : select_rank<K>(a, W::M, zmin, zmax));
    return true;
}

// Growth level for window sizes beyond the compile-time set (k > 11), bytes from the tile.
__device__ bool level_generic(const uint8_t* __restrict__ B, const Geo& geo, int ty, int tx, int k, uint8_t* out) {
    const int rk = k / 2;
    const uint8_t* base = B + (size_t)(ty + geo.R - rk) * geo.BS + (tx + geo.CP - rk);
    uint32_t zmin = 255, zmax = 0;
    for (int r = 0; r < k; ++r)
        for (int c = 0; c < k; ++c) {
            const uint32_t v = base[(size_t)r * geo.BS + c];
            zmin = min(zmin, v);
            zmax = max(zmax, v);
        }
    if (zmin == zmax) return false;
    const int m = (k * k - 1) / 2;
    int cmin = 0, cmax = 0;
    for (int r = 0; r < k; ++r)
        for (int c = 0; c < k; ++c) {
            const uint32_t v = base[(size_t)r * geo.BS + c];
            cmin += v == zmin;
            cmax += v == zmax;
        }
    if (cmin > m || cmax > m) return false;
    const uint32_t g = B[(size_t)(ty + geo.R) * geo.BS + tx + geo.CP];
    if (g != zmin && g != zmax) {
        *out = (uint8_t)g;
        return true;
    }
    const int hb = 31 - __clz(zmin ^ zmax);
    uint32_t prefix = zmin & ~((2u << hb) - 1u);
    int below = 0;
    for (int b = hb; b >= 0; --b) {
        const uint32_t mask = (0xFFu << b) & 0xFFu;
        int c = 0;
        for (int r = 0; r < k; ++r)
            for (int cc = 0; cc < k; ++cc) c += ((base[(size_t)r * geo.BS + cc] ^ prefix) & mask) == 0;
        if (below + c <= m) {
            below += c;
            prefix |= 1u << b;
        }
    }
    *out = (uint8_t)prefix;
    return true;
}

struct AmfArgs {
    const uint8_t* src;
    size_t spitch, sslice;
    uint8_t* dst;
    size_t dpitch, dslice;
    uint8_t* fin;
    size_t fpitch, fslice;
    int rows, cols;          // source buffer (clamping bounds)
    int row_begin, row_end;  // output rows (source coordinates)
    int n_slices, smax;
    int tiles_x, tiles_y;
    int has_fin;
};

// Issues the TMA loads of one tile's byte box (x offsets are multiples of 16 bytes -- TMA on this
// stack faults on unaligned inner-dimension starts, tests/cuda/tma_probe2.cu; out-of-bounds
// cells arrive zero-filled and are rebuilt by edge replication).
__device__ __forceinline__ void issue_tile_load(const CUtensorMap* tm, const Geo& geo, uint8_t* Bbuf, uint64_t* bar,
                                                int x0, int y0, int z) {
    mbar_expect_tx(bar, (uint32_t)(geo.box_w * geo.nbx * geo.box_h * geo.nby));
    for (int by = 0; by < geo.nby; ++by)
        for (int bx = 0; bx < geo.nbx; ++bx)
            tma_load_3d(Bbuf + (size_t)by * geo.box_h * geo.BS + (size_t)bx * geo.box_w, tm, bar,
                        x0 - geo.CP + bx * geo.box_w, y0 - geo.R + by * geo.box_h, z);
}

__global__ void __launch_bounds__(NT, 4)
    amf_kernel(const __grid_constant__ CUtensorMap tm_src, const __grid_constant__ CUtensorMap tm_dst,
               const __grid_constant__ CUtensorMap tm_fin, const AmfArgs args) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    const Geo geo = make_geo(args.smax);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
    int* qcount = reinterpret_cast<int*>(smem + 16);
    size_t off = 640;
    uint8_t* Bbuf[2];
    Bbuf[0] = smem + off;
    Bbuf[1] = smem + off + (geo.nbuf == 2 ? geo.b_bytes : 0);
    off += geo.nbuf * geo.b_bytes;
    uint32_t* PR = reinterpret_cast<uint32_t*>(smem + off);
    uint16_t* Q1 = reinterpret_cast<uint16_t*>(smem + off);  // aliases PR after k = 3
    off += rup((size_t)(TH + 2) * PS * 4, 128);
    uint8_t* O = smem + off;
    off += TH * TW;
    uint8_t* F = smem + off;
    off += TH * TW;
    uint16_t* Q0 = reinterpret_cast<uint16_t*>(smem + off);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rows = args.rows, cols = args.cols;
    const int per_slice = args.tiles_x * args.tiles_y;
    const int ntiles = per_slice * args.n_slices;
    int t = blockIdx.x;
    if (t >= ntiles) return;

    auto tile_xyz = [&](int tt, int& x0, int& y0, int& z) {
        z = tt / per_slice;
        const int rem = tt - z * per_slice;
        const int by = rem / args.tiles_x;
        x0 = (rem - by * args.tiles_x) * TW;
        y0 = args.row_begin + by * TH;
    };

    if (tid == 0) {
        prefetch_tmap(&tm_src);
        prefetch_tmap(&tm_dst);
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
        int x0, y0, z;
        tile_xyz(t, x0, y0, z);
        issue_tile_load(&tm_src, geo, Bbuf[0], &mbar[0], x0, y0, z);
    }
    __syncthreads();
    uint32_t phase_bits = 0;  // per-buffer mbarrier parity

    for (int it = 0; t < ntiles; ++it, t += gridDim.x) {
        const int buf = geo.nbuf == 2 ? (it & 1) : 0;
        int x0, y0, z;
        tile_xyz(t, x0, y0, z);
        if (geo.nbuf == 2 && tid == 0 && t + (int)gridDim.x < ntiles) {
            int nx, ny, nz;
            tile_xyz(t + gridDim.x, nx, ny, nz);
            issue_tile_load(&tm_src, geo, Bbuf[buf ^ 1], &mbar[buf ^ 1], nx, ny, nz);
        }
        uint8_t* B = Bbuf[buf];
        if (tid < MAX_LEVELS) qcount[tid] = 0;
        mbar_wait(&mbar[buf], (phase_bits >> buf) & 1u);
        phase_bits ^= 1u << buf;

        // ---- border tiles: edge replication in place of TMA's zero fill ----
        const int sx0 = x0 - geo.CP, sy0 = y0 - geo.R;
        if (sx0 < 0 || sx0 + geo.BS > cols || sy0 < 0 || sy0 + geo.BH > rows) {
            const int c_lo = max(0, -sx0), c_hi = min(geo.BS, cols - sx0);
            const int r_lo = max(0, -sy0), r_hi = min(geo.BH, rows - sy0);
            if (c_lo > 0 || c_hi < geo.BS) {
                for (int rr = r_lo + warp; rr < r_hi; rr += NT / 32) {
                    uint8_t* row = B + (size_t)rr * geo.BS;
                    const uint8_t lv = row[c_lo], rv = row[c_hi - 1];
                    for (int cc = lane; cc < geo.BS; cc += 32) {
                        if (cc < c_lo) row[cc] = lv;
                        else if (cc >= c_hi) row[cc] = rv;
                    }
                }
                __syncthreads();
            }
            const int words = geo.BS >> 2;
            for (int idx = tid; idx < geo.BH * words; idx += NT) {
                const int rr = idx / words, q = idx - rr * words;
                const int src_r = rr < r_lo ? r_lo : (rr >= r_hi ? r_hi - 1 : rr);
                if (src_r != rr)
                    reinterpret_cast<uint32_t*>(B + (size_t)rr * geo.BS)[q] =
                        reinterpret_cast<const uint32_t*>(B + (size_t)src_r * geo.BS)[q];
            }
        }
        if (tid == 0) tma_store_wait_read();  // previous tile's O / F no longer read by TMA
        __syncthreads();

        // ---- row-pair tile: PR[pr][cc'] = (t(pr-1, cc'-PO), t(pr, cc'-PO)) in tile coordinates ----
        {
            constexpr int PW4 = PS / 4;
#pragma unroll 1
            for (int idx = tid; idx < (TH + 1) * PW4; idx += NT) {
                const int pr = idx / PW4, q = idx - pr * PW4;
                const int boff = 4 * q - PO + geo.CP;  // multiple of 4
                const uint32_t a = *reinterpret_cast<const uint32_t*>(B + (size_t)(pr - 1 + geo.R) * geo.BS + boff);
                const uint32_t b = *reinterpret_cast<const uint32_t*>(B + (size_t)(pr + geo.R) * geo.BS + boff);
                const uint32_t x = prmt(a, b, 0x5140), y = prmt(a, b, 0x7362);
                *reinterpret_cast<uint4*>(PR + (size_t)pr * PS + 4 * q) =
                    make_uint4(prmt(x, 0, 0x4140), prmt(x, 0, 0x4342), prmt(y, 0, 0x4140), prmt(y, 0, 0x4342));
            }
        }
        __syncthreads();

        // ---- k = 3 on every pixel: thread = rows (r0, r0+1) x columns c0..c0+7 ----
        const int r0 = 2 * (tid >> 4), c0 = 8 * (tid & 15);
        {
            uint32_t lo[10], hi[10], mid[10], gm[10];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                // pair words for tile columns c0-1 .. c0+8 are words PO-1 .. PO+8 of PR[r0+j][c0 ..]
                const uint4* rp = reinterpret_cast<const uint4*>(PR + (size_t)(r0 + j) * PS + c0);
                uint32_t w[10];
                {
                    const uint4 t0 = rp[0], t1 = rp[1], t2 = rp[2], t3 = rp[3];
                    w[0] = t0.w;
                    w[1] = t1.x;
                    w[2] = t1.y;
                    w[3] = t1.z;
                    w[4] = t1.w;
                    w[5] = t2.x;
                    w[6] = t2.y;
                    w[7] = t2.z;
                    w[8] = t2.w;
                    w[9] = t3.x;
                }
#pragma unroll
                for (int i = 0; i < 10; ++i) {
                    if (j == 0) {
                        lo[i] = hi[i] = mid[i] = w[i];
                    } else if (j == 1) {
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
                const uint32_t zmed = a ^ b ^ c ^ ml ^ mh;
                const uint32_t g = gm[j + 1];
                // lane masks: mA = level A holds, mB = g strictly inside (zmin, zmax)
                const uint32_t mA = lane_mask(__vminu2(zmed - zmin, zmax - zmed) + 0x7FFF7FFFu);
                const uint32_t mB = lane_mask(__vminu2(g - zmin, zmax - g) + 0x7FFF7FFFu);
                const uint32_t sel = mA & ~mB;
                o[j] = (zmed & sel) | (g & ~sel);
                fz[j] = mA & 0x00030003u;  // 3 where finalised at k = 3, 0 = queue
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t t01 = prmt(o[4 * h], o[4 * h + 1], 0x6240);
                const uint32_t t23 = prmt(o[4 * h + 2], o[4 * h + 3], 0x6240);
                *reinterpret_cast<uint32_t*>(O + (size_t)r0 * TW + c0 + 4 * h) = prmt(t01, t23, 0x5410);
                *reinterpret_cast<uint32_t*>(O + (size_t)(r0 + 1) * TW + c0 + 4 * h) = prmt(t01, t23, 0x7632);
                const uint32_t f01 = prmt(fz[4 * h], fz[4 * h + 1], 0x6240);
                const uint32_t f23 = prmt(fz[4 * h + 2], fz[4 * h + 3], 0x6240);
                *reinterpret_cast<uint32_t*>(F + (size_t)r0 * TW + c0 + 4 * h) = prmt(f01, f23, 0x5410);
                *reinterpret_cast<uint32_t*>(F + (size_t)(r0 + 1) * TW + c0 + 4 * h) = prmt(f01, f23, 0x7632);
            }
        }
        __syncthreads();  // F complete; PR dead from here on (Q1 aliases it)

        // ---- compact level-A failures (F == 0) inside the output range into queue 0 ----
        {
            const int qr = tid >> 3, qc = 16 * (tid & 7);  // 16 F bytes per thread
            const uint4 fw = *reinterpret_cast<const uint4*>(F + (size_t)qr * TW + qc);
            const uint32_t wv[4] = {fw.x, fw.y, fw.z, fw.w};
            uint32_t m = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t tz = (wv[j] & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
                const uint32_t z80 = ~(tz | wv[j]) & 0x80808080u;  // 0x80 in zero bytes
                m |= ((z80 >> 7) & 1u | (z80 >> 14) & 2u | (z80 >> 21) & 4u | (z80 >> 28) & 8u) << (4 * j);
            }
            const int row_lim = args.row_end - y0, col_lim = cols - x0;
            if (qr >= row_lim) m = 0;
            if (qc + 16 > col_lim) m &= col_lim <= qc ? 0u : ((1u << (col_lim - qc)) - 1u);
            const int nf = __popc(m);
            int incl = nf;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= d) incl += v;
            }
            int base = 0;
            if (lane == 31 && incl > 0) base = atomicAdd(&qcount[0], incl);
            base = __shfl_sync(0xFFFFFFFFu, base, 31);
            int pos = base + incl - nf;
            while (m) {
                const int bit = __ffs(m) - 1;
                m &= m - 1;
                Q0[pos++] = (uint16_t)(qr * TW + qc + bit);
            }
        }

        // ---- growth levels k = 5..smax over the compacted queue ----
        int lvl = 0;
        for (int k = 5; k <= args.smax; k += 2, ++lvl) {
            __syncthreads();
            const int n = qcount[lvl];
            if (n == 0) break;
            const uint16_t* qin = (lvl & 1) ? Q1 : Q0;
            uint16_t* qout = (lvl & 1) ? Q0 : Q1;
            if (k <= 7) {
                const int npairs = (n + 1) >> 1;
                for (int base = warp * 32; base < npairs; base += NT) {
                    const int i = base + lane;
                    uint32_t keep = 0;
                    int pa = 0, pb = 0;
                    if (i < npairs) {
                        pa = qin[2 * i];
                        const bool hasb = 2 * i + 1 < n;
                        pb = hasb ? qin[2 * i + 1] : pa;
                        uint32_t done, outw;
                        if (k == 5) level_pair<5>(B, geo, pa, pb, done, outw);
                        else level_pair<7>(B, geo, pa, pb, done, outw);
                        if (done & 1u) {
                            O[pa] = (uint8_t)outw;
                            F[pa] = (uint8_t)k;
                        } else {
                            keep |= 1u;
                        }
                        if (hasb) {
                            if (done & 2u) {
                                O[pb] = (uint8_t)(outw >> 8);
                                F[pb] = (uint8_t)k;
                            } else {
                                keep |= 2u;
                            }
                        }
                    }
                    const uint32_t balA = __ballot_sync(0xFFFFFFFFu, keep & 1u);
                    const uint32_t balB = __ballot_sync(0xFFFFFFFFu, keep & 2u);
                    const int cnt = __popc(balA) + __popc(balB);
                    if (cnt) {
                        int wbase = 0;
                        if (lane == 0) wbase = atomicAdd(&qcount[lvl + 1], cnt);
                        wbase = __shfl_sync(0xFFFFFFFFu, wbase, 0);
                        const uint32_t below = (1u << lane) - 1u;
                        if (keep & 1u) qout[wbase + __popc(balA & below)] = (uint16_t)pa;
                        if (keep & 2u) qout[wbase + __popc(balA) + __popc(balB & below)] = (uint16_t)pb;
                    }
                }
            } else {
                for (int base = warp * 32; base < n; base += NT) {
                    const int i = base + lane;
                    bool keep = false;
                    int pix = 0;
                    if (i < n) {
                        pix = qin[i];
                        const int ty = pix / TW, tx = pix % TW;
                        uint8_t o = 0;
                        bool done;
                        switch (k) {
                            case 9: done = level_fixed<9>(B, geo, ty, tx, &o); break;
                            case 11: done = level_fixed<11>(B, geo, ty, tx, &o); break;
                            default: done = level_generic(B, geo, ty, tx, k, &o); break;
                        }
                        if (done) {
                            O[pix] = o;
                            F[pix] = (uint8_t)k;
                        } else {
                            keep = true;
                        }
                    }
                    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
                    if (bal) {
                        int wbase = 0;
                        if (lane == 0) wbase = atomicAdd(&qcount[lvl + 1], __popc(bal));
                        wbase = __shfl_sync(0xFFFFFFFFu, wbase, 0);
                        if (keep) qout[wbase + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)pix;
                    }
                }
            }
        }

        // ---- output tile (and finalized_at): TMA store for whole tiles, plain stores at the edges ----
        const int orow = y0 - args.row_begin;
        const int out_rows = args.row_end - args.row_begin;
        const bool full = x0 + TW <= cols && orow + TH <= out_rows;
        if (full) fence_proxy_async_smem();
        __syncthreads();
        if (full) {
            if (tid == 0) {
                tma_store_3d(&tm_dst, O, x0, orow, z);
                if (args.has_fin) tma_store_3d(&tm_fin, F, x0, orow, z);
                tma_store_commit();
            }
        } else {
            const int rl = min(TH, out_rows - orow), cl = min(TW, cols - x0);
            uint8_t* dbase = args.dst + (size_t)z * args.dslice + (size_t)orow * args.dpitch + x0;
            uint8_t* fbase = args.has_fin ? args.fin + (size_t)z * args.fslice + (size_t)orow * args.fpitch + x0 : nullptr;
            for (int idx = tid; idx < TH * TW; idx += NT) {
                const int r = idx >> 7, c = idx & (TW - 1);
                if (r < rl && c < cl) {
                    dbase[(size_t)r * args.dpitch + c] = O[idx];
                    if (fbase) fbase[(size_t)r * args.fpitch + c] = F[idx];
                }
            }
            __syncthreads();  // O / F are rewritten by the next tile
        }
        if (geo.nbuf == 1 && tid == 0 && t + (int)gridDim.x < ntiles) {
            int nx, ny, nz;
            tile_xyz(t + gridDim.x, nx, ny, nz);
            issue_tile_load(&tm_src, geo, Bbuf[0], &mbar[0], nx, ny, nz);
        }
    }
    if (tid == 0) tma_store_wait_all();
}

int g_num_sms = 0;

}  // namespace

cudaError_t launch_amf(const Plane& p, int smax, uint8_t* fin, size_t fpitch, size_t fslice, cudaStream_t stream) {
    const Geo geo = make_geo(smax);
    const size_t smem = smem_bytes(geo);
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(amf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int out_rows = p.row_end - p.row_begin;
    CUtensorMap tm_src, tm_dst, tm_fin;
    cudaError_t e = make_tmap_u8(&tm_src, p.src, p.cols, p.rows, p.n_slices, p.spitch, p.sslice,
                                 geo.box_w, geo.box_h);
    if (e != cudaSuccess) return e;
    e = make_tmap_u8(&tm_dst, p.dst, p.cols, out_rows, p.n_slices, p.dpitch, p.dslice, TW, TH);
    if (e != cudaSuccess) return e;
    if (fin) {
        e = make_tmap_u8(&tm_fin, fin, p.cols, out_rows, p.n_slices, fpitch, fslice, TW, TH);
        if (e != cudaSuccess) return e;
    } else {
        tm_fin = tm_dst;
    }
    AmfArgs a;
    a.src = p.src;
    a.spitch = p.spitch;
    a.sslice = p.sslice;
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
    a.smax = smax;
    a.tiles_x = (p.cols + TW - 1) / TW;
    a.tiles_y = (out_rows + TH - 1) / TH;
    a.has_fin = fin != nullptr;
    static size_t occ_smem = 0;
    static int per_sm = 1;
    if (occ_smem != smem) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, amf_kernel, NT, smem);
        if (per_sm < 1) per_sm = 1;
        occ_smem = smem;
    }
    const long long ntiles = (long long)a.tiles_x * a.tiles_y * a.n_slices;
    const int grid = (int)std::min<long long>(ntiles, (long long)g_num_sms * per_sm);
    amf_kernel<<<grid, NT, smem, stream>>>(tm_src, tm_dst, tm_fin, a);
    count_launch();
    return cudaGetLastError();
}

}  // namespace hyb
