// amf.cu -- adaptive median filter (AMF) for sm_100a.
//
// Semantics: detail::adaptive_median_rows, reference proj/src/adaptive_median.cpp:123-215
// (windows k = 3..smax over the pristine input, edge replication, level A/B, unresolved
// pixels keep their input).  Design:
//
//   * one CTA per 128 x 32 output tile; the tile plus a halo of R = (smax-1)/2 pixels is
//     staged once in shared memory with coordinates clamped to the source bounds, so every
//     later window (any k <= smax) reads on-chip data and edge replication is free;
//   * k = 3 (95-99.7% of pixels finalise here) runs on every pixel with u16x2 SIMD: the
//     tile is re-laid out as row PAIRS (word = pixel(r,c) | pixel(r+1,c) << 16) so one
//     VIMNMX3.U16x2 serves two output rows; each thread owns 2 rows x 8 columns and sorts
//     each 3-tall column once (min3 / max3 / xor-median), reusing it for 3 outputs;
//   * pixels failing level A are compacted into a per-CTA shared-memory work queue
//     (warp ballot + scan, one shared atomic per warp); each growth level k = 5..smax then
//     processes only the queue, warp-uniformly, and re-queues its survivors;
//   * growth levels test level A with counts instead of a median: zmin < zmed < zmax
//     <=> #(v == zmin) <= m and #(v == zmax) <= m (m = (k^2-1)/2), computed with SWAR
//     zero-byte counting on 4 pixels per 32-bit word; the median itself (needed only when
//     level A passes and g is an extreme) comes from an 8-step bitwise radix select.
#include <cstdint>

#include "hyb_internal.cuh"

namespace hyb {
namespace {

constexpr int TW = 128;  // tile columns
constexpr int TH = 32;   // tile rows
constexpr int NT = 256;  // threads per CTA
constexpr int PS = TW + 4;  // pair-tile row stride (words)
constexpr int MAX_LEVELS = 128;

struct Geo {
    int R;   // halo radius of the byte tile
    int CP;  // column pad of the byte tile (>= R, == 1 mod 4 so pair words align)
    int BH;  // byte-tile rows
    int BS;  // byte-tile row stride in bytes (multiple of 16)
};

__host__ __device__ inline Geo make_geo(int smax) {
    Geo g;
    g.R = (smax - 1) / 2;
    int cp = g.R < 1 ? 1 : g.R;
    while ((cp & 3) != 1) ++cp;
    g.CP = cp;
    g.BH = TH + 2 * g.R;
    g.BS = ((TW + 2 * cp + 4) + 15) & ~15;
    return g;
}

__host__ __device__ inline size_t smem_bytes(const Geo& g) {
    size_t b = (size_t)g.BH * g.BS;           // byte tile
    b = (b + 15) & ~(size_t)15;
    b += (size_t)(TH + 2) * PS * 4;           // pair tile (aliased by queue 1 after k = 3)
    b += (size_t)TH * TW;                     // output tile
    b += (size_t)TH * TW;                     // finalized_at tile
    b += (size_t)TH * TW * 2;                 // queue 0
    b += MAX_LEVELS * 4;                      // per-level queue counters
    return b;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
    return __byte_perm(a, b, s);
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
                                         : (TAIL == 1 ? 0x00000080u
                                                      : (TAIL == 2 ? 0x00008080u : 0x00808080u));
    }
};

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

// Element of rank `rank` (0-based) of the window: bitwise radix select.  All values lie in
// [lo, hi], so the bits above the highest bit where lo and hi differ are fixed.
template <int K>
__device__ __forceinline__ uint32_t select_rank(const uint32_t (&a)[K][Win<K>::AW], int rank,
                                                uint32_t lo, uint32_t hi) {
    const int hb = 31 - __clz(lo ^ hi);  // lo != hi whenever this is called
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

// One growth level with a compile-time window size.  Returns true when the pixel is
// finalised (and writes its output), false to re-queue it.
template <int K>
__device__ __forceinline__ bool level_fixed(const uint8_t* __restrict__ B, const Geo& geo, int ty,
                                            int tx, uint8_t* out) {
    using W = Win<K>;
    const int start = tx + geo.CP - W::RK;
    const int sh = 8 * (start & 3);
    const uint32_t* rowp =
        reinterpret_cast<const uint32_t*>(B + (size_t)(ty + geo.R - W::RK) * geo.BS) + (start >> 2);
    uint32_t a[K][W::AW];
#pragma unroll
    for (int r = 0; r < K; ++r) {
        uint32_t raw[W::NRAW];
#pragma unroll
        for (int j = 0; j < W::NRAW; ++j) raw[j] = rowp[r * (geo.BS >> 2) + j];
#pragma unroll
        for (int j = 0; j < W::AW; ++j)
            a[r][j] = __funnelshift_r(raw[j], (j + 1 < W::NRAW) ? raw[j + 1] : 0u, sh);
    }
    // zmin / zmax with u16x2 lanes (duplicated bytes cannot change a min or max).
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
    if (count_eq<K>(a, zmin) > W::M || count_eq<K>(a, zmax) > W::M) return false;  // level A fails
    const uint32_t g = B[(size_t)(ty + geo.R) * geo.BS + tx + geo.CP];
    *out = (uint8_t)((g != zmin && g != zmax) ? g : select_rank<K>(a, W::M, zmin, zmax));
    return true;
}

// Growth level for window sizes beyond the compile-time set (k > 11): same algorithm on
// bytes read straight from the shared tile.
__device__ bool level_generic(const uint8_t* __restrict__ B, const Geo& geo, int ty, int tx, int k,
                              uint8_t* out) {
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

__global__ void __launch_bounds__(NT) amf_kernel(Plane p, int smax, uint8_t* __restrict__ fin,
                                                 size_t fpitch, size_t fslice) {
    extern __shared__ __align__(16) uint8_t smem[];
    const Geo geo = make_geo(smax);
    uint8_t* B = smem;
    size_t off = ((size_t)geo.BH * geo.BS + 15) & ~(size_t)15;
    uint32_t* PR = reinterpret_cast<uint32_t*>(smem + off);
    uint16_t* Q1 = reinterpret_cast<uint16_t*>(smem + off);  // aliases PR after k = 3
    off += (size_t)(TH + 2) * PS * 4;
    uint8_t* O = smem + off;
    off += TH * TW;
    uint8_t* F = smem + off;
    off += TH * TW;
    uint16_t* Q0 = reinterpret_cast<uint16_t*>(smem + off);
    off += TH * TW * 2;
    int* qcount = reinterpret_cast<int*>(smem + off);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int x0 = blockIdx.x * TW;
    const int y0 = p.row_begin + blockIdx.y * TH;  // source row of tile row 0
    const uint8_t* __restrict__ src = p.src + (size_t)blockIdx.z * p.sslice;
    const int rows = p.rows, cols = p.cols;

    if (tid < MAX_LEVELS) qcount[tid] = 0;

    // ---- stage the clamped byte tile: B[rr][cc] = src(clamp(y0-R+rr), clamp(x0-CP+cc)) ----
    {
        const int words = geo.BS >> 2;
        const bool interior_x = (x0 - geo.CP >= 0) && (x0 - geo.CP + geo.BS <= cols);
        for (int idx = tid; idx < geo.BH * words; idx += NT) {
            const int rr = idx / words, q = idx - rr * words;
            const int sr = min(max(y0 - geo.R + rr, 0), rows - 1);
            const uint8_t* srow = src + (size_t)sr * p.spitch;
            const int c = x0 - geo.CP + 4 * q;
            uint32_t w;
            if (interior_x) {
                w = (uint32_t)srow[c] | ((uint32_t)srow[c + 1] << 8) | ((uint32_t)srow[c + 2] << 16) |
                    ((uint32_t)srow[c + 3] << 24);
            } else {
                w = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    w |= (uint32_t)srow[min(max(c + b, 0), cols - 1)] << (8 * b);
            }
            reinterpret_cast<uint32_t*>(B + (size_t)rr * geo.BS)[q] = w;
        }
    }
    __syncthreads();

    // ---- row-pair tile: PR[pr][cc'] = (t(pr-1, cc'-1), t(pr, cc'-1)) in tile coordinates ----
    {
        constexpr int PW4 = PS / 4;
        for (int idx = tid; idx < (TH + 1) * PW4; idx += NT) {
            const int pr = idx / PW4, q = idx - pr * PW4;
            const int boff = 4 * q - 1 + geo.CP;  // multiple of 4
            const uint32_t a = *reinterpret_cast<const uint32_t*>(B + (size_t)(pr - 1 + geo.R) * geo.BS + boff);
            const uint32_t b = *reinterpret_cast<const uint32_t*>(B + (size_t)(pr + geo.R) * geo.BS + boff);
            const uint32_t x = prmt(a, b, 0x5140), y = prmt(a, b, 0x7362);
            uint4 v;
            v.x = prmt(x, 0, 0x4140);
            v.y = prmt(x, 0, 0x4342);
            v.z = prmt(y, 0, 0x4140);
            v.w = prmt(y, 0, 0x4342);
            *reinterpret_cast<uint4*>(PR + (size_t)pr * PS + 4 * q) = v;
        }
    }
    __syncthreads();

    // ---- k = 3 on every pixel: thread = rows (r0, r0+1) x columns c0..c0+7 ----
    const int r0 = 2 * (tid >> 4), c0 = 8 * (tid & 15);
    const int row_lim = p.row_end - y0;  // tile rows < row_lim are in range
    const int col_lim = cols - x0;
    uint32_t fail_mask = 0;
    {
        uint32_t lo[10], hi[10], mid[10], gm[10];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const uint4* rp = reinterpret_cast<const uint4*>(PR + (size_t)(r0 + j) * PS + c0);
            uint32_t w[12];
#pragma unroll
            for (int v = 0; v < 3; ++v) {
                const uint4 t = rp[v];
                w[4 * v] = t.x;
                w[4 * v + 1] = t.y;
                w[4 * v + 2] = t.z;
                w[4 * v + 3] = t.w;
            }
#pragma unroll
            for (int i = 0; i < 10; ++i) {
                if (j == 0) {
                    lo[i] = w[i];
                    hi[i] = w[i];
                    mid[i] = w[i];
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
            const uint32_t okA = __vminu2(__vminu2(zmed - zmin, zmax - zmed), 0x00010001u);
            const uint32_t gext = 0x00010001u - __vminu2(__vminu2(g - zmin, zmax - g), 0x00010001u);
            const uint32_t sel = (okA & gext) * 0xFFFFu;
            o[j] = (zmed & sel) | (g & ~sel);
            fz[j] = okA * 3u;
            const uint32_t fl = okA ^ 0x00010001u;  // 1 in lanes that fail level A
            fail_mask |= ((fl & 1u) << (2 * j)) | ((fl >> 16) << (2 * j + 1));
        }
        // lanes outside the output range never enter the queue
        uint32_t valid = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const bool cv = c0 + j < col_lim;
            valid |= (uint32_t)(cv && r0 < row_lim) << (2 * j);
            valid |= (uint32_t)(cv && r0 + 1 < row_lim) << (2 * j + 1);
        }
        fail_mask &= valid;
        // pack rows r0 (u16 lane 0) and r0+1 (lane 1) back to bytes
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
    __syncthreads();  // qcount init visible; PR dead from here on (Q1 aliases it)

    // ---- compact level-A failures into queue 0 (warp scan + one shared atomic per warp) ----
    {
        const int nf = __popc(fail_mask);
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
        uint32_t m = fail_mask;
        while (m) {
            const int bit = __ffs(m) - 1;
            m &= m - 1;
            const int j = bit >> 1, rr = r0 + (bit & 1);
            Q0[pos++] = (uint16_t)(rr * TW + c0 + j);
        }
    }

    // ---- growth levels k = 5..smax over the compacted queue ----
    int lvl = 0;
    for (int k = 5; k <= smax; k += 2, ++lvl) {
        __syncthreads();
        const int n = qcount[lvl];
        if (n == 0) break;
        const uint16_t* qin = (lvl & 1) ? Q1 : Q0;
        uint16_t* qout = (lvl & 1) ? Q0 : Q1;
        for (int base = warp * 32; base < n; base += NT) {
            const int i = base + lane;
            bool keep = false;
            int pix = 0;
            if (i < n) {
                pix = qin[i];
                const int ty = pix / TW, tx = pix - (pix / TW) * TW;
                uint8_t o = 0;
                bool done;
                switch (k) {
                    case 5: done = level_fixed<5>(B, geo, ty, tx, &o); break;
                    case 7: done = level_fixed<7>(B, geo, ty, tx, &o); break;
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
    __syncthreads();

    // ---- write the output (and finalized_at) tile ----
    uint8_t* __restrict__ dst = p.dst + (size_t)blockIdx.z * p.dslice;
    const int rl = min(TH, row_lim), cl = min(TW, col_lim);
    const int orow0 = y0 - p.row_begin;
    const bool vec = ((p.dpitch & 15) == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
    for (int idx = tid; idx < TH * (TW / 16); idx += NT) {
        const int r = idx >> 3, q = idx & 7;
        if (r >= rl) continue;
        uint8_t* drow = dst + (size_t)(orow0 + r) * p.dpitch + x0;
        const uint8_t* orow = O + (size_t)r * TW;
        if (vec && 16 * q + 16 <= cl) {
            *reinterpret_cast<uint4*>(drow + 16 * q) = *reinterpret_cast<const uint4*>(orow + 16 * q);
        } else {
            for (int c = 16 * q; c < min(16 * q + 16, cl); ++c) drow[c] = orow[c];
        }
    }
    if (fin) {
        uint8_t* fbase = fin + (size_t)blockIdx.z * fslice;
        for (int idx = tid; idx < TH * TW; idx += NT) {
            const int r = idx / TW, c = idx - (idx / TW) * TW;
            if (r < rl && c < cl) fbase[(size_t)(orow0 + r) * fpitch + x0 + c] = F[idx];
        }
    }
}

}  // namespace

cudaError_t launch_amf(const Plane& p, int smax, uint8_t* fin, size_t fpitch, size_t fslice,
                       cudaStream_t stream) {
    const Geo geo = make_geo(smax);
    const size_t smem = smem_bytes(geo);
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e =
            cudaFuncSetAttribute(amf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    const dim3 grid((p.cols + TW - 1) / TW, (p.row_end - p.row_begin + TH - 1) / TH, p.n_slices);
    amf_kernel<<<grid, NT, smem, stream>>>(p, smax, fin, fpitch, fslice);
    count_launch();
    return cudaGetLastError();
}

size_t amf_smem_bytes(int smax) { return smem_bytes(make_geo(smax)); }

}  // namespace hyb
