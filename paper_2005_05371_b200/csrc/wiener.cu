// wiener.cu -- W1 local-statistics Wiener filter for sm_100a.
//
// The reference has no local Wiener (its stage-2 slot, proj/src/pipeline.cpp:45-53, runs an
// FFT spectral-subtraction filter).  This file implements the north_star's W1
// (SURVEY.md 8(a)): per pixel S1 = sum f, S2 = sum f^2 over a win x win window (edge
// replication), V = n*S2 - S1^2 exact in integers; the noise estimate is the mean local
// variance nu = W / (n^2 P) with W = sum V (exact int64 -> independent of partitioning);
// y = mu + max(v - nu, 0)/v * (f - mu), rounded half away from zero.
//
// Two launches (nu is global): `stats` (separable box sums in shared memory, warp-shuffle +
// block reduction, one 64-bit atomic per CTA into W) and `gain` (same box sums, then the gain).
// The gain runs in fp32 and falls back to an exact __int128 comparison only when the fp32
// result lies within 2^-11 of a rounding boundary, so the output equals the exact rational
// result bit for bit.
#include <cuda.h>

#include <algorithm>
#include <cstdint>

#include "hyb_internal.cuh"
#include "tma.cuh"
#include "w1_core.cuh"

namespace hyb {
namespace {

constexpr int TW = 128;
constexpr int TH = 32;
constexpr int NT = 256;

struct WGeo {
    int RW;    // window radius
    int NC;    // staged columns = TW + 2 RW
    int FH;    // staged rows = TH + 2 RW
    int FS;    // staged row stride (bytes, multiple of 16)
};

__host__ __device__ inline WGeo make_wgeo(int win) {
    WGeo g;
    g.RW = win / 2;
    g.NC = TW + 2 * g.RW;
    g.FH = TH + 2 * g.RW;
    g.FS = (g.NC + 4 + 15) & ~15;
    return g;
}

__host__ __device__ inline size_t wsmem_bytes(const WGeo& g) {
    size_t b = ((size_t)g.FH * g.FS + 15) & ~(size_t)15;
    b += (size_t)TH * g.NC * 4 * 2;  // column sums S1, S2
    b += 64;                          // reduction scratch
    return b;
}

// wq = floor(W / P): for integer V, V * P <= W  <=>  V <= floor(W / P).
__device__ __forceinline__ uint8_t gain_pixel(int f, int s1, long long v, int n, long long W,
                                              long long wq, long long P, float a_n) {
    if (v <= wq) return (uint8_t)((2 * s1 + n) / (2 * n));  // v <= nu: y = mu
    const int d = n * f - s1;
    const float t = (float)d * a_n / (float)v;                  // D W / (n V P)
    const float h = (float)f - t + 0.5f;
    const float fl = floorf(h);
    const float fr = h - fl;
    int q = (int)fl;
    if (fr < kTieEps || fr > 1.0f - kTieEps) {
        // exact: y >= m - 1/2  <=>  (2 (f - m) + 1) * n V P >= 2 D W
        const int m = fr < 0.5f ? q : q + 1;
        const __int128 Q = (__int128)((long long)n * v) * P;
        const __int128 lhs = (__int128)(2 * (f - m) + 1) * Q;
        const __int128 rhs = (__int128)(2 * (long long)d) * W;
        q = lhs >= rhs ? m : m - 1;
    }
    return (uint8_t)min(max(q, 0), 255);
}

template <bool GAIN>
__global__ void __launch_bounds__(NT) wiener_kernel(Plane p, int win,
                                                    unsigned long long* __restrict__ wsum,
                                                    const long long* __restrict__ wread,
                                                    long long pixel_count) {
    extern __shared__ __align__(16) uint8_t smem[];
    grid_dep_wait();  // f (and the zeroed noise sums) come from the previous grids
    const WGeo geo = make_wgeo(win);
    uint8_t* Ft = smem;
    size_t off = ((size_t)geo.FH * geo.FS + 15) & ~(size_t)15;
    uint32_t* C1 = reinterpret_cast<uint32_t*>(smem + off);
    off += (size_t)TH * geo.NC * 4;
    uint32_t* C2 = reinterpret_cast<uint32_t*>(smem + off);
    off += (size_t)TH * geo.NC * 4;
    unsigned long long* red = reinterpret_cast<unsigned long long*>(smem + off);

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * TW;
    const int y0 = p.row_begin + blockIdx.y * TH;
    const uint8_t* __restrict__ src = p.src + (size_t)blockIdx.z * p.sslice;
    const int rows = p.rows, cols = p.cols;
    const int RW = geo.RW;

    // stage f with clamped coordinates: Ft[rr][cc] = f(clamp(y0-RW+rr), clamp(x0-RW+cc))
    {
        const int words = geo.FS >> 2;
        for (int idx = tid; idx < geo.FH * words; idx += NT) {
            const int rr = idx / words, q = idx - rr * words;
            const int sr = min(max(y0 - RW + rr, 0), rows - 1);
            const uint8_t* srow = src + (size_t)sr * p.spitch;
            const int c = x0 - RW + 4 * q;
            uint32_t w = 0;
            if (c >= 0 && c + 3 < cols) {
                w = (uint32_t)srow[c] | ((uint32_t)srow[c + 1] << 8) | ((uint32_t)srow[c + 2] << 16) |
                    ((uint32_t)srow[c + 3] << 24);
            } else {
#pragma unroll
                for (int b = 0; b < 4; ++b) w |= (uint32_t)srow[min(max(c + b, 0), cols - 1)] << (8 * b);
            }
            reinterpret_cast<uint32_t*>(Ft + (size_t)rr * geo.FS)[q] = w;
        }
    }
    __syncthreads();

    // vertical sums: C[r][cc] = sum_{dr < win} Ft[r + dr][cc], 8 output rows per item
    for (int idx = tid; idx < geo.NC * (TH / 8); idx += NT) {
        const int cc = idx % geo.NC, r0 = (idx / geo.NC) * 8;
        uint32_t s1 = 0, s2 = 0;
        for (int dr = 0; dr < win - 1; ++dr) {
            const uint32_t v = Ft[(size_t)(r0 + dr) * geo.FS + cc];
            s1 += v;
            s2 += v * v;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const uint32_t vin = Ft[(size_t)(r0 + r + win - 1) * geo.FS + cc];
            s1 += vin;
            s2 += vin * vin;
            C1[(r0 + r) * geo.NC + cc] = s1;
            C2[(r0 + r) * geo.NC + cc] = s2;
            const uint32_t vout = Ft[(size_t)(r0 + r) * geo.FS + cc];
            s1 -= vout;
            s2 -= vout * vout;
        }
    }
    __syncthreads();

    // horizontal sums + per-pixel work: thread = row r, 16 columns
    const int r = tid >> 3, c0 = 16 * (tid & 7);
    const int n = win * win;
    const bool row_ok = (y0 + r) < p.row_end;
    const int col_lim = cols - x0;
    const uint32_t* c1 = C1 + r * geo.NC + c0;
    const uint32_t* c2 = C2 + r * geo.NC + c0;
    long long s1 = 0, s2 = 0;
    for (int dc = 0; dc < win - 1; ++dc) {
        s1 += c1[dc];
        s2 += c2[dc];
    }
    unsigned long long vsum = 0;
    long long W = 0, wq = 0;
    float a_n = 0.f;
    if (GAIN) {
        W = wread[blockIdx.z];
        wq = W / pixel_count;
        a_n = (float)((double)W / ((double)pixel_count * (double)n));
    }
    uint32_t outw[4] = {0, 0, 0, 0};
#pragma unroll 4
    for (int j = 0; j < 16; ++j) {
        s1 += c1[j + win - 1];
        s2 += c2[j + win - 1];
        const long long V = (long long)n * s2 - s1 * s1;
        if (!GAIN) {
            if (row_ok && c0 + j < col_lim) vsum += (unsigned long long)V;
        } else {
            const int f = Ft[(size_t)(r + RW) * geo.FS + c0 + j + RW];
            const uint8_t y = gain_pixel(f, (int)s1, V, n, W, wq, pixel_count, a_n);
            outw[j >> 2] |= (uint32_t)y << (8 * (j & 3));
        }
        s1 -= c1[j];
        s2 -= c2[j];
    }

    if (!GAIN) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) vsum += __shfl_down_sync(0xFFFFFFFFu, vsum, d);
        if ((tid & 31) == 0) red[tid >> 5] = vsum;
        __syncthreads();
        if (tid == 0) {
            unsigned long long s = 0;
            for (int w = 0; w < NT / 32; ++w) s += red[w];
            if (s) atomicAdd(wsum + blockIdx.z, s);
        }
    } else if (row_ok) {
        uint8_t* __restrict__ drow = p.dst + (size_t)blockIdx.z * p.dslice +
                                     (size_t)(y0 + r - p.row_begin) * p.dpitch + x0 + c0;
        if (c0 + 16 <= col_lim && ((reinterpret_cast<uintptr_t>(drow) & 15) == 0)) {
            *reinterpret_cast<uint4*>(drow) = make_uint4(outw[0], outw[1], outw[2], outw[3]);
        } else {
            for (int j = 0; j < 16 && c0 + j < col_lim; ++j) drow[j] = (uint8_t)(outw[j >> 2] >> (8 * (j & 3)));
        }
    }
}

template <bool GAIN>
cudaError_t launch(const Plane& p, int win, unsigned long long* wsum, const long long* wread,
                   long long pixel_count, cudaStream_t stream) {
    const WGeo geo = make_wgeo(win);
    const size_t smem = wsmem_bytes(geo);
    static PerDevice attr;
    {
        const cudaError_t e = ensure_smem_attr(attr, (const void*)wiener_kernel<GAIN>, smem);
        if (e != cudaSuccess) return e;
    }
    const dim3 grid((p.cols + TW - 1) / TW, (p.row_end - p.row_begin + TH - 1) / TH, p.n_slices);
    cudaError_t e = launch_pdl(wiener_kernel<GAIN>, dim3(grid), dim3(NT), smem, stream, p, win, wsum, wread,
                               pixel_count);
    if (e != cudaSuccess) return e;
    count_launch();
    return cudaGetLastError();
}


// ------------------------------------------------------------------------------------------
// Fast path for win in {1, 3, 5, 7} (every BASELINE config): warp-autonomous 128 x 32 tiles.
// Each warp owns one tile at a time (TMA box of the tile plus an RW halo into a warp-private
// double-buffered slot), each lane 4 columns.  Per input row a lane forms, for each of its 4
// pixels, the horizontal window sums of f and f^2 with IDP.4A (dp4a) on byte-aligned words,
// and slides them down the tile through an N-deep register ring, so every pixel costs a few
// integer ops; statistics stay exact int32 per pixel.
// ------------------------------------------------------------------------------------------
constexpr int FNW = 8;           // warps per CTA
// Tile rows for images >= 16 MPix (8 below): a tile pays N - 1 prologue rows of box sums, so taller tiles
// amortise them, at the cost of shared memory per warp.  Measured (W1 ms, config 2 = 5x5 / config 4 = 7x7):
// 16 rows 0.168 / 0.667, 24 rows 0.160 / 0.682, 32 rows 0.178 / 0.663.  With the four-pixel sums (w1_core.cuh hsums4):
// 24 rows everywhere 0.146 / 0.617, 32 rows 0.163 / 0.598, the default 0.146 / 0.595; 4 gain CTAs per SM 0.149 / 0.606.
#ifndef HYB_W1_FH
#define HYB_W1_FH(RW) ((RW) <= 2 ? 24 : 16)
#endif
#ifndef HYB_W1_GAIN_MINB
#define HYB_W1_GAIN_MINB 3  // gain CTAs per SM (register budget; 4: config 4 W1 +1.4 %)
#endif
__host__ __device__ constexpr int kFastSmemSlot(int rw, int fh) { return ((FBS * (fh + 2 * rw)) + 127) / 128 * 128; }

struct FastArgs {
    uint8_t* dst;
    size_t dpitch, dslice;
    int rows, cols, row_begin, row_end, n_slices;
    int tiles_x, tiles_y;
    uint32_t mx, ms;           // ceil(2^32 / tiles_x), ceil(2^32 / per_slice): tile index -> coordinates
    unsigned long long* wsum;  // stats
    const long long* wread;    // gain
    long long pixel_count;
    unsigned* mm;              // gain, MM: [0] = min y, [1] = 255 - max y (atomicMin; 0xFFFFFFFF when empty)
};

template <int RW, bool GAIN, int FH, bool MM = false>
__global__ void __launch_bounds__(FNW * 32, GAIN ? HYB_W1_GAIN_MINB : 3) wiener_fast_kernel(const __grid_constant__ CUtensorMap tm,
                                                               const __grid_constant__ FastArgs a) {
    constexpr int SROWS = FH + 2 * RW;
    constexpr int SLOT = kFastSmemSlot(RW, FH);
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem) + 2 * warp;  // 2 per warp
    uint8_t* slots = smem + 128 + (size_t)warp * 2 * SLOT;
    const int per_slice = a.tiles_x * a.tiles_y;
    const int ntiles = per_slice * a.n_slices;
    const int gw = blockIdx.x * FNW + warp, nw = gridDim.x * FNW;  // global warp id / count
    if (gw >= ntiles) return;
    // t / d as a multiply-high by m = min(ceil(2^32 / d), 2^32 - 1) plus a correction step each way
    // (the estimate is off by at most one; d = 1 clamps m); the integer divisions were ~5 % of the W1
    // passes' stall samples at config 4
    auto fdiv = [](uint32_t t, uint32_t d, uint32_t m) {
        uint32_t q = __umulhi(t, m);
        if (q * d > t) --q;
        if ((q + 1) * d <= t) ++q;
        return q;
    };
    auto coords = [&](int t, int& x0, int& y0, int& z) {
        z = a.n_slices == 1 ? 0 : (int)fdiv((uint32_t)t, (uint32_t)per_slice, a.ms);
        const int rem = t - z * per_slice;
        const int by = (int)fdiv((uint32_t)rem, (uint32_t)a.tiles_x, a.mx);
        x0 = (rem - by * a.tiles_x) * FW;
        y0 = a.row_begin + by * FH;
    };
    auto issue = [&](int t, int slot) {
        int x0, y0, z;
        coords(t, x0, y0, z);
        mbar_expect_tx(&bar[slot], FBS * SROWS);
        tma_load_3d(slots + slot * SLOT, &tm, &bar[slot], x0 - FCP, y0 - RW, z);
    };
    grid_dep_wait();  // f (and the zeroed noise sums) come from the previous grids
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
        issue(gw, 0);
        if (gw + nw < ntiles) issue(gw + nw, 1);
    }
    __syncwarp();

    W1Gain kg = {};
    unsigned long long vsum = 0;
    uint32_t ymn = 0xFFFFFFFFu, ymx = 0u;  // MM: byte-SIMD range of the y written by this lane
    int zprev = -1;
    int it = 0;
    for (int t = gw; t < ntiles; t += nw, ++it) {
        const int slot = it & 1;
        mbar_wait_warp(&bar[slot], (uint32_t)(it >> 1) & 1u);
        int x0, y0, z;
        coords(t, x0, y0, z);
        uint8_t* T = slots + slot * SLOT;
        if (GAIN && z != zprev) {  // per-slice noise sums
            kg = w1_gain_consts(a.wread[z], a.pixel_count);
            zprev = z;
        }
        if (!GAIN && z != zprev) {
            if (zprev >= 0) {
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) vsum += __shfl_down_sync(0xFFFFFFFFu, vsum, d);
                if (lane == 0 && vsum) atomicAdd(a.wsum + zprev, vsum);
                vsum = 0;
            }
            zprev = z;
        }

        // ---- border tiles: replicate edges into the zero-filled halo (warp-private slot) ----
        const int sx0 = x0 - FCP, sy0 = y0 - RW;
        if (sx0 < 0 || sx0 + FBS > a.cols || sy0 < 0 || sy0 + SROWS > a.rows)
            replicate_edges<32>(T, FBS, max(0, -sx0), min(FBS, a.cols - sx0), max(0, -sy0),
                                min(SROWS, a.rows - sy0), 0, SROWS, RW);

        const int col_lim = a.cols - x0, row_lim = a.row_end - y0;
        if (!GAIN) {
            vsum += (unsigned long long)w1_tile_stats<RW, FH>(T, x0, y0, a.rows, a.cols, a.row_begin, a.row_end);
        } else {
            w1_tile_gain<RW, FH, MM>(T, x0, col_lim, row_lim, kg,
                                     a.dst + (size_t)z * a.dslice + (size_t)(y0 - a.row_begin) * a.dpitch + x0,
                                     a.dpitch, &ymn, &ymx);
        }
        __syncwarp();
        // refill this slot with the warp's tile after next
        if (lane == 0 && t + 2 * nw < ntiles) {
            fence_proxy_async_smem();
            issue(t + 2 * nw, slot);
        }
    }
    if (!GAIN && zprev >= 0) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) vsum += __shfl_down_sync(0xFFFFFFFFu, vsum, d);
        if (lane == 0 && vsum) atomicAdd(a.wsum + zprev, vsum);
    }
    if (MM) {  // the warp's y range -> the image range (one min atomic each for lo and 255 - hi)
        uint32_t lo = min(min(ymn & 0xFFu, (ymn >> 8) & 0xFFu), min((ymn >> 16) & 0xFFu, ymn >> 24));
        uint32_t hi = max(max(ymx & 0xFFu, (ymx >> 8) & 0xFFu), max((ymx >> 16) & 0xFFu, ymx >> 24));
        lo = __reduce_min_sync(0xFFFFFFFFu, lo);
        hi = __reduce_max_sync(0xFFFFFFFFu, hi);
        if (lane == 0 && lo <= hi) {
            atomicMin(&a.mm[0], lo);
            atomicMin(&a.mm[1], 255u - hi);
        }
    }
}

template <int RW, bool GAIN, int FH, bool MM = false>
cudaError_t launch_fast(const Plane& p, unsigned long long* wsum, const long long* wread, long long pixel_count,
                        cudaStream_t stream, unsigned* mm = nullptr) {
    constexpr int SLOT = kFastSmemSlot(RW, FH);
    constexpr size_t smem = 128 + (size_t)FNW * 2 * SLOT + 128;
    static PerDevice attr, occ;
    {
        const cudaError_t e = ensure_smem_attr(attr, (const void*)wiener_fast_kernel<RW, GAIN, FH, MM>, smem);
        if (e != cudaSuccess) return e;
    }
    CUtensorMap tm;
    cudaError_t e = make_tmap_u8(&tm, p.src, p.cols, p.rows, p.n_slices, p.spitch, p.sslice, FBS, FH + 2 * RW);
    if (e != cudaSuccess) return e;
    FastArgs a;
    a.dst = p.dst;
    a.dpitch = p.dpitch;
    a.dslice = p.dslice;
    a.rows = p.rows;
    a.cols = p.cols;
    a.row_begin = p.row_begin;
    a.row_end = p.row_end;
    a.n_slices = p.n_slices;
    a.tiles_x = (p.cols + FW - 1) / FW;
    a.tiles_y = (p.row_end - p.row_begin + FH - 1) / FH;
    {
        auto magic = [](unsigned long long d) {
            return (uint32_t)std::min<unsigned long long>(((1ull << 32) + d - 1) / d, 0xFFFFFFFFull);
        };
        a.mx = magic((unsigned long long)a.tiles_x);
        a.ms = magic((unsigned long long)a.tiles_x * a.tiles_y);
    }
    a.wsum = wsum;
    a.wread = wread;
    a.pixel_count = pixel_count;
    a.mm = mm;
    const int per_sm = occupancy(occ, (const void*)wiener_fast_kernel<RW, GAIN, FH, MM>, FNW * 32, smem);
    const long long ntiles = (long long)a.tiles_x * a.tiles_y * a.n_slices;
    const long long warps = std::min<long long>(ntiles, (long long)device_sms() * per_sm * FNW);
    const int grid = (int)((warps + FNW - 1) / FNW);
    const cudaError_t le =
        launch_pdl(wiener_fast_kernel<RW, GAIN, FH, MM>, dim3(grid), dim3(FNW * 32), smem, stream, tm, a);
    if (le != cudaSuccess) return le;
    count_launch();
    return cudaGetLastError();
}

template <bool GAIN>
cudaError_t dispatch(const Plane& p, int win, unsigned long long* wsum, const long long* wread,
                     long long pixel_count, cudaStream_t stream, unsigned* mm = nullptr) {
    if (tma_compatible(p.src, p.spitch, p.sslice)) {
        const long long px = (long long)(p.row_end - p.row_begin) * p.cols * p.n_slices;
        const bool small = px < (16ll << 20);
        // small images: 8-row tiles, twice the warps in flight and half the per-warp chain
#define HYB_FAST(RW)                                                                                          \
    if constexpr (GAIN) {                                                                                     \
        if (mm)                                                                                               \
            return small ? launch_fast<RW, true, 8, true>(p, wsum, wread, pixel_count, stream, mm)           \
                         : launch_fast<RW, true, HYB_W1_FH(RW), true>(p, wsum, wread, pixel_count, stream, mm); \
    }                                                                                                         \
    return small ? launch_fast<RW, GAIN, 8>(p, wsum, wread, pixel_count, stream)                              \
                 : launch_fast<RW, GAIN, HYB_W1_FH(RW)>(p, wsum, wread, pixel_count, stream);
        switch (win) {
            case 1: HYB_FAST(0)
            case 3: HYB_FAST(1)
            case 5: HYB_FAST(2)
            case 7: HYB_FAST(3)
            default: break;
        }
#undef HYB_FAST
    }
    cudaError_t e = launch<GAIN>(p, win, wsum, wread, pixel_count, stream);
    if (e != cudaSuccess || !GAIN || !mm) return e;
    // generic gain: the range of the rows it wrote by a separate pass (same result, one more read)
    for (int z = 0; z < p.n_slices && e == cudaSuccess; ++z)
        e = launch_stretch_minmax(p.dst + (size_t)z * p.dslice, p.dpitch, p.row_end - p.row_begin, p.cols, mm, stream);
    return e;
}

}  // namespace

cudaError_t launch_wiener_stats(const Plane& p, int win, unsigned long long* noise_sum,
                                cudaStream_t stream) {
    return dispatch<false>(p, win, noise_sum, nullptr, 0, stream);
}

cudaError_t launch_wiener_gain(const Plane& p, int win, const long long* noise_sum,
                               long long pixel_count, cudaStream_t stream, unsigned* mm) {
    return dispatch<true>(p, win, nullptr, noise_sum, pixel_count, stream, mm);
}

}  // namespace hyb
