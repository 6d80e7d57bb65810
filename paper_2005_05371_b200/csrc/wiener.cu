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
#include <cstdint>

#include "hyb_internal.cuh"

namespace hyb {
namespace {

constexpr int TW = 128;
constexpr int TH = 32;
constexpr int NT = 256;
constexpr float kTieEps = 1.0f / 2048.0f;

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
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(wiener_kernel<GAIN>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    const dim3 grid((p.cols + TW - 1) / TW, (p.row_end - p.row_begin + TH - 1) / TH, p.n_slices);
    wiener_kernel<GAIN><<<grid, NT, smem, stream>>>(p, win, wsum, wread, pixel_count);
    count_launch();
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_wiener_stats(const Plane& p, int win, unsigned long long* noise_sum,
                                cudaStream_t stream) {
    return launch<false>(p, win, noise_sum, nullptr, 0, stream);
}

cudaError_t launch_wiener_gain(const Plane& p, int win, const long long* noise_sum,
                               long long pixel_count, cudaStream_t stream) {
    return launch<true>(p, win, nullptr, noise_sum, pixel_count, stream);
}

}  // namespace hyb
