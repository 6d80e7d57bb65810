// w1_core.cuh -- W1 local-statistics Wiener tile bodies shared by the W1 kernels (wiener.cu) and the
// fused small-image kernel (small.cu).  Reference: the Wiener slot of proj/src/pipeline.cpp:45-53 with
// the W1 estimator of SURVEY.md 8 (oracle/hyb_oracle.c restates it); see wiener.cu for the derivation.
//
// A tile is FW = 128 columns x FH rows; its staged bytes T hold FH + 2 RW rows (image rows
// y0 - RW ..) of FBS = 160 bytes (image column x0 at byte FCP), edges already replicated.  One warp
// per tile, 4 columns per lane.
#pragma once
#include <cstdint>

namespace hyb {
namespace {

constexpr float kTieEps = 1.0f / 2048.0f;
constexpr int FW = 128;            // tile columns
constexpr int FCP = 16;            // column pad (TMA box x offsets must be 16-byte aligned)
constexpr int FBS = FW + 2 * FCP;  // staged row bytes (160)

// 4 bytes starting at byte S of the 12-byte window [w0 w1 w2] (S compile-time, 0..11).
template <int S>
__device__ __forceinline__ uint32_t bytes4(uint32_t w0, uint32_t w1, uint32_t w2) {
    if constexpr (S == 0) return w0;
    else if constexpr (S == 4) return w1;
    else if constexpr (S == 8) return w2;
    else if constexpr (S < 4) return __funnelshift_r(w0, w1, 8 * S);
    else if constexpr (S < 8) return __funnelshift_r(w1, w2, 8 * (S - 4));
    else return w2 >> (8 * (S - 8));  // only the low 12 - S bytes are meaningful
}

// Horizontal window sums (f, f^2) of pixel I (0..3) of the lane's 4 columns.
template <int RW, int I>
__device__ __forceinline__ void hsums(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t& h1, uint32_t& h2) {
    constexpr int N = 2 * RW + 1;
    constexpr int S = 4 + I - RW;  // first window byte in [w0 w1 w2] (w1 = the lane's own word)
    if (N == 1) {
        const uint32_t x = (bytes4<S>(w0, w1, w2)) & 0xFFu;
        h1 = x;
        h2 = x * x;
    } else if (N == 3) {
        const uint32_t x = bytes4<S>(w0, w1, w2) & 0x00FFFFFFu;
        h1 = __dp4a(x, 0x01010101u, 0u);
        h2 = __dp4a(x, x, 0u);
    } else {
        const uint32_t lo = bytes4<S>(w0, w1, w2);
        constexpr uint32_t hm = N == 5 ? 0x000000FFu : 0x00FFFFFFu;
        const uint32_t hi = bytes4<S + 4>(w0, w1, w2) & hm;
        h1 = __dp4a(hi, 0x01010101u, __dp4a(lo, 0x01010101u, 0u));
        h2 = __dp4a(hi, hi, __dp4a(lo, lo, 0u));
    }
}

// Horizontal window sum of f only (statistics pass); window bytes beyond N get weight 0.
template <int RW, int I>
__device__ __forceinline__ uint32_t hsum1(uint32_t w0, uint32_t w1, uint32_t w2) {
    constexpr int N = 2 * RW + 1;
    constexpr int S = 4 + I - RW;
    if (N == 1) return bytes4<S>(w0, w1, w2) & 0xFFu;
    if (N == 3) return __dp4a(bytes4<S>(w0, w1, w2), 0x00010101u, 0u);
    constexpr uint32_t hw = N == 5 ? 0x00000001u : 0x00010101u;
    return __dp4a(bytes4<S + 4>(w0, w1, w2), hw, __dp4a(bytes4<S>(w0, w1, w2), 0x01010101u, 0u));
}

// Horizontal window sums of the lane's 4 pixels at once.  5 x 5 and 7 x 7 windows: the sums of the two
// pixels whose windows are made of whole words (plus masked neighbour words) come from dp4a, the other two
// follow by adding the byte that enters and subtracting the byte that leaves (squares on the FMA pipe):
// 6 (7 x 7) / 2 (5 x 5) dp4a per row instead of 16 -- the dp4a issue rate bounded the gain pass.
__device__ __forceinline__ uint32_t byte_of(uint32_t w, int i) { return (w >> (8 * i)) & 0xFFu; }
#ifndef HYB_W1_LOWDP
#define HYB_W1_LOWDP 0  // 1: 7 x 7 edge sums from single bytes too (2 dp4a per row): measured slower, config 4 W1 0.618 vs 0.594 ms
#endif

template <int RW>
__device__ __forceinline__ void hsums4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t (&h1)[4], uint32_t (&h2)[4]) {
    if constexpr (RW == 3) {
        // windows: bytes 1..7, 2..8, 3..9, 4..10 of [w0 w1 w2]
        const uint32_t m1 = __dp4a(w1, 0x01010101u, 0u), m2 = __dp4a(w1, w1, 0u);
        const uint32_t b1 = byte_of(w0, 1), b3 = byte_of(w0, 3), b8 = byte_of(w2, 0), b10 = byte_of(w2, 2);
#if HYB_W1_LOWDP
        const uint32_t b2 = byte_of(w0, 2), b9 = byte_of(w2, 1);
        h1[0] = m1 + b1 + b2 + b3;
        h1[3] = m1 + b8 + b9 + b10;
        h2[0] = m2 + b1 * b1 + b2 * b2 + b3 * b3;
        h2[3] = m2 + b8 * b8 + b9 * b9 + b10 * b10;
#else
        const uint32_t l = w0 & 0xFFFFFF00u, r = w2 & 0x00FFFFFFu;
        h1[0] = __dp4a(l, 0x01010101u, m1);
        h1[3] = __dp4a(r, 0x01010101u, m1);
        h2[0] = __dp4a(l, l, m2);
        h2[3] = __dp4a(r, r, m2);
#endif
        h1[1] = h1[0] - b1 + b8;
        h1[2] = h1[3] + b3 - b10;
        h2[1] = h2[0] - b1 * b1 + b8 * b8;
        h2[2] = h2[3] + b3 * b3 - b10 * b10;
    } else if constexpr (RW == 2) {
        // windows: bytes 2..6, 3..7, 4..8, 5..9
        const uint32_t m1 = __dp4a(w1, 0x01010101u, 0u), m2 = __dp4a(w1, w1, 0u);
        const uint32_t b2 = byte_of(w0, 2), b3 = byte_of(w0, 3), b4 = byte_of(w1, 0), b7 = byte_of(w1, 3);
        const uint32_t b8 = byte_of(w2, 0), b9 = byte_of(w2, 1);
        h1[1] = m1 + b3;
        h1[2] = m1 + b8;
        h1[0] = h1[1] + b2 - b7;
        h1[3] = h1[2] + b9 - b4;
        h2[1] = m2 + b3 * b3;
        h2[2] = m2 + b8 * b8;
        h2[0] = h2[1] + b2 * b2 - b7 * b7;
        h2[3] = h2[2] + b9 * b9 - b4 * b4;
    } else {
        hsums<RW, 0>(w0, w1, w2, h1[0], h2[0]);
        hsums<RW, 1>(w0, w1, w2, h1[1], h2[1]);
        hsums<RW, 2>(w0, w1, w2, h1[2], h2[2]);
        hsums<RW, 3>(w0, w1, w2, h1[3], h2[3]);
    }
}

// The same for the sums of f only (statistics pass).
template <int RW>
__device__ __forceinline__ void hsum1x4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t (&h)[4]) {
    if constexpr (RW == 3) {
        const uint32_t m1 = __dp4a(w1, 0x01010101u, 0u);
        h[0] = __dp4a(w0 & 0xFFFFFF00u, 0x01010101u, m1);
        h[3] = __dp4a(w2 & 0x00FFFFFFu, 0x01010101u, m1);
        h[1] = h[0] - byte_of(w0, 1) + byte_of(w2, 0);
        h[2] = h[3] + byte_of(w0, 3) - byte_of(w2, 2);
    } else if constexpr (RW == 2) {
        const uint32_t m1 = __dp4a(w1, 0x01010101u, 0u);
        h[1] = m1 + byte_of(w0, 3);
        h[2] = m1 + byte_of(w2, 0);
        h[0] = h[1] + byte_of(w0, 2) - byte_of(w1, 3);
        h[3] = h[2] + byte_of(w2, 1) - byte_of(w1, 0);
    } else {
        h[0] = hsum1<RW, 0>(w0, w1, w2);
        h[1] = hsum1<RW, 1>(w0, w1, w2);
        h[2] = hsum1<RW, 2>(w0, w1, w2);
        h[3] = hsum1<RW, 3>(w0, w1, w2);
    }
}

// Number of (output position p in [lo, hi), offset d in [-RW, RW]) pairs whose clamped coordinate
// clamp(p + d, 0, n - 1) equals r: how many output windows cover row (or column) r.
__device__ __forceinline__ int win_count(int r, int lo, int hi, int n, int RW) {
    int cnt = 0;
    for (int d = -RW; d <= RW; ++d) {
        int plo, phi;
        if (n == 1) {
            plo = lo;
            phi = hi - 1;
        } else if (r == 0) {
            plo = lo;
            phi = -d;
        } else if (r == n - 1) {
            plo = n - 1 - d;
            phi = hi - 1;
        } else {
            plo = phi = r - d;
        }
        plo = max(plo, lo);
        phi = min(phi, hi - 1);
        cnt += max(0, phi - plo + 1);
    }
    return cnt;
}

// Packed f32x2 arithmetic (FFMA2 / FADD2 on sm_100a): two pixels per instruction.
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ uint64_t f2splat(float a) { return f2pack(a, a); }
__device__ __forceinline__ void f2unpack(uint64_t v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t fadd2_rd(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

// Statistics of one tile: this lane's share of n * sum S2 - sum S1^2 over the tile's output pixels
// (two's complement; the warp / grid sum is W).  FAST: the tile's rows and the lane's columns are all
// interior (every f^2 of the tile's output rows is covered by n windows, no image or range border
// within reach), so the coverage-weighted sum is n^2 times a plain 32-bit sum of f^2 over the output
// rows -- no per-row window counts (they were a quarter of this pass's instructions).
template <int RW, int FH, bool FAST>
__device__ __forceinline__ long long w1_tile_stats_body(const uint8_t* __restrict__ T, int x0, int y0, int rows,
                                                        int cols, int row_begin, int row_end, const uint32_t (&wc)[4],
                                                        bool wc_full) {
    constexpr int N = 2 * RW + 1;
    constexpr int NN = N * N;
    constexpr int SROWS = FH + 2 * RW;
    const int lane = threadIdx.x & 31;
    const int c = 4 * lane;
    const int col_lim = cols - x0, row_lim = row_end - y0;
    const uint32_t* base = reinterpret_cast<const uint32_t*>(T + FCP + c - 4);
    const int own_lo = (y0 == row_begin) ? max(0, row_begin - RW) : y0;
    const int own_hi = (y0 + FH >= row_end) ? min(rows, row_end + RW) : y0 + FH;
    uint32_t r1[N][4], s1[4] = {0, 0, 0, 0};
    long long tile_sq = 0, tile_s1sq = 0;
    uint32_t sq32 = 0;  // FAST: sum of f^2 over the output rows (<= 16 * 4 * 255^2)
    auto take_row = [&](int rr, uint32_t (&h)[4]) {
        const uint32_t* rp = base + rr * (FBS / 4);
        const uint32_t w0 = rp[0], w1 = rp[1], w2 = rp[2];
        hsum1x4<RW>(w0, w1, w2, h);
        if constexpr (FAST) {
            if (rr >= RW && rr < RW + FH) sq32 = __dp4a(w1, w1, sq32);
        } else {
            const int r = y0 - RW + rr;  // image row of this tile row
            if (r >= own_lo && r < own_hi) {
                const bool interior = r - RW >= max(row_begin, 0) && r + RW < min(row_end, rows);
                const uint32_t wr = interior ? (uint32_t)N : (uint32_t)win_count(r, row_begin, row_end, rows, RW);
                uint32_t q;
                if (wc_full) {
                    q = (uint32_t)N * __dp4a(w1, w1, 0u);
                } else {
                    q = 0;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t f = (w1 >> (8 * i)) & 0xFFu;
                        q += wc[i] * f * f;
                    }
                }
                tile_sq += (long long)wr * q;
            }
        }
    };
#pragma unroll
    for (int rr = 0; rr < N - 1; ++rr) {
        take_row(rr, r1[rr]);
#pragma unroll
        for (int i = 0; i < 4; ++i) s1[i] += r1[rr][i];
    }
#pragma unroll 1
    for (int yg = 0; yg < FH; yg += N) {
#pragma unroll
        for (int u = 0; u < N; ++u) {
            const int y = yg + u;
            if (y >= FH) break;
            uint32_t h[4];
            take_row(y + N - 1, h);
            uint32_t sq4 = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                s1[i] += h[i];
                r1[(u + N - 1) % N][i] = h[i];
                if (FAST || c + i < col_lim) sq4 += s1[i] * s1[i];  // <= 4 * 12495^2 < 2^32
            }
            if (FAST || y < row_lim) tile_s1sq += sq4;
#pragma unroll
            for (int i = 0; i < 4; ++i) s1[i] -= r1[u][i];
        }
    }
    if constexpr (FAST) return (long long)NN * NN * sq32 - tile_s1sq;
    // the last rows of the tile box (below the window of the last output row) hold halo f^2
#pragma unroll
    for (int rr = FH + N - 1; rr < SROWS; ++rr) {
        uint32_t h[4];
        take_row(rr, h);
    }
    return (long long)NN * tile_sq - tile_s1sq;
}

template <int RW, int FH>
__device__ __forceinline__ long long w1_tile_stats(const uint8_t* __restrict__ T, int x0, int y0, int rows, int cols,
                                                   int row_begin, int row_end) {
    constexpr int N = 2 * RW + 1;
    // ---- statistics: W = n * sum_p S2(p) - sum_p S1(p)^2 with sum_p S2(p) = sum_q f(q)^2 WR(q_r) WC(q_c)
    // (WR / WC = how many output windows cover a row / column, clamping included), so only S1
    // needs a per-pixel box sum.  Each image pixel's f^2 is owned by exactly one tile: its output
    // rows, plus the RW halo rows outside the output range for the first / last tile.
    const int c = 4 * (threadIdx.x & 31);
    uint32_t wc[4];
    bool wc_full = true;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int cc = x0 + c + i;
        wc[i] = cc < cols ? (uint32_t)win_count(cc, 0, cols, cols, RW) : 0u;
        wc_full &= wc[i] == (uint32_t)N;
    }
    // rows: output rows y0 .. y0 + FH - 1 all in range and all RW away from the image and range borders
    const bool rows_interior = y0 - RW >= max(row_begin, 0) && y0 + FH - 1 + RW < min(row_end, rows) &&
                               y0 != row_begin && y0 + FH < row_end;
    if (__all_sync(0xFFFFFFFFu, wc_full) && rows_interior)
        return w1_tile_stats_body<RW, FH, true>(T, x0, y0, rows, cols, row_begin, row_end, wc, true);
    return w1_tile_stats_body<RW, FH, false>(T, x0, y0, rows, cols, row_begin, row_end, wc, wc_full);
}

// Gain constants of one image: W = sum of V, wq32 = min(floor(W / P), 2^31 - 1), kq = W / P.
struct W1Gain {
    long long W;
    long long pixel_count;
    int wq32;
    float kq;
};

__device__ __forceinline__ W1Gain w1_gain_consts(long long W, long long pixel_count) {
    W1Gain k;
    k.W = W;
    k.pixel_count = pixel_count;
    const long long wq = W / pixel_count;
    k.wq32 = wq > 0x7FFFFFFFll ? 0x7FFFFFFF : (int)wq;
    k.kq = (float)((double)W / (double)pixel_count);
    return k;
}

// y of the 4 pixels of a lane from their window sums (S1, S2) and f (bytes of own): the float chain
// as packed f32x2 pairs; exact fix-up near rounding boundaries.
template <int NN>
__device__ __forceinline__ uint32_t w1_gain4(const W1Gain& k, uint32_t own, const uint32_t (&s1)[4],
                                             const uint32_t (&s2)[4], float inv_n) {
    uint32_t out = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // pixels (2h, 2h + 1): the float chain runs as packed f32x2 ops
        int S1[2], V[2], d[2];
        uint32_t f[2];
        float rv[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int i = 2 * h + j;
            f[j] = (own >> (8 * i)) & 0xFFu;
            S1[j] = (int)s1[i];
            V[j] = (int)(NN * s2[i] - s1[i] * s1[i]);
            d[j] = (int)(NN * f[j]) - S1[j];  // n (f - mu), |d| <= 49 * 255 < 2^14
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rv[j]) : "f"((float)V[j]));
        }
        // y + 1/2 = (S1 + g d) / n + 1/2, g = max(0, 1 - (W/P) / V): exponent-trick conversions, one
        // FFMA chain; within 2^-11 of a rounding boundary the exact integer test decides.
        const uint64_t s1f = fadd2(f2pack(__int_as_float(0x4B000000 | S1[0]), __int_as_float(0x4B000000 | S1[1])),
                                   f2splat(-8388608.0f));
        const uint64_t df = fadd2(f2pack(__int_as_float(0x4B000000 + d[0] + 16384),
                                         __int_as_float(0x4B000000 + d[1] + 16384)),
                                  f2splat(-8404992.0f));
        float t0, t1;
        f2unpack(ffma2(f2splat(-k.kq), f2pack(rv[0], rv[1]), f2splat(1.0f)), t0, t1);
        const uint64_t gg = f2pack(fmaxf(0.0f, t0), fmaxf(0.0f, t1));
        const uint64_t hh = ffma2(ffma2(gg, df, s1f), f2splat(inv_n), f2splat(0.5f));
        const uint64_t hb = fadd2_rd(hh, f2splat(12582912.0f));  // floor in the mantissa
        const uint64_t fr = ffma2(fadd2(hb, f2splat(-12582912.0f)), f2splat(-1.0f), hh);
        float frj[2], hbf[2], tie[2];
        f2unpack(fr, frj[0], frj[1]);
        f2unpack(hb, hbf[0], hbf[1]);
        f2unpack(fadd2(fr, f2splat(-0.5f)), tie[0], tie[1]);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            int q = __float_as_int(hbf[j]) - 0x4B400000;
            if (fabsf(tie[j]) > 0.5f - kTieEps) {
                if (V[j] <= k.wq32) {
                    q = (int)((2u * (uint32_t)S1[j] + NN) / (2u * NN));  // v <= nu: y = mu, half up
                } else {
                    // y >= m - 1/2  <=>  (2 (f - m) + 1) n V P >= 2 D W
                    const int m = frj[j] < 0.5f ? q : q + 1;
                    const __int128 Q = (__int128)((long long)NN * V[j]) * k.pixel_count;
                    const __int128 lhs = (__int128)(2 * ((int)f[j] - m) + 1) * Q;
                    const __int128 rhs = (__int128)(2 * (long long)d[j]) * k.W;
                    q = lhs >= rhs ? m : m - 1;
                }
            }
            out |= (uint32_t)q << (8 * (2 * h + j));  // y in [min(mu, f), max(mu, f)] -> 0..255
        }
    }
    return out;
}

// Gain of one tile: y for the tile's output pixels (rows < row_lim, columns < col_lim) through
// dst_tile (image row y0, column x0).
// MM: also fold the written y bytes into the byte-SIMD running minimum / maximum mn / mx (the contrast
// stretch's image range, fused into the gain).
template <int RW, int FH, bool MM = false>
__device__ __forceinline__ void w1_tile_gain(const uint8_t* __restrict__ T, int x0, int col_lim, int row_lim,
                                             const W1Gain& k, uint8_t* dst_tile, size_t dpitch,
                                             uint32_t* mn = nullptr, uint32_t* mx = nullptr) {
    constexpr int N = 2 * RW + 1;
    constexpr int NN = N * N;
    const int lane = threadIdx.x & 31;
    const int c = 4 * lane;
    const float inv_n = 1.0f / (float)NN;
    const uint32_t* base = reinterpret_cast<const uint32_t*>(T + FCP + c - 4);
    // ---- gain: per-pixel S1, S2 by horizontal dp4a sums slid down the tile; the leaving row is
    // re-read from the tile (small code, high occupancy) rather than kept in a register ring ----
    uint32_t s1[4] = {0, 0, 0, 0}, s2[4] = {0, 0, 0, 0};
    auto add_row = [&](int rr, bool sub) {
        const uint32_t* rp = base + rr * (FBS / 4);
        const uint32_t w0 = rp[0], w1 = rp[1], w2 = rp[2];
        uint32_t h1[4], h2[4];
        hsums4<RW>(w0, w1, w2, h1, h2);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            s1[i] = sub ? s1[i] - h1[i] : s1[i] + h1[i];
            s2[i] = sub ? s2[i] - h2[i] : s2[i] + h2[i];
        }
    };
#pragma unroll
    for (int rr = 0; rr < N - 1; ++rr) add_row(rr, false);
    uint8_t* drow = dst_tile + c;
    const bool vec_store = c + 4 <= col_lim && ((reinterpret_cast<uintptr_t>(drow) & 3) == 0) && (dpitch & 3) == 0;
#pragma unroll 1
    for (int y = 0; y < FH; ++y) {
        add_row(y + N - 1, false);  // window of output row y = tile rows y .. y + N - 1
        const uint32_t own = *(base + (y + RW) * (FBS / 4) + 1);  // f of the 4 output pixels
        const uint32_t out = w1_gain4<NN>(k, own, s1, s2, inv_n);
        if (y < row_lim) {
            if (MM) {
                // bytes outside the image (ragged last tile) are neutral: 0xFF for the min, 0 for the max
                const uint32_t keep = c + 4 <= col_lim ? 0xFFFFFFFFu
                                                       : (c >= col_lim ? 0u : (1u << (8 * (col_lim - c))) - 1u);
                *mn = __vminu4(*mn, out | ~keep);
                *mx = __vmaxu4(*mx, out & keep);
            }
            if (vec_store) {
                *reinterpret_cast<uint32_t*>(drow) = out;
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (c + i < col_lim) drow[i] = (uint8_t)(out >> (8 * i));
            }
        }
        drow += dpitch;
        add_row(y, true);  // drop tile row y
    }
}

// 3 x 3 windows, statistics and gain sharing one box-sum pass (fused small-image kernel): the
// statistics pass stores each pixel's S1 (<= 2295, 12 bits) and S2 (<= 585225, 20 bits) packed in one
// word, sums[y * 128 + column], and returns this lane's share of sum V over the valid pixels; the gain
// pass reads them back instead of recomputing the box sums.
template <int FH>
__device__ __forceinline__ long long w1_tile_sums3(const uint8_t* __restrict__ T, int col_lim, int row_lim,
                                                   uint32_t* __restrict__ sums) {
    constexpr int RW = 1, N = 3, NN = 9;
    const int lane = threadIdx.x & 31;
    const int c = 4 * lane;
    const uint32_t* base = reinterpret_cast<const uint32_t*>(T + FCP + c - 4);
    uint32_t s1[4] = {0, 0, 0, 0}, s2[4] = {0, 0, 0, 0};
    auto add_row = [&](int rr, bool sub) {
        const uint32_t* rp = base + rr * (FBS / 4);
        const uint32_t w0 = rp[0], w1 = rp[1], w2 = rp[2];
        uint32_t h1[4], h2[4];
        hsums4<RW>(w0, w1, w2, h1, h2);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            s1[i] = sub ? s1[i] - h1[i] : s1[i] + h1[i];
            s2[i] = sub ? s2[i] - h2[i] : s2[i] + h2[i];
        }
    };
#pragma unroll
    for (int rr = 0; rr < N - 1; ++rr) add_row(rr, false);
    long long vsum = 0;
#pragma unroll 1
    for (int y = 0; y < FH; ++y) {
        add_row(y + N - 1, false);
        uint4 pk;
        pk.x = s1[0] | (s2[0] << 12);
        pk.y = s1[1] | (s2[1] << 12);
        pk.z = s1[2] | (s2[2] << 12);
        pk.w = s1[3] | (s2[3] << 12);
        *reinterpret_cast<uint4*>(sums + y * FW + c) = pk;
        if (y < row_lim) {
            int v = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (c + i < col_lim) v += (int)(NN * s2[i] - s1[i] * s1[i]);  // <= 4 * 9 * 585225 < 2^31
            vsum += v;
        }
        add_row(y, true);
    }
    return vsum;
}

template <int FH>
__device__ __forceinline__ void w1_tile_gain3(const uint8_t* __restrict__ T, const uint32_t* __restrict__ sums,
                                              int col_lim, int row_lim, const W1Gain& k, uint8_t* dst_tile,
                                              size_t dpitch) {
    constexpr int RW = 1;
    const int lane = threadIdx.x & 31;
    const int c = 4 * lane;
    const uint32_t* base = reinterpret_cast<const uint32_t*>(T + FCP + c - 4);
    uint8_t* drow = dst_tile + c;
    const bool vec_store = c + 4 <= col_lim && ((reinterpret_cast<uintptr_t>(drow) & 3) == 0) && (dpitch & 3) == 0;
    const float inv_n = 1.0f / 9.0f;
#pragma unroll 1
    for (int y = 0; y < FH && y < row_lim; ++y) {
        const uint4 pk = *reinterpret_cast<const uint4*>(sums + y * FW + c);
        const uint32_t s1[4] = {pk.x & 0xFFFu, pk.y & 0xFFFu, pk.z & 0xFFFu, pk.w & 0xFFFu};
        const uint32_t s2[4] = {pk.x >> 12, pk.y >> 12, pk.z >> 12, pk.w >> 12};
        const uint32_t own = *(base + (y + RW) * (FBS / 4) + 1);
        const uint32_t out = w1_gain4<9>(k, own, s1, s2, inv_n);
        if (vec_store) {
            *reinterpret_cast<uint32_t*>(drow) = out;
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (c + i < col_lim) drow[i] = (uint8_t)(out >> (8 * i));
        }
        drow += dpitch;
    }
}

}  // namespace
}  // namespace hyb
