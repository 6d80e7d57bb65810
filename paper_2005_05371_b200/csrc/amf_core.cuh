// amf_core.cuh -- AMF building blocks shared by the AMF kernels (amf.cu) and the fused small-image
// kernel (small.cu): tile geometry, u16x2 pair-word helpers, the k = 3 strip, and the growth
// windows / selection networks / radix select for k >= 5.  Semantics: reference
// proj/src/adaptive_median.cpp:123-215 (see amf.cu).
#pragma once
#include <cstdint>

#include "networks.cuh"

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

// k = 3 for one 4-row strip of a 128 x 32 tile (one warp).  B: the tile's byte rows at stride BS,
// row 0 = image row y0 - 1, column CP = image column x0 (edges already replicated).  Writes the
// strip's output rows through dst_tile / fin_tile (image row y0, column x0; rows >= tile_row_lim or
// columns >= col_lim are outside the output), stages them in the warp's O / F areas, and, when
// bm_tile is set, the level-A failure bits of the strip into the tile's 512-byte bitmap.  Returns the
// strip's failure count (warp-uniform).
template <bool FIN>
__device__ __forceinline__ int k3_strip(const uint8_t* __restrict__ B, uint8_t* O, uint8_t* F, int sub,
                                        uint8_t* bm_tile, uint8_t* dst_tile, size_t dpitch, uint8_t* fin_tile,
                                        size_t fpitch, int tile_row_lim, int col_lim) {
    const int lane = threadIdx.x & 31;
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
    const int row_lim = tile_row_lim - sub * WR;  // strip rows < row_lim are in range

    // ---- level-A failures (inside the output range) -> the tile's failure bitmap (no atomics:
    //      every bitmap byte of the tile is written by exactly one lane) ----
    int nf = 0;
    if (bm_tile) {
        const uint32_t rv = __brev(failbits);                     // bit 16+j: row lr; bit j: row lr+1
        uint32_t m = ((rv >> 16) & 0xFFu) | ((rv & 0xFFu) << 8);  // bit j: row lr; bit 8+j: row lr+1
        if (lr >= row_lim) m &= 0xFF00u;
        if (lr + 1 >= row_lim) m &= 0x00FFu;
        if (c0 + 8 > col_lim) {
            const uint32_t cm = col_lim <= c0 ? 0u : ((1u << (col_lim - c0)) - 1u);
            m &= cm | (cm << 8);
        }
        uint8_t* bm = bm_tile + (sub * WR + lr) * 16 + (c0 >> 3);
        bm[0] = (uint8_t)m;
        bm[16] = (uint8_t)(m >> 8);
        nf = __reduce_add_sync(0xFFFFFFFFu, __popc(m));
    }
    __syncwarp();

    // ---- the strip's 4 output rows (and finalized_at): one 16-byte store per lane ----
    {
        const int sr = lane >> 3, sc = 16 * (lane & 7);
        if (sr < row_lim) {
            uint8_t* drow = dst_tile + (size_t)(sub * WR + sr) * dpitch + sc;
            uint8_t* frow = FIN ? fin_tile + (size_t)(sub * WR + sr) * fpitch + sc : nullptr;
            if (sc + 16 <= col_lim) {
                *reinterpret_cast<uint4*>(drow) = *reinterpret_cast<const uint4*>(O + sr * TW + sc);
                if (FIN) *reinterpret_cast<uint4*>(frow) = *reinterpret_cast<const uint4*>(F + sr * TW + sc);
            } else {
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    if (sc + c < col_lim) {
                        drow[c] = O[sr * TW + sc + c];
                        if (FIN) frow[c] = F[sr * TW + sc + c];
                    }
                }
            }
        }
    }
    __syncwarp();
    return nf;
}

// Tile geometry of the growth kernel: the 128 x 64 tile plus a halo of R = (smax-1)/2.
struct GGeo {
    int R, CP, BS, BH;          // halo, column pad (multiple of 16), row stride, rows
    int box_w, nbx, box_h, nby;  // TMA boxes (<= 256 per dimension)
    int b_bytes;                 // bytes per tile buffer (128-aligned)
};

inline GGeo make_ggeo(int smax) {
    GGeo g;
    g.R = (smax - 1) / 2;
    g.CP = 16 * ((g.R + 15) / 16 > 0 ? (g.R + 15) / 16 : 1);
    const int need = TW + 2 * g.CP;
    g.box_w = need <= 256 ? need : 128;
    g.nbx = (need + g.box_w - 1) / g.box_w;
    g.BS = g.box_w * g.nbx;
    g.BH = TH + 2 * g.R;
    g.box_h = g.BH <= 256 ? g.BH : 128;
    g.nby = (g.BH + g.box_h - 1) / g.box_h;
    g.b_bytes = (g.BS * g.box_h * g.nby + 127) / 128 * 128;
    return g;
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

// The K x K window around tile pixel (ty, tx) as K rows of AW byte-aligned words from the tile.
template <int K>
__device__ __forceinline__ void load_window(const uint8_t* __restrict__ B, const GGeo& geo, int ty, int tx,
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

// k = 5, 7: two queued pixels in the u16x2 lanes of one thread, generated selection network.
template <int K>
__device__ __forceinline__ void level_pair(const uint8_t* __restrict__ B, const GGeo& geo, int pa, int pb,
                                           uint32_t& done, uint32_t& outw) {
    using W = Win<K>;
    uint32_t A[K][W::AW], Bw[K][W::AW];
    load_window<K>(B, geo, pa >> 7, pa & 127, A);
    load_window<K>(B, geo, pb >> 7, pb & 127, Bw);
    uint32_t v[K * K];
#pragma unroll
    for (int r = 0; r < K; ++r)
#pragma unroll
        for (int e = 0; e < K; ++e) v[r * K + e] = pairw_rt(A[r][e >> 2], Bw[r][e >> 2], e & 3);
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

// Same with the two pixels in different tile slots.
template <int K>
__device__ __forceinline__ void level_pair2(const uint8_t* __restrict__ BA, const uint8_t* __restrict__ BB,
                                            const GGeo& geo, int pa, int pb, uint32_t& done, uint32_t& outw) {
    using W = Win<K>;
    uint32_t A[K][W::AW], Bw[K][W::AW];
    load_window<K>(BA, geo, pa >> 7, pa & 127, A);
    load_window<K>(BB, geo, pb >> 7, pb & 127, Bw);
    uint32_t v[K * K];
#pragma unroll
    for (int r = 0; r < K; ++r)
#pragma unroll
        for (int e = 0; e < K; ++e) v[r * K + e] = pairw_rt(A[r][e >> 2], Bw[r][e >> 2], e & 3);
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
__device__ __forceinline__ bool level_radix(const uint8_t* __restrict__ B, const GGeo& geo, int ty, int tx,
                                            uint8_t* out) {
    using W = Win<K>;
    uint32_t w[K][W::AW];
    load_window<K>(B, geo, ty, tx, w);
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
    if (zmin == zmax || count_eq<K>(w, zmin) > W::M || count_eq<K>(w, zmax) > W::M) return false;
    const uint32_t g = B[(size_t)(ty + geo.R) * geo.BS + tx + geo.CP];
    *out = (uint8_t)((g != zmin && g != zmax) ? g : select_rank<K>(w, W::M, zmin, zmax));
    return true;
}

// k > 11: same algorithm on byte reads from the tile.
__device__ __noinline__ bool level_generic(const uint8_t* __restrict__ B, const GGeo& geo, int ty, int tx, int k, uint8_t* out) {
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

}  // namespace
}  // namespace hyb
