// amf_core.cuh -- AMF building blocks shared by the AMF kernels (amf.cu) and the fused small-image
// kernel (small.cu): tile geometry, u16x2 pair-word helpers, the k = 3 strip, and the growth
// windows / selection networks / radix select for k >= 5.  Semantics: reference
// proj/src/adaptive_median.cpp:123-215 (see amf.cu).
#pragma once
#include <cstdint>

#include "networks.cuh"
#include "tma.cuh"
#include "trace.cuh"

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

// 128 x the number of zero bytes of x among the byte lanes flagged (0x80) in v80, added to acc.  The flag
// bytes are summed by dp4a: a POPC per window word (XU pipe, a quarter of the ALU rate) bounded the radix
// selects once the plane tests left them as the deep levels' only work.
#ifndef HYB_ZB_POPC
#define HYB_ZB_POPC 0  // 1: the POPC form (A/B)
#endif
__device__ __forceinline__ uint32_t zero_bytes_acc(uint32_t x, uint32_t v80, uint32_t acc) {
    const uint32_t t = (x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
#if HYB_ZB_POPC
    return acc + 128u * (uint32_t)__popc(~(t | x) & v80);
#else
    return __dp4a(~(t | x) & v80, 0x01010101u, acc);
#endif
}

// Compact growth windows (sparse strips, smax <= 7): a strip with at most `thresh` level-A failures
// writes each failure's whole 7 x 7 window (clamped to the source bounds) with its coordinates as one
// 64-byte entry instead of setting bitmap bits, so the growth never reloads its tile: words 2r, 2r + 1
// = window row r (bytes 0..6 = columns x - 3 .. x + 3), word 14 = x (0xFFFFFFFF: no entry), word 15 =
// slice * out_rows + output row.  B: the tile buffer with a 3-row halo (row 0 = image row y0 - 3).
struct CompactOut {
    uint4* ent;
    int* ctr;
    int cap, thresh;
    const uint8_t* B;
    uint32_t x0, key0;  // tile column, slice * out_rows + tile output row
};
constexpr uint32_t CQ_NONE = 0xFFFFFFFFu;
#ifndef HYB_COMPACT_COOP
#define HYB_COMPACT_COOP 0  // 1: warp-cooperative entry writes (measured slower: config 3 k = 3 kernel 236 vs 213 us)
#endif

__device__ __forceinline__ void compact_emit(const CompactOut& co, int tr, int tc, int pos) {
    const int start = CP + tc - 3;
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(co.B + tr * BS + (start & ~3));
    const int sh = 8 * (start & 3);
    uint32_t w[16];
#pragma unroll
    for (int r = 0; r < 7; ++r) {
        const uint32_t a = wp[r * (BS / 4)], b = wp[r * (BS / 4) + 1], c = wp[r * (BS / 4) + 2];
        w[2 * r] = __funnelshift_r(a, b, sh);
        w[2 * r + 1] = __funnelshift_r(b, c, sh);
    }
    w[14] = co.x0 + (uint32_t)tc;
    w[15] = co.key0 + (uint32_t)tr;
    uint4* e = co.ent + (size_t)pos * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) e[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
}

// k = 3 for one 4-row strip of a 128 x 32 tile (one warp).  B: the tile's byte rows at stride BS,
// row 0 = image row y0 - 1, column CP = image column x0 (edges already replicated).  Writes the
// strip's output rows through dst_tile / fin_tile (image row y0, column x0; rows >= tile_row_lim or
// columns >= col_lim are outside the output), stages them in the warp's O / F areas, and, when
// bm_tile is set, the level-A failure bits of the strip into the tile's 512-byte bitmap.  Returns the
// strip's failure count (warp-uniform).
// With q set, the failures are also appended to the shared-memory queue q (entries qslot | pixel, one
// shared atomic on *qctr per strip) -- the fused kernel's growth queue, built without a bitmap pass.
template <bool FIN>
__device__ __forceinline__ int k3_strip(const uint8_t* __restrict__ B, uint8_t* O, uint8_t* F, int sub,
                                        uint8_t* bm_tile, uint8_t* dst_tile, size_t dpitch, uint8_t* fin_tile,
                                        size_t fpitch, int tile_row_lim, int col_lim, uint16_t* q = nullptr,
                                        int* qctr = nullptr, uint32_t qslot = 0, const CompactOut* co = nullptr) {
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
                    mid[i] = add_fma(mid[i], w[i]);
                } else {
                    const uint32_t l = __vminu2(lo[i], w[i]), h = __vmaxu2(hi[i], w[i]);
                    // median of 3 = a + b + c - min - max (IMADs: exact on packed lanes, FMA pipe)
                    mid[i] = sub_fma(sub_fma(add_fma(mid[i], w[i]), l), h);
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
            // median of 9 = med3(max lo, med mid, min hi)
            const uint32_t zmed = sub_fma(sub_fma(add_fma(add_fma(a, b), c), ml), mh);
            const uint32_t g = gm[j + 1];
            // flags in bit 15 of each lane (values are v * 257): tA = level A holds, tB = zmin < g < zmax;
            // one sign-replicating PRMT turns tA & ~tB into the lane select mask
            const uint32_t tA = fadd(__vimin3_u16x2(fsub(zmed, zmin), fsub(zmax, zmed), 0x01010101u), 0x7FFF7FFFu);
            const uint32_t tB = fadd(__vimin3_u16x2(fsub(g, zmin), fsub(zmax, g), 0x01010101u), 0x7FFF7FFFu);
            const uint32_t sel = lane_mask(tA & ~tB);
            o[j] = (zmed & sel) | (g & ~sel);
            if (FIN) fz[j] = lane_mask(tA) & 0x00030003u;  // 3 where finalised at k = 3
            failbits |= (~tA & 0x80008000u) >> j;          // lane 0 -> bit 15 - j, lane 1 -> bit 31 - j
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
    if (bm_tile || q) {
        const uint32_t rv = __brev(failbits);                     // bit 16+j: row lr; bit j: row lr+1
        uint32_t m = ((rv >> 16) & 0xFFu) | ((rv & 0xFFu) << 8);  // bit j: row lr; bit 8+j: row lr+1
        if (lr >= row_lim) m &= 0xFF00u;
        if (lr + 1 >= row_lim) m &= 0x00FFu;
        if (c0 + 8 > col_lim) {
            const uint32_t cm = col_lim <= c0 ? 0u : ((1u << (col_lim - c0)) - 1u);
            m &= cm | (cm << 8);
        }
        if (co) {  // sparse strip: windows to the compact list (all or none of the strip's failures)
            const int cl = __popc(m);
            const int nfw = __reduce_add_sync(0xFFFFFFFFu, cl);
            if (nfw > 0 && nfw <= co->thresh) {
                int base = 0;
                if (lane == 0) base = atomicAdd(co->ctr, nfw);
                base = __shfl_sync(0xFFFFFFFFu, base, 0);
                if (base + nfw <= co->cap) {
#if HYB_COMPACT_COOP
                    // warp-cooperative: one failure at a time, lanes 0..6 copy its window rows, lane 7 the
                    // coordinates -- one coalesced 64-byte store per failure
                    uint32_t act = __ballot_sync(0xFFFFFFFFu, m != 0);
                    int pos = base;
                    const uint32_t* rowp = nullptr;
                    int sh = 0;
                    while (act) {
                        const int src = __ffs(act) - 1;
                        act &= act - 1;
                        uint32_t mm = __shfl_sync(0xFFFFFFFFu, m, src);
                        const int tr0 = sub * WR + 2 * (src >> 4), tc0 = 8 * (src & 15);
                        while (mm) {
                            const int b = __ffs(mm) - 1;
                            mm &= mm - 1;
                            const int tr = tr0 + (b >> 3), tc = tc0 + (b & 7);
                            if (lane < 8) {
                                uint2 val;
                                if (lane < 7) {
                                    const int start = CP + tc - 3;
                                    rowp = reinterpret_cast<const uint32_t*>(co->B + (tr + lane) * BS + (start & ~3));
                                    sh = 8 * (start & 3);
                                    const uint32_t x = rowp[0], y = rowp[1], z = rowp[2];
                                    val = make_uint2(__funnelshift_r(x, y, sh), __funnelshift_r(y, z, sh));
                                } else {
                                    val = make_uint2(co->x0 + (uint32_t)tc, co->key0 + (uint32_t)tr);
                                }
                                reinterpret_cast<uint2*>(co->ent + (size_t)pos * 4)[lane] = val;
                            }
                            ++pos;
                        }
                    }
                    m = 0;
#else
                    int incl = cl;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const int v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                        if (lane >= d) incl += v;
                    }
                    int pos = base + incl - cl;
                    while (m) {
                        const int b = __ffs(m) - 1;
                        m &= m - 1;
                        compact_emit(*co, sub * WR + lr + (b >> 3), c0 + (b & 7), pos++);
                    }
#endif
                } else if (lane < co->cap - base) {  // reservation straddles the end: void its entries
                    co->ent[(size_t)(base + lane) * 4 + 3].z = CQ_NONE;
                }
            }
        }
        if (bm_tile) {
            uint8_t* bm = bm_tile + (sub * WR + lr) * 16 + (c0 >> 3);
            bm[0] = (uint8_t)m;
            bm[16] = (uint8_t)(m >> 8);
        }
        const int c = __popc(m);
        if (q) {
            int incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= d) incl += v;
            }
            int base = 0;
            if (lane == 31 && incl) base = atomicAdd(qctr, incl);
            base = __shfl_sync(0xFFFFFFFFu, base, 31);
            int pos = base + incl - c;
            const uint32_t pbase = qslot | (uint32_t)((sub * WR + lr) * TW + c0);
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                q[pos++] = (uint16_t)(pbase + (uint32_t)((b >> 3) * TW + (b & 7)));
            }
            nf = __shfl_sync(0xFFFFFFFFu, incl, 31);
        } else {
            nf = __reduce_add_sync(0xFFFFFFFFu, c);
        }
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
template <>
__device__ __forceinline__ void select_net<9>(uint32_t (&v)[81], uint32_t& a, uint32_t& b, uint32_t& c) {
    select_net9(v, a, b, c);
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

// Level k = K (5 or 7) of two compact entries (CompactOut; in shared or global memory) in the u16x2
// lanes of one thread: the k = 5 window is the entry's centre 5 x 5, k = 7 its whole window.  `pend` bit l: entry l still open (and
// valid); out(x, key, value) stores a resolved pixel.  Returns the entries still open after level K
// (unresolved pixels keep the input the k = 3 pass wrote).
template <int K, class Out>
__device__ __forceinline__ uint32_t compact_level(const uint4* __restrict__ ea, const uint4* __restrict__ eb,
                                                  uint32_t pend, Out out) {
    const uint4 ca = ea[3], cb = eb[3];  // row 6 + coordinates
    constexpr int O = (7 - K) / 2;                          // window offset in the 7 x 7 entry
    uint32_t v[K * K];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (2 * q + 1 < O || 2 * q >= O + K) continue;
        const uint4 x = q < 3 ? ea[q] : ca, y = q < 3 ? eb[q] : cb;
        const uint32_t A[4] = {x.x, x.y, x.z, x.w}, Bw[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // entry row 2q + h = words 4q + 2h, 4q + 2h + 1
            const int r = 2 * q + h - O;
            if (r >= 0 && r < K) {
#pragma unroll
                for (int e = 0; e < K; ++e)
                    v[r * K + e] = pairw_rt(A[2 * h + ((e + O) >> 2)], Bw[2 * h + ((e + O) >> 2)], (e + O) & 3);
            }
        }
    }
    const uint32_t g = v[(K * K) / 2];
    uint32_t zmin, zmed, zmax;
    select_net<K>(v, zmin, zmed, zmax);
#pragma unroll
    for (int l = 0; l < 2; ++l) {
        const uint32_t zn = (zmin >> (16 * l)) & 0xFFu, zd = (zmed >> (16 * l)) & 0xFFu;
        const uint32_t zx = (zmax >> (16 * l)) & 0xFFu, gl = (g >> (16 * l)) & 0xFFu;
        if ((pend >> l & 1u) && zn < zd && zd < zx) {
            out(l ? cb.z : ca.z, l ? cb.w : ca.w, (zn < gl && gl < zx) ? gl : zd);
            pend &= ~(1u << l);
        }
    }
    return pend;
}

// Count of window values equal to v (SWAR over the aligned window words).
template <int K>
__device__ __forceinline__ int count_eq(const uint32_t (&w)[K][Win<K>::AW], uint32_t v) {
    const uint32_t P = v * 0x01010101u;
    uint32_t c = 0;
#pragma unroll
    for (int r = 0; r < K; ++r)
#pragma unroll
        for (int j = 0; j < Win<K>::AW; ++j) c = zero_bytes_acc(w[r][j] ^ P, Win<K>::v80(j), c);
    return (int)(c >> 7);
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
        uint32_t c128 = 0;
#pragma unroll
        for (int r = 0; r < K; ++r)
#pragma unroll
            for (int j = 0; j < Win<K>::AW; ++j) c128 = zero_bytes_acc((w[r][j] ^ P) & M, Win<K>::v80(j), c128);
        const int c = (int)(c128 >> 7);
        if (below + c <= rank) {
            below += c;
            prefix |= 1u << b;
        }
    }
    return prefix;
}

// Window extremes of a K x K window (aligned words): zmin / zmax.
template <int K>
__device__ __forceinline__ void window_minmax(const uint32_t (&w)[K][Win<K>::AW], uint32_t& zmin, uint32_t& zmax) {
    using W = Win<K>;
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
    zmin = min(mn & 0xFFFFu, mn >> 16);
    zmax = max(mx & 0xFFFFu, mx >> 16);
}

// k = 9, 11, one pixel per thread, first pass: level A from SWAR counts without a median
// (zmin < zmed < zmax <=> zmin < zmax, #(v == zmin) <= m and #(v == zmax) <= m).  Returns 0: level A
// fails; 1: resolved, *out = g (zmin < g < zmax); 2: resolved to the median, which the caller computes
// in a second, compacted pass (level_radix_median) so the radix select runs on full warps.
template <int K>
__device__ __forceinline__ int level_radix_test(const uint8_t* __restrict__ B, const GGeo& geo, int ty, int tx,
                                                uint8_t* out) {
    using W = Win<K>;
    uint32_t w[K][W::AW];
    load_window<K>(B, geo, ty, tx, w);
    uint32_t zmin, zmax;
    window_minmax<K>(w, zmin, zmax);
    if (zmin == zmax || count_eq<K>(w, zmin) > W::M || count_eq<K>(w, zmax) > W::M) return 0;
    const uint32_t g = B[(size_t)(ty + geo.R) * geo.BS + tx + geo.CP];
    if (g != zmin && g != zmax) {
        *out = (uint8_t)g;
        return 1;
    }
    return 2;
}

// Second pass: the window median by bitwise radix select (values within [zmin, zmax]).
template <int K, bool FULL = false>
__device__ __forceinline__ uint8_t level_radix_median(const uint8_t* __restrict__ B, const GGeo& geo, int ty, int tx) {
    using W = Win<K>;
    uint32_t w[K][W::AW];
    load_window<K>(B, geo, ty, tx, w);
    uint32_t zmin = 0u, zmax = 255u;  // FULL: the window is known to hold a 0 and a 255 (plane tests)
    if (!FULL) window_minmax<K>(w, zmin, zmax);
    return (uint8_t)select_rank<K>(w, W::M, zmin, zmax);
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

// Failure bitmaps (nwords 32-bit words, 128 per 128 x 32 tile: word 4 r + q = row r, columns
// 32 q ..) -> queue entries slot << 12 | pixel in raster order, CTA-wide: a block scan gives every
// word its output base, then each warp emits one word per step, one bit per lane (no per-thread
// serial bit loops).  wbase: nwords u16 scratch; wsum: NTHR / 32 ints.  Returns the entry count.
template <int NTHR>
__device__ __forceinline__ int cta_bitmap_queue(const uint32_t* words, int nwords, uint16_t* Q, uint16_t* wbase,
                                                int* wsum) {
    constexpr int NWARP = NTHR / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (nwords + NTHR - 1) / NTHR;
    int c = 0;
    for (int i = 0; i < per; ++i) {
        const int w = tid * per + i;
        if (w < nwords) c += __popc(words[w]);
    }
    int incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= d) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int off = incl - c, total = 0;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) {
        off += w < warp ? wsum[w] : 0;
        total += wsum[w];
    }
    for (int i = 0; i < per; ++i) {
        const int w = tid * per + i;
        if (w < nwords) {
            wbase[w] = (uint16_t)off;
            off += __popc(words[w]);
        }
    }
    __syncthreads();
    for (int w = warp; w < nwords; w += NWARP) {
        const uint32_t word = words[w];
        if ((word >> lane) & 1u) {
            const int lw = w & 127;
            Q[wbase[w] + __popc(word & ((1u << lane) - 1u))] =
                (uint16_t)(((w >> 7) << 12) | ((lw >> 2) * 128 + 32 * (lw & 3) + lane));
        }
    }
    __syncthreads();
    return total;
}

__device__ __forceinline__ void grow_tile_load(const CUtensorMap* tm, const GGeo& geo, uint8_t* Bbuf, uint64_t* bar,
                                               int x0, int y0, int z) {
    mbar_expect_tx(bar, (uint32_t)(geo.box_w * geo.nbx * geo.box_h * geo.nby));
    for (int by = 0; by < geo.nby; ++by)
        for (int bx = 0; bx < geo.nbx; ++bx)
            tma_load_3d(Bbuf + (size_t)by * geo.box_h * geo.BS + (size_t)bx * geo.box_w, tm, bar,
                        x0 - geo.CP + bx * geo.box_w, y0 - geo.R + by * geo.box_h, z);
}

// Growth work records (amf_k3_kernel -> growth): one per tile with level-A failures, weighted
// offsets (a tile load counts REC_W failures) so a range split balances loads and failures.
constexpr int REC_SHIFT = 40;
constexpr int REC_W = 128;  // growth balancing weight of one tile load, in failures
constexpr unsigned long long REC_MASK = (1ull << REC_SHIFT) - 1;
#ifndef HYB_GSLOTS
#define HYB_GSLOTS 8
#endif
#ifndef HYB_GCAP
#define HYB_GCAP 8192
#endif
constexpr int GSLOTS = HYB_GSLOTS;  // tile segments per growth batch
constexpr int GCAP = HYB_GCAP;      // pooled queue capacity
constexpr int MAX_LEVELS = 128;

__device__ __forceinline__ long long rec_off(const unsigned long long* rec, long long i) {
    return (long long)(__ldcg(rec + i) >> 24);
}

// Growth levels k = 5..smax over a pooled queue Q0[0, n) of entries slot << 12 | pixel (pixel =
// row * 128 + column of a 128 x 32 tile whose window bytes start at slot(slot), laid out as geo).  CTA-wide
// (NTHR threads, every thread calls it; qcount[1..] zero on entry); level k resolves what it can through
// out(slot, pixel, value, k) and re-queues the rest for k + 2.  Ends with __syncthreads.
#ifndef HYB_GUIDED
#define HYB_GUIDED 1  // guided (shrinking) dynamic growth claims; needs the k = 3 chunk table at 2048 units
#endif
#ifndef HYB_STATIC_Q
#define HYB_STATIC_Q 3  // quarters of the growth work split statically (the rest claimed dynamically)
#endif
#ifndef HYB_GUIDED_DIV
#define HYB_GUIDED_DIV 2  // a guided claim takes remaining / (HYB_GUIDED_DIV * CTAs) units
#endif
#ifndef HYB_GROW_NETMAX
#define HYB_GROW_NETMAX 9  // largest window grown with a selection network (k <= 9); radix above
#endif
#ifndef HYB_NET9_MIN
#define HYB_NET9_MIN 1  // the k = 9 network needs >= HYB_NET9_MIN * NTHR queued pixels (else radix, 1 px/thread)
#endif
template <bool FIN, int NTHR, class Slot, class Out, int NETMAX = HYB_GROW_NETMAX>
__device__ __forceinline__ void grow_levels_at(Slot slot, const GGeo& geo, uint16_t* Q0, uint16_t* Q1, int* qcount,
                                               int n, int smax, Out out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int lvl = 0;
    for (int k = 5; k <= smax; k += 2, ++lvl) {
#ifdef HYB_TRACE
        unsigned long long t_lvl = 0;
        if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_lvl));
#endif
        const uint16_t* qin = (lvl & 1) ? Q1 : Q0;
        uint16_t* qout = (lvl & 1) ? Q0 : Q1;
        const bool last = k + 2 > smax;
        if (k <= NETMAX && (k < 9 || n >= HYB_NET9_MIN * NTHR)) {
            const int npairs = (n + 1) >> 1;
            for (int base = warp * 32; base < npairs; base += NTHR) {
                const int i = base + lane;
                uint32_t keep = 0;
                int ea = 0, eb = 0;
                if (i < npairs) {
                    ea = qin[2 * i];
                    const bool hasb = 2 * i + 1 < n;
                    eb = hasb ? qin[2 * i + 1] : ea;
                    const int sa = ea >> 12, pa = ea & 4095, sb = eb >> 12, pb = eb & 4095;
                    uint32_t done, outw;
                    const uint8_t* BA = slot(sa);
                    const uint8_t* BB = slot(sb);
                    if (k == 5) level_pair2<5>(BA, BB, geo, pa, pb, done, outw);
                    else if (k == 7) level_pair2<7>(BA, BB, geo, pa, pb, done, outw);
                    else if constexpr (NETMAX >= 9) level_pair2<9>(BA, BB, geo, pa, pb, done, outw);
                    if (done & 1u) {
                        out(sa, pa, (uint8_t)outw, k);
                    } else {
                        keep |= 1u;
                    }
                    if (hasb) {
                        if (done & 2u) {
                            out(sb, pb, (uint8_t)(outw >> 8), k);
                        } else {
                            keep |= 2u;
                        }
                    }
                }
                if (!last) {
                    const uint32_t balA = __ballot_sync(0xFFFFFFFFu, keep & 1u);
                    const uint32_t balB = __ballot_sync(0xFFFFFFFFu, keep & 2u);
                    const int c = __popc(balA) + __popc(balB);
                    if (c) {
                        int qb = 0;
                        if (lane == 0) qb = atomicAdd(&qcount[lvl + 1], c);
                        qb = __shfl_sync(0xFFFFFFFFu, qb, 0);
                        const uint32_t below = (1u << lane) - 1u;
                        if (keep & 1u) qout[qb + __popc(balA & below)] = (uint16_t)ea;
                        if (keep & 2u) qout[qb + __popc(balA) + __popc(balB & below)] = (uint16_t)eb;
                    }
                }
            }
        } else {
            // one pixel per thread.  k = 9 / 11: the level-A test first; pixels resolved to the median
            // (g at a window extreme) are compacted per warp over the warp's already consumed queue
            // slots (entry s at qw[warp * 32 + (s / 32) * NTHR + s % 32]) and get their radix select in a
            // second pass on full warps -- in one pass, every warp with any such lane paid the whole select.
            const bool radix = k == 9 || k == 11;
            uint16_t* qw = const_cast<uint16_t*>(qin);
            int nmed = 0;  // warp-uniform
            for (int base = warp * 32; base < n; base += NTHR) {
                const int i = base + lane;
                bool keep = false, med = false;
                int e = 0;
                if (i < n) {
                    e = qin[i];
                    const int sl = e >> 12, pix = e & 4095, ty = pix >> 7, tx = pix & 127;
                    const uint8_t* B = slot(sl);
                    uint8_t o = 0;
                    if (radix) {
                        const int st = k == 9 ? level_radix_test<9>(B, geo, ty, tx, &o)
                                              : level_radix_test<11>(B, geo, ty, tx, &o);
                        if (st == 1) out(sl, pix, o, k);
                        med = st == 2;
                        keep = st == 0;
                    } else if (level_generic(B, geo, ty, tx, k, &o)) {
                        out(sl, pix, o, k);
                    } else {
                        keep = true;
                    }
                }
                if (radix) {
                    const uint32_t bm = __ballot_sync(0xFFFFFFFFu, med);
                    if (med) {
                        const int s = nmed + __popc(bm & ((1u << lane) - 1u));
                        qw[warp * 32 + (s >> 5) * NTHR + (s & 31)] = (uint16_t)e;
                    }
                    nmed += __popc(bm);
                }
                if (!last) {
                    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
                    if (bal) {
                        int qb = 0;
                        if (lane == 0) qb = atomicAdd(&qcount[lvl + 1], __popc(bal));
                        qb = __shfl_sync(0xFFFFFFFFu, qb, 0);
                        if (keep) qout[qb + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)e;
                    }
                }
            }
            __syncwarp();
            for (int s0 = 0; s0 < nmed; s0 += 32) {
                const int s = s0 + lane;
                if (s < nmed) {
                    const int e = qw[warp * 32 + (s >> 5) * NTHR + (s & 31)];
                    const int sl = e >> 12, pix = e & 4095, ty = pix >> 7, tx = pix & 127;
                    const uint8_t* B = slot(sl);
                    const uint8_t o = k == 9 ? level_radix_median<9>(B, geo, ty, tx) : level_radix_median<11>(B, geo, ty, tx);
                    out(sl, pix, o, k);
                }
            }
        }
        __syncthreads();
#ifdef HYB_TRACE
        // growth-level profile (kernel id 1): slots 5 + lvl += level time, 9 + lvl += level pixels
        if (threadIdx.x == 0 && blockIdx.x < 1024 && lvl < 4) {
            unsigned long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            g_trace[(1024 + blockIdx.x) * 16 + 5 + lvl] += t1 - t_lvl;
            g_trace[(1024 + blockIdx.x) * 16 + 9 + lvl] += (unsigned long long)n;
        }
#endif
        if (last) break;
        n = qcount[lvl + 1];
        if (n == 0) break;
    }
}

// Slots at a fixed stride in local shared memory.
template <bool FIN, int NTHR, class Out, int NETMAX = HYB_GROW_NETMAX>
__device__ __forceinline__ void grow_levels(const uint8_t* bufs, const GGeo& geo, uint16_t* Q0, uint16_t* Q1,
                                            int* qcount, int n, int smax, Out out) {
    auto slot = [&](int sl) { return bufs + (size_t)sl * geo.b_bytes; };
    grow_levels_at<FIN, NTHR, decltype(slot), Out, NETMAX>(slot, geo, Q0, Q1, qcount, n, smax, out);
}

// ------------------------------------------------------------------------------------------
// Fast growth levels: zero / 255 bit planes
// ------------------------------------------------------------------------------------------
//
// Under heavy salt & pepper nearly every window of a growing pixel holds both a 0 and a 255, so
// zmin = 0 and zmax = 255 are known without looking at the values, level A (zmin < zmed < zmax) is
// #(v == 0) <= m and #(v == 255) <= m, and level B keeps g unless g is 0 or 255 -- the window median
// is needed only at the level where A passes, and only for an impulse centre.  The counts come from
// two bit planes of the staged tile (bit = byte is 0 / byte is 255; build_planes), a few funnel
// shifts and one POPC per 32 window bits instead of a selection network per level.  Windows are
// nested, so a pixel whose 5 x 5 window lacks a 0 or a 255 is the only kind the shortcut cannot
// decide: it is flagged (entry bit 15) and takes the generic zmin / zmed / zmax test at every level,
// sharing the median pass with the flagged-free entries.

// Bit planes of `ns` staged tiles: planes[sl][row * PW + w] = (zero bits, 255 bits) of the 32 tile
// bytes at 32 (row * PW + w) (BS = 32 PW, so plane words and tile bytes are both linear).
template <int NTHR>
__device__ __forceinline__ void build_planes(const uint8_t* bufs, const GGeo& geo, uint2* planes, int pstride, int ns) {
    const int per = geo.BH * (geo.BS >> 5);
    for (int t = threadIdx.x; t < ns * per; t += NTHR) {
        const int sl = t / per, q = t - sl * per;
        const uint4* src = reinterpret_cast<const uint4*>(bufs + (size_t)sl * geo.b_bytes + 32 * q);
        const uint4 lo = src[0], hi = src[1];
        const uint32_t x[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
        // the four byte MSBs are gathered into the top nibble by one multiply (bits 24..27 of the product stay
        // zero) and shifted into the plane word; even and odd words in separate chains (half the dependent depth)
        uint32_t a0 = 0, b0 = 0, a1 = 0, b1 = 0;
#pragma unroll
        for (int j = 7; j >= 0; --j) {
            const uint32_t t7 = x[j] & 0x7F7F7F7Fu;
            const uint32_t z = ~((t7 + 0x7F7F7F7Fu) | x[j]) & 0x80808080u;  // byte MSB: byte == 0
            const uint32_t f = (t7 + 0x01010101u) & x[j] & 0x80808080u;      // byte MSB: byte == 255
            if (j & 1) {
                a0 = __funnelshift_l(z * 0x00204081u, a0, 8);
                a1 = __funnelshift_l(f * 0x00204081u, a1, 8);
            } else {
                b0 = __funnelshift_l(z * 0x00204081u, b0, 8);
                b1 = __funnelshift_l(f * 0x00204081u, b1, 8);
            }
        }
        planes[(size_t)sl * pstride + q] = make_uint2(a0 | (b0 >> 4), a1 | (b1 >> 4));
    }
}

// #(v == 0) and #(v == 255) of the K x K window around tile pixel (ty, tx), from the tile's planes.
template <int K>
__device__ __forceinline__ void plane_counts(const uint2* __restrict__ P, const GGeo& geo, int ty, int tx, int& c0,
                                             int& c255) {
    constexpr int RK = K / 2, RPW = 32 / K;  // window rows packed per 32-bit word
    constexpr uint32_t MASK = (1u << K) - 1u;
    const int PW = geo.BS >> 5, cs = tx + geo.CP - RK, sh = cs & 31;
    const uint2* row = P + (size_t)(ty + geo.R - RK) * PW + (cs >> 5);
    uint32_t a0 = 0, a1 = 0;
    c0 = 0;
    c255 = 0;
#pragma unroll
    for (int r = 0; r < K; ++r) {
        const uint2 lo = row[r * PW], hi = row[r * PW + 1];  // (the plane is padded by one word)
        a0 = a0 * (1u << K) + (__funnelshift_r(lo.x, hi.x, sh) & MASK);
        a1 = a1 * (1u << K) + (__funnelshift_r(lo.y, hi.y, sh) & MASK);
        if ((r + 1) % RPW == 0 || r == K - 1) {
            c0 += __popc(a0);
            c255 += __popc(a1);
            a0 = a1 = 0;
        }
    }
}

// Bit-sliced box counts of one plane for one tile row: e[i][j] = plane word j (of 5) of window row i (of
// 5).  For every column, le12 / any = the 5 x 5 window holds <= 12 / >= 1 set bits.  Vertical sums as
// 3-bit numbers (two full adders per word), five horizontally shifted copies added by carry-save adders:
// ~45 LOP3 / SHF per 32 pixels, against one selection network per pixel.
__device__ __forceinline__ uint32_t xor3(uint32_t a, uint32_t b, uint32_t c) { return a ^ b ^ c; }
__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (c & (a | b)); }

__device__ __forceinline__ void box5_counts(const uint32_t (&e)[5][5], uint32_t (&le12)[5], uint32_t (&any)[5]) {
    uint32_t v[3][7];  // vertical sums, bit b of word j at v[b][j + 1]; zero words either side
#pragma unroll
    for (int b = 0; b < 3; ++b) v[b][0] = v[b][6] = 0u;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const uint32_t s1 = xor3(e[0][j], e[1][j], e[2][j]), c1 = maj3(e[0][j], e[1][j], e[2][j]);
        v[0][j + 1] = xor3(s1, e[3][j], e[4][j]);
        const uint32_t c2 = maj3(s1, e[3][j], e[4][j]);
        v[1][j + 1] = c1 ^ c2;
        v[2][j + 1] = c1 & c2;
    }
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        uint32_t t[3], c[3], d[3];
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const uint32_t A = __funnelshift_l(v[b][j], v[b][j + 1], 2);      // column - 2
            const uint32_t B = __funnelshift_l(v[b][j], v[b][j + 1], 1);      // column - 1
            const uint32_t C = v[b][j + 1];
            const uint32_t D = __funnelshift_r(v[b][j + 1], v[b][j + 2], 1);  // column + 1
            const uint32_t E = __funnelshift_r(v[b][j + 1], v[b][j + 2], 2);  // column + 2
            const uint32_t s = xor3(A, B, C);
            c[b] = maj3(A, B, C);
            t[b] = xor3(s, D, E);
            d[b] = maj3(s, D, E);
        }
        // t[b] weighs 2^b, c[b] and d[b] 2^(b+1)
        const uint32_t r0 = t[0];
        const uint32_t r1 = xor3(t[1], c[0], d[0]), k1 = maj3(t[1], c[0], d[0]);
        const uint32_t u = xor3(t[2], c[1], d[1]), ku = maj3(t[2], c[1], d[1]);
        const uint32_t r2 = u ^ k1, kv = u & k1;
        const uint32_t w = xor3(c[2], d[2], ku), kw = maj3(c[2], d[2], ku);
        const uint32_t r3 = w ^ kv, kx = w & kv;
        const uint32_t r4 = kw | kx;
        le12[j] = ~(r4 | (r3 & r2 & (r1 | r0)));  // count < 13
        any[j] = r0 | r1 | r2 | r3 | r4;
    }
}

// Level k = 5 for a whole tile at once, one warp per staged tile, lane = tile row (geo.CP == 16, BS == 160).
// bm[128] holds the tile's level-A failures of k = 3 (bitmap words 4 row + q), [lo, hi) the in-tile rank
// range of the segment this batch grows.  Returns, for the lane's row, m = the pixels whose k = 5 median
// is needed (impulse centres that pass level A, and every pixel whose window lacks a 0 or a 255 -- the
// generic test decides those) and s = the pixels still open.  Pixels that pass with a non-impulse centre
// keep g, which f already holds (FIN: they go through the median pass so finalized_at gets its 5).
template <bool FIN>
__device__ __forceinline__ void dense_level5(const uint2* P0, const GGeo& geo, const uint32_t* __restrict__ bm, int lo,
                                             int hi, uint4& m, uint4& s) {
    static_assert(TH == 32, "one warp = the rows of one tile");
    const int row = threadIdx.x & 31;
    uint4 f = reinterpret_cast<const uint4*>(bm)[row];
    {
        const int nf = __popc(f.x) + __popc(f.y) + __popc(f.z) + __popc(f.w);
        int incl = nf;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
            if (row >= d) incl += v;
        }
        int rank = incl - nf;
        if (rank < lo || incl > hi) {  // the segment boundary crosses this row
            uint32_t wb[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t bits = wb[j], keepw = 0;
                while (bits) {
                    const uint32_t low = bits & (0u - bits);
                    if (rank >= lo && rank < hi) keepw |= low;
                    bits ^= low;
                    ++rank;
                }
                wb[j] = keepw;
            }
            f = make_uint4(wb[0], wb[1], wb[2], wb[3]);
        }
    }
    const uint2* P = P0 + (row + geo.R - 2) * 5;
    uint32_t e0[5][5], e1[5][5];
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const uint2 w = P[i * 5 + j];
            e0[i][j] = w.x;
            e1[i][j] = w.y;
        }
    uint32_t le0[5], any0[5], le1[5], any1[5], dm[5], ds[5];
    box5_counts(e0, le0, any0);
    box5_counts(e1, le1, any1);
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const uint32_t pass = le0[j] & le1[j], elig = any0[j] & any1[j], ext = e0[2][j] | e1[2][j];
        dm[j] = FIN ? (~elig | pass) : (~elig | (pass & ext));
        ds[j] = elig & ~pass;
    }
    // plane bit 16 + c = tile column c
    m = make_uint4(f.x & __funnelshift_r(dm[0], dm[1], 16), f.y & __funnelshift_r(dm[1], dm[2], 16),
                   f.z & __funnelshift_r(dm[2], dm[3], 16), f.w & __funnelshift_r(dm[3], dm[4], 16));
    s = make_uint4(f.x & __funnelshift_r(ds[0], ds[1], 16), f.y & __funnelshift_r(ds[1], ds[2], 16),
                   f.z & __funnelshift_r(ds[2], ds[3], 16), f.w & __funnelshift_r(ds[3], ds[4], 16));
}

// One whole level K (9 or 11) of one pixel, out of line (the rare flagged pixels of the chained intervals):
// 0: level A fails; else *out = the result.
template <int K>
__device__ __noinline__ int level_radix_full(const uint8_t* __restrict__ B, const GGeo& geo, int ty, int tx, uint8_t* out) {
    const int st = level_radix_test<K>(B, geo, ty, tx, out);
    if (st == 2) *out = level_radix_median<K>(B, geo, ty, tx);
    return st;
}

// Median of a K x K window known to hold a 0 and a 255, by a pair of lanes (half = lane & 1): each loads half of
// the window rows and counts its share per radix step, one shuffle adds the two.  The deep levels hold a few
// hundred pixels per batch; at one pixel per lane they fill a warp or two whose ~1 000-instruction selects the
// other warps wait for, at one pixel per lane pair the work spreads over twice the warps at half the length.
// Every lane of the warp must call it (full-mask shuffle); both lanes return the median.
template <int K>
__device__ __forceinline__ uint32_t radix_median_pair(const uint8_t* __restrict__ B, const GGeo& geo, int ty, int tx,
                                                      int half) {
    using W = Win<K>;
    constexpr int NR = (K + 1) / 2;  // row slots per lane; the last slot of half 1 lies beyond the window
    const int start = tx + geo.CP - W::RK;
    const int sh = 8 * (start & 3);
    const uint32_t* rowp =
        reinterpret_cast<const uint32_t*>(B + (size_t)(ty + geo.R - W::RK) * geo.BS) + (start >> 2);
    uint32_t w[NR][W::AW];
#pragma unroll
    for (int s = 0; s < NR; ++s) {
        const int r = min(half * NR + s, K - 1);
        uint32_t raw[W::NRAW];
#pragma unroll
        for (int j = 0; j < W::NRAW; ++j) raw[j] = rowp[r * (geo.BS >> 2) + j];
#pragma unroll
        for (int j = 0; j < W::AW; ++j) w[s][j] = __funnelshift_r(raw[j], (j + 1 < W::NRAW) ? raw[j + 1] : 0u, sh);
    }
    const uint32_t lastm = (half * NR + NR - 1 < K) ? 0xFFFFFFFFu : 0u;
    uint32_t prefix = 0;
    int below = 0;
#pragma unroll 1
    for (int b = 7; b >= 0; --b) {
        const uint32_t M = ((0xFFu << b) & 0xFFu) * 0x01010101u;
        const uint32_t P = prefix * 0x01010101u;
        uint32_t c128 = 0;
#pragma unroll
        for (int s = 0; s < NR; ++s)
#pragma unroll
            for (int j = 0; j < W::AW; ++j)
                c128 = zero_bytes_acc((w[s][j] ^ P) & M, s == NR - 1 ? (W::v80(j) & lastm) : W::v80(j), c128);
        c128 += __shfl_xor_sync(0xFFFFFFFFu, c128, 1);
        const int c = (int)(c128 >> 7);
        if (below + c <= W::M) {
            below += c;
            prefix |= 1u << b;
        }
    }
    return prefix;
}

// Queues of the fast levels.  Level index l <-> k = 5 + 2 l; |S_k| = qcount[2 l], |M_k| = qcount[2 l + 1].
// S_k (open pixels, unflagged, plane-testable) sits at the front of a buffer, M_k (pixels whose level-k
// median is needed: impulse centres that passed A, and every flagged pixel) at its tail, growing down.
constexpr int FAST_FLAG = 0x8000;
#ifndef HYB_FAST_PAIRS
#define HYB_FAST_PAIRS 0  // 1: the side-by-side deep median passes take one pixel per lane pair (radix_median_pair);
                          // measured slower, config 4 AMF 1.753 vs 1.739 ms per lane
#endif

// Pass A of level K: plane test of S_K = X[0, nS) -> S_K+2 (front of Y), M_K (tail of Y), or the pixel keeps g.
// CHAIN (K + 2 is the last level): a pixel that fails level K takes the K + 2 test at once, and the front list
// becomes M_K+2 -- the next interval then runs the median passes of both levels side by side.
template <bool FIN, int NTHR, int CAP, int K, bool CHAIN, class Slot, class PlaneOf, class Out>
__device__ __forceinline__ void fast_pass_a(Slot slot, PlaneOf plane, const GGeo& geo, const uint16_t* X, uint16_t* Y,
                                            int nS, int* cSn, int* cM, bool last, int wrot, Out out) {
    constexpr int NWARP = NTHR / 32;
    const int lane = threadIdx.x & 31, warp = ((threadIdx.x >> 5) + NWARP - wrot) % NWARP;
    const uint32_t below = (1u << lane) - 1u;
    constexpr int M = (K * K - 1) / 2;
    for (int base = warp * 32; base < nS; base += NTHR) {
        const int i = base + lane;
        int cls = 0, e = 0;  // 1: still open, 2: median needed
        if (i < nS) {
            e = X[i];
            const int sl = e >> 12, pix = e & 4095, ty = pix >> 7, tx = pix & 127;
            if (K <= 11) {
                int c0, c255;
                plane_counts<(K <= 11 ? K : 11)>(plane(sl), geo, ty, tx, c0, c255);
                if (c0 > M || c255 > M) {
                    if constexpr (CHAIN && K <= 9) {
                        constexpr int M2 = ((K + 2) * (K + 2) - 1) / 2;
                        plane_counts<(K <= 9 ? K + 2 : 11)>(plane(sl), geo, ty, tx, c0, c255);
                        if (c0 <= M2 && c255 <= M2) {
                            const uint32_t g = slot(sl)[(size_t)(ty + geo.R) * geo.BS + tx + geo.CP];
                            if (g != 0u && g != 255u) {
                                if (FIN) out(sl, pix, (uint8_t)g, K + 2);
                            } else {
                                cls = 1;  // front list: M_K+2
                            }
                        }
                    } else {
                        cls = last ? 0 : 1;
                    }
                } else {
                    const uint32_t g = slot(sl)[(size_t)(ty + geo.R) * geo.BS + tx + geo.CP];
                    if (g != 0u && g != 255u) {
                        if (FIN) out(sl, pix, (uint8_t)g, K);  // f already holds g (the k = 3 pass wrote it)
                    } else {
                        cls = 2;
                    }
                }
            } else {
                cls = 2;  // beyond the plane tests: the generic level decides
            }
        }
        const uint32_t balS = __ballot_sync(0xFFFFFFFFu, cls == 1);
        const uint32_t balM = __ballot_sync(0xFFFFFFFFu, cls == 2);
        if (balS) {
            int qb = 0;
            if (lane == 0) qb = atomicAdd(cSn, __popc(balS));
            qb = __shfl_sync(0xFFFFFFFFu, qb, 0);
            if (cls == 1) Y[qb + __popc(balS & below)] = (uint16_t)e;
        }
        if (balM) {
            int qb = 0;
            if (lane == 0) qb = atomicAdd(cM, __popc(balM));
            qb = __shfl_sync(0xFFFFFFFFu, qb, 0);
            if (cls == 2) Y[CAP - 1 - (qb + __popc(balM & below))] = (uint16_t)e;
        }
    }
}

// Pass B of level K: the median pass over M_K = tail of X, nM entries; flagged pixels that fail the
// generic level A move to M_K+2 (tail of Y, flagged).
// FRONT: the list sits at the front of X instead (entry j at X[j]; see fast_pass_a CHAIN), the warps rotated by wrot.
// INL (K + 2 is the last level and its median pass runs beside this one): a flagged pixel that fails here takes
// level K + 2 at once, in its own thread (rare), instead of moving to M_K+2.
template <bool FIN, int NTHR, int CAP, int K, int NETMAX, bool FRONT, bool INL, class Slot, class Out>
__device__ __forceinline__ void fast_pass_b(Slot slot, const GGeo& geo, const uint16_t* X, uint16_t* Y, int nM, int* cMn,
                                            bool last, int wrot, Out out) {
    constexpr int NWARP = NTHR / 32;
    const int lane = threadIdx.x & 31, warp = ((threadIdx.x >> 5) + NWARP - wrot) % NWARP;
    const uint32_t below = (1u << lane) - 1u;
    const uint16_t* Mq = FRONT ? X : X + CAP - 1;  // entry j at Mq[-j] (FRONT: Mq[j])
    constexpr int DIR = FRONT ? -1 : 1;
    if constexpr (K <= NETMAX && K <= 9) {
        const int npairs = (nM + 1) >> 1;
        for (int base = warp * 32; base < npairs; base += NTHR) {
            const int i = base + lane;
            uint32_t keep = 0;
            int ea = 0, eb = 0;
            if (i < npairs) {
                ea = Mq[-DIR * 2 * i];
                const bool hasb = 2 * i + 1 < nM;
                eb = hasb ? Mq[-DIR * (2 * i + 1)] : ea;
                const int sa = (ea >> 12) & 7, pa = ea & 4095, sb = (eb >> 12) & 7, pb = eb & 4095;
                uint32_t done, outw;
                level_pair2<K>(slot(sa), slot(sb), geo, pa, pb, done, outw);
                if (done & 1u) out(sa, pa, (uint8_t)outw, K);
                else keep |= 1u;
                if (hasb) {
                    if (done & 2u) out(sb, pb, (uint8_t)(outw >> 8), K);
                    else keep |= 2u;
                }
            }
            if constexpr (INL && (K == 7 || K == 9)) {
#pragma unroll
                for (int l = 0; l < 2; ++l) {
                    if (keep >> l & 1u) {
                        const int e = l ? eb : ea, sl = (e >> 12) & 7, pix = e & 4095;
                        uint8_t o = 0;
                        if (level_radix_full<K + 2>(slot(sl), geo, pix >> 7, pix & 127, &o)) out(sl, pix, o, K + 2);
                    }
                }
            } else if (!last) {  // only pixels whose windows lack a 0 or a 255 can fail here
                const uint32_t balA = __ballot_sync(0xFFFFFFFFu, keep & 1u);
                const uint32_t balB = __ballot_sync(0xFFFFFFFFu, keep & 2u);
                const int c = __popc(balA) + __popc(balB);
                if (c) {
                    int qb = 0;
                    if (lane == 0) qb = atomicAdd(cMn, c);
                    qb = __shfl_sync(0xFFFFFFFFu, qb, 0);
                    if (keep & 1u) Y[CAP - 1 - (qb + __popc(balA & below))] = (uint16_t)(ea | FAST_FLAG);
                    if (keep & 2u) Y[CAP - 1 - (qb + __popc(balA) + __popc(balB & below))] = (uint16_t)(eb | FAST_FLAG);
                }
            }
        }
    } else {
        for (int base = warp * 32; base < nM; base += NTHR) {
            const int i = base + lane;
            bool keep = false;
            int e = 0;
            if (i < nM) {
                e = Mq[-DIR * i];
                const int sl = (e >> 12) & 7, pix = e & 4095, ty = pix >> 7, tx = pix & 127;
                const uint8_t* B = slot(sl);
                uint8_t o = 0;
                if constexpr (K == 9 || K == 11) {
                    int st = 2;  // unflagged: level A passed and g is an impulse -> the median (values span 0..255)
                    if (e & FAST_FLAG) {
                        st = level_radix_full<K>(B, geo, ty, tx, &o);
                    } else {
                        o = level_radix_median<K, true>(B, geo, ty, tx);
                    }
                    if (st) out(sl, pix, o, K);
                    keep = st == 0;
                    if constexpr (INL && K == 9) {
                        if (keep) {
                            if (level_radix_full<11>(B, geo, ty, tx, &o)) out(sl, pix, o, 11);
                            keep = false;
                        }
                    }
                } else {
                    keep = true;  // generic levels: fast_pass_generic
                }
            }
            if (!last && !(INL && K == 9)) {
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
                if (bal) {
                    int qb = 0;
                    if (lane == 0) qb = atomicAdd(cMn, __popc(bal));
                    qb = __shfl_sync(0xFFFFFFFFu, qb, 0);
                    if (keep) Y[CAP - 1 - (qb + __popc(bal & below))] = (uint16_t)(e | FAST_FLAG);
                }
            }
        }
    }
}

// Pass B of level K (9 or 11) in the interval where the k = smax - 2 and k = smax median passes run side by side:
// one pixel per lane pair (radix_median_pair), 16 per warp round.  Nothing is queued here: FRONT (K = smax) is the
// last level, and a flagged pixel that fails the generic level K = smax - 2 takes level smax at once (out of line).
template <bool FIN, int NTHR, int CAP, int K, bool FRONT, class Slot, class Out>
__device__ __forceinline__ void fast_pass_b_pair(Slot slot, const GGeo& geo, const uint16_t* X, int nM, int wrot, Out out) {
    constexpr int NWARP = NTHR / 32;
    const int lane = threadIdx.x & 31, warp = ((threadIdx.x >> 5) + NWARP - wrot) % NWARP;
    const int half = lane & 1;
    for (int base = warp * 16; base < nM; base += NWARP * 16) {
        const int idx = base + (lane >> 1);
        const bool act = idx < nM;
        const int j = act ? idx : nM - 1;
        const int e = FRONT ? X[j] : X[CAP - 1 - j];
        const int sl = (e >> 12) & 7, pix = e & 4095, ty = pix >> 7, tx = pix & 127;
        const uint8_t* B = slot(sl);
        const uint32_t med = radix_median_pair<K>(B, geo, ty, tx, half);
        if (act && half == 0) {
            if (!(e & FAST_FLAG)) {
                out(sl, pix, (uint8_t)med, K);
            } else {
                uint8_t o = 0;
                if (level_radix_full<K>(B, geo, ty, tx, &o)) {
                    out(sl, pix, o, K);
                } else if constexpr (!FRONT && K == 9) {
                    if (level_radix_full<11>(B, geo, ty, tx, &o)) out(sl, pix, o, 11);
                }
            }
        }
    }
}

// Levels k >= 13 (beyond the plane tests and the unrolled selects): every entry of S_k (front of X) and
// M_k (tail of X) takes the generic level; failures move to M_k+2 (tail of Y).
template <int NTHR, int CAP, class Slot, class Out>
__device__ __forceinline__ void fast_pass_generic(Slot slot, const GGeo& geo, const uint16_t* X, uint16_t* Y, int nS, int nM,
                                                  int* cMn, int k, bool last, Out out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t below = (1u << lane) - 1u;
    for (int base = warp * 32; base < nS + nM; base += NTHR) {
        const int i = base + lane;
        bool keep = false;
        int e = 0;
        if (i < nS + nM) {
            e = i < nS ? X[i] : X[CAP - 1 - (i - nS)];
            const int sl = (e >> 12) & 7, pix = e & 4095;
            uint8_t o = 0;
            if (level_generic(slot(sl), geo, pix >> 7, pix & 127, k, &o)) out(sl, pix, o, k);
            else keep = true;
        }
        if (!last) {
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, keep);
            if (bal) {
                int qb = 0;
                if (lane == 0) qb = atomicAdd(cMn, __popc(bal));
                qb = __shfl_sync(0xFFFFFFFFu, qb, 0);
                if (keep) Y[CAP - 1 - (qb + __popc(bal & below))] = (uint16_t)(e | FAST_FLAG);
            }
        }
    }
}

// Growth levels with the plane shortcut, after dense_level5 and the queue build: Q0 holds S_7 at its
// front (qcount[2] entries) and M_5 at its tail (qcount[1]); qcount[3..] zero.  Interval i runs pass B of
// level kB = 5 + 2 i and pass A of level kB + 2 between two barriers (both read one buffer and write
// the other; the selection network of one level and the plane test of the next share the instruction
// cache, and the short tests fill the median pass's tail).  CTA-wide; ends with __syncthreads.
template <bool FIN, int NTHR, int CAP, class Slot, class PlaneOf, class Out, int NETMAX = HYB_GROW_NETMAX>
__device__ __forceinline__ void grow_levels_fast(Slot slot, PlaneOf plane, const GGeo& geo, uint16_t* Q0, uint16_t* Q1,
                                                 int* qcount, int smax, Out out) {
    constexpr int NWARP = NTHR / 32;
    constexpr bool PAIRS = HYB_FAST_PAIRS != 0;
    bool chained = false;  // the previous interval's pass A covered the last two levels: X's front list is M_kA
    for (int i = 0;; ++i) {
        const int kB = 5 + 2 * i, kA = kB + 2;
        if (kB > smax) break;
#ifdef HYB_TRACE
        unsigned long long t_iv = 0;
        if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_iv));
#endif
        const uint16_t* X = (i & 1) ? Q1 : Q0;
        uint16_t* Y = (i & 1) ? Q0 : Q1;
        const int nM = qcount[2 * i + 1], nS = kA <= smax ? qcount[2 * i + 2] : 0;
        int* cMn = &qcount[2 * i + 3];  // |M_kA|
        int* cSn = &qcount[2 * i + 4];  // |S_kA+2|
        const bool lastB = kB + 2 > smax, lastA = kA + 2 > smax;
        if (kB > 11) {
            // S_kB is empty unless this is the first generic level (pass A below routes everything to M)
            fast_pass_generic<NTHR, CAP>(slot, geo, X, Y, 0, nM, cMn, kB, lastB, out);
        } else if (kB == 5) {
            fast_pass_b<FIN, NTHR, CAP, 5, NETMAX, false, false>(slot, geo, X, Y, nM, cMn, lastB, 0, out);
        } else if (kB == 7) {
            if (chained) fast_pass_b<FIN, NTHR, CAP, 7, NETMAX, false, true>(slot, geo, X, Y, nM, cMn, lastB, 0, out);
            else fast_pass_b<FIN, NTHR, CAP, 7, NETMAX, false, false>(slot, geo, X, Y, nM, cMn, lastB, 0, out);
        } else if (kB == 9) {
            if (chained && PAIRS && NETMAX < 9) fast_pass_b_pair<FIN, NTHR, CAP, 9, false>(slot, geo, X, nM, 0, out);
            else if (chained) fast_pass_b<FIN, NTHR, CAP, 9, NETMAX, false, true>(slot, geo, X, Y, nM, cMn, lastB, 0, out);
            else fast_pass_b<FIN, NTHR, CAP, 9, NETMAX, false, false>(slot, geo, X, Y, nM, cMn, lastB, 0, out);
        } else {
            fast_pass_b<FIN, NTHR, CAP, 11, NETMAX, false, false>(slot, geo, X, Y, nM, cMn, lastB, 0, out);
        }
        // the warps with one median round fewer start the second pass
        const int per = (kB <= NETMAX && kB <= 9) ? 64 : (chained && PAIRS && kB == 9) ? 16 : 32;
        const int wrot = ((nM + per - 1) / per) % NWARP;
        const bool chain = !chained && kA + 2 == smax && smax <= 11;
        if (chained) {
            // kA = smax: the medians of the front list, beside pass B of kB
            if (PAIRS && NETMAX < 9) {
                if (kA == 9) fast_pass_b_pair<FIN, NTHR, CAP, 9, true>(slot, geo, X, nS, wrot, out);
                else fast_pass_b_pair<FIN, NTHR, CAP, 11, true>(slot, geo, X, nS, wrot, out);
            } else if (kA == 9) {
                fast_pass_b<FIN, NTHR, CAP, 9, NETMAX, true, false>(slot, geo, X, Y, nS, cMn, true, wrot, out);
            } else {
                fast_pass_b<FIN, NTHR, CAP, 11, NETMAX, true, false>(slot, geo, X, Y, nS, cMn, true, wrot, out);
            }
        } else if (nS > 0) {
            if (kA == 7) {
                if (chain) fast_pass_a<FIN, NTHR, CAP, 7, true>(slot, plane, geo, X, Y, nS, cSn, cMn, lastA, wrot, out);
                else fast_pass_a<FIN, NTHR, CAP, 7, false>(slot, plane, geo, X, Y, nS, cSn, cMn, lastA, wrot, out);
            } else if (kA == 9) {
                if (chain) fast_pass_a<FIN, NTHR, CAP, 9, true>(slot, plane, geo, X, Y, nS, cSn, cMn, lastA, wrot, out);
                else fast_pass_a<FIN, NTHR, CAP, 9, false>(slot, plane, geo, X, Y, nS, cSn, cMn, lastA, wrot, out);
            } else if (kA == 11) {
                fast_pass_a<FIN, NTHR, CAP, 11, false>(slot, plane, geo, X, Y, nS, cSn, cMn, lastA, wrot, out);
            } else {
                fast_pass_a<FIN, NTHR, CAP, 13, false>(slot, plane, geo, X, Y, nS, cSn, cMn, lastA, wrot, out);
            }
        }
        chained = chain;
        __syncthreads();
#ifdef HYB_TRACE
        // fast-level profile (kernel id 1): slots 5 + i += interval time (pass B of k = 5 + 2 i, pass A of k + 2)
        if (threadIdx.x == 0 && blockIdx.x < 1024 && i < 4) {
            unsigned long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            g_trace[(1024 + blockIdx.x) * 16 + 5 + i] += t1 - t_iv;
        }
#endif
        if (*cMn == 0 && (lastA || *cSn == 0)) break;  // (after a chained pass A, *cSn = |M_smax|)
    }
}

// Growth over the failure range [gbeg, gend) of the weighted record order (records: (offset << 24) |
// tile, offsets increasing; record r spans REC_W units for its tile load, then its failures): batches
// of up to GSLOTS tile segments / GCAP failures; each segment's tile (+ R halo) is TMA-loaded into
// its own slot, its failures (bitmap bits with in-tile rank in the segment) are pooled into one queue
// and the levels run over the whole pool (grow_levels).  CTA-wide (NTHR threads); out(si, pix, v, k)
// stores a result, si = {x0, y0, z, ...} of the pixel's tile.  `phases` carries the slot mbarrier
// parities across calls.
struct GrowSmem {
    uint64_t* bar;   // [SLOTS] tile slots (initialised by the caller)
    int* sinfo;      // [SLOTS][8]: x0 y0 z tile lo hi qbase border -- the batch being grown
    long long* cur;  // [4]: record, position of the next choice, end of the claimed range, static range taken
    int* ctl;        // [4]: segments, queue n, more, bitmaps issued -- the batch being grown
    int* qcount;     // [MAX_LEVELS]
    uint8_t* bufs;   // [SLOTS][geo.b_bytes]
    uint16_t* Q0;    // [CAP]
    uint16_t* Q1;    // [CAP]
    int* sinfo_n;    // [SLOTS][8] the next batch (chosen one batch ahead)
    int* ctl_n;      // [4]
    uint32_t* bms;   // [SLOTS][128] the next batch's failure bitmaps (bulk-copied ahead)
    uint64_t* bmbar; // [1] their mbarrier (initialised by the caller)
    uint2* planes = nullptr;  // [SLOTS][pstride] zero / 255 bit planes (nullptr: plain grow_levels); with planes,
                              // bms is [2][SLOTS][128] and bmbar [2]: the bitmaps stay until the dense k = 5 pass
    int pstride = 0;          // plane words per slot (>= BH * BS / 32 + 1)
};

template <bool FIN, int NTHR, class Out, int SLOTS = GSLOTS, int CAP = GCAP, int NETMAX = HYB_GROW_NETMAX,
          bool DYN = true, long long CHUNK = CAP>
__device__ __forceinline__ void grow_range(const CUtensorMap* tm, const GGeo& geo, const GrowSmem& sm,
                                           const uint8_t* bitmap, const unsigned long long* records, long long R,
                                           long long T, const int* chunk_rec, int* chunk_ctr, int per_slice,
                                           int tiles_x, int row_begin, int rows, int cols, int smax,
                                           uint32_t& phases, Out out) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NWARP = NTHR / 32;
    uint64_t* bar = sm.bar;
    int* sinfo = sm.sinfo;
    long long* cur = sm.cur;
    int* ctl = sm.ctl;
    int* qcount = sm.qcount;
    uint8_t* bufs = sm.bufs;
    uint16_t* Q0 = sm.Q0;
    uint16_t* Q1 = sm.Q1;
    uint32_t bmphase = 0;
#ifdef HYB_TRACE
    // growth batch profile (kernel id 1): slot 1 += promotion + tile loads issued, 2 += queue build,
    // 3 += tile wait + edges, 4 += batches, 13 += kernel entry to the first batch
    unsigned long long tt0 = 0, tt1 = 0;
    auto tnow = [] { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; };
    auto tacc = [&](int slot) {
        if (tid == 0 && blockIdx.x < 1024) { tt1 = tnow(); g_trace[(1024 + blockIdx.x) * 16 + slot] += tt1 - tt0; tt0 = tt1; }
    };
    if (tid == 0) tt0 = tnow();
#define GTRACE(slot) tacc(slot)
#else
#define GTRACE(slot) do {} while (0)
#endif
    if (tid == 0) {
        cur[0] = 0;
        cur[1] = 0;
        cur[2] = 0;  // nothing claimed yet
        cur[3] = 0;  // static range not taken yet
    }
    // Work split: the first 3/4 of the chunks (CHUNK weighted units each) are split statically, CTA j
    // taking a contiguous run; with DYN the rest is claimed chunk by chunk from a global counter by
    // whichever CTA runs out first -- the cost of a failure depends on how deep it grows, which no
    // static split sees (config 4: static-only CTAs finished 1.70 .. 2.22 ms; with the dynamic quarter
    // 2.03 .. 2.17 ms and a 3 % shorter step).  Without DYN everything is static (configs 2 / 3, where
    // the failures are shallow and a claimed chunk's half-filled batches cost more than the tail).
    const long long nchunks = (T + CHUNK - 1) / CHUNK, nstatic = DYN ? nchunks * HYB_STATIC_Q / 4 : nchunks;
    __syncthreads();

    // One warp chooses the next batch (lane l: record cur + l) into sinfo_n / ctl_n and bulk-copies its
    // tiles' failure bitmaps into bms.  Positions are weighted: record r spans [off, next) = REC_W units
    // for its tile load, then its failures.  Work is claimed in chunks of CHUNK weighted units from a
    // global counter (chunk_rec gives each chunk's first record), so CTAs that meet cheap failures take
    // more chunks -- the cost of a failure depends on how deep it grows, which no static split sees.
    const bool dbl = sm.planes != nullptr;  // two bitmap buffers
    auto choose = [&](int nbuf) {
        uint32_t* bms_n = sm.bms + nbuf * SLOTS * 128;
        uint64_t* bmbar_n = sm.bmbar + nbuf;
        if (cur[1] >= cur[2]) {  // range exhausted: the static run, then chunks from the counter
            bool have = false;
            if (!cur[3]) {
                // static run: [Ts j / G, Ts (j + 1) / G) of the first Ts weighted units; its first record by a
                // 32-ary search (the last record whose offset is <= the start)
                const long long Ts = min(T, nstatic * CHUNK);
                const long long b0 = Ts * blockIdx.x / gridDim.x, b1 = Ts * (blockIdx.x + 1) / gridDim.x;
                have = b0 < b1;
                long long lo = 0, hi = R;
                while (have && hi - lo > 1) {
                    const long long step = (hi - lo + 31) / 32, idx = lo + lane * step;
                    const bool le = idx < hi && rec_off(records, idx) <= b0;
                    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, le);
                    lo += (31 - __clz(bal)) * step;  // lane 0 always qualifies
                    hi = min(hi, lo + step);
                }
                __syncwarp();
                if (lane == 0) {
                    cur[3] = 1;
                    if (have) {
                        cur[0] = lo;
                        cur[1] = b0;
                        cur[2] = b1;
                    }
                }
                __syncwarp();
            }
#if HYB_GUIDED
            if (!have && DYN) {
                // guided dynamic claims: k table units of 2048 (the k = 3 kernel's chunk table granularity),
                // k = remaining units / (2 x CTAs) clamped to [1, CHUNK / 2048] -- big claims first, single units
                // at the end, so the CTAs' finishing times close up (config 4 AMF 2.127 -> 2.096 ms with CHUNK 2^15;
                // 4 x CTAs: 2.134, 1 x: 2.116 at CHUNK 2^13; half the work static: 2.170; strips of N = 4 / 8:
                // 790 -> 764 / 440 -> 423 us)
                constexpr long long U = 2048;
                const long long Ts = min(T, nstatic * CHUNK), nu = (T - Ts + U - 1) / U;
                long long c = 0, k = 1;
                if (lane == 0) {
                    const long long rem = nu - (long long)*(volatile int*)chunk_ctr;
                    const long long d = (long long)HYB_GUIDED_DIV * gridDim.x;
                    k = min(max((rem + d - 1) / d, 1ll), CHUNK / U);
                    c = atomicAdd(chunk_ctr, (int)k);
                }
                c = __shfl_sync(0xFFFFFFFFu, c, 0);
                k = __shfl_sync(0xFFFFFFFFu, k, 0);
                if (c >= nu) {
                    if (lane == 0) {
                        sm.ctl_n[0] = 0;
                        sm.ctl_n[1] = 0;
                        sm.ctl_n[2] = 0;  // no more work
                    }
                    __syncwarp();
                    return;
                }
                if (lane == 0) {
                    cur[0] = __ldcg(chunk_rec + ((Ts + c * U) >> 11));
                    cur[1] = Ts + c * U;
                    cur[2] = min(Ts + (c + k) * U, T);
                }
                __syncwarp();
            } else
#endif
            if (!have) {
                long long ch = nchunks;  // without DYN: no dynamic chunks
                if (DYN) {
                    if (lane == 0) ch = nstatic + atomicAdd(chunk_ctr, 1);
                    ch = __shfl_sync(0xFFFFFFFFu, ch, 0);
                }
                if (ch >= nchunks) {
                    if (lane == 0) {
                        sm.ctl_n[0] = 0;
                        sm.ctl_n[1] = 0;
                        sm.ctl_n[2] = 0;  // no more work
                    }
                    __syncwarp();
                    return;
                }
                if (lane == 0) {
                    cur[0] = __ldcg(chunk_rec + ch);
                    cur[1] = ch * CHUNK;
                    cur[2] = min((ch + 1) * CHUNK, T);
                }
                __syncwarp();
            }
        }
        const long long gend = cur[2];
        const long long rec = cur[0] + lane, pos = cur[1];
        long long take = 0, off = 0, nxt = 0, flo = 0, whi = 0;
        int tile = 0;
        bool valid = false;
        if (rec < R && lane < SLOTS) {
            const unsigned long long rv = __ldcg(records + rec);
            off = (long long)(rv >> 24);
            tile = (int)(rv & 0xFFFFFFu);
            nxt = rec + 1 < R ? rec_off(records, rec + 1) : T;
            const long long wlo = max(off, pos);
            whi = min(nxt, gend);
            valid = wlo < whi;
            const long long c = nxt - off - REC_W;  // failures of the tile
            flo = min(max(wlo - off - REC_W, 0ll), c);
            take = valid ? min(max(whi - off - REC_W, 0ll), c) - flo : 0;
        }
        // inclusive prefix of the segment sizes, capped by the queue capacity
        long long incl = take;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const long long v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
            if (lane >= d) incl += v;
        }
        const long long excl = incl - take;
        const bool within = valid && excl < CAP;
        const long long mine = within ? min(take, (long long)CAP - excl) : 0;
        const uint32_t segs = __ballot_sync(0xFFFFFFFFu, mine > 0);
        const uint32_t inside = __ballot_sync(0xFFFFFFFFu, within);  // lanes 0..k (lane 0 always)
        const int ns = __popc(segs);
        if (lane == 0 && ns) mbar_expect_tx(bmbar_n, (uint32_t)(ns * 512));
        __syncwarp();
        if (mine > 0) {
            const int sl = __popc(segs & ((1u << lane) - 1u));
            const int z = tile / per_slice, rem = tile - z * per_slice, by = rem / tiles_x;
            int* si = sm.sinfo_n + 8 * sl;
            si[0] = (rem - by * tiles_x) * TW;
            si[1] = row_begin + by * TH;
            si[2] = z;
            si[3] = tile;
            si[4] = (int)flo;  // in-tile failure rank range [lo, hi)
            si[5] = (int)(flo + mine);
            si[6] = (int)excl;  // queue base
            const int sx0 = si[0] - geo.CP, sy0 = si[1] - geo.R;
            si[7] = sx0 < 0 || sx0 + geo.BS > cols || sy0 < 0 || sy0 + geo.BH > rows;
            fence_proxy_async_smem();  // the previous batch's generic reads of bms before the async write
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
                    smem_u32(bms_n + 128 * sl)),
                "l"(bitmap + (size_t)tile * 512), "r"(smem_u32(bmbar_n))
                : "memory");
        }
        const int last = 31 - __clz(inside);
        if (lane == last) {
            const long long end_pos = mine == take ? whi : off + REC_W + flo + mine;
            cur[1] = end_pos;
            cur[0] = rec + (end_pos >= nxt ? 1 : 0);
            sm.ctl_n[0] = ns;
            sm.ctl_n[1] = (int)(excl + mine);
            sm.ctl_n[2] = 1;  // the next choice claims a new chunk or reports the end
        }
        __syncwarp();
    };
    if (warp == 0) choose(0);
    __syncthreads();
    GTRACE(13);

    for (int it = 0;; ++it) {
        const int cb = dbl ? (it & 1) : 0, nbuf = dbl ? ((it + 1) & 1) : 0;  // this batch's / the next batch's bitmaps
        // ---- 1. promote the chosen batch; warp 0 issues its tile loads ----
        if (tid < MAX_LEVELS) qcount[tid] = 0;
        if (tid < 8 * SLOTS) sinfo[tid] = sm.sinfo_n[tid];
        if (tid < 3) ctl[tid] = sm.ctl_n[tid];
        __syncthreads();
        const int ns = ctl[0];
        const bool more = ctl[2] != 0;
        if (ns == 0) {  // only tile-load weight in this stretch of the range
            if (!more) break;
            if (warp == 0) choose(nbuf);
            __syncthreads();
            continue;
        }
        if (warp == 0 && lane < ns) {
            const int* si = sinfo + 8 * lane;
            fence_proxy_async_smem();  // the slot's previous generic reads/writes before the async write
            grow_tile_load(tm, geo, bufs + (size_t)lane * geo.b_bytes, &bar[lane], si[0], si[1], si[2]);
        }
        GTRACE(1);
        // ---- 2. queue: warp w collects slot w's failures with in-tile rank in [lo, hi) (with planes: after
        //      the dense k = 5 pass below, from its bitmaps) ----
        if (!dbl) {
        if (warp < ns) {
            mbar_wait_warp(sm.bmbar, bmphase);
            const int* si = sinfo + 8 * warp;
            const uint4 w4 = reinterpret_cast<const uint4*>(sm.bms + 128 * warp)[lane];
            const uint32_t wb[4] = {w4.x, w4.y, w4.z, w4.w};
            const int nf = __popc(w4.x) + __popc(w4.y) + __popc(w4.z) + __popc(w4.w);
            int incl = nf;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= d) incl += v;
            }
            int rank = incl - nf;
            const int lo = si[4], hi = si[5], qb = si[6] - lo;
            const uint32_t sbase = (uint32_t)warp << 12;
            if (rank < hi && incl > lo) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int w = lane * 4 + j;  // bitmap word: tile row w >> 2, columns 32 (w & 3) ..
                    const uint32_t base = sbase | (uint32_t)((w >> 2) * TW + 32 * (w & 3));
                    uint32_t bits = wb[j];
                    while (bits) {
                        const int b = __ffs(bits) - 1;
                        bits &= bits - 1;
                        if (rank >= lo && rank < hi) Q0[qb + rank] = (uint16_t)(base + b);
                        ++rank;
                    }
                }
            }
        }
        bmphase ^= 1u;
        __syncthreads();  // bms consumed
        }
        GTRACE(2);
        // ---- 3. the last warp chooses the next batch (its record loads and bitmap copies overlap the
        //      tile wait and the levels); tiles landed; border tiles get edge replication ----
        if (warp == NWARP - 1) choose(nbuf);
        for (int sl = 0; sl < ns; ++sl) mbar_wait(&bar[sl], (phases >> sl) & 1u);
        phases ^= (1u << ns) - 1u;
        bool anyb = false;
        for (int sl = 0; sl < ns; ++sl) {
            if (!sinfo[8 * sl + 7]) continue;  // uniform
            anyb = true;
            const int sx0 = sinfo[8 * sl] - geo.CP, sy0 = sinfo[8 * sl + 1] - geo.R;
            replicate_edges<NTHR>(bufs + (size_t)sl * geo.b_bytes, geo.BS, max(0, -sx0), min(geo.BS, cols - sx0),
                                  max(0, -sy0), min(geo.BH, rows - sy0), 0, geo.BH, geo.R);
        }
        if (anyb || !dbl) __syncthreads();  // (every thread waited for the tiles itself)
        GTRACE(3);
        // ---- 4. levels, pooled over the batch ----
        int n = ctl[1];
        auto slot_out = [&](int sl, int pix, uint8_t v, int k) { out(sinfo + 8 * sl, pix, v, k); };
        if (sm.planes) {
            build_planes<NTHR>(bufs, geo, sm.planes, sm.pstride, ns);
            __syncthreads();
            GTRACE(9);
            // warp w: the dense k = 5 pass of slot w, then its queue entries -- S_7 at the front of Q0, M_5 at its
            // tail (slot order as the warps arrive); the row masks stay in registers
            if (warp < ns) {
                mbar_wait_warp(sm.bmbar + cb, (bmphase >> cb) & 1u);
                uint4 m4, s4;
                dense_level5<FIN>(sm.planes + (size_t)warp * sm.pstride, geo, sm.bms + (cb * SLOTS + warp) * 128,
                                  sinfo[8 * warp + 4], sinfo[8 * warp + 5], m4, s4);
                const uint32_t mb[4] = {m4.x, m4.y, m4.z, m4.w}, sb[4] = {s4.x, s4.y, s4.z, s4.w};
                const int mine = (__popc(s4.x) + __popc(s4.y) + __popc(s4.z) + __popc(s4.w)) |
                                 ((__popc(m4.x) + __popc(m4.y) + __popc(m4.z) + __popc(m4.w)) << 16);
                int incl = mine;  // open count | medians << 16 (each <= 4096)
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                    if (lane >= d) incl += v;
                }
                const int tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
                int bS = 0, bM = 0;
                if (lane == 0) {
                    bS = atomicAdd(&qcount[2], tot & 0xFFFF);
                    bM = atomicAdd(&qcount[1], tot >> 16);
                }
                bS = __shfl_sync(0xFFFFFFFFu, bS, 0);
                bM = __shfl_sync(0xFFFFFFFFu, bM, 0);
                int rs = bS + ((incl - mine) & 0xFFFF), rm = CAP - 1 - (bM + ((incl - mine) >> 16));
                const uint32_t sbase = ((uint32_t)warp << 12) | (uint32_t)(lane * TW);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint32_t bits = sb[j];
                    while (bits) {
                        const int b = __ffs(bits) - 1;
                        bits &= bits - 1;
                        Q0[rs++] = (uint16_t)(sbase + 32 * j + b);
                    }
                    bits = mb[j];
                    while (bits) {
                        const int b = __ffs(bits) - 1;
                        bits &= bits - 1;
                        Q0[rm--] = (uint16_t)(sbase + 32 * j + b);
                    }
                }
            }
            bmphase ^= 1u << cb;
            __syncthreads();
            GTRACE(11);
            auto slot = [&](int sl) { return bufs + (size_t)sl * geo.b_bytes; };
            auto plane = [&](int sl) { return sm.planes + (size_t)sl * sm.pstride; };
            grow_levels_fast<FIN, NTHR, CAP, decltype(slot), decltype(plane), decltype(slot_out), NETMAX>(
                slot, plane, geo, Q0, Q1, qcount, smax, slot_out);
        } else {
            grow_levels<FIN, NTHR, decltype(slot_out), NETMAX>(bufs, geo, Q0, Q1, qcount, n, smax, slot_out);
        }
        __syncthreads();  // slots, queues and counters are reused by the next batch
#ifdef HYB_TRACE
        if (tid == 0 && blockIdx.x < 1024) g_trace[(1024 + blockIdx.x) * 16 + 4] += 1;
        if (tid == 0) tt0 = tnow();
#endif
    }
#undef GTRACE
}

}  // namespace
}  // namespace hyb
