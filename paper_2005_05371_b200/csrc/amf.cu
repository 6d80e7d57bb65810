// amf.cu -- adaptive median filter (AMF) for sm_100a.
//
// Semantics: detail::adaptive_median_rows, reference proj/src/adaptive_median.cpp:123-215
// (windows k = 3..smax over the pristine input, edge replication, level A/B, unresolved pixels
// keep their input).  Design:
//
//   * amf_k3_kernel (persistent, 8 compute warps + 1 producer warp): 95-99.7 % of pixels finalise
//     at k = 3, so k = 3 runs on every pixel.  The producer claims 128 x 32 tiles and TMA-loads
//     them (+ 1-pixel halo) into a 4-deep full/empty mbarrier ring; compute warps claim 4-row
//     strips (amf_core.cuh k3_strip: u16x2 row pairs, column sorts reused by 3 outputs, level A/B
//     as lane masks).  Level-A failures go to a per-tile bitmap; the tile's last strip appends one
//     weighted work record (64-bit atomic).
//   * amf_grow_kernel (persistent): every CTA takes an equal weighted range of the records, loads
//     the tiles it touches (+ R halo) by TMA, pools their failures in shared memory and runs the
//     levels k = 5..smax over the pool (amf_core.cuh grow_range / grow_levels): pruned selection
//     networks on u16x2 pairs for k = 5, 7; SWAR level-A counts + radix select for k >= 9.
#include <cuda.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "amf_core.cuh"
#include "hyb_internal.cuh"
#include "tma.cuh"
#include "trace.cuh"

namespace hyb {
namespace {

#ifndef HYB_COMPACT_T_DEF
#define HYB_COMPACT_T_DEF 32  // strips with at most this many level-A failures use compact growth entries
#endif
constexpr int KHMAX = 3;         // largest k = 3 tile halo (3 rows: compact growth windows, amf_core.cuh CompactOut)
constexpr int BBYTES = (BS * (TH + 2 * KHMAX) + 127) / 128 * 128;  // ring slot (TMA destinations 128-byte aligned)
constexpr int NBUF = 4;          // TMA ring depth
constexpr int HDR = 384;         // mbarriers, counters, tile coordinates, per-strip failure counts
constexpr int K3T = NT + 32;     // + one producer warp (tile claims and TMA loads)
constexpr int WAREA = 2 * WPIX;  // per warp: output strip, finalized_at strip
constexpr size_t SMEM = HDR + NBUF * BBYTES + NW * WAREA + 128;

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
    int grow;                // record level-A failures (smax >= 5)
    uint8_t* bitmap;         // per tile 32 rows x 16 bytes: bit c%8 of byte c/8 = pixel (row, c) failed level A
    int dynamic;             // tiles claimed from `claim` (else blockIdx.x + i * gridDim.x)
    int* claim;              // global tile-claim counter (reset by the last CTA to finish)
    int* done;               // CTAs finished
    unsigned long long* rec_ctr;  // (records << 40) | weighted failures (+REC_W per tile), once per tile with failures
    unsigned long long* records;  // [record] = (weighted offset << 24) | tile
    int* chunk_rec;               // [chunk] = record holding weighted position chunk << chunk_shift
    int chunk_shift;              // log2 of the growth chunk (the growth variant's queue capacity)
    int halo;                     // tile rows loaded above / below: 1, or 3 with compact windows
    uint4* cq;                    // compact growth entries (nullptr: bitmaps only)
    int* cq_ctr;
    int cq_cap, cq_thresh;
    int out_rows;
};


__device__ __forceinline__ void issue_tile_load(const CUtensorMap* tm, uint8_t* Bbuf, uint64_t* bar, int x0, int y0,
                                                int z, int halo) {
    mbar_expect_tx(bar, BS * (TH + 2 * halo));
    tma_load_3d(Bbuf, tm, bar, x0 - CP, y0 - halo, z);
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
__global__ void __launch_bounds__(K3T, 3)
    amf_k3_kernel(const __grid_constant__ CUtensorMap tm_src, const __grid_constant__ K3Args args) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);        // [NBUF] tile landed (or: no tile)
    uint64_t* empty = reinterpret_cast<uint64_t*>(smem + 32);  // [NBUF] all strips of the slot done
    int* done_cnt = reinterpret_cast<int*>(smem + 64);           // [NBUF] strips finished
    int* tinfo = reinterpret_cast<int*>(smem + 128);             // [NBUF][4]: x0, y0, z, tile (-1: none)
    int* fcnt = reinterpret_cast<int*>(smem + 256);              // [NBUF][NW] level-A failures per strip
    uint8_t* bufs = smem + HDR;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    const int rows = args.rows, cols = args.cols;
    const int ntiles = args.tiles_x * args.tiles_y * args.n_slices;

    if (tid == 0) {
        prefetch_tmap(&tm_src);
        for (int s = 0; s < NBUF; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], TH / WR);
            done_cnt[s] = 0;
        }
        fence_mbar_init();
    }
    __syncthreads();
    grid_dep_wait();  // the previous grid (e.g. the last step's gain reading dst) has completed
    TRACE(0, 0);

    if (warp == NW) {
        // ---- producer: claims tiles from the global counter in ring order (so the first empty
        //      claim ends the CTA's sequence) and TMA-loads them ----
        if (lane == 0) {
            for (int ti = 0;; ++ti) {
                const int s = ti & (NBUF - 1);
                if (ti >= NBUF) mbar_wait(&empty[s], (uint32_t)(ti / NBUF - 1) & 1u);
                // few tiles per CTA: static round-robin (a prefetching dynamic claimer would grab up
                // to NBUF tiles per CTA up front); many: dynamic claims balance the SMs
                const int t = args.dynamic ? atomicAdd(args.claim, 1) : (int)blockIdx.x + ti * (int)gridDim.x;
                if (t >= ntiles) {
                    tinfo[4 * s + 3] = -1;
                    mbar_arrive(&full[s]);
                    break;
                }
                tile_coords(args, t, tinfo + 4 * s);
                tinfo[4 * s + 3] = t;
                fence_proxy_async_smem();
                issue_tile_load(&tm_src, bufs + s * BBYTES, &full[s], tinfo[4 * s], tinfo[4 * s + 1],
                                tinfo[4 * s + 2], args.halo);
            }
            __threadfence();
            if (args.dynamic && atomicAdd(args.done, 1) == (int)gridDim.x - 1) {  // every CTA stopped claiming
                *args.claim = 0;
                *args.done = 0;
            }
        }
        return;
    }
    uint8_t* O = bufs + NBUF * BBYTES + warp * WAREA;
    uint8_t* F = O + WPIX;

    // Warp w takes strip w (rows 4w .. 4w + 3) of every tile of the ring: k = 3 costs the same on every
    // strip, so a static split balances without a strip-claim atomic per strip (the dynamic claim's atomics
    // held ~10 % of this kernel's stall samples, but the kernel is ALU-bound and measured the same time
    // either way -- configs 3 / 4 AMF 0.241 / 2.136 ms; the static split is the simpler code).
    const int sub = warp;
    for (int ti = 0;; ++ti) {
        const int s = ti & (NBUF - 1);
        mbar_wait_warp(&full[s], (uint32_t)(ti / NBUF) & 1u);
        const int t = tinfo[4 * s + 3];
        if (t < 0) break;
        const int x0 = tinfo[4 * s], y0 = tinfo[4 * s + 1], z = tinfo[4 * s + 2];
        const int H = args.halo;
        uint8_t* Bfull = bufs + s * BBYTES;  // row 0 = image row y0 - H
        uint8_t* B = Bfull + (H - 1) * BS;   // row 0 = image row y0 - 1

        // ---- border tiles: edge replication (this strip's rows, reach H) in place of TMA's zero fill ----
        const int sx0 = x0 - CP, sy0 = y0 - H, bh = TH + 2 * H;
        if (sx0 < 0 || sx0 + BS > cols || sy0 < 0 || sy0 + bh > rows)
            replicate_edges<32>(Bfull, BS, max(0, -sx0), min(BS, cols - sx0), max(0, -sy0), min(bh, rows - sy0),
                                sub * WR, sub * WR + WR + 2 * H, H);

        CompactOut co;
        if (args.cq) {
            co.ent = args.cq;
            co.ctr = args.cq_ctr;
            co.cap = args.cq_cap;
            co.thresh = args.cq_thresh;
            co.B = Bfull;
            co.x0 = (uint32_t)x0;
            co.key0 = (uint32_t)(z * args.out_rows + (y0 - args.row_begin));
        }
        const int nf = k3_strip<FIN>(B, O, F, sub, args.grow ? args.bitmap + (size_t)t * 512 : nullptr,
                                     args.dst + (size_t)z * args.dslice + (size_t)(y0 - args.row_begin) * args.dpitch + x0,
                                     args.dpitch,
                                     FIN ? args.fin + (size_t)z * args.fslice + (size_t)(y0 - args.row_begin) * args.fpitch + x0
                                         : nullptr,
                                     args.fpitch, args.row_end - y0, cols - x0, nullptr, nullptr, 0,
                                     args.cq ? &co : nullptr);

        // ---- release the slot; the tile's last strip publishes its failure record ----
        if (lane == 0) {
            fcnt[s * NW + sub] = nf;
            __threadfence_block();
            if (atomicAdd(&done_cnt[s], 1) == TH / WR - 1) {
                done_cnt[s] = 0;
                __threadfence_block();  // the other strips' counts (written before their done_cnt adds)
                int c = 0;
#pragma unroll
                for (int w = 0; w < NW; ++w) c += ((volatile int*)fcnt)[s * NW + w];
                if (c) {
                    const unsigned long long old =
                        atomicAdd(args.rec_ctr, (1ull << REC_SHIFT) | (unsigned)(c + REC_W));
                    const long long rec = (long long)(old >> REC_SHIFT), off = (long long)(old & REC_MASK);
                    args.records[rec] = ((unsigned long long)off << 24) | (unsigned)t;
                    // chunk boundaries inside this record's weighted span [off, off + c + REC_W)
                    const int sh = args.chunk_shift;
                    for (long long ch = (off + (1ll << sh) - 1) >> sh; ch <= (off + c + REC_W - 1) >> sh; ++ch)
                        args.chunk_rec[ch] = (int)rec;
                }
            }
            mbar_arrive(&empty[s]);
        }
    }
    TRACE(0, 15);
}

// ------------------------------------------------------------------------------------------
// growth kernel (k = 5..smax): tile-wise, all levels from shared memory
// ------------------------------------------------------------------------------------------

#ifndef HYB_GNT
#define HYB_GNT 256
#endif
constexpr int GNT = HYB_GNT;     // threads per growth CTA

constexpr int GHDR = 1536;       // mbarriers, tile coordinates, level counters, scan scratch


struct GArgs {
    GGeo geo;
    uint8_t* dst;
    size_t dpitch, dslice;
    uint8_t* fin;
    size_t fpitch, fslice;
    const uint8_t* bitmap;
    int rows, cols, row_begin, row_end, n_slices, smax;
    int tiles_x, tiles_y;    // k = 3 tiles
    unsigned long long* rec_ctr;        // written by amf_k3_kernel; reset here by the last CTA
    const unsigned long long* records;  // (failure offset << 24) | tile, offsets increasing
    const int* chunk_rec;               // [chunk] = record holding its first weighted position
    int* chunk_ctr;                     // growth chunk claims; reset here by the last CTA
    int* done;
    const uint4* cq;                    // compact entries of the sparse strips (nullptr: none)
    int* cq_ctr;                        // their count (may exceed cq_cap); reset here by the last CTA
    int* cq_claim;                      // compact chunk claims; reset here by the last CTA
    int cq_cap, out_rows;
    int fast;                           // plane words per slot of the fast growth levels (0: plain levels)
};


// Sparse growth, balanced by failures.  amf_k3_kernel publishes one record per tile with level-A
// failures (its failure offset in a global order); CTA j takes the failures [jT/G, (j+1)T/G) and
// walks the records covering them in batches of up to GSLOTS tile segments / GCAP failures: each
// segment's tile (+ R halo) is TMA-loaded into its own slot, its failures (bitmap bits whose
// in-tile rank falls in the segment) are pooled into one shared-memory queue (entry = slot << 12 |
// pixel), and every level round k = 5..smax runs over the whole pool.

// Two growth variants, chosen per call by smax: "wide" (k = 9 by selection network, 114 registers,
// 2 CTAs/SM, batches of 8 tiles / 8192 failures) pays off when the k = 9 level is dense (BASELINE
// config 4: smax 11, S&P 0.5); "lean" (networks up to k = 7, radix above, <= 80 registers, 3 CTAs/SM,
// batches of 8 tiles / 4096 failures) when it is sparse or absent (config 2: 6 % faster step).
template <int NETMAX_, int MINB_, int SLOTS_, int CAP_, bool DYN_, int CHUNK_SHIFT_, int NT_ = GNT>
struct GrowCfg {
    static constexpr int NETMAX = NETMAX_, MINB = MINB_, SLOTS = SLOTS_, CAP = CAP_;
    static constexpr int NT = NT_;     // threads per CTA
    static constexpr bool DYN = DYN_;  // dynamic last quarter of the work (amf_core.cuh grow_range)
    static constexpr int CHUNK_SHIFT = CHUNK_SHIFT_;  // log2 of a claim, in weighted units
};
#ifndef HYB_LEAN_DYN
#define HYB_LEAN_DYN 0
#endif
#ifndef HYB_WIDE_MINB
#define HYB_WIDE_MINB 2  // CTAs / SM
#endif
#ifndef HYB_WIDE_SLOTS
#define HYB_WIDE_SLOTS 8  // tiles per batch
#endif
#ifndef HYB_WIDE_CAP
#define HYB_WIDE_CAP 8192  // pooled queue capacity
#endif
#ifndef HYB_WIDE_CHUNK
#define HYB_WIDE_CHUNK 15  // log2 of the static chunk (the guided claims take at most this many units)
#endif
// With the bit-plane levels (amf_core.cuh grow_levels_fast) the k = 9 medians are few (config 4: ~270 per batch), so
// the wide variant keeps networks to k = 7 (80 registers) and spends the registers on 12 warps per CTA instead:
// measured config 4 AMF 1.864 ms (k = 9 network, 256 threads) / 1.860 (radix, 256) / 1.813 (radix, 384); 3 CTAs / SM of
// 5- or 6-tile batches 2.04 / 2.11 ms -- the pool size matters more than the warps.  On the final levels: 384 threads
// 1.739 ms, 448 (72 registers) 1.747, 512 (64 registers, small spills) 1.793; half the work static 1.751.
#ifndef HYB_WIDE_NETMAX
#define HYB_WIDE_NETMAX 7  // largest window the wide variant grows with a selection network
#endif
#ifndef HYB_WIDE_NT
#define HYB_WIDE_NT 384
#endif
using GrowWide = GrowCfg<HYB_WIDE_NETMAX, HYB_WIDE_MINB, HYB_WIDE_SLOTS, HYB_WIDE_CAP, true, HYB_WIDE_CHUNK, HYB_WIDE_NT>;
#ifndef HYB_LEAN_SLOTS
#define HYB_LEAN_SLOTS 8
#endif
#ifndef HYB_WIDE_MIN_SMAX
#define HYB_WIDE_MIN_SMAX 11  // smallest smax grown by the wide variant
#endif
#ifndef HYB_LEAN_CHUNK
#define HYB_LEAN_CHUNK 11
#endif
using GrowLean = GrowCfg<7, 3, HYB_LEAN_SLOTS, 4096, HYB_LEAN_DYN != 0, HYB_LEAN_CHUNK>;
static_assert(GrowWide::SLOTS <= 8 && GrowLean::SLOTS <= 8, "header layout");
static_assert(GrowWide::SLOTS <= GrowWide::NT / 32 && GrowLean::SLOTS <= GrowLean::NT / 32, "queue build: one warp per slot");
static_assert(GrowWide::CHUNK_SHIFT >= 11 && GrowLean::CHUNK_SHIFT >= 11, "chunk table sized for chunks >= 2048");

// plane words (uint2) per slot of the fast growth levels: one per 32 tile bytes, one of padding, 16-byte multiple
inline int plane_stride(const GGeo& g) { return (g.BH * (g.BS >> 5) + 2) & ~1; }

template <class C>
inline size_t grow_smem(const GGeo& g, bool fast = false) {
    return GHDR + (size_t)C::SLOTS * g.b_bytes + 2 * C::CAP * 2 + (size_t)C::SLOTS * 512 + 128 +
           (fast ? (size_t)C::SLOTS * (plane_stride(g) * 8 + 512) : 0);  // planes + the second bitmap buffer
}


template <bool FIN, class C>
__global__ void __launch_bounds__(C::NT, C::MINB) amf_grow_kernel(const __grid_constant__ CUtensorMap tm,
                                                      const __grid_constant__ GArgs args) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    const GGeo& geo = args.geo;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);            // [SLOTS]
    int* sinfo = reinterpret_cast<int*>(smem + 64);                // [SLOTS][8]: x0 y0 z tile lo hi qbase border
    long long* cur = reinterpret_cast<long long*>(smem + 320);     // [4] record, position, range end, static taken
    int* ctl = reinterpret_cast<int*>(smem + 368);                 // [4] segments, queue n, more
    int* qcount = reinterpret_cast<int*>(smem + 384);              // [MAX_LEVELS]
    uint8_t* bufs = smem + GHDR;
    uint16_t* Q0 = reinterpret_cast<uint16_t*>(bufs + (size_t)C::SLOTS * geo.b_bytes);
    uint16_t* Q1 = Q0 + C::CAP;
    int* sinfo_n = reinterpret_cast<int*>(smem + 1024);            // [SLOTS][8] next batch
    int* ctl_n = reinterpret_cast<int*>(smem + 1280);              // [4]
    uint64_t* bmbar = reinterpret_cast<uint64_t*>(smem + 1344);    // [2] next batch's bitmap copies
    uint32_t* bms = reinterpret_cast<uint32_t*>(Q1 + C::CAP);      // [SLOTS][128]
    uint64_t* cbar = reinterpret_cast<uint64_t*>(smem + 1416);     // [2] compact entry staging
    const int tid = threadIdx.x;
    const int per_slice = args.tiles_x * args.tiles_y;
    if (tid == 0) {
        for (int i = 0; i < C::SLOTS; ++i) mbar_init(&bar[i], 1);
        mbar_init(bmbar, 1);
        mbar_init(bmbar + 1, 1);
        mbar_init(&cbar[0], 1);
        mbar_init(&cbar[1], 1);
        prefetch_tmap(&tm);
        fence_mbar_init();
    }
    grid_dep_wait();  // records and bitmap come from the k = 3 grid
    const unsigned long long ctr = __ldcg(args.rec_ctr);
    const long long R = (long long)(ctr >> REC_SHIFT), T = (long long)(ctr & REC_MASK);
    uint32_t phases = 0;
    GrowSmem sm{bar, sinfo, cur, ctl, qcount, bufs, Q0, Q1, sinfo_n, ctl_n, bms, bmbar};
    if (args.fast) {  // zero / 255 bit planes behind the bitmaps (16-byte aligned)
        sm.planes = reinterpret_cast<uint2*>(bms + 2 * C::SLOTS * 128);
        sm.pstride = args.fast;
    }
    auto out = [&](const int* si, int pix, uint8_t v, int k) {
        const size_t row = (size_t)(si[1] - args.row_begin + (pix >> 7));
        args.dst[(size_t)si[2] * args.dslice + row * args.dpitch + si[0] + (pix & 127)] = v;
        if (FIN) args.fin[(size_t)si[2] * args.fslice + row * args.fpitch + si[0] + (pix & 127)] = (uint8_t)k;
    };
    // tile records first: the CTAs that have some join the compact chunk claims below late
    grow_range<FIN, C::NT, decltype(out), C::SLOTS, C::CAP, C::NETMAX, C::DYN, 1ll << C::CHUNK_SHIFT>(&tm, geo, sm, args.bitmap, args.records, R, T,
                                                                     args.chunk_rec, args.chunk_ctr, per_slice,
                                                                     args.tiles_x,
                                                                     args.row_begin, args.rows, args.cols, args.smax,
                                                                     phases, out);
    if (args.cq) {
        // The sparse strips' failures (compact entries): chunks of ch entries claimed from a global counter
        // (so CTAs busy with tile records above take fewer), bulk-copied into the tile slots, double-buffered;
        // k = 5 from shared memory, two entries per thread.  The entries still open are listed in shared
        // memory (Q0 / Q1 as int scratch) and get k = 7 from global memory on full warps afterwards (inline
        // when the list is full).
        __syncthreads();  // the slots and queues are free
        const int nc = min(__ldcg(args.cq_ctr), args.cq_cap);
        const uint4* cq = args.cq;
        int* sc = reinterpret_cast<int*>(smem + 1408);
        int* cclaim = reinterpret_cast<int*>(smem + 1432);  // [2] chunk in each staging buffer
        int* open7 = reinterpret_cast<int*>(Q0);
        constexpr int OCAP = C::CAP;  // 2 * CAP u16 = CAP ints
        const int ch = min((C::SLOTS * geo.b_bytes / 128) & ~1, 512);  // entries per staging buffer
        const int ntot = (nc + ch - 1) / ch;
        uint4* stg = reinterpret_cast<uint4*>(bufs);  // [2][ch] entries
        auto claim_issue = [&](int b) {
            const int c = atomicAdd(args.cq_claim, 1);
            cclaim[b] = c;
            if (c < ntot) {
                const int n = min(ch, nc - c * ch);
                mbar_expect_tx(&cbar[b], (uint32_t)n * 64);
                bulk_g2s(stg + (size_t)b * ch * 4, cq + (size_t)c * ch * 4, (uint32_t)n * 64, &cbar[b]);
            }
        };
        if (tid == 0) {
            *sc = 0;
            fence_proxy_async_smem();
            claim_issue(0);
            claim_issue(1);
        }
        __syncthreads();
        auto cout = [&](int k) {
            return [&, k](uint32_t x, uint32_t key, uint32_t v) {
                const uint32_t z = key / (uint32_t)args.out_rows, row = key - z * (uint32_t)args.out_rows;
                args.dst[(size_t)z * args.dslice + (size_t)row * args.dpitch + x] = (uint8_t)v;
                if (FIN) args.fin[(size_t)z * args.fslice + (size_t)row * args.fpitch + x] = (uint8_t)k;
            };
        };
        const int lane = tid & 31;
        for (int it = 0;; ++it) {
            const int b = it & 1, c = cclaim[b];
            if (c >= ntot) break;
            mbar_wait(&cbar[b], (uint32_t)(it >> 1) & 1u);
            const int n = min(ch, nc - c * ch);
            const uint4* sb = stg + (size_t)b * ch * 4;
            for (int p0 = 0; 2 * p0 < n; p0 += C::NT) {
                const int pi = p0 + tid;
                uint32_t pend = 0;
                int ia = 2 * pi, ib = 2 * pi + 1;
                if (ia < n) {
                    const bool hasb = ib < n;
                    if (!hasb) ib = ia;
                    pend = (sb[ia * 4 + 3].z != CQ_NONE ? 1u : 0u) | (hasb && sb[ib * 4 + 3].z != CQ_NONE ? 2u : 0u);
                    if (pend) pend = compact_level<5>(sb + ia * 4, sb + ib * 4, pend, cout(5));
                }
                if (args.smax >= 7) {
                    const uint32_t balA = __ballot_sync(0xFFFFFFFFu, pend & 1u);
                    const uint32_t balB = __ballot_sync(0xFFFFFFFFu, pend & 2u);
                    const int tot = __popc(balA) + __popc(balB);
                    int base = 0;
                    if (lane == 0 && tot) base = atomicAdd(sc, tot);
                    base = __shfl_sync(0xFFFFFFFFu, base, 0);
                    const uint32_t below = (1u << lane) - 1u;
                    const int pa = base + __popc(balA & below), pb = base + __popc(balA) + __popc(balB & below);
                    const int ga = c * ch + ia, gb = c * ch + ib;
                    if (base + tot <= OCAP) {
                        if (pend & 1u) open7[pa] = ga;
                        if (pend & 2u) open7[pb] = gb;
                    } else if (pend) {
                        compact_level<7>(cq + (size_t)ga * 4, cq + (size_t)gb * 4, pend, cout(7));
                    }
                }
            }
            fence_proxy_async_smem();  // this buffer's generic reads before its next bulk copy
            __syncthreads();           // (also publishes the claims made after the previous barrier)
            if (tid == 0) claim_issue(b);
        }
        __syncthreads();
        const int n7 = min(*sc, OCAP);
        for (int j = tid; 2 * j < n7; j += C::NT) {
            const int ia = open7[2 * j], ib = 2 * j + 1 < n7 ? open7[2 * j + 1] : ia;
            compact_level<7>(cq + (size_t)ia * 4, cq + (size_t)ib * 4, 2 * j + 1 < n7 ? 3u : 1u, cout(7));
        }
    }
    TRACE(1, 15);
    // the last CTA resets the record counter for the next k = 3 launch
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(args.done, 1) == (int)gridDim.x - 1) {
            *args.rec_ctr = 0;
            *args.chunk_ctr = 0;
            if (args.cq) {
                *args.cq_ctr = 0;
                *args.cq_claim = 0;
            }
            *args.done = 0;
        }
    }
}

// ------------------------------------------------------------------------------------------
// fused AMF kernel: k = 3 and the growth of a batch of tiles in one CTA
// ------------------------------------------------------------------------------------------
//
// The separate kernels above write f, record the level-A failures in a global bitmap, and reload every
// tile with failures (+ R halo) for the growth: the growth re-reads g (with halo), re-reads the bitmap
// and rewrites the f sectors it touches (read-for-ownership) -- 3.7x the image in DRAM reads at config 4.
// Here one CTA owns a batch of BT consecutive tiles end to end: TMA-loads them once with the growth halo
// R, runs the k = 3 strips (k3_strip: f stored, failures appended straight to a shared-memory queue),
// then the growth levels k = 5..smax over the batch's pooled queue from the resident tiles (grow_levels),
// whose f byte stores land in L2 lines the k = 3 stores of the same CTA just wrote.  g is read once, f
// written once; no bitmap, no records, no second launch.  Batches are claimed from a global counter, so
// SMs that meet cheap batches take more.  Tile geometry: R <= 16 (smax <= 33), so the k = 3 byte-tile
// layout (CP = 16, BS = 160) is the growth tile's.
template <int NETMAX_, int MINB_, int BT_, int NSET_, int CAP_>
struct FusedCfg {
    static constexpr int NETMAX = NETMAX_, MINB = MINB_, BT = BT_;
    static constexpr int NSET = NSET_;  // slot sets: 2 = the next batch's tiles load while this one computes
    // growth queue capacity (entries per buffer); below BT * 4096 the k = 3 pass runs tile by tile and the
    // growth runs whenever the queue could overflow on the next tile (and at the batch end)
    static constexpr int CAP = CAP_;
    static constexpr bool CAPPED = CAP_ < BT_ * TW * TH;
};
// Measured (config 2 / 3 / 4 AMF ms): one slot set with 3 / 4 tiles per batch 0.182 / 0.270 / 2.26; two sets
// (the next batch's tiles load during this one) with 2 / 3 tiles 0.197 / 0.286 / 2.47 -- the growth pool size
// matters more than the exposed load latency, which the co-resident CTAs cover.
#ifndef HYB_FUSED_BT_WIDE
#define HYB_FUSED_BT_WIDE 4
#endif
#ifndef HYB_FUSED_BT_LEAN
#define HYB_FUSED_BT_LEAN 3
#endif
#ifndef HYB_FUSED_NSET
#define HYB_FUSED_NSET 1
#endif
#ifndef HYB_FUSED_CAP_WIDE
#define HYB_FUSED_CAP_WIDE (HYB_FUSED_BT_WIDE * TW * TH)
#endif
#ifndef HYB_FUSED_CAP_LEAN
#define HYB_FUSED_CAP_LEAN (HYB_FUSED_BT_LEAN * TW * TH)
#endif
// k = 9 network (~115 registers): 2 CTAs / SM
using FusedWide = FusedCfg<9, 2, HYB_FUSED_BT_WIDE, HYB_FUSED_NSET, HYB_FUSED_CAP_WIDE>;
// networks to k = 7, radix above: 3 CTAs / SM
using FusedLean = FusedCfg<7, 3, HYB_FUSED_BT_LEAN, HYB_FUSED_NSET, HYB_FUSED_CAP_LEAN>;
static_assert(FusedWide::BT * FusedWide::NSET <= 16 && FusedLean::BT * FusedLean::NSET <= 16, "header layout");
static_assert(FusedWide::BT <= 8 && FusedLean::BT <= 8, "3-bit queue slots");
static_assert(FusedWide::CAP >= TW * TH && FusedLean::CAP >= TW * TH, "one tile's failures fit the queue");

constexpr int FHDR = 1024;  // mbarriers [16], tile info [16][4], level counters [128], batch claims [2]

struct FArgs {
    GGeo geo;
    uint8_t* dst;
    size_t dpitch, dslice;
    uint8_t* fin;
    size_t fpitch, fslice;
    int rows, cols, row_begin, row_end, n_slices, smax;
    int tiles_x, tiles_y;
    int* claim;  // batch claims (reset by the last CTA)
    int* done;
};

template <bool FIN, class C>
inline size_t fused_smem(const GGeo& g) {  // header, tile sets, k = 3 staging (+ finalized_at), two queues
    return FHDR + (size_t)C::NSET * C::BT * g.b_bytes + (size_t)NW * (FIN ? 2 : 1) * WPIX + 2 * (size_t)C::CAP * 2 +
           128;
}

template <bool FIN, class C>
__global__ void __launch_bounds__(NT, C::MINB) amf_fused_kernel(const __grid_constant__ CUtensorMap tm,
                                                              const __grid_constant__ FArgs a) {
    constexpr int BT = C::BT, NSET = C::NSET;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    const GGeo& geo = a.geo;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);     // [NSET][BT] tile loads
    int* tinfo = reinterpret_cast<int*>(smem + 128);        // [NSET][BT][4]: x0, y0, z, border
    int* qcount = reinterpret_cast<int*>(smem + 384);       // [MAX_LEVELS]
    int* batch = reinterpret_cast<int*>(smem + 896);        // [NSET] claimed first tile
    uint8_t* slots = smem + FHDR;                           // [NSET][BT][geo.b_bytes]
    uint8_t* stage = slots + (size_t)NSET * BT * geo.b_bytes;  // [NW][1 + FIN][WPIX] k = 3 output / finalized_at
    uint16_t* Q0 = reinterpret_cast<uint16_t*>(stage + NW * (FIN ? 2 : 1) * WPIX);
    uint16_t* Q1 = Q0 + C::CAP;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int per_slice = a.tiles_x * a.tiles_y;
    const int ntiles = per_slice * a.n_slices;
    const bool grow = a.smax >= 5;
    if (tid == 0) {
        for (int i = 0; i < NSET * BT; ++i) mbar_init(&bar[i], 1);
        prefetch_tmap(&tm);
        fence_mbar_init();
    }
    if (tid < MAX_LEVELS) qcount[tid] = 0;
    grid_dep_wait();  // the previous grid (e.g. the last step's gain reading dst) has completed
    // thread 0: claim the next BT tiles for slot set `set` and start their TMA loads (+ growth halo R)
    auto claim_issue = [&](int set) {
        const int t0 = atomicAdd(a.claim, BT);
        batch[set] = t0;
        if (t0 >= ntiles) return;
        fence_proxy_async_smem();  // the slot set's previous generic accesses before the async writes
        for (int i = 0; i < min(BT, ntiles - t0); ++i) {
            const int t = t0 + i, z = t / per_slice, rem = t - z * per_slice, by = rem / a.tiles_x;
            int* ti = tinfo + 4 * (set * BT + i);
            ti[0] = (rem - by * a.tiles_x) * TW;
            ti[1] = a.row_begin + by * TH;
            ti[2] = z;
            const int sx0 = ti[0] - geo.CP, sy0 = ti[1] - geo.R;
            ti[3] = sx0 < 0 || sx0 + geo.BS > a.cols || sy0 < 0 || sy0 + geo.BH > a.rows;
            grow_tile_load(&tm, geo, slots + (size_t)(set * BT + i) * geo.b_bytes, &bar[set * BT + i], ti[0], ti[1],
                           z);
        }
    };
    uint8_t* O = stage + warp * (FIN ? 2 : 1) * WPIX;
    uint8_t* F = FIN ? O + WPIX : O;
    uint32_t phases = 0;  // bit s: parity of slot set s's next wait
    if (tid == 0) claim_issue(0);
    for (int it = 0;; ++it) {
        const int cur = NSET == 2 ? (it & 1) : 0;
        if (NSET == 1 && it > 0 && tid == 0) claim_issue(0);
        __syncthreads();  // batch / tile info of this set; the previous batch's slot and queue use complete
        const int t0 = batch[cur];
        if (t0 >= ntiles) break;
        if (NSET == 2 && tid == 0) claim_issue(cur ^ 1);  // the next batch loads while this one computes
        const int nt = min(BT, ntiles - t0);
        uint8_t* bufs = slots + (size_t)cur * BT * geo.b_bytes;
        const int* tset = tinfo + 4 * cur * BT;
        for (int i = 0; i < nt; ++i) mbar_wait(&bar[cur * BT + i], (phases >> cur) & 1u);
        phases ^= 1u << cur;
        for (int i = 0; i < nt; ++i) {  // border tiles: edge replication within the growth reach R
            const int* ti = tset + 4 * i;
            if (!ti[3]) continue;  // uniform
            const int sx0 = ti[0] - geo.CP, sy0 = ti[1] - geo.R;
            replicate_edges<NT>(bufs + (size_t)i * geo.b_bytes, geo.BS, max(0, -sx0), min(geo.BS, a.cols - sx0),
                                max(0, -sy0), min(geo.BH, a.rows - sy0), 0, geo.BH, geo.R);
        }
        // ---- k = 3 on every pixel of the batch: f stored, level-A failures queued; growth k = 5..smax over
        //      the pooled failures, from the resident tiles ----
        auto out = [&](int sl, int pix, uint8_t v, int k) {
            const int* ti = tset + 4 * sl;
            const size_t row = (size_t)(ti[1] - a.row_begin + (pix >> 7));
            a.dst[(size_t)ti[2] * a.dslice + row * a.dpitch + ti[0] + (pix & 127)] = v;
            if (FIN) a.fin[(size_t)ti[2] * a.fslice + row * a.fpitch + ti[0] + (pix & 127)] = (uint8_t)k;
        };
        auto k3 = [&](int i, int sub) {
            const int* ti = tset + 4 * i;
            const int x0 = ti[0], y0 = ti[1], z = ti[2];
            const uint8_t* B = bufs + (size_t)i * geo.b_bytes + (size_t)(geo.R - 1) * geo.BS;  // row 0 = y0 - 1
            k3_strip<FIN>(B, O, F, sub, nullptr,
                          a.dst + (size_t)z * a.dslice + (size_t)(y0 - a.row_begin) * a.dpitch + x0, a.dpitch,
                          FIN ? a.fin + (size_t)z * a.fslice + (size_t)(y0 - a.row_begin) * a.fpitch + x0 : nullptr,
                          a.fpitch, a.row_end - y0, a.cols - x0, grow ? Q0 : nullptr, qcount, (uint32_t)i << 12);
        };
        if constexpr (!C::CAPPED) {
            for (int j = warp; j < nt * NW; j += NW) k3(j / NW, j % NW);
            __syncthreads();
            const int total = qcount[0];
            if (grow && total > 0) grow_levels<FIN, NT, decltype(out), C::NETMAX>(bufs, geo, Q0, Q1, qcount, total, a.smax, out);
            __syncthreads();
            if (tid < MAX_LEVELS) qcount[tid] = 0;
        } else {
            // tile by tile (one strip per warp); the pooled growth runs when the next tile's failures might
            // not fit, and at the batch end
            for (int i = 0; i < nt; ++i) {
                k3(i, warp);
                __syncthreads();
                const int total = qcount[0];
                if (grow && total > 0 && (i == nt - 1 || total > C::CAP - TW * TH)) {
                    grow_levels<FIN, NT, decltype(out), C::NETMAX>(bufs, geo, Q0, Q1, qcount, total, a.smax, out);
                    if (tid < MAX_LEVELS) qcount[tid] = 0;
                    __syncthreads();
                }
            }
            if (!grow && tid == 0) qcount[0] = 0;
        }
    }
    // the last CTA resets the claim counter for the next launch
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(a.done, 1) == (int)gridDim.x - 1) {
            *a.claim = 0;
            *a.done = 0;
        }
    }
}

template <bool FIN, class C>
cudaError_t launch_fused_amf(const Plane& p, int smax, uint8_t* fin, size_t fpitch, size_t fslice, const AmfWork& work,
                             cudaStream_t stream) {
    static PerDevice attr, occ;
    const GGeo geo = make_ggeo(smax);
    const size_t smem = fused_smem<FIN, C>(geo);
    auto kern = amf_fused_kernel<FIN, C>;
    cudaError_t e = ensure_smem_attr(attr, (const void*)kern, smem);
    if (e != cudaSuccess) return e;
    CUtensorMap tm;
    e = make_tmap_u8(&tm, p.src, p.cols, p.rows, p.n_slices, p.spitch, p.sslice, geo.box_w, geo.box_h);
    if (e != cudaSuccess) return e;
    FArgs a;
    a.geo = geo;
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
    a.tiles_y = (p.row_end - p.row_begin + TH - 1) / TH;
    a.claim = work.counters + 2;
    a.done = work.counters + 3;
    const long long ntiles = (long long)a.tiles_x * a.tiles_y * a.n_slices;
    const int per_sm = occupancy(occ, (const void*)kern, NT, smem);
    const int grid = (int)std::min<long long>((ntiles + C::BT - 1) / C::BT, (long long)device_sms() * per_sm);
    e = launch_pdl(kern, dim3(grid), dim3(NT), smem, stream, tm, a);
    count_launch();
    return e;
}

}  // namespace

// Compact growth entries: one per 128 image pixels (at least 1024, at most 2^21 = 128 MiB); strips that
// find the list full fall back to their tile's bitmap.
inline int compact_cap(const Plane& p) {
    static const int forced = getenv("HYB_COMPACT_CAP") ? atoi(getenv("HYB_COMPACT_CAP")) : 0;  // tests: overflow
    if (forced > 0) return forced;
    const long long npix = (long long)p.cols * (p.row_end - p.row_begin) * p.n_slices;
    return (int)std::min<long long>(std::max<long long>(npix / 128, 1024), 1ll << 21);
}

size_t amf_work_bytes(const Plane& p) {
    const size_t tiles = (size_t)((p.cols + TW - 1) / TW) * ((p.row_end - p.row_begin + TH - 1) / TH) * p.n_slices;
    // chunk table: weighted total <= tiles * (TW * TH + REC_W) over chunks of >= 2048 -> <= 2.07 tiles + 1
    const size_t head = 64 + (tiles * 8 + 63) / 64 * 64 + tiles * 512 + (tiles * 3 + 16) * sizeof(int);
    return (head + 127) / 128 * 128 + (size_t)compact_cap(p) * 64;
}

AmfWork amf_work(uint8_t* base, const Plane& p) {
    const size_t tiles = (size_t)((p.cols + TW - 1) / TW) * ((p.row_end - p.row_begin + TH - 1) / TH) * p.n_slices;
    AmfWork w;
    w.counters = reinterpret_cast<int*>(base);
    w.records = reinterpret_cast<unsigned long long*>(base + 64);
    w.bitmap = base + 64 + (tiles * 8 + 63) / 64 * 64;
    w.chunk_rec = reinterpret_cast<int*>(w.bitmap + tiles * 512);
    const size_t head = 64 + (tiles * 8 + 63) / 64 * 64 + tiles * 512 + (tiles * 3 + 16) * sizeof(int);
    w.cq = reinterpret_cast<uint4*>(base + (head + 127) / 128 * 128);
    w.cq_cap = compact_cap(p);
    return w;
}

cudaError_t launch_amf(const Plane& p, int smax, uint8_t* fin, size_t fpitch, size_t fslice, const AmfWork& work,
                       cudaStream_t stream) {
    // k = 3 + growth in one kernel per tile batch (amf_fused_kernel) for single images with smax 5..9
    // (config 2: -6 % AMF time); the two-kernel path (pipelined k = 3 kernel, pooled growth over 8-tile
    // batches) for smax >= 11 and for stacks, where it measured faster (config 4
    // 2.13 vs 2.26 ms, config 3 0.24 vs 0.27 ms).  HYB_AMF_SPLIT / HYB_AMF_FUSED force one path (A/B).
    static const bool force_split = getenv("HYB_AMF_SPLIT") != nullptr;
    static const bool force_fused = getenv("HYB_AMF_FUSED") != nullptr;
    static const bool lean11 = getenv("HYB_FUSED_LEAN11") != nullptr;
    const bool fusable = smax >= 5 && (smax - 1) / 2 <= 16;
    if (fusable && !force_split && (force_fused || (smax <= 9 && p.n_slices == 1))) {
        if (smax >= 11 && !lean11)
            return fin ? launch_fused_amf<true, FusedWide>(p, smax, fin, fpitch, fslice, work, stream)
                       : launch_fused_amf<false, FusedWide>(p, smax, fin, fpitch, fslice, work, stream);
        return fin ? launch_fused_amf<true, FusedLean>(p, smax, fin, fpitch, fslice, work, stream)
                   : launch_fused_amf<false, FusedLean>(p, smax, fin, fpitch, fslice, work, stream);
    }
    static PerDevice attr_k3[2], occ_k3;
    cudaError_t e = ensure_smem_attr(attr_k3[0], (const void*)amf_k3_kernel<false>, SMEM);
    if (e == cudaSuccess) e = ensure_smem_attr(attr_k3[1], (const void*)amf_k3_kernel<true>, SMEM);
    if (e != cudaSuccess) return e;
    const int num_sms = device_sms();
    const int out_rows = p.row_end - p.row_begin;
    const bool grow = smax >= 5;
    // compact growth windows for sparse strips (smax <= 7: 7 x 7 windows; key = slice * out_rows + row
    // must fit 32 bits).  HYB_COMPACT_T = per-strip failure threshold (0: off; A/B).
    static const int cq_thresh = getenv("HYB_COMPACT_T") ? atoi(getenv("HYB_COMPACT_T")) : HYB_COMPACT_T_DEF;
    const bool compact = grow && smax <= 7 && cq_thresh > 0 && (long long)p.n_slices * out_rows < (1ll << 31) &&
                         p.cols < (1 << 30);
    const int halo = compact ? 3 : 1;
    CUtensorMap tm_src;
    e = make_tmap_u8(&tm_src, p.src, p.cols, p.rows, p.n_slices, p.spitch, p.sslice, BS, TH + 2 * halo);
    if (e != cudaSuccess) return e;
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
    a.bitmap = work.bitmap;
    a.claim = work.counters + 2;
    a.done = work.counters + 3;
    a.rec_ctr = reinterpret_cast<unsigned long long*>(work.counters);
    a.records = work.records;
    a.chunk_rec = work.chunk_rec;
    // the chunk table of the growth variant below: 2048-unit entries for guided claims
    a.chunk_shift = HYB_GUIDED ? 11 : smax >= HYB_WIDE_MIN_SMAX ? GrowWide::CHUNK_SHIFT : GrowLean::CHUNK_SHIFT;
    a.halo = halo;
    a.cq = compact ? work.cq : nullptr;
    a.cq_ctr = work.counters + 6;
    a.cq_cap = work.cq_cap;
    a.cq_thresh = std::min(cq_thresh, 32);
    a.out_rows = out_rows;
    const int per_sm = occupancy(occ_k3, (const void*)amf_k3_kernel<false>, K3T, SMEM);
    const long long ntiles = (long long)a.tiles_x * a.tiles_y * a.n_slices;
    const int grid = (int)std::min<long long>(ntiles, (long long)num_sms * per_sm);
    a.dynamic = ntiles > 8ll * grid;
    e = launch_pdl(fin ? amf_k3_kernel<true> : amf_k3_kernel<false>, dim3(grid), dim3(K3T), SMEM, stream, tm_src, a);
    count_launch();
    if (e != cudaSuccess || !grow) return e;

    // ---- growth: one batched launch for every window size k = 5..smax ----
    const GGeo geo = make_ggeo(smax);
    const bool wide = smax >= HYB_WIDE_MIN_SMAX;
    // zero / 255 bit-plane levels (amf_core.cuh grow_levels_fast) for the wide variant; HYB_GROW_FAST=0: plain levels (A/B)
    static const bool fast_env = !(getenv("HYB_GROW_FAST") && atoi(getenv("HYB_GROW_FAST")) == 0);
    // HYB_GROW_FAST_LEAN=1: the lean variant too (experiment)
    static const bool fast_lean = getenv("HYB_GROW_FAST_LEAN") && atoi(getenv("HYB_GROW_FAST_LEAN")) != 0;
    const bool fast = (wide || fast_lean) && fast_env && (smax - 1) / 2 <= 16;
    const size_t gsm = wide ? grow_smem<GrowWide>(geo, fast) : grow_smem<GrowLean>(geo, fast);
    auto kern = wide ? (fin ? amf_grow_kernel<true, GrowWide> : amf_grow_kernel<false, GrowWide>)
                     : (fin ? amf_grow_kernel<true, GrowLean> : amf_grow_kernel<false, GrowLean>);
    const int vi = (fin ? 1 : 0) + (wide ? 2 : 0);
    static PerDevice gattr[4], gocc[4];
    e = ensure_smem_attr(gattr[vi], (const void*)kern, gsm);
    if (e != cudaSuccess) return e;
    CUtensorMap tm_g;
    e = make_tmap_u8(&tm_g, p.src, p.cols, p.rows, p.n_slices, p.spitch, p.sslice, geo.box_w, geo.box_h);
    if (e != cudaSuccess) return e;
    GArgs g;
    g.geo = geo;
    g.dst = p.dst;
    g.dpitch = p.dpitch;
    g.dslice = p.dslice;
    g.fin = fin;
    g.fpitch = fpitch;
    g.fslice = fslice;
    g.bitmap = work.bitmap;
    g.rows = p.rows;
    g.cols = p.cols;
    g.row_begin = p.row_begin;
    g.row_end = p.row_end;
    g.n_slices = p.n_slices;
    g.smax = smax;
#ifdef HYB_EXP_GROW_SMAX_CAP  // timing experiment only: the growth stops at this window (output incomplete)
    g.smax = std::min(smax, HYB_EXP_GROW_SMAX_CAP);
#endif
    g.tiles_x = a.tiles_x;
    g.tiles_y = a.tiles_y;
    g.rec_ctr = a.rec_ctr;
    g.records = work.records;
    g.chunk_rec = work.chunk_rec;
    g.chunk_ctr = work.counters + 5;
    g.done = work.counters + 4;
    g.cq = a.cq;
    g.cq_ctr = a.cq_ctr;
    g.cq_claim = work.counters + 7;
    g.cq_cap = a.cq_cap;
    g.out_rows = out_rows;
    g.fast = fast ? plane_stride(geo) : 0;
    const int gnt = wide ? GrowWide::NT : GrowLean::NT;
    const int gper_sm = occupancy(gocc[vi], (const void*)kern, gnt, gsm);
    // every resident CTA slot busy; each CTA takes a contiguous run of tiles
    const int ggrid = (int)std::min<long long>(ntiles, (long long)num_sms * gper_sm);
    e = launch_pdl(kern, dim3(ggrid), dim3(gnt), gsm, stream, tm_g, g);
    count_launch();
    return e;
}

}  // namespace hyb

#ifdef HYB_TRACE
extern "C" int hyb_trace_read(unsigned long long* host) {
    return (int)cudaMemcpyFromSymbol(host, hyb::g_trace, sizeof(hyb::g_trace));
}
extern "C" int hyb_trace_clear() {
    static unsigned long long zero[2 * 1024 * 16];
    return (int)cudaMemcpyToSymbol(hyb::g_trace, zero, sizeof(zero));
}
#endif
