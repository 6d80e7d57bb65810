// small.cu -- the whole hybrid step (AMF k = 3..smax, W1 statistics, W1 gain) in ONE persistent
// kernel for images small enough that every CTA keeps its 128 x 32 tiles resident in shared memory
// (BASELINE config 1: 1600 x 1600 = 650 tiles on 296 CTAs).
//
// Per CTA (tiles t = blockIdx.x + i * gridDim.x, i < STPC):
//   A  TMA-load each tile of g with the growth halo R = (smax-1)/2, replicate edges, run the k = 3
//      strips (warp w: strip w of every tile; amf_core.cuh k3_strip) writing f to global memory and
//      appending their level-A failures to one shared-memory queue (one shared atomic per strip);
//   B  run the growth levels k = 5..smax over that pooled queue from the resident tiles
//      (amf_core.cuh grow_levels) -- no second launch, no reload, no bitmap pass;
//   -- grid barrier (f complete; CTA 0 has zeroed W) --
//   C  TMA-load each tile of f with the W1 halo into the same slots, statistics per 128 x 8
//      sub-tile (w1_core.cuh), one atomic per CTA into W;
//   -- grid barrier (W complete) --
//   D  gain per sub-tile from the resident f tiles, y written once.
// The separate-kernel path (amf.cu, wiener.cu) computes the same thing; this one removes three
// launches, the growth reload and the second f read for latency-bound small images.  The grid is
// launched cooperatively (all CTAs co-resident) because of the two grid barriers.  (A variant that
// balanced the growth over the grid through failure records and a third barrier measured slower at
// config 1: its per-batch search / reload latency exceeded the imbalance it removed.)
#include <cuda.h>

#include <algorithm>
#include <cstdint>

#include "amf_core.cuh"
#include "hyb_internal.cuh"
#include "tma.cuh"
#include "trace.cuh"
#include "w1_core.cuh"

namespace hyb {
namespace {

// CTA size: 256 threads, 3 CTAs/SM (2 tiles each).  HYB_SMALL_NT=768 (one CTA per SM, all 24 warps
// pooling the SM's growth failures) shortened the in-kernel growth tail by 1.8 us at config 1 but
// measured 1.8 us slower per launch (30.8 vs 29.0 us; 512: 30.8 us) -- kept as a build option.
#ifndef HYB_SMALL_NT
#define HYB_SMALL_NT 256
#endif
constexpr int SNT = HYB_SMALL_NT;                            // threads per CTA
constexpr int SNW = SNT / 32;                                // warps per CTA
constexpr int SMIN = SNT >= 768 ? 1 : (SNT >= 512 ? 2 : 3);  // CTAs per SM (register budget)
constexpr int STPC = SNT >= 768 ? 6 : (SNT >= 512 ? 3 : 2);  // tiles per CTA (max)
static_assert(STPC <= 8 && SNW <= 32, "header layout");
constexpr int SHDR = 1024;  // mbarriers, tile coordinates, level counters
constexpr int SFH = 8;     // W1 sub-tile rows

struct SArgs {
    GGeo geo;                 // growth tile geometry (halo R)
    int slot_bytes;           // per-tile slot: max(g tile with halo R, f tile with halo RW)
    int rows, cols, smax;
    int tiles_x, ntiles;
    uint8_t* f;               // AMF output (TMA-compatible pitch)
    size_t fpitch;
    uint8_t* y;
    size_t ypitch;
    unsigned long long* wsum;  // W (two's complement), zeroed in the kernel
    unsigned* bar_count;      // grid barrier: arrivals / exits (zero when allocated; reset by the last exit)
    unsigned* bar_gen;
    unsigned long long* times;  // globaltimer: [0] start (CTA 0), [1] after the AMF barrier, [2] last CTA end
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Grid barrier number k (0, 1, ...) of this launch: arrivals accumulate on one counter (fire-and-forget
// release adds), every CTA polls it with acquire loads until all gridDim.x * (k + 1) arrivals are in.
// The last CTA to exit resets the counter for the next launch.
__device__ __forceinline__ void grid_barrier(unsigned* count, int k) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
        const unsigned target = gridDim.x * (unsigned)(k + 1);
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

__device__ __forceinline__ void grid_exit(unsigned* count, unsigned* exits) {
    if (threadIdx.x == 0 && atomicAdd(exits, 1u) == gridDim.x - 1) {  // every CTA is past its last barrier
        *count = 0;
        *exits = 0;
    }
}

// Edge replication of the border tiles among the first nt slots (org[i] = box origin), CTA-wide.
__device__ __forceinline__ void cta_replicate_edges(uint8_t* slots, int slot_bytes, int nt, const int* org, int width,
                                                    int height, int rows, int cols, int reach) {
    for (int i = 0; i < nt; ++i) {
        const int sx0 = org[2 * i], sy0 = org[2 * i + 1];
        if (sx0 < 0 || sx0 + width > cols || sy0 < 0 || sy0 + height > rows)
            replicate_edges<SNT>(slots + (size_t)i * slot_bytes, width, max(0, -sx0), min(width, cols - sx0),
                                 max(0, -sy0), min(height, rows - sy0), 0, height, reach);
    }
}

template <int RW>
__global__ void __launch_bounds__(SNT, SMIN) hybrid_small_kernel(const __grid_constant__ CUtensorMap tm_g,
                                                             const __grid_constant__ CUtensorMap tm_f,
                                                             const __grid_constant__ SArgs a) {
    constexpr int FROWS = TH + 2 * RW;  // f tile rows with the W1 halo
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    const GGeo& geo = a.geo;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);           // [STPC] own tiles (g, then f)
    int* tinfo = reinterpret_cast<int*>(smem + 64);               // [STPC][2]: x0, y0
    int* org = reinterpret_cast<int*>(smem + 128);                // [STPC][2]: box origin (edge fix-up)
    unsigned long long* wred = reinterpret_cast<unsigned long long*>(smem + 256);  // [SNW] warp partial W
    int* qcount = reinterpret_cast<int*>(smem + 512);             // [MAX_LEVELS]
    uint8_t* slots = smem + SHDR;                                // [STPC][slot_bytes] g tiles, then f tiles
    uint8_t* bitmaps = slots + (size_t)STPC * a.slot_bytes;     // [STPC][512]
    uint8_t* stage = bitmaps + STPC * 512;                      // [SNW][WPIX] k = 3 output staging
    uint16_t* Q0 = reinterpret_cast<uint16_t*>(stage + SNW * WPIX);
    uint16_t* Q1 = Q0 + STPC * 4096;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nt = (a.ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;  // my tiles (<= STPC)

    TRACE(0, 0);
    // ---- A: own g tiles (+ growth halo R) by TMA, edges, k = 3 (f; failures queued in Q0) ----
    if (tid == 0) {
        if (blockIdx.x == 0) {
            a.times[0] = gtimer();
            a.times[2] = 0;
        }
        for (int i = 0; i < STPC; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
        for (int i = 0; i < nt; ++i) {
            // snake order: block i of G consecutive tiles is dealt forwards for even i, backwards for odd i
            // (for two tiles per CTA: the second is the point mirror of the first), so a CTA's tiles come
            // from opposite parts of the image -- failure density follows the image content and its
            // column gradient
            const int G = (int)gridDim.x, b = (int)blockIdx.x;
            const int t = (i & 1) ? min((i + 1) * G, a.ntiles) - 1 - b : i * G + b;
            const int by = t / a.tiles_x;
            tinfo[2 * i] = (t - by * a.tiles_x) * TW;
            tinfo[2 * i + 1] = by * TH;
            org[2 * i] = tinfo[2 * i] - geo.CP;
            org[2 * i + 1] = tinfo[2 * i + 1] - geo.R;
            uint8_t* B = slots + (size_t)i * a.slot_bytes;
            mbar_expect_tx(&bar[i], (uint32_t)(geo.box_w * geo.nbx * geo.box_h * geo.nby));
            for (int yb = 0; yb < geo.nby; ++yb)
                for (int xb = 0; xb < geo.nbx; ++xb)
                    tma_load_3d(B + (size_t)yb * geo.box_h * geo.BS + (size_t)xb * geo.box_w, &tm_g, &bar[i],
                                org[2 * i] + xb * geo.box_w, org[2 * i + 1] + yb * geo.box_h, 0);
        }
    }
    if (tid < MAX_LEVELS) qcount[tid] = 0;
    __syncthreads();
    for (int i = 0; i < nt; ++i) mbar_wait(&bar[i], 0);
    TRACE(0, 1);
    cta_replicate_edges(slots, a.slot_bytes, nt, org, geo.BS, geo.BH, a.rows, a.cols, geo.R);
    TRACE(0, 2);
    {
        uint8_t* O = stage + warp * WPIX;
        for (int j = warp; j < nt * NW; j += SNW) {  // strip j % NW of tile j / NW
            const int i = j / NW;
            const int x0 = tinfo[2 * i], y0 = tinfo[2 * i + 1];
            const uint8_t* B = slots + (size_t)i * a.slot_bytes + (size_t)(geo.R - 1) * geo.BS;  // row 0 = y0 - 1
            k3_strip<false>(B, O, O, j % NW, nullptr, a.f + (size_t)y0 * a.fpitch + x0, a.fpitch, nullptr, 0,
                            a.rows - y0, a.cols - x0, a.smax >= 5 ? Q0 : nullptr, qcount, (uint32_t)i << 12);
        }
    }
    __syncthreads();
    TRACE(0, 3);

    // ---- B: growth over the pooled failures of the resident tiles ----
    if (a.smax >= 5) {
        const int total = qcount[0];  // the k = 3 strips appended their failures to Q0
        TRACE(0, 4);
#ifdef HYB_TRACE
        if (tid == 0 && blockIdx.x < 1024) {
            g_trace[blockIdx.x * 16 + 12] = (unsigned long long)total;
            g_trace[blockIdx.x * 16 + 13] = (unsigned long long)nt;
        }
#endif
        if (total > 0)
        {
            auto out = [&](int sl, int pix, uint8_t v, int) {
                a.f[(size_t)(tinfo[2 * sl + 1] + (pix >> 7)) * a.fpitch + tinfo[2 * sl] + (pix & 127)] = v;
            };
            // networks up to k = 7 here (the k = 9 one needs more registers than 3 CTAs/SM allow)
            grow_levels<false, SNT, decltype(out), 7>(slots, geo, Q0, Q1, qcount, total, a.smax, out);
        }
    }
    TRACE(0, 5);
    if (blockIdx.x == 0 && tid == 0) *a.wsum = 0;
    asm volatile("fence.proxy.async.global;" ::: "memory");  // f stores -> the TMA reads of phase C
    grid_barrier(a.bar_count, 0);  // f complete
    TRACE(0, 6);
    if (blockIdx.x == 0 && tid == 0) a.times[1] = gtimer();

    // ---- C: own f tiles (+ RW halo) by TMA, W1 statistics ----
    if (tid == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        fence_proxy_async_smem();  // the slots' generic accesses before the async writes
        for (int i = 0; i < nt; ++i) {
            org[2 * i] = tinfo[2 * i] - FCP;
            org[2 * i + 1] = tinfo[2 * i + 1] - RW;
            mbar_expect_tx(&bar[i], (uint32_t)(FBS * FROWS));
            tma_load_3d(slots + (size_t)i * a.slot_bytes, &tm_f, &bar[i], org[2 * i], org[2 * i + 1], 0);
        }
    }
    __syncthreads();
    for (int i = 0; i < nt; ++i) mbar_wait(&bar[i], 1);
    TRACE(0, 7);
    cta_replicate_edges(slots, a.slot_bytes, nt, org, FBS, FROWS, a.rows, a.cols, RW);
    TRACE(0, 8);
    unsigned long long vsum = 0;
    uint32_t* sums = reinterpret_cast<uint32_t*>(Q0);  // [STPC][32][128] packed S1 | S2 << 12 (RW == 1)
    for (int j = warp; j < nt * (TH / SFH); j += SNW) {
        const int i = j / (TH / SFH), k = j % (TH / SFH);
        const uint8_t* T = slots + (size_t)i * a.slot_bytes + (size_t)k * SFH * FBS;
        const int y0 = tinfo[2 * i + 1] + k * SFH;
        if (y0 >= a.rows) continue;
        if constexpr (RW == 1)
            vsum += (unsigned long long)w1_tile_sums3<SFH>(T, a.cols - tinfo[2 * i], a.rows - y0,
                                                           sums + ((size_t)i * TH + k * SFH) * FW);
        else
            vsum += (unsigned long long)w1_tile_stats<RW, SFH>(T, tinfo[2 * i], y0, a.rows, a.cols, 0, a.rows);
    }
    TRACE(0, 9);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) vsum += __shfl_down_sync(0xFFFFFFFFu, vsum, d);
    if (lane == 0) wred[warp] = vsum;
    __syncthreads();
    if (tid == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < SNW; ++w) s += wred[w];
        if (s) atomicAdd(a.wsum, s);
    }
    grid_barrier(a.bar_count, 1);  // W complete

    TRACE(0, 10);
    // ---- D: gain from the resident f tiles ----
    const W1Gain kg = w1_gain_consts((long long)__ldcg(a.wsum), (long long)a.rows * a.cols);
    for (int j = warp; j < nt * (TH / SFH); j += SNW) {
        const int i = j / (TH / SFH), k = j % (TH / SFH);
        const uint8_t* T = slots + (size_t)i * a.slot_bytes + (size_t)k * SFH * FBS;
        const int x0 = tinfo[2 * i], y0 = tinfo[2 * i + 1] + k * SFH;
        if (y0 >= a.rows) continue;
        if constexpr (RW == 1)
            w1_tile_gain3<SFH>(T, sums + ((size_t)i * TH + k * SFH) * FW, a.cols - x0, a.rows - y0, kg,
                               a.y + (size_t)y0 * a.ypitch + x0, a.ypitch);
        else
            w1_tile_gain<RW, SFH>(T, x0, a.cols - x0, a.rows - y0, kg, a.y + (size_t)y0 * a.ypitch + x0, a.ypitch);
    }
    __syncthreads();
    TRACE(0, 11);
    if (tid == 0) atomicMax(&a.times[2], gtimer());
    grid_exit(a.bar_count, a.bar_gen);
}

size_t small_smem(int slot_bytes) {
    return SHDR + (size_t)STPC * slot_bytes + STPC * 512 + SNW * WPIX + 2 * STPC * 4096 * 2 + 128;
}

template <int RW>
cudaError_t launch_small_rw(const SmallPlan& pl, const SmallBufs& bf, int rows, int cols, int smax,
                            bool cooperative, cudaStream_t stream) {
    SArgs a;
    a.geo = make_ggeo(smax);
    a.slot_bytes = pl.slot_bytes;
    const GGeo box = a.geo;
    a.geo.b_bytes = pl.slot_bytes;  // the growth windows address the slots at this stride
    a.rows = rows;
    a.cols = cols;
    a.smax = smax;
    a.tiles_x = (cols + TW - 1) / TW;
    a.ntiles = a.tiles_x * ((rows + TH - 1) / TH);
    a.f = bf.f;
    a.fpitch = bf.fpitch;
    a.y = bf.y;
    a.ypitch = bf.ypitch;
    a.wsum = bf.wsum;
    a.bar_count = bf.sbar;
    a.bar_gen = bf.sbar + 1;
    a.times = reinterpret_cast<unsigned long long*>(bf.sbar + 2);
    CUtensorMap tm_g, tm_f;
    cudaError_t e = make_tmap_u8(&tm_g, bf.g, cols, rows, 1, bf.gpitch, bf.gpitch * rows, box.box_w, box.box_h);
    if (e == cudaSuccess) e = make_tmap_u8(&tm_f, bf.f, cols, rows, 1, bf.fpitch, bf.fpitch * rows, FBS, TH + 2 * RW);
    if (e != cudaSuccess) return e;
    auto kern = hybrid_small_kernel<RW>;
    const size_t smem = small_smem(pl.slot_bytes);
    static PerDevice smem_attr;
    e = ensure_smem_attr(smem_attr, (const void*)kern, smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.grid);
    cfg.blockDim = dim3(SNT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cooperative ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, kern, tm_g, tm_f, a);
    count_launch();
    return e;
}

}  // namespace

// Whether the fused kernel takes this image, and with which grid (all CTAs must be co-resident).
SmallPlan plan_small(int rows, int cols, int smax, int win) {
    SmallPlan pl{};
    if (smax > 11 || win > 7 || win < 1 || (win & 1) == 0) return pl;
    const GGeo geo = make_ggeo(smax);
    const int rw = (win - 1) / 2;
    pl.slot_bytes = std::max(geo.b_bytes, (FBS * (TH + 2 * rw) + 127) / 128 * 128);
    static PerDevice attr[4], occ[4];
    const size_t smem = small_smem(pl.slot_bytes);
    const void* k = rw == 0   ? (const void*)hybrid_small_kernel<0>
                    : rw == 1 ? (const void*)hybrid_small_kernel<1>
                    : rw == 2 ? (const void*)hybrid_small_kernel<2>
                              : (const void*)hybrid_small_kernel<3>;
    static PerDevice carve[4];
    const int dev = current_device();
    if (dev >= kMaxDevices || !carve[rw].v[dev].load(std::memory_order_acquire)) {
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);  // a hint; before occupancy
        if (dev < kMaxDevices) carve[rw].v[dev].store(1, std::memory_order_release);
    }
    if (ensure_smem_attr(attr[rw], k, smem) != cudaSuccess) {
        cudaGetLastError();
        return pl;
    }
    const int per_sm = occupancy(occ[rw], k, SNT, smem);
    const long long ntiles = (long long)((cols + TW - 1) / TW) * ((rows + TH - 1) / TH);
    const long long capacity = (long long)device_sms() * per_sm;
    if (capacity <= 0 || ntiles > capacity * STPC) return pl;
    pl.grid = (int)std::min<long long>(capacity, ntiles);
    pl.ok = true;
    return pl;
}

cudaError_t launch_small(const SmallPlan& pl, const SmallBufs& bf, int rows, int cols, int smax, int win,
                         bool cooperative, cudaStream_t stream) {
    switch ((win - 1) / 2) {
        case 0: return launch_small_rw<0>(pl, bf, rows, cols, smax, cooperative, stream);
        case 1: return launch_small_rw<1>(pl, bf, rows, cols, smax, cooperative, stream);
        case 2: return launch_small_rw<2>(pl, bf, rows, cols, smax, cooperative, stream);
        default: return launch_small_rw<3>(pl, bf, rows, cols, smax, cooperative, stream);
    }
}

}  // namespace hyb

#ifdef HYB_TRACE
extern "C" int hyb_trace_read_small(unsigned long long* host) {
    return (int)cudaMemcpyFromSymbol(host, hyb::g_trace, sizeof(hyb::g_trace));
}
#endif
