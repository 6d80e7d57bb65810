// tma.cuh -- Tensor Memory Accelerator (cp.async.bulk.tensor) and mbarrier helpers for sm_100a,
// plus host-side tensor-map encoding through the driver entry point (no libcuda link needed).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace hyb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Plain arrival (release semantics at CTA scope).
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Programmatic dependent launch: wait for the preceding grid's memory (no-op without the attribute),
// and let the next grid start its prologue early.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Waits for the phase with the given parity; backs off so waiting warps leave issue slots free.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) __nanosleep(64);
}

// Warp-convergent wait: the warp leaves the loop together (every lane has observed the completed
// phase itself, i.e. has its own acquire), so code after it may rely on a converged warp.
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
    while (!__all_sync(0xFFFFFFFFu, mbar_try_wait(bar, parity))) __nanosleep(32);
}

// Edge replication in a TMA-loaded byte tile (`width` bytes per row, out-of-image bytes zero-filled
// by TMA; in-image columns [c_lo, c_hi), rows [r_lo, r_hi)), restricted to rows [row0, row1) and to
// the `reach` columns / rows next to the image -- the only out-of-image bytes a window of radius
// <= reach around an in-image pixel reads: those columns take the nearest in-image column, then
// those rows copy the nearest in-image row.  NTHR cooperating threads (32: one warp; else the CTA)
// with uniform trip counts (a lane-strided loop with a ragged tail would leave a warp diverged while
// the caller reads the tile); ends with a warp / CTA barrier.
template <int NTHR>
__device__ __forceinline__ void replicate_edges(uint8_t* T, int width, int c_lo, int c_hi, int r_lo, int r_hi, int row0,
                                                int row1, int reach) {
    const int tid = NTHR == 32 ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
    const int cl0 = max(0, c_lo - reach), cr1 = min(width, c_hi + reach);
    const int nl = c_lo - cl0, nfix = nl + (cr1 - c_hi);
    const int ra = max(row0, r_lo), rb = min(row1, r_hi);
    if (nfix > 0 && rb > ra) {
        const int n = (rb - ra) * nfix;
        for (int i0 = 0; i0 < n; i0 += NTHR) {
            const int i = i0 + tid;
            if (i < n) {
                const int rr = ra + i / nfix, j = i - (rr - ra) * nfix;
                uint8_t* row = T + rr * width;
                if (j < nl) row[cl0 + j] = row[c_lo];
                else row[c_hi + (j - nl)] = row[c_hi - 1];
            }
        }
        if (NTHR == 32) __syncwarp();
        else __syncthreads();
    }
    const int wpr = width / 4;
    const int a0 = max(row0, r_lo - reach), a1 = min(row1, r_lo);  // rows above the image
    const int b0 = max(row0, r_hi), b1 = min(row1, r_hi + reach);  // rows below
    const int above = max(0, a1 - a0), below = max(0, b1 - b0);
    const int n = (above + below) * wpr;
    for (int i0 = 0; i0 < n; i0 += NTHR) {
        const int i = i0 + tid;
        if (i < n) {
            const int k = i / wpr, q = i - k * wpr;
            const int rr = k < above ? a0 + k : b0 + (k - above);
            const int src = rr < r_lo ? r_lo : r_hi - 1;
            reinterpret_cast<uint32_t*>(T + rr * width)[q] = reinterpret_cast<const uint32_t*>(T + src * width)[q];
        }
    }
    if (NTHR == 32) __syncwarp();
    else __syncthreads();
}

// Bulk copy global -> shared (cp.async.bulk, 16-byte aligned, bytes a multiple of 16), completing on bar.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// 3-D tiled TMA load (x = column, y = row, z = slice); out-of-bounds elements read as zero.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                            int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
        : "memory");
}

// 3-D tiled TMA store from shared memory; out-of-bounds elements are not written.
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int x, int y, int z) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
                 "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
                 : "memory");
}

__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

__device__ __forceinline__ void tma_store_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Order this thread's generic-proxy shared-memory writes before later async-proxy (TMA) reads.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// Host: encode a 3-D uint8 tensor map {cols, rows, slices} with byte strides {pitch, slice}
// and box {box_w, box_h, 1}.  Requires a 16-byte aligned base and pitch/slice multiples of 16.
cudaError_t make_tmap_u8(CUtensorMap* map, const void* base, int cols, int rows, int slices, size_t pitch,
                         size_t slice_stride, int box_w, int box_h);

inline bool tma_compatible(const void* base, size_t pitch, size_t slice_stride) {
    return (reinterpret_cast<uintptr_t>(base) & 15) == 0 && (pitch & 15) == 0 && (slice_stride & 15) == 0;
}

}  // namespace hyb
