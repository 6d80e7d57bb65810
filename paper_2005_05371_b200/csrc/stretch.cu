// stretch.cu -- contrast_stretch (reference proj/src/pipeline.cpp:10-21), the step right after the
// path: the image's min / max, then out = (v - lo) / (hi - lo) scaled to
// 0..255 and rounded half up, the image unchanged when hi == lo (oracle: hyb_oracle_contrast_stretch_u8).
//
// Two HBM-streaming kernels: minmax (1 B/px read; 16 bytes per thread per step with byte-SIMD
// VIMNMX.U8x4, one min atomic per CTA for lo and for 255 - hi so one memset initialises both) and
// map (1 B/px read + 1 B/px write through a 256-entry shared-memory table of exact quotients).
#include <cstdint>

#include "hyb_internal.cuh"
#include "tma.cuh"

namespace hyb {
namespace {

constexpr int XT = 256;  // threads per CTA

// Per-thread byte-SIMD min / max over rows [blockIdx.y-strided], columns in 16-byte chunks.
__global__ void __launch_bounds__(XT) minmax_kernel(const uint8_t* __restrict__ src, size_t pitch, int rows, int cols,
                                                   unsigned* __restrict__ mm) {
    grid_dep_wait();
    uint32_t lo = 0xFFFFFFFFu, hi = 0u;
    const bool vec = (pitch & 15) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0;
    const int chunks = vec ? cols / 16 : 0;
    const long long total = (long long)rows * chunks;
    for (long long i = (long long)blockIdx.x * XT + threadIdx.x; i < total; i += (long long)gridDim.x * XT) {
        const int r = (int)(i / chunks), k = (int)(i - (long long)r * chunks);
        const uint4 v = __ldcs(reinterpret_cast<const uint4*>(src + (size_t)r * pitch) + k);
        lo = __vminu4(lo, __vminu4(__vminu4(v.x, v.y), __vminu4(v.z, v.w)));
        hi = __vmaxu4(hi, __vmaxu4(__vmaxu4(v.x, v.y), __vmaxu4(v.z, v.w)));
    }
    // columns outside the 16-byte chunks (ragged tail or unaligned rows), byte by byte
    const int c0 = chunks * 16, tail = cols - c0;
    const long long ttotal = (long long)rows * tail;
    for (long long i = (long long)blockIdx.x * XT + threadIdx.x; i < ttotal; i += (long long)gridDim.x * XT) {
        const int r = (int)(i / tail), c = c0 + (int)(i - (long long)r * tail);
        const uint32_t v = src[(size_t)r * pitch + c] * 0x01010101u;
        lo = __vminu4(lo, v);
        hi = __vmaxu4(hi, v);
    }
    unsigned l = min(min(lo & 0xFF, (lo >> 8) & 0xFF), min((lo >> 16) & 0xFF, lo >> 24));
    unsigned h = max(max(hi & 0xFF, (hi >> 8) & 0xFF), max((hi >> 16) & 0xFF, hi >> 24));
    l = __reduce_min_sync(0xFFFFFFFFu, l);
    h = __reduce_max_sync(0xFFFFFFFFu, h);
    __shared__ unsigned sl[XT / 32], sh[XT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        sl[warp] = l;
        sh[warp] = h;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < XT / 32; ++w) {
            l = min(l, sl[w]);
            h = max(h, sh[w]);
        }
        atomicMin(&mm[0], l);
        atomicMin(&mm[1], 255u - h);
    }
}

__global__ void __launch_bounds__(XT) map_kernel(const uint8_t* __restrict__ src, size_t spitch, int rows, int cols,
                                                uint8_t* __restrict__ dst, size_t dpitch, const unsigned* __restrict__ mm) {
    __shared__ uint8_t lut[256];
    grid_dep_wait();
    const int lo = (int)__ldcg(&mm[0]), hi = 255 - (int)__ldcg(&mm[1]);
    {
        const int v = threadIdx.x;
        lut[v] = hi == lo ? (uint8_t)v
                          : (uint8_t)(v <= lo ? 0 : (v >= hi ? 255 : (510 * (v - lo) + (hi - lo)) / (2 * (hi - lo))));
    }
    __syncthreads();
    const bool vec = (spitch & 3) == 0 && (dpitch & 3) == 0 && (reinterpret_cast<uintptr_t>(src) & 3) == 0 &&
                     (reinterpret_cast<uintptr_t>(dst) & 3) == 0;
    const int words = vec ? cols / 4 : 0;
    const long long total = (long long)rows * words;
    for (long long i = (long long)blockIdx.x * XT + threadIdx.x; i < total; i += (long long)gridDim.x * XT) {
        const int r = (int)(i / words), k = (int)(i - (long long)r * words);
        const uint32_t v = reinterpret_cast<const uint32_t*>(src + (size_t)r * spitch)[k];
        const uint32_t o = (uint32_t)lut[v & 0xFF] | ((uint32_t)lut[(v >> 8) & 0xFF] << 8) |
                           ((uint32_t)lut[(v >> 16) & 0xFF] << 16) | ((uint32_t)lut[v >> 24] << 24);
        reinterpret_cast<uint32_t*>(dst + (size_t)r * dpitch)[k] = o;
    }
    const int c0 = words * 4, tail = cols - c0;
    const long long ttotal = (long long)rows * tail;
    for (long long i = (long long)blockIdx.x * XT + threadIdx.x; i < ttotal; i += (long long)gridDim.x * XT) {
        const int r = (int)(i / tail), c = c0 + (int)(i - (long long)r * tail);
        dst[(size_t)r * dpitch + c] = lut[src[(size_t)r * spitch + c]];
    }
}

}  // namespace

cudaError_t launch_stretch_minmax(const uint8_t* src, size_t spitch, int rows, int cols, unsigned* mm,
                                  cudaStream_t stream) {
    const long long px = (long long)rows * cols;
    const int grid = (int)std::max(1ll, std::min((long long)device_sms() * 8, (px + XT * 16 - 1) / (XT * 16)));
    const cudaError_t e = launch_pdl(minmax_kernel, dim3(grid), dim3(XT), 0, stream, src, spitch, rows, cols, mm);
    count_launch();
    return e;
}

cudaError_t launch_stretch_map(const uint8_t* src, size_t spitch, int rows, int cols, uint8_t* dst, size_t dpitch,
                               const unsigned* mm, cudaStream_t stream) {
    const long long px = (long long)rows * cols;
    const int mgrid = (int)std::max(1ll, std::min((long long)device_sms() * 8, (px + XT * 4 - 1) / (XT * 4)));
    const cudaError_t e = launch_pdl(map_kernel, dim3(mgrid), dim3(XT), 0, stream, src, spitch, rows, cols, dst,
                                     dpitch, mm);
    count_launch();
    return e;
}

cudaError_t launch_contrast_stretch(const uint8_t* src, size_t spitch, int rows, int cols, uint8_t* dst,
                                    size_t dpitch, unsigned* mm, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(mm, 0xFF, 2 * sizeof(unsigned), stream);  // lo = 255+, 255 - hi = 255+
    if (e != cudaSuccess) return e;
    e = launch_stretch_minmax(src, spitch, rows, cols, mm, stream);
    if (e != cudaSuccess) return e;
    return launch_stretch_map(src, spitch, rows, cols, dst, dpitch, mm, stream);
}

}  // namespace hyb
