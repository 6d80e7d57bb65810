// wstats.cu -- window_stats (reference proj/src/adaptive_median.cpp:96-119, declared
// proj/include/denoise/adaptive_median.hpp:16-24): per pixel the minimum, the
// median (sorted index (k^2 - 1) / 2) and the maximum of its k x k window, borders by edge replication
// (proj/src/adaptive_median.cpp:20-41 clamps the coordinates).  Not on the hybrid path -- the AMF kernels
// compute these only where a pixel needs them -- but the reference exports the full planes for its
// estimator tests, so this is the dense form of the same selection.
//
// One CTA per 32 x 32 output tile: the tile plus a halo of R = (k-1)/2 rows / columns is staged in shared
// memory with clamped coordinates (coalesced row loads), then every thread selects four outputs (one
// column, rows ty, ty + 8, ..): window min / max in one pass; if they differ, the median by a bitwise
// radix select over the bits where min and max differ (all values lie in [min, max]).  Windows too
// large for shared memory (k > 2 * kMaxR + 1) read the clamped pixels from global memory instead.
#include <cstdint>

#include "hyb_internal.cuh"
#include "tma.cuh"

namespace hyb {
namespace {

constexpr int WT = 32;     // output tile edge
constexpr int WTY = 8;     // thread rows (4 outputs per thread)
constexpr int kMaxR = 96;  // largest radius staged in shared memory ((32 + 192)^2 = 50 KB)

struct WsArgs {
    const uint8_t* src;
    size_t pitch;
    int rows, cols, k;
    uint8_t *zmin, *zmed, *zmax;  // each nullable
    size_t opitch;
};

template <bool SMEM>
__global__ void __launch_bounds__(WT* WTY) window_stats_kernel(const WsArgs a) {
    extern __shared__ uint8_t patch[];
    const int R = a.k / 2, pw = WT + 2 * R;
    const int x0 = blockIdx.x * WT, y0 = blockIdx.y * WT;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * WT + tx;
    grid_dep_wait();
    if (SMEM) {
        for (int i = tid; i < pw * pw; i += WT * WTY) {
            const int pr = i / pw, pc = i - pr * pw;
            const int r = min(max(y0 - R + pr, 0), a.rows - 1), c = min(max(x0 - R + pc, 0), a.cols - 1);
            patch[i] = a.src[(size_t)r * a.pitch + c];
        }
        __syncthreads();
    }
    // window pixel (dr, dc) of output (y, x): patch row y - y0 + dr, column x - x0 + dc (0 <= dr, dc < k)
    auto px = [&](int y, int x, int dr, int dc) -> uint32_t {
        if (SMEM) return patch[(y - y0 + dr) * pw + (x - x0 + dc)];
        const int r = min(max(y - R + dr, 0), a.rows - 1), c = min(max(x - R + dc, 0), a.cols - 1);
        return __ldg(a.src + (size_t)r * a.pitch + c);
    };
    const int x = x0 + tx;
    const int m = (a.k * a.k - 1) / 2;
    for (int i = 0; i < WT / WTY; ++i) {
        const int y = y0 + ty + WTY * i;
        if (x >= a.cols || y >= a.rows) continue;
        uint32_t lo = 255, hi = 0;
        for (int dr = 0; dr < a.k; ++dr)
            for (int dc = 0; dc < a.k; ++dc) {
                const uint32_t v = px(y, x, dr, dc);
                lo = min(lo, v);
                hi = max(hi, v);
            }
        uint32_t med = lo;
        if (lo != hi) {
            // bits above the highest bit where lo and hi differ are common to every window value
            const int hb = 31 - __clz(lo ^ hi);
            uint32_t prefix = lo & ~((2u << hb) - 1u);
            int below = 0;
            for (int b = hb; b >= 0; --b) {
                const uint32_t mask = (0xFFu << b) & 0xFFu;
                int c = 0;  // values with the current prefix and bit b clear
                for (int dr = 0; dr < a.k; ++dr)
                    for (int dc = 0; dc < a.k; ++dc) c += ((px(y, x, dr, dc) ^ prefix) & mask) == 0;
                if (below + c <= m) {
                    below += c;
                    prefix |= 1u << b;
                }
            }
            med = prefix;
        }
        const size_t o = (size_t)y * a.opitch + x;
        if (a.zmin) a.zmin[o] = (uint8_t)lo;
        if (a.zmed) a.zmed[o] = (uint8_t)med;
        if (a.zmax) a.zmax[o] = (uint8_t)hi;
    }
}

}  // namespace

cudaError_t launch_window_stats(const uint8_t* src, size_t pitch, int rows, int cols, int k, uint8_t* zmin,
                                uint8_t* zmed, uint8_t* zmax, size_t opitch, cudaStream_t stream) {
    WsArgs a{src, pitch, rows, cols, k, zmin, zmed, zmax, opitch};
    const dim3 grid((cols + WT - 1) / WT, (rows + WT - 1) / WT), block(WT, WTY);
    const int R = k / 2;
    cudaError_t e;
    if (R <= kMaxR) {
        static PerDevice attr;
        const size_t smem = (size_t)(WT + 2 * R) * (WT + 2 * R);
        e = ensure_smem_attr(attr, (const void*)window_stats_kernel<true>, smem);
        if (e != cudaSuccess) return e;
        e = launch_pdl(window_stats_kernel<true>, grid, block, smem, stream, a);
    } else {
        e = launch_pdl(window_stats_kernel<false>, grid, block, 0, stream, a);
    }
    count_launch();
    return e;
}

}  // namespace hyb
