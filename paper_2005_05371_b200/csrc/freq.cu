// freq.cu -- the reference's own Wiener stage: the frequency-domain Wiener
// filter (proj/src/wiener.cpp:54-77 over proj/src/dft2.cpp:32-56) and its noise estimates
// (proj/src/wiener.cpp:30-52), in double precision like the reference.
//
//   wiener_filter: forward real-to-complex 2-D DFT (cuFFT D2Z; the Hermitian half carries every bin
//   the reference's full complex spectrum has, and the gain is symmetric), per-bin gain
//   (P - N0) / P or 0 with N0 = rows * cols * sigma2 (one fused kernel), inverse C2R, x 1/(rows cols),
//   optional clamp to [0, 1] (fused into the scale kernel).  sigma2 == 0 returns the input.
//   Robust estimate: per pixel |p - median3(p)| (3x3, replicated borders, a 19-exchange network in
//   registers) -> keys sorted on the device (CUB radix sort) -> median (even counts average the two
//   middle values) / 0.6745, squared.  Reference estimate: mean squared difference (block
//   reduction, one double atomic per CTA).
#include <cub/cub.cuh>
#include <cufft.h>

#include <cstdint>

#include "hyb_internal.cuh"

namespace hyb {
namespace {

constexpr int FT = 256;

__global__ void __launch_bounds__(FT) pack_kernel(const double* __restrict__ in, size_t ipitch, int rows, int cols,
                                                 double* __restrict__ out) {
    const long long n = (long long)rows * cols;
    for (long long i = (long long)blockIdx.x * FT + threadIdx.x; i < n; i += (long long)gridDim.x * FT) {
        const int r = (int)(i / cols), c = (int)(i - (long long)r * cols);
        out[i] = in[(size_t)r * ipitch + c];
    }
}

__global__ void __launch_bounds__(FT) gain_kernel(double2* __restrict__ bins, long long n, double n0) {
    for (long long i = (long long)blockIdx.x * FT + threadIdx.x; i < n; i += (long long)gridDim.x * FT) {
        double2 b = bins[i];
        const double p = b.x * b.x + b.y * b.y;  // std::norm
        const double g = p > n0 ? (p - n0) / p : 0.0;
        b.x *= g;
        b.y *= g;
        bins[i] = b;
    }
}

__device__ __forceinline__ double clamp01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

__global__ void __launch_bounds__(FT) scale_kernel(const double* __restrict__ in, int rows, int cols, double norm,
                                                  bool clamp, double* __restrict__ out, size_t opitch) {
    const long long n = (long long)rows * cols;
    for (long long i = (long long)blockIdx.x * FT + threadIdx.x; i < n; i += (long long)gridDim.x * FT) {
        const int r = (int)(i / cols), c = (int)(i - (long long)r * cols);
        const double v = in[i] * norm;
        out[(size_t)r * opitch + c] = clamp ? clamp01(v) : v;
    }
}

// sigma2 == 0: the input itself (clamped on request), wiener.cpp:58-66
__global__ void __launch_bounds__(FT) copy_kernel(const double* __restrict__ in, size_t ipitch, int rows, int cols,
                                                 bool clamp, double* __restrict__ out, size_t opitch) {
    const long long n = (long long)rows * cols;
    for (long long i = (long long)blockIdx.x * FT + threadIdx.x; i < n; i += (long long)gridDim.x * FT) {
        const int r = (int)(i / cols), c = (int)(i - (long long)r * cols);
        const double v = in[(size_t)r * ipitch + c];
        out[(size_t)r * opitch + c] = clamp ? clamp01(v) : v;
    }
}

__global__ void single_kernel(const double* __restrict__ in, double sigma2, bool clamp, double* __restrict__ out) {
    const double v = in[0], p = v * v;
    const double g = p > sigma2 ? (p - sigma2) / p : 0.0;
    const double o = v * g;
    out[0] = clamp ? clamp01(o) : o;
}

__device__ __forceinline__ void cx(double& a, double& b) {
    const double lo = fmin(a, b), hi = fmax(a, b);
    a = lo;
    b = hi;
}

// |p - median3(p)| per pixel (3x3 window, coordinates clamped to the image)
__global__ void __launch_bounds__(FT) residual_kernel(const double* __restrict__ in, size_t ipitch, int rows, int cols,
                                                     double* __restrict__ res) {
    const long long n = (long long)rows * cols;
    for (long long i = (long long)blockIdx.x * FT + threadIdx.x; i < n; i += (long long)gridDim.x * FT) {
        const int r = (int)(i / cols), c = (int)(i - (long long)r * cols);
        double v[9];
        int k = 0;
        for (int dr = -1; dr <= 1; ++dr) {
            const int rr = min(max(r + dr, 0), rows - 1);
            for (int dc = -1; dc <= 1; ++dc) {
                const int cc = min(max(c + dc, 0), cols - 1);
                v[k++] = in[(size_t)rr * ipitch + cc];
            }
        }
        // median of 9 (Paeth's 19-exchange network)
        cx(v[1], v[2]); cx(v[4], v[5]); cx(v[7], v[8]); cx(v[0], v[1]); cx(v[3], v[4]);
        cx(v[6], v[7]); cx(v[1], v[2]); cx(v[4], v[5]); cx(v[7], v[8]); cx(v[0], v[3]);
        cx(v[5], v[8]); cx(v[4], v[7]); cx(v[3], v[6]); cx(v[1], v[4]); cx(v[2], v[5]);
        cx(v[4], v[7]); cx(v[4], v[2]); cx(v[6], v[4]); cx(v[4], v[2]);
        res[i] = fabs(in[(size_t)r * ipitch + c] - v[4]);
    }
}

__global__ void __launch_bounds__(FT) sqdiff_kernel(const double* __restrict__ a, size_t ap, const double* __restrict__ b,
                                                   size_t bp, int rows, int cols, double* __restrict__ acc) {
    const long long n = (long long)rows * cols;
    double s = 0.0;
    for (long long i = (long long)blockIdx.x * FT + threadIdx.x; i < n; i += (long long)gridDim.x * FT) {
        const int r = (int)(i / cols), c = (int)(i - (long long)r * cols);
        const double d = a[(size_t)r * ap + c] - b[(size_t)r * bp + c];
        s += d * d;
    }
    using BR = cub::BlockReduce<double, FT>;
    __shared__ typename BR::TempStorage tmp;
    s = BR(tmp).Sum(s);
    if (threadIdx.x == 0) atomicAdd(acc, s);
}

__global__ void median_kernel(const double* __restrict__ sorted, long long n, double* __restrict__ out) {
    const double m = sorted[n / 2];
    out[0] = (n % 2 == 0) ? (m + sorted[n / 2 - 1]) / 2.0 : m;
}

// contrast_stretch on doubles (proj/src/pipeline.cpp:10-21): per-CTA min / max partials, one CTA folds
// them, then (p - lo) / (hi - lo) -- the reference's own operations, so bit-identical results.
__global__ void __launch_bounds__(FT) minmax_f64_kernel(const double* __restrict__ in, size_t ipitch, int rows,
                                                       int cols, double* __restrict__ part) {
    const long long n = (long long)rows * cols;
    double lo = INFINITY, hi = -INFINITY;
    for (long long i = (long long)blockIdx.x * FT + threadIdx.x; i < n; i += (long long)gridDim.x * FT) {
        const int r = (int)(i / cols), c = (int)(i - (long long)r * cols);
        const double v = in[(size_t)r * ipitch + c];
        lo = fmin(lo, v);
        hi = fmax(hi, v);
    }
    using BR = cub::BlockReduce<double, FT>;
    __shared__ typename BR::TempStorage t0, t1;
    lo = BR(t0).Reduce(lo, cub::Min());
    hi = BR(t1).Reduce(hi, cub::Max());
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = lo;
        part[2 * blockIdx.x + 1] = hi;
    }
}

__global__ void __launch_bounds__(FT) fold_kernel(double* __restrict__ part, int nparts) {
    double lo = INFINITY, hi = -INFINITY;
    for (int i = threadIdx.x; i < nparts; i += FT) {
        lo = fmin(lo, part[2 * i]);
        hi = fmax(hi, part[2 * i + 1]);
    }
    using BR = cub::BlockReduce<double, FT>;
    __shared__ typename BR::TempStorage t0, t1;
    lo = BR(t0).Reduce(lo, cub::Min());
    hi = BR(t1).Reduce(hi, cub::Max());
    if (threadIdx.x == 0) {
        part[0] = lo;
        part[1] = hi;
    }
}

__global__ void __launch_bounds__(FT) stretch_f64_kernel(const double* __restrict__ in, size_t ipitch, int rows,
                                                        int cols, const double* __restrict__ mm,
                                                        double* __restrict__ out, size_t opitch) {
    const double lo = mm[0], hi = mm[1], range = hi - lo;
    const long long n = (long long)rows * cols;
    for (long long i = (long long)blockIdx.x * FT + threadIdx.x; i < n; i += (long long)gridDim.x * FT) {
        const int r = (int)(i / cols), c = (int)(i - (long long)r * cols);
        const double p = in[(size_t)r * ipitch + c];
        out[(size_t)r * opitch + c] = hi == lo ? p : (p - lo) / range;
    }
}

int grid_for(long long n) {
    const int sms = device_sms();
    return (int)std::max(1ll, std::min((long long)sms * 8, (n + FT - 1) / FT));
}

}  // namespace

FreqWork::~FreqWork() { release(); }

void FreqWork::release() {
    if (plan_f) cufftDestroy((cufftHandle)plan_f);
    if (plan_i) cufftDestroy((cufftHandle)plan_i);
    plan_f = plan_i = 0;
    if (real) cudaFree(real);
    if (bins) cudaFree(bins);
    if (keys) cudaFree(keys);
    if (tmp) cudaFree(tmp);
    real = nullptr;
    bins = nullptr;
    keys = nullptr;
    tmp = nullptr;
    rows = cols = 0;
    real_n = bins_n = keys_n = tmp_n = 0;
}

static cudaError_t grow(void** p, size_t* have, size_t want) {
    if (want <= *have) return cudaSuccess;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *have = 0;
    cudaError_t e = cudaMalloc(p, want);
    if (e == cudaSuccess) *have = want;
    return e;
}

// cuFFT plans for rows x cols (real <-> Hermitian half); 1-D when one side is 1.
static int ensure_plans(FreqWork& w, int rows, int cols) {
    if (w.plan_f && w.rows == rows && w.cols == cols) return 0;
    if (w.plan_f) cufftDestroy((cufftHandle)w.plan_f);
    if (w.plan_i) cufftDestroy((cufftHandle)w.plan_i);
    w.plan_f = w.plan_i = 0;
    cufftHandle f = 0, i = 0;
    cufftResult r;
    if (rows == 1 || cols == 1) {
        const int n = rows * cols;
        r = cufftPlan1d(&f, n, CUFFT_D2Z, 1);
        if (r == CUFFT_SUCCESS) r = cufftPlan1d(&i, n, CUFFT_Z2D, 1);
    } else {
        r = cufftPlan2d(&f, rows, cols, CUFFT_D2Z);
        if (r == CUFFT_SUCCESS) r = cufftPlan2d(&i, rows, cols, CUFFT_Z2D);
    }
    if (r != CUFFT_SUCCESS) return (int)r;
    w.plan_f = (unsigned long long)f;
    w.plan_i = (unsigned long long)i;
    w.rows = rows;
    w.cols = cols;
    return 0;
}

cudaError_t launch_wiener_freq(const double* in, size_t ipitch, int rows, int cols, double sigma2, bool clamp,
                               double* out, size_t opitch, FreqWork& w, cudaStream_t stream, int* cufft_status) {
    *cufft_status = 0;
    const long long n = (long long)rows * cols;
    if (sigma2 == 0.0) {
        copy_kernel<<<grid_for(n), FT, 0, stream>>>(in, ipitch, rows, cols, clamp, out, opitch);
        count_launch();
        return cudaGetLastError();
    }
    if (n == 1) {  // the 1 x 1 DFT is the identity
        single_kernel<<<1, 1, 0, stream>>>(in, sigma2, clamp, out);
        count_launch();
        return cudaGetLastError();
    }
    const bool one_d = rows == 1 || cols == 1;
    const long long half = one_d ? (n / 2 + 1) : (long long)rows * (cols / 2 + 1);
    cudaError_t e = grow((void**)&w.real, &w.real_n, (size_t)n * sizeof(double));
    if (e == cudaSuccess) e = grow((void**)&w.bins, &w.bins_n, (size_t)half * sizeof(double2));
    if (e != cudaSuccess) return e;
    if ((*cufft_status = ensure_plans(w, rows, cols))) return cudaSuccess;
    cufftSetStream((cufftHandle)w.plan_f, stream);
    cufftSetStream((cufftHandle)w.plan_i, stream);
    pack_kernel<<<grid_for(n), FT, 0, stream>>>(in, ipitch, rows, cols, w.real);
    count_launch();
    if ((*cufft_status = (int)cufftExecD2Z((cufftHandle)w.plan_f, w.real, (cufftDoubleComplex*)w.bins)))
        return cudaSuccess;
    gain_kernel<<<grid_for(half), FT, 0, stream>>>((double2*)w.bins, half, (double)rows * cols * sigma2);
    count_launch();
    if ((*cufft_status = (int)cufftExecZ2D((cufftHandle)w.plan_i, (cufftDoubleComplex*)w.bins, w.real)))
        return cudaSuccess;
    scale_kernel<<<grid_for(n), FT, 0, stream>>>(w.real, rows, cols, 1.0 / ((double)rows * cols), clamp, out, opitch);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_noise_robust(const double* in, size_t ipitch, int rows, int cols, FreqWork& w, double* d_sigma_med,
                                cudaStream_t stream) {
    const long long n = (long long)rows * cols;
    cudaError_t e = grow((void**)&w.keys, &w.keys_n, (size_t)2 * n * sizeof(double));
    if (e != cudaSuccess) return e;
    double* res = w.keys;
    double* sorted = w.keys + n;
    size_t need = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, need, res, sorted, (int)n, 0, 64, stream);
    if ((e = grow(&w.tmp, &w.tmp_n, need)) != cudaSuccess) return e;
    residual_kernel<<<grid_for(n), FT, 0, stream>>>(in, ipitch, rows, cols, res);
    count_launch();
    if ((e = cub::DeviceRadixSort::SortKeys(w.tmp, need, res, sorted, (int)n, 0, 64, stream)) != cudaSuccess) return e;
    count_launch();
    median_kernel<<<1, 1, 0, stream>>>(sorted, n, d_sigma_med);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_contrast_stretch_f64(const double* in, size_t ipitch, int rows, int cols, double* out,
                                        size_t opitch, FreqWork& w, cudaStream_t stream) {
    const long long n = (long long)rows * cols;
    const int grid = grid_for(n);
    cudaError_t e = grow((void**)&w.keys, &w.keys_n, (size_t)2 * grid * sizeof(double));
    if (e != cudaSuccess) return e;
    minmax_f64_kernel<<<grid, FT, 0, stream>>>(in, ipitch, rows, cols, w.keys);
    fold_kernel<<<1, FT, 0, stream>>>(w.keys, grid);
    stretch_f64_kernel<<<grid, FT, 0, stream>>>(in, ipitch, rows, cols, w.keys, out, opitch);
    count_launch();
    count_launch();
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_noise_reference(const double* a, size_t ap, const double* b, size_t bp, int rows, int cols,
                                   double* d_acc, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(d_acc, 0, sizeof(double), stream);
    if (e != cudaSuccess) return e;
    sqdiff_kernel<<<grid_for((long long)rows * cols), FT, 0, stream>>>(a, ap, b, bp, rows, cols, d_acc);
    count_launch();
    return cudaGetLastError();
}

}  // namespace hyb
