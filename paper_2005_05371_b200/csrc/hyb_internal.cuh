// hyb_internal.cuh -- shared declarations of libhybrid_cuda (kernels + launchers).
#pragma once
#include <algorithm>
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace hyb {

// ---- per-device launch setup ----
// Function attributes (the >48 KB dynamic shared-memory opt-in), occupancies and SM counts belong to
// one device; a process may drive several devices (one context each, or a multi-device context) from
// several host threads.  Each call site keeps one PerDevice cache (static storage: zero-initialised);
// racing threads may compute the same value twice, which is harmless.
constexpr int kMaxDevices = 64;
struct PerDevice {
    std::atomic<long long> v[kMaxDevices];
};
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}
inline int device_sms() {
    static PerDevice cache;
    const int d = current_device();
    if (d < kMaxDevices) {
        const long long c = cache.v[d].load(std::memory_order_acquire);
        if (c) return (int)c;
    }
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    if (n < 1) n = 1;
    if (d < kMaxDevices) cache.v[d].store(n, std::memory_order_release);
    return n;
}
// Dynamic shared-memory opt-in of `kern` on the current device, raised to at least `smem` bytes.
inline cudaError_t ensure_smem_attr(PerDevice& pd, const void* kern, size_t smem) {
    const int d = current_device();
    if (d < kMaxDevices && (size_t)pd.v[d].load(std::memory_order_acquire) >= smem) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess && d < kMaxDevices) {
        long long cur = pd.v[d].load(std::memory_order_relaxed);
        while (cur < (long long)smem && !pd.v[d].compare_exchange_weak(cur, (long long)smem)) {
        }
    }
    return e;
}
// Resident blocks per SM of `kern` on the current device at (threads, smem), cached per device (the
// cache entry is keyed by smem; at least 1).
inline int occupancy(PerDevice& pd, const void* kern, int threads, size_t smem) {
    const int d = current_device();
    const long long key = (long long)smem << 16;
    if (d < kMaxDevices) {
        const long long c = pd.v[d].load(std::memory_order_acquire);
        if (c && (c & ~0xFFFFll) == key) return (int)(c & 0xFFFF);
    }
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    if (n < 1) n = 1;
    if (d < kMaxDevices) pd.v[d].store(key | n, std::memory_order_release);
    return n;
}

// Geometry of one filtering launch: `n_slices` images of rows x cols with byte
// pitches and slice strides.  Output row i corresponds to input row row_begin + i.
struct Plane {
    const uint8_t* src;
    size_t spitch;
    size_t sslice;
    uint8_t* dst;
    size_t dpitch;
    size_t dslice;
    int rows, cols;
    int row_begin, row_end;
    int n_slices;
};

// Device workspace of the AMF (amf_work_bytes(p) bytes, carved by amf_work): 64 bytes of counters
// (zero when allocated; every launch leaves them zero), one failure record per k = 3 tile with
// level-A failures, and the per-tile failure bitmap (512 bytes per 128 x 32 tile).
struct AmfWork {
    int* counters;                 // [0..1] record counter (u64), [2] tile claims, [3] / [4] CTAs done,
                                   // [5] growth chunk claims, [6] compact growth entries, [7] their chunk claims
    unsigned long long* records;   // (failure offset << 24) | tile
    uint8_t* bitmap;
    int* chunk_rec;                // [chunk]: the record holding weighted position chunk * CHUNK
    uint4* cq;                     // compact growth entries (64 bytes each), counter = counters[6]
    int cq_cap;
};
size_t amf_work_bytes(const Plane& p);
AmfWork amf_work(uint8_t* base, const Plane& p);

// Launch with programmatic stream serialization: the kernel's prologue may overlap the previous
// kernel's tail; every kernel launched this way calls griddepcontrol.wait before touching memory
// the previous grids produce or consume.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<Args&&>(args)...);
}

// AMF launch (amf.cu): k = 3 tile kernel + one tile-wise growth kernel (k = 5..smax).  fin may be null.
cudaError_t launch_amf(const Plane& p, int smax, uint8_t* fin, size_t fpitch, size_t fslice,
                       const AmfWork& work, cudaStream_t stream);

// W1 statistics launch (wiener.cu): adds sum of V over the rows into noise_sum[slice].
cudaError_t launch_wiener_stats(const Plane& p, int win, unsigned long long* noise_sum,
                                cudaStream_t stream);
// W1 gain launch: noise_sum[slice] read on the device; pixel_count per slice.  mm (nullable, device, 2 u32):
// also fold the range of the y it writes into mm[0] = min, mm[1] = 255 - max (atomicMin; the caller
// initialises both to 0xFFFFFFFF) -- contrast_stretch's min / max fused into the gain.
cudaError_t launch_wiener_gain(const Plane& p, int win, const long long* noise_sum,
                               long long pixel_count, cudaStream_t stream, unsigned* mm = nullptr);

// Fused single-kernel hybrid step for small single images (small.cu): every CTA keeps its tiles
// resident; two grid barriers (cooperative launch).  plan_small says whether it applies.
struct SmallPlan {
    bool ok;
    int grid;
    int slot_bytes;
};
SmallPlan plan_small(int rows, int cols, int smax, int win);
struct SmallBufs {
    const uint8_t* g;  // TMA-compatible
    size_t gpitch;
    uint8_t* f;        // AMF output scratch, TMA-compatible
    size_t fpitch;
    uint8_t* y;
    size_t ypitch;
    unsigned long long* wsum;      // W (zeroed in the kernel)
    unsigned* sbar;                // 32 bytes, zero when allocated: barrier / exit counters, 3 globaltimer stamps
};
// cooperative: launch with cudaLaunchAttributeCooperative (co-residency guaranteed by the driver);
// otherwise a plain launch whose grid never exceeds the occupancy (caller: exclusive device).
cudaError_t launch_small(const SmallPlan& pl, const SmallBufs& bufs, int rows, int cols, int smax, int win,
                         bool cooperative, cudaStream_t stream);

// contrast_stretch (stretch.cu): mm = 2 u32 device scratch; src == dst allowed.
cudaError_t launch_contrast_stretch(const uint8_t* src, size_t spitch, int rows, int cols, uint8_t* dst,
                                    size_t dpitch, unsigned* mm, cudaStream_t stream);
// its two passes: fold src's range into mm (mm[0] = min, mm[1] = 255 - max, atomicMin: initialise both to
// 0xFFFFFFFF first), and the exact LUT map with the range mm holds
cudaError_t launch_stretch_minmax(const uint8_t* src, size_t spitch, int rows, int cols, unsigned* mm,
                                  cudaStream_t stream);
cudaError_t launch_stretch_map(const uint8_t* src, size_t spitch, int rows, int cols, uint8_t* dst, size_t dpitch,
                               const unsigned* mm, cudaStream_t stream);
// multi-device stretch: out[0..1] = the elementwise min of the n devices' mm pairs (peer reads)
struct MmPartials {
    const unsigned* p[kMaxDevices];
    int n;
};
cudaError_t launch_min_partials(const MmPartials& parts, unsigned* out, cudaStream_t stream);

// window_stats (wstats.cu): min / median / max planes of the k x k windows; outputs nullable.
cudaError_t launch_window_stats(const uint8_t* src, size_t pitch, int rows, int cols, int k, uint8_t* zmin,
                                uint8_t* zmed, uint8_t* zmax, size_t opitch, cudaStream_t stream);

// Frequency-domain Wiener + noise estimates (freq.cu, doubles like the reference).
struct FreqWork {
    unsigned long long plan_f = 0, plan_i = 0;  // cufftHandle
    int rows = 0, cols = 0;
    double* real = nullptr;
    void* bins = nullptr;  // double2 (Hermitian half)
    double* keys = nullptr;
    void* tmp = nullptr;   // CUB scratch
    size_t real_n = 0, bins_n = 0, keys_n = 0, tmp_n = 0;
    ~FreqWork();
    void release();
};
// pitches in elements; cufft_status != 0 reports a cuFFT failure
cudaError_t launch_wiener_freq(const double* in, size_t ipitch, int rows, int cols, double sigma2, bool clamp,
                               double* out, size_t opitch, FreqWork& w, cudaStream_t stream, int* cufft_status);
// d_sigma_med <- median(|p - median3(p)|) (device double)
cudaError_t launch_noise_robust(const double* in, size_t ipitch, int rows, int cols, FreqWork& w, double* d_sigma_med,
                                cudaStream_t stream);
// contrast_stretch on doubles (in == out allowed)
cudaError_t launch_contrast_stretch_f64(const double* in, size_t ipitch, int rows, int cols, double* out,
                                        size_t opitch, FreqWork& w, cudaStream_t stream);
// d_acc <- sum (a - b)^2 (device double)
cudaError_t launch_noise_reference(const double* a, size_t ap, const double* b, size_t bp, int rows, int cols,
                                   double* d_acc, cudaStream_t stream);

// Multi-device noise reduction (multi.cu): *out = sum of the n int64 partials, each in this device's
// memory or in a peer device's memory readable over NVLink (peer access enabled).
struct Partials {
    const long long* p[kMaxDevices];
    int n;
};
cudaError_t launch_sum_partials(const Partials& parts, long long* out, cudaStream_t stream);

// Kernel-launch counter (bench evidence), incremented by every launcher.
void count_launch();

}  // namespace hyb
