/*
 * hybrid_cuda.h -- C ABI of libhybrid_cuda: the B200 (sm_100a) hybrid
 * adaptive-median + local-Wiener denoiser of arXiv 2005.05371.
 *
 * The reference (`denoise`, proj/ in the reference tree) is a static C++
 * library of free functions; there is no plugin registry.  Each entry point
 * below replaces one reference call site (file:line into the reference's
 * proj/ directory) with plain pointers and sizes.  No C++ exceptions cross
 * this boundary: every call returns a status code, and hyb_last_error()
 * returns the message text the reference would have thrown.
 *
 * Pixels are uint8 (the reference's doubles k/255, proj/src/pgm_io.cpp:73,88;
 * the AMF commutes with that map exactly, so results are bit-identical).
 * Every image pointer may be HOST or DEVICE memory (detected per call):
 *   - device pointers: work is enqueued on the context stream and the call
 *     returns without synchronising (unless a host-side output such as a
 *     hyb_stats struct or a host noise_sum must be filled);
 *   - host pointers: the call stages through context-owned pitched device
 *     buffers and returns after the result is back in host memory.
 * The context owns all device scratch; callers own their buffers.
 */
#ifndef HYBRID_CUDA_H
#define HYBRID_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. */
#define HYB_OK 0
#define HYB_EINVAL 1 /* reference throws std::invalid_argument */
#define HYB_ECUDA 2  /* CUDA runtime error (std::runtime_error on the host side) */
#define HYB_ENCCL 3  /* reserved: collective failure */
#define HYB_ENOMEM 4 /* device allocation failed */

typedef struct hyb_ctx hyb_ctx;

/* Per-call statistics (reference HybridResult, proj/include/denoise/pipeline.hpp:12-18). */
typedef struct hyb_stats {
    int64_t noise_sum;   /* W = sum of V = n*S2 - S1^2 over all pixels (exact) */
    int64_t pixel_count; /* P */
    double sigma2;       /* nu / 255^2 = W / (n^2 P) / 255^2, intensity^2 units like HybridResult.sigma2 */
    double t_adaptive;   /* seconds, device time of the AMF stage (CUDA events) */
    double t_wiener;     /* seconds, device time of the Wiener stage */
    double t_total;      /* seconds, device time of the whole call incl. staging copies */
} hyb_stats;

/* Context: one CUDA device, one stream, pooled device scratch.  Not
 * thread-safe per context (one context per host thread), like the
 * reference's per-call pool (proj/src/parallel.cpp:62-65). */
hyb_ctx* hyb_create(int device, int* status);
int hyb_destroy(hyb_ctx* ctx);
/* Multi-device context: the paper's 2/4/8-partition scheme on one box, behind the same entry points
 * (reference FilterConfig.parts / workers, proj/include/denoise/parallel.hpp:13-19, executed by
 * adaptive_median_parallel proj/src/parallel.cpp:27-70; SURVEY.md 8(b) sketched hyb_create(n_gpus,
 * device_ids)).  Strip i of an image runs on device_ids[i] (ids may repeat: several strips on one
 * GPU); peer access is enabled between all pairs of distinct devices that support it (NVLink).
 * hyb_hybrid_u8 on this context splits the image into n_devices horizontal strips (split_bands
 * geometry, halo (smax-1)/2 + (win-1)/2 rows read straight from the caller's buffer), filters them
 * concurrently, reduces the exact int64 noise sum over NVLink (each device reads its peers'
 * partials) and applies the gain -- bit-identical to one device for every n.  hyb_hybrid_batch_u8
 * shards the slices of a stack by contiguous chunks, one per device.  Every other entry point runs on
 * device_ids[0].  hyb_destroy releases all devices' resources. */
hyb_ctx* hyb_create_multi(int n_devices, const int* device_ids, int* status);
/* Number of devices a context drives (1 for hyb_create); device_ids (nullable) receives them. */
int hyb_context_devices(const hyb_ctx* ctx, int* device_ids);
/* Use a caller-owned cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); NULL restores the context stream. */
int hyb_set_stream(hyb_ctx* ctx, void* stream);
/* exclusive != 0: the caller guarantees that no other kernels run on this device while this
 * context's calls execute (a dedicated GPU).  The fused small-image kernel, whose CTAs meet at
 * grid barriers, is then launched as a plain (graph-capturable) kernel sized to the device's
 * occupancy instead of a cooperative launch (~4-6 us cheaper per call).  Default 0: cooperative
 * launch, which guarantees co-residency even with concurrent work.  (Library extension; the
 * reference has no device.) */
int hyb_set_exclusive(hyb_ctx* ctx, int exclusive);
/* async_host != 0: hyb_hybrid_u8 calls (parts = 1, no hyb_stats) on PINNED host buffers return as soon
 * as the work is enqueued.  Device staging is double-buffered, so the next call's upload overlaps this
 * call's download (a stream of images keeps both PCIe directions busy).  The caller must not touch the
 * buffers of a pending call; results are complete after hyb_synchronize() (or hyb_set_async(ctx, 0)).
 * Other calls and pageable buffers keep the synchronous behaviour.  (Library extension.) */
int hyb_set_async(hyb_ctx* ctx, int async_host);
/* Waits for every call enqueued on the context (all its streams, all its devices). */
int hyb_synchronize(hyb_ctx* ctx);
const char* hyb_last_error(const hyb_ctx* ctx);
/* Number of kernels this context has launched so far (bench evidence). */
int64_t hyb_kernel_launches(const hyb_ctx* ctx);

/* validate_smax -- reference proj/src/adaptive_median.cpp:11-16.
 * HYB_EINVAL unless smax is odd and > 1 ("smax must be an odd integer > 1, got N"). */
int hyb_validate_smax(int smax);
/* validate_config -- reference proj/src/parallel.cpp:16-25 (smax, parts >= 1, workers >= 1). */
int hyb_validate_config(int smax, int parts, int workers);

/* detail::adaptive_median_rows -- reference proj/include/denoise/adaptive_median.hpp:47-48,
 * proj/src/adaptive_median.cpp:123-215; called from proj/src/adaptive_median.cpp:222 and the band
 * worker at proj/src/parallel.cpp:49-50.  Filters rows [row_begin, row_end) of src (rows x cols)
 * into dst ((row_end-row_begin) x cols); windows clamp to src's bounds (edge replication).
 * finalized_at (nullable) receives the finalizing window size per pixel, 0 if never finalized. */
int hyb_amf_u8(hyb_ctx* ctx, const uint8_t* src, size_t src_pitch, int rows, int cols,
               int row_begin, int row_end, int smax, uint8_t* dst, size_t dst_pitch,
               uint8_t* finalized_at, size_t fin_pitch);

/* Batched AMF over n_slices images of rows x cols each (slice strides in bytes);
 * whole slices (row range [0, rows)).  Serves the CT-stack configuration. */
int hyb_amf_batch_u8(hyb_ctx* ctx, const uint8_t* src, size_t src_pitch, size_t src_slice_stride,
                     int n_slices, int rows, int cols, int smax, uint8_t* dst, size_t dst_pitch,
                     size_t dst_slice_stride);

/* window_stats -- reference proj/src/adaptive_median.cpp:96-119 (proj/include/denoise/adaptive_median.hpp:16-24):
 * per pixel the min, median (sorted index (k^2-1)/2) and max of its k x k window, edge replication.
 * k odd >= 3 (HYB_EINVAL "window size must be an odd integer >= 3, got N").  The three output planes share
 * out_pitch; any of them may be NULL (not computed). */
int hyb_window_stats_u8(hyb_ctx* ctx, const uint8_t* src, size_t pitch, int rows, int cols, int k,
                        uint8_t* zmin, uint8_t* zmed, uint8_t* zmax, size_t out_pitch);

/* W1 local-Wiener noise statistics (replaces estimate_noise_variance, reference
 * proj/include/denoise/wiener.hpp:23, call site proj/src/pipeline.cpp:46-50).
 * Adds W = sum of V over rows [row_begin, row_end) of f to *noise_sum (host or device int64);
 * windows win x win (odd, 1..63) clamp to f's bounds. */
int hyb_wiener_stats_u8(hyb_ctx* ctx, const uint8_t* f, size_t pitch, int rows, int cols,
                        int row_begin, int row_end, int win, int64_t* noise_sum);

/* W1 gain (replaces wiener_filter, reference proj/include/denoise/wiener.hpp:29, call site
 * proj/src/pipeline.cpp:51): y = mu + max(v - nu, 0)/v * (f - mu), nu = W/(n^2 P), rounded half
 * away from zero, for rows [row_begin, row_end) of f into y.  noise_sum may be host or device. */
int hyb_wiener_gain_u8(hyb_ctx* ctx, const uint8_t* f, size_t pitch, int rows, int cols,
                       int row_begin, int row_end, int win, const int64_t* noise_sum,
                       int64_t pixel_count, uint8_t* y, size_t y_pitch);

/* Whole-image W1 (stats, then gain).  noise_sum_out (nullable, host) receives W. */
int hyb_wiener_u8(hyb_ctx* ctx, const uint8_t* f, size_t pitch, int rows, int cols, int win,
                  uint8_t* y, size_t y_pitch, int64_t* noise_sum_out);

/* hybrid_denoise stages 1-2 -- reference proj/src/pipeline.cpp:23-53 (call sites
 * proj/tools/hybridfilter.cpp:96-97,228,240) with adaptive_median_parallel's band split
 * (proj/src/parallel.cpp:27-70, proj/src/tiling.cpp:10-45): `parts` horizontal strips with halo
 * (smax-1)/2 + (win-1)/2, each filtered as an independent sub-launch from its own strip copy,
 * one exact int64 noise reduction, then the gain per strip.  Bit-identical for every parts.
 * stats (nullable) is filled on return (forces a synchronisation). */
int hyb_hybrid_u8(hyb_ctx* ctx, const uint8_t* g, size_t pitch, int rows, int cols, int smax,
                  int win, int parts, uint8_t* y, size_t y_pitch, hyb_stats* stats);

/* Batched hybrid over a CT-like stack: each slice is an independent image with its own noise
 * estimate (no cross-slice reduction).  noise_sums (nullable, host, n_slices entries). */
int hyb_hybrid_batch_u8(hyb_ctx* ctx, const uint8_t* g, size_t pitch, size_t slice_stride,
                        int n_slices, int rows, int cols, int smax, int win, uint8_t* y,
                        size_t y_pitch, size_t y_slice_stride, int64_t* noise_sums);

/* contrast_stretch -- reference proj/src/pipeline.cpp:10-21: out = (v - lo)
 * / (hi - lo) over the image min / max, as uint8 = floor((510 (v - lo) + (hi - lo)) / (2 (hi - lo)))
 * (the exact rational rounded half up; lo -> 0, hi -> 255); unchanged when hi == lo.  src == dst
 * allowed (in place). */
int hyb_contrast_stretch_u8(hyb_ctx* ctx, const uint8_t* src, size_t pitch, int rows, int cols,
                            uint8_t* dst, size_t dst_pitch);

/* hybrid_denoise stages 1-3 (stretch_after_each = false): hyb_hybrid_u8, then the final
 * contrast_stretch (proj/src/pipeline.cpp:55). */
int hyb_hybrid_stretch_u8(hyb_ctx* ctx, const uint8_t* g, size_t pitch, int rows, int cols, int smax,
                          int win, int parts, uint8_t* y, size_t y_pitch, hyb_stats* stats);

/* The reference's own Wiener stage, doubles like the reference; pitches
 * in elements; host or device pointers.
 * wiener_filter proj/src/wiener.cpp:54-77 (+ dft2 proj/src/dft2.cpp:32-56): per-bin gain
 * (P - N0) / P, N0 = rows * cols * sigma2, zero where noise dominates; output clamped to [0, 1]
 * when clamp != 0; sigma2 == 0 returns the input; sigma2 < 0 -> HYB_EINVAL. */
int hyb_wiener_freq_f64(hyb_ctx* ctx, const double* f, size_t pitch, int rows, int cols, double sigma2,
                        int clamp, double* out, size_t out_pitch);
/* contrast_stretch on doubles, proj/src/pipeline.cpp:10-21 (the reference's operations: bit-identical). */
int hyb_contrast_stretch_f64(hyb_ctx* ctx, const double* src, size_t pitch, int rows, int cols, double* dst,
                             size_t dst_pitch);
/* estimate_noise_variance without a reference, proj/src/wiener.cpp:44-51:
 * sigma = median(|p - median3(p)|) / 0.6745 (3x3, replicated borders), sigma2 = sigma^2. */
int hyb_noise_robust_f64(hyb_ctx* ctx, const double* f, size_t pitch, int rows, int cols, double* sigma2);
/* estimate_noise_variance with a reference, proj/src/wiener.cpp:31-42: mean squared difference. */
int hyb_noise_reference_f64(hyb_ctx* ctx, const double* f, size_t pitch, const double* ref, size_t ref_pitch,
                            int rows, int cols, double* sigma2);

/* Synthetic phantom of BASELINE.json's configs (host only, deterministic):
 * background 20, n_ellipses ellipses (full axes 20-200 px, rotation U[0,pi), intensity
 * U[40,220]), +-15 linear gradient along columns, Gaussian sigma (rounded, clipped), then salt &
 * pepper at `density` with the reference's threshold rule (proj/src/noise.cpp:40-57).
 * Rng64 = mt19937_64, top-53-bit uniforms, Marsaglia polar normals (proj/include/denoise/noise.hpp:24-40). */
int hyb_make_phantom_u8(int rows, int cols, int n_ellipses, double sigma, double density,
                        uint64_t seed, uint8_t* out, size_t pitch);

#ifdef __cplusplus
}
#endif
#endif /* HYBRID_CUDA_H */
