// denoise_cuda.hpp -- C++ host driver with the reference's filter API, on libhybrid_cuda.
//
// Mirrors the reference's `namespace denoise` signatures for the hot path
// (proj/include/denoise/{image,adaptive_median,parallel,tiling,pipeline}.hpp) so a caller of the
// reference can switch by changing the namespace: same names, argument meaning and exception
// types (std::invalid_argument with the reference's message texts, std::runtime_error for device
// failures).  Pixels travel to the GPU as uint8: the reference's Image doubles are k/255 values
// (proj/src/pgm_io.cpp:73,88); images with <= 256 distinct values that are not on that grid are
// rank-compressed, which is exact for the AMF (it only compares and selects).  The Wiener stage is
// the north_star's local-statistics W1 (the reference's stage-2 slot, proj/src/pipeline.cpp:45-53).
#pragma once

#include <cstddef>
#include <cstdint>
#include <filesystem>
#include <vector>

namespace denoise_cuda {

/// Row-major double raster, reference proj/include/denoise/image.hpp:13-50.
class Image {
public:
    Image() = default;
    Image(int rows, int cols, double fill = 0.0);
    static Image from_pixels(int rows, int cols, std::vector<double> px);

    int rows() const noexcept { return rows_; }
    int cols() const noexcept { return cols_; }
    std::size_t size() const noexcept { return px_.size(); }
    double& at(int r, int c) noexcept { return px_[idx(r, c)]; }
    double at(int r, int c) const noexcept { return px_[idx(r, c)]; }
    double* row(int r) noexcept { return px_.data() + idx(r, 0); }
    const double* row(int r) const noexcept { return px_.data() + idx(r, 0); }
    std::vector<double>& pixels() noexcept { return px_; }
    const std::vector<double>& pixels() const noexcept { return px_; }
    bool same_size(const Image& o) const noexcept { return rows_ == o.rows_ && cols_ == o.cols_; }
    friend bool operator==(const Image&, const Image&) = default;

private:
    std::size_t idx(int r, int c) const noexcept {
        return static_cast<std::size_t>(r) * static_cast<std::size_t>(cols_) + static_cast<std::size_t>(c);
    }
    int rows_ = 0;
    int cols_ = 0;
    std::vector<double> px_;
};

/// validate_smax -- proj/src/adaptive_median.cpp:11-16.
void validate_smax(int smax);

/// EstimateMode -- proj/include/denoise/wiener.hpp:8.  For the W1 Wiener: robust = the north_star's
/// estimator (nu = mean of the local variances, exact int64 W); reference = the mean squared difference
/// between the AMF output and the reference image (proj/src/wiener.cpp:31-42).
enum class EstimateMode { robust, reference };

/// FilterConfig -- proj/include/denoise/parallel.hpp:13-19, same fields and defaults, plus the W1 window
/// and where it runs: `device` (one GPU), or `gpus` > 1 strips on devices device .. device + gpus - 1,
/// or an explicit `device_ids` list (ids may repeat) -- a multi-device context (hyb_create_multi), one
/// strip per device, NVLink exchange of the noise sums, bit-identical to one GPU.  final_stretch: the
/// reference pipeline's closing contrast_stretch (proj/src/pipeline.cpp:55-57) after the W1 stage.
struct FilterConfig {
    int smax = 11;
    int parts = 1;
    int workers = 1;
    EstimateMode estimate_mode = EstimateMode::robust;
    bool use_halo = true;
    int wiener_window = 3;
    int device = 0;
    int gpus = 1;
    std::vector<int> device_ids;
    bool final_stretch = false;
};

/// Device used by the entry points that take no FilterConfig (reference signatures: adaptive_median_serial,
/// detail::adaptive_median_rows, wiener_local, contrast_stretch, estimate_noise_variance, wiener_filter);
/// per host thread, default 0.
void set_default_device(int device);
int default_device();

/// validate_config -- proj/src/parallel.cpp:16-25.
void validate_config(const FilterConfig& config);

/// WindowStats / window_stats -- proj/include/denoise/adaptive_median.hpp:16-24: per-pixel min / median /
/// max planes of the k x k window (edge replication), on the GPU (hyb_window_stats_u8).
struct WindowStats {
    Image zmin;
    Image zmax;
    Image zmed;
    int k = 0;
};
WindowStats window_stats(const Image& image, int k);

/// adaptive_median_serial -- proj/include/denoise/adaptive_median.hpp:35.
Image adaptive_median_serial(const Image& image, int smax);

namespace detail {
/// adaptive_median_rows -- proj/include/denoise/adaptive_median.hpp:47-48.
void adaptive_median_rows(const Image& src, int smax, int row_begin, int row_end, Image& dst,
                          std::vector<int>* finalized_at = nullptr);
}  // namespace detail

/// adaptive_median_parallel -- proj/include/denoise/parallel.hpp:31 (bands = strips on the GPU).
Image adaptive_median_parallel(const Image& image, const FilterConfig& config);

/// W1 local-statistics Wiener; *sigma2 (nullable) receives nu / 255^2.
Image wiener_local(const Image& filtered, int window, double* sigma2 = nullptr);

/// HybridResult -- proj/include/denoise/pipeline.hpp:12-18 (+ the exact noise sum W).
struct HybridResult {
    Image image;
    double sigma2 = 0.0;
    double t_adaptive = 0.0;
    double t_wiener = 0.0;
    double t_stretch = 0.0;
    long long noise_sum = 0;
};

/// hybrid_denoise -- proj/include/denoise/pipeline.hpp:25-27, same signature: the adaptive median (parts
/// bands, on config's device(s)), [contrast stretch when stretch_after_each], the W1 Wiener in the Wiener
/// slot with the noise from config.estimate_mode (reference mode needs `reference`, same errors as
/// proj/src/pipeline.cpp:25-31), [final contrast stretch when config.final_stretch].
HybridResult hybrid_denoise(const Image& noisy, const FilterConfig& config, const Image* reference = nullptr,
                            bool stretch_after_each = false);

/// uint8 <-> reference doubles (k/255).  to_u8 throws std::invalid_argument off the grid.
std::vector<uint8_t> to_u8(const Image& image);
Image from_u8(const uint8_t* px, int rows, int cols);

/// The reference's own Wiener stage and pipeline tail on the GPU (doubles, like the reference):
/// contrast_stretch proj/src/pipeline.cpp:10-21 (bit-identical), estimate_noise_variance
/// proj/src/wiener.cpp:30-52, wiener_filter proj/src/wiener.cpp:54-77 (cuFFT, double).
enum class NoiseSource { given, reference, robust };
struct NoiseEstimate {
    double sigma2 = 0.0;
    NoiseSource source = NoiseSource::given;
};
Image contrast_stretch(const Image& image);
NoiseEstimate estimate_noise_variance(const Image& image, const Image* reference = nullptr);
Image wiener_filter(const Image& image, const NoiseEstimate& noise, bool clamp = true);

/// The reference's full hybrid_denoise (proj/src/pipeline.cpp:23-57): adaptive median bands,
/// [stretch], noise estimate (reference image if given, else robust), frequency Wiener, final stretch.
HybridResult hybrid_denoise_reference(const Image& noisy, const FilterConfig& config, const Image* reference = nullptr,
                                      bool stretch_after_each = false);

/// load_pgm / save_pgm -- proj/src/pgm_io.cpp:49-122: P5 or P2, maxval
/// 1..65535, samples / maxval; writer P5 maxval 255, round half away from zero.  Same error texts
/// ("pgm <path>: ...", std::runtime_error).  P5/P2 files with maxval 255 load exactly onto the
/// k/255 grid, i.e. straight into the uint8 path (to_u8).
Image load_pgm(const std::filesystem::path& path);
void save_pgm(const Image& image, const std::filesystem::path& path);

}  // namespace denoise_cuda
