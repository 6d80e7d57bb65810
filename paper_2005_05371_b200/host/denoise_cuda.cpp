// denoise_cuda.cpp -- C++ host driver (reference filter API) on the libhybrid_cuda C ABI.
#include "denoise_cuda.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <map>
#include <stdexcept>
#include <string>

#include "../../include/hybrid_cuda.h"

namespace denoise_cuda {
namespace {

// One hyb_ctx per (host thread, device list), like the reference's per-call pool (proj/src/parallel.cpp:62-65):
// a single device, or a multi-device context (hyb_create_multi) for a strip partition over several GPUs.
struct Contexts {
    std::map<std::vector<int>, hyb_ctx*> by_devices;
    int default_device = 0;
    ~Contexts() {
        for (auto& kv : by_devices) hyb_destroy(kv.second);
    }
};

Contexts& contexts() {
    thread_local Contexts ctxs;
    return ctxs;
}

hyb_ctx* context_for(const std::vector<int>& devices) {
    Contexts& ctxs = contexts();
    auto it = ctxs.by_devices.find(devices);
    if (it != ctxs.by_devices.end()) return it->second;
    int st = 0;
    hyb_ctx* c = devices.size() == 1 ? hyb_create(devices[0], &st)
                                     : hyb_create_multi((int)devices.size(), devices.data(), &st);
    if (!c) {
        std::string ids;
        for (int d : devices) ids += (ids.empty() ? "" : ",") + std::to_string(d);
        throw std::runtime_error("libhybrid_cuda: cannot open CUDA device(s) " + ids);
    }
    ctxs.by_devices[devices] = c;
    return c;
}

hyb_ctx* context(int device) { return context_for({device}); }
hyb_ctx* context() { return context(contexts().default_device); }

// The devices a FilterConfig asks for: device_ids, else gpus consecutive devices from `device`.
std::vector<int> config_devices(const FilterConfig& config) {
    if (!config.device_ids.empty()) return config.device_ids;
    if (config.gpus < 1) throw std::invalid_argument("gpus must be >= 1, got " + std::to_string(config.gpus));
    std::vector<int> ids;
    for (int i = 0; i < config.gpus; ++i) ids.push_back(config.device + i);
    return ids;
}

void check(int status, hyb_ctx* ctx) {
    if (status == HYB_OK) return;
    const std::string msg = hyb_last_error(ctx);
    if (status == HYB_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("libhybrid_cuda: " + msg);
}

// uint8 view of an Image for the AMF: the k/255 grid, or a rank code when the image has at most 256
// distinct values (order-isomorphic, exact for an order-statistics filter).
struct Coded {
    std::vector<uint8_t> px;
    std::vector<double> table;  // empty: grid coding (value k/255)
    double decode(uint8_t k) const { return table.empty() ? k / 255.0 : table[k]; }
};

bool on_grid(const Image& img, std::vector<uint8_t>* out) {
    if (out) out->resize(img.size());
    const auto& px = img.pixels();
    for (std::size_t i = 0; i < px.size(); ++i) {
        const long q = std::lround(px[i] * 255.0);
        if (q < 0 || q > 255 || q / 255.0 != px[i]) return false;
        if (out) (*out)[i] = static_cast<uint8_t>(q);
    }
    return true;
}

Coded encode_for_amf(const Image& img) {
    Coded c;
    if (on_grid(img, &c.px)) return c;
    std::vector<double> vals = img.pixels();
    std::sort(vals.begin(), vals.end());
    vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
    if (vals.size() > 256)
        throw std::invalid_argument("image has " + std::to_string(vals.size()) +
                                    " distinct values off the 8-bit grid; the uint8 filter path cannot represent it");
    c.table = vals;
    c.px.resize(img.size());
    const auto& px = img.pixels();
    for (std::size_t i = 0; i < px.size(); ++i)
        c.px[i] = static_cast<uint8_t>(std::lower_bound(vals.begin(), vals.end(), px[i]) - vals.begin());
    return c;
}

}  // namespace

Image::Image(int rows, int cols, double fill) : rows_(rows), cols_(cols) {
    if (rows < 1 || cols < 1)
        throw std::invalid_argument("image dimensions must be at least 1x1, got " + std::to_string(rows) + "x" +
                                    std::to_string(cols));
    px_.assign(static_cast<std::size_t>(rows) * static_cast<std::size_t>(cols), fill);
}

Image Image::from_pixels(int rows, int cols, std::vector<double> px) {
    Image img(rows, cols);
    if (px.size() != img.size())
        throw std::invalid_argument("pixel buffer length " + std::to_string(px.size()) + " does not match " +
                                    std::to_string(rows) + "x" + std::to_string(cols));
    img.px_ = std::move(px);
    return img;
}

void set_default_device(int device) { contexts().default_device = device; }
int default_device() { return contexts().default_device; }

void validate_smax(int smax) {
    if (hyb_validate_smax(smax) != HYB_OK)
        throw std::invalid_argument("smax must be an odd integer > 1, got " + std::to_string(smax));
}

void validate_config(const FilterConfig& config) {
    validate_smax(config.smax);
    if (config.parts < 1) throw std::invalid_argument("parts must be >= 1, got " + std::to_string(config.parts));
    if (config.workers < 1)
        throw std::invalid_argument("workers must be >= 1, got " + std::to_string(config.workers));
}

std::vector<uint8_t> to_u8(const Image& image) {
    std::vector<uint8_t> px;
    if (!on_grid(image, &px)) throw std::invalid_argument("image values are not on the k/255 grid");
    return px;
}

Image from_u8(const uint8_t* px, int rows, int cols) {
    Image img(rows, cols);
    for (std::size_t i = 0; i < img.size(); ++i) img.pixels()[i] = px[i] / 255.0;
    return img;
}

namespace detail {

void adaptive_median_rows(const Image& src, int smax, int row_begin, int row_end, Image& dst,
                          std::vector<int>* finalized_at) {
    validate_smax(smax);
    const int rows = src.rows(), cols = src.cols();
    if (row_begin < 0 || row_end > rows || row_begin >= row_end)
        throw std::invalid_argument("bad row range [" + std::to_string(row_begin) + ", " + std::to_string(row_end) +
                                    ") for " + std::to_string(rows) + " rows");
    const Coded in = encode_for_amf(src);
    const int out_rows = row_end - row_begin;
    std::vector<uint8_t> out((std::size_t)out_rows * cols), fin;
    if (finalized_at) fin.resize(out.size());
    hyb_ctx* ctx = context();
    check(hyb_amf_u8(ctx, in.px.data(), cols, rows, cols, row_begin, row_end, smax, out.data(), cols,
                     finalized_at ? fin.data() : nullptr, cols),
          ctx);
    if (dst.rows() != out_rows || dst.cols() != cols) dst = Image(out_rows, cols);
    for (std::size_t i = 0; i < out.size(); ++i) dst.pixels()[i] = in.decode(out[i]);
    if (finalized_at) finalized_at->assign(fin.begin(), fin.end());
}

}  // namespace detail

WindowStats window_stats(const Image& image, int k) {
    if (k < 3 || k % 2 == 0)  // proj/src/adaptive_median.cpp:97-100
        throw std::invalid_argument("window size must be an odd integer >= 3, got " + std::to_string(k));
    const int rows = image.rows(), cols = image.cols();
    const Coded in = encode_for_amf(image);  // order statistics commute with the rank coding
    std::vector<uint8_t> planes(3 * (std::size_t)rows * cols);
    uint8_t* zmin = planes.data();
    uint8_t* zmed = zmin + (std::size_t)rows * cols;
    uint8_t* zmax = zmed + (std::size_t)rows * cols;
    hyb_ctx* ctx = context();
    check(hyb_window_stats_u8(ctx, in.px.data(), cols, rows, cols, k, zmin, zmed, zmax, cols), ctx);
    WindowStats ws;
    ws.k = k;
    ws.zmin = Image(rows, cols);
    ws.zmed = Image(rows, cols);
    ws.zmax = Image(rows, cols);
    for (std::size_t i = 0; i < (std::size_t)rows * cols; ++i) {
        ws.zmin.pixels()[i] = in.decode(zmin[i]);
        ws.zmed.pixels()[i] = in.decode(zmed[i]);
        ws.zmax.pixels()[i] = in.decode(zmax[i]);
    }
    return ws;
}

Image adaptive_median_serial(const Image& image, int smax) {
    validate_smax(smax);
    Image out;
    detail::adaptive_median_rows(image, smax, 0, image.rows(), out);
    return out;
}

Image adaptive_median_parallel(const Image& image, const FilterConfig& config) {
    validate_config(config);
    const int rows = image.rows(), cols = image.cols();
    if (config.parts > rows)
        throw std::invalid_argument("parts " + std::to_string(config.parts) + " exceeds image rows " +
                                    std::to_string(rows));
    const Coded in = encode_for_amf(image);
    std::vector<uint8_t> out((std::size_t)rows * cols);
    hyb_ctx* ctx = context(config.device);
    if (config.use_halo) {
        // With the halo every band's output equals the serial filter's rows (proj/include/denoise/
        // parallel.hpp:27-28), so the GPU filters the whole image in one upload and one launch: the
        // bands are the kernel's tiles, `workers` its CTAs.
        check(hyb_amf_u8(ctx, in.px.data(), cols, rows, cols, 0, rows, config.smax, out.data(), cols, nullptr, cols),
              ctx);
    } else {
        // the literal halo-free split (use_halo = false): each band filtered as its own image, which
        // clamps its windows at the band edges (proj/src/parallel.cpp:34)
        const int base = rows / config.parts, extra = rows % config.parts;
        int start = 0;
        for (int i = 0; i < config.parts; ++i) {
            const int core = base + (i < extra ? 1 : 0);
            check(hyb_amf_u8(ctx, in.px.data() + (std::size_t)start * cols, cols, core, cols, 0, core, config.smax,
                             out.data() + (std::size_t)start * cols, cols, nullptr, cols),
                  ctx);
            start += core;
        }
    }
    Image res(rows, cols);
    for (std::size_t i = 0; i < out.size(); ++i) res.pixels()[i] = in.decode(out[i]);
    return res;
}

Image wiener_local(const Image& filtered, int window, double* sigma2) {
    const std::vector<uint8_t> f = to_u8(filtered);
    std::vector<uint8_t> y(f.size());
    int64_t w = 0;
    hyb_ctx* ctx = context();
    check(hyb_wiener_u8(ctx, f.data(), filtered.cols(), filtered.rows(), filtered.cols(), window, y.data(),
                        filtered.cols(), &w),
          ctx);
    if (sigma2) {
        const double n = (double)window * window;
        *sigma2 = (double)w / (n * n * (double)f.size()) / (255.0 * 255.0);
    }
    return from_u8(y.data(), filtered.rows(), filtered.cols());
}

HybridResult hybrid_denoise(const Image& noisy, const FilterConfig& config, const Image* reference,
                            bool stretch_after_each) {
    validate_config(config);
    if (config.estimate_mode == EstimateMode::reference && reference == nullptr)
        throw std::invalid_argument("reference mode requires a reference image");
    if (reference && !noisy.same_size(*reference))
        throw std::invalid_argument("reference image dimensions do not match");
    const int rows = noisy.rows(), cols = noisy.cols();
    const std::vector<uint8_t> g = to_u8(noisy);
    std::vector<uint8_t> y(g.size());
    hyb_ctx* ctx = context_for(config_devices(config));
    HybridResult r;
    const long long P = (long long)rows * cols;
    const int win = config.wiener_window;
    if (config.estimate_mode == EstimateMode::robust && !stretch_after_each) {
        // the hot path: AMF + W1 in one call (strips over every configured device); with final_stretch the
        // stretch rides along (its min / max folded into the gain, the range reduced across the devices)
        hyb_stats st{};
        auto hybrid = config.final_stretch ? hyb_hybrid_stretch_u8 : hyb_hybrid_u8;
        check(hybrid(ctx, g.data(), cols, rows, cols, config.smax, win, config.parts, y.data(), cols, &st), ctx);
        r.sigma2 = st.sigma2;
        r.t_adaptive = st.t_adaptive;
        r.t_wiener = st.t_wiener;
        r.noise_sum = st.noise_sum;
    } else {
        using clock = std::chrono::steady_clock;
        auto secs = [](clock::time_point a, clock::time_point b) { return std::chrono::duration<double>(b - a).count(); };
        std::vector<uint8_t> f(g.size());
        auto t0 = clock::now();
        check(hyb_amf_u8(ctx, g.data(), cols, rows, cols, 0, rows, config.smax, f.data(), cols, nullptr, cols), ctx);
        auto t1 = clock::now();
        r.t_adaptive = secs(t0, t1);
        if (stretch_after_each) {  // proj/src/pipeline.cpp:39-43 (uint8 stretch, rounded half up)
            check(hyb_contrast_stretch_u8(ctx, f.data(), cols, rows, cols, f.data(), cols), ctx);
            r.t_stretch += secs(t1, clock::now());
        }
        auto t2 = clock::now();
        int64_t W = 0;
        long long Pn = P;
        const double n = (double)win * win;
        if (config.estimate_mode == EstimateMode::reference) {
            // sigma2 = mean((f - reference)^2) in [0, 1] intensity units (proj/src/wiener.cpp:31-42); the W1 gain
            // takes it as W / (n^2 P) with P scaled by K so the rounding of W costs < 2^-6 / (n^2 P)
            double acc = 0.0;
            for (std::size_t i = 0; i < f.size(); ++i) {
                const double d = f[i] / 255.0 - reference->pixels()[i];
                acc += d * d;
            }
            r.sigma2 = acc / (double)P;
            constexpr long long K = 64;
            Pn = P * K;
            W = std::llround(r.sigma2 * 255.0 * 255.0 * n * n * (double)Pn);
        } else {
            check(hyb_wiener_stats_u8(ctx, f.data(), cols, rows, cols, 0, rows, win, &W), ctx);
            r.sigma2 = (double)W / (n * n * (double)P) / (255.0 * 255.0);
        }
        check(hyb_wiener_gain_u8(ctx, f.data(), cols, rows, cols, 0, rows, win, &W, Pn, y.data(), cols), ctx);
        r.t_wiener = secs(t2, clock::now());
        r.noise_sum = config.estimate_mode == EstimateMode::reference ? 0 : W;
    }
    const bool stretched = config.estimate_mode == EstimateMode::robust && !stretch_after_each;
    if (config.final_stretch && !stretched) {  // proj/src/pipeline.cpp:55-57
        const auto t = std::chrono::steady_clock::now();
        check(hyb_contrast_stretch_u8(ctx, y.data(), cols, rows, cols, y.data(), cols), ctx);
        r.t_stretch += std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
    }
    r.image = from_u8(y.data(), rows, cols);
    return r;
}

Image contrast_stretch(const Image& image) {
    Image out(image.rows(), image.cols());
    hyb_ctx* ctx = context();
    check(hyb_contrast_stretch_f64(ctx, image.pixels().data(), image.cols(), image.rows(), image.cols(),
                                   out.pixels().data(), out.cols()),
          ctx);
    return out;
}

NoiseEstimate estimate_noise_variance(const Image& image, const Image* reference) {
    hyb_ctx* ctx = context();
    NoiseEstimate est;
    if (reference) {
        if (reference->rows() != image.rows() || reference->cols() != image.cols())
            throw std::invalid_argument("reference image dimensions do not match");
        check(hyb_noise_reference_f64(ctx, image.pixels().data(), image.cols(), reference->pixels().data(),
                                      reference->cols(), image.rows(), image.cols(), &est.sigma2),
              ctx);
        est.source = NoiseSource::reference;
    } else {
        check(hyb_noise_robust_f64(ctx, image.pixels().data(), image.cols(), image.rows(), image.cols(), &est.sigma2),
              ctx);
        est.source = NoiseSource::robust;
    }
    return est;
}

Image wiener_filter(const Image& image, const NoiseEstimate& noise, bool clamp) {
    Image out(image.rows(), image.cols());
    hyb_ctx* ctx = context();
    check(hyb_wiener_freq_f64(ctx, image.pixels().data(), image.cols(), image.rows(), image.cols(), noise.sigma2,
                              clamp ? 1 : 0, out.pixels().data(), out.cols()),
          ctx);
    return out;
}

HybridResult hybrid_denoise_reference(const Image& noisy, const FilterConfig& config, const Image* reference,
                                      bool stretch_after_each) {
    validate_config(config);
    if (reference && (reference->rows() != noisy.rows() || reference->cols() != noisy.cols()))
        throw std::invalid_argument("reference image dimensions do not match");
    using clock = std::chrono::steady_clock;
    auto secs = [](clock::time_point a, clock::time_point b) { return std::chrono::duration<double>(b - a).count(); };
    HybridResult r;
    auto t0 = clock::now();
    Image filtered = adaptive_median_parallel(noisy, config);
    auto t1 = clock::now();
    r.t_adaptive = secs(t0, t1);
    if (stretch_after_each) {
        filtered = contrast_stretch(filtered);
        r.t_stretch += secs(t1, clock::now());
    }
    auto t2 = clock::now();
    const NoiseEstimate est = estimate_noise_variance(filtered, reference);
    r.sigma2 = est.sigma2;
    Image denoised = wiener_filter(filtered, est);
    auto t3 = clock::now();
    r.t_wiener = secs(t2, t3);
    r.image = contrast_stretch(denoised);
    r.t_stretch += secs(t3, clock::now());
    return r;
}

}  // namespace denoise_cuda
