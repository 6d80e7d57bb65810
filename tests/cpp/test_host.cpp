// test_host.cpp -- the reference's hot-path unit tests re-expressed against the C++ host driver
// (denoise_cuda, on the GPU) with the C oracle (oracle/hyb_oracle.c) as the checker.  Mirrors
// proj/tests/test_adaptive_median.cpp and proj/tests/test_parallel.cpp case by case.
// Exit code = number of failed checks (like the reference acceptance gate).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../paper_2005_05371_b200/host/denoise_cuda.hpp"

extern "C" {
int hyb_oracle_amf_u8(const uint8_t*, size_t, int, int, int, int, int, uint8_t*, size_t, uint8_t*, size_t);
int hyb_oracle_hybrid_u8(const uint8_t*, size_t, int, int, int, int, uint8_t*, uint8_t*, size_t, int64_t*);
int hyb_make_phantom_u8(int, int, int, double, double, uint64_t, uint8_t*, size_t);
int hyb_oracle_wiener_stats_u8(const uint8_t*, size_t, int, int, int, int, int, int64_t*);
int hyb_oracle_wiener_gain_u8(const uint8_t*, size_t, int, int, int, int, int, int64_t, int64_t, uint8_t*, size_t);
int hyb_oracle_contrast_stretch_u8(const uint8_t*, size_t, int, int, uint8_t*, size_t);
int hyb_oracle_window_stats_u8(const uint8_t*, size_t, int, int, int, uint8_t*, uint8_t*, uint8_t*, size_t);
}

using namespace denoise_cuda;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        ++g_checks;                                                            \
        if (!(cond)) {                                                         \
            ++g_fail;                                                          \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);        \
        }                                                                      \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                               \
    do {                                                                       \
        bool thrown_ = false;                                                  \
        try {                                                                  \
            (void)(expr);                                                      \
        } catch (const T&) {                                                   \
            thrown_ = true;                                                    \
        } catch (...) {                                                        \
        }                                                                      \
        CHECK(thrown_ && #expr);                                               \
    } while (0)

static Image random_grid_image(int rows, int cols, uint64_t seed, double sp) {
    std::mt19937_64 gen(seed);
    Image img(rows, cols);
    for (double& p : img.pixels()) {
        const double u = (gen() >> 11) * 0x1.0p-53;
        const double v = (gen() >> 11) * 0x1.0p-53;
        p = std::lround(u * 255.0) / 255.0;
        if (v < sp / 2) p = 0.0;
        else if (v < sp) p = 1.0;
    }
    return img;
}

static Image oracle_amf(const Image& img, int smax) {
    std::vector<uint8_t> in = to_u8(img), out(in.size());
    hyb_oracle_amf_u8(in.data(), img.cols(), img.rows(), img.cols(), 0, img.rows(), smax, out.data(), img.cols(),
                      nullptr, 0);
    return from_u8(out.data(), img.rows(), img.cols());
}

int main() {
    // validate_smax (proj/tests/test_adaptive_median.cpp:17-24)
    validate_smax(3);
    validate_smax(11);
    CHECK_THROWS_AS(validate_smax(4), std::invalid_argument);
    CHECK_THROWS_AS(validate_smax(1), std::invalid_argument);
    CHECK_THROWS_AS(validate_smax(0), std::invalid_argument);
    CHECK_THROWS_AS(validate_smax(-3), std::invalid_argument);
    try {
        validate_smax(4);
    } catch (const std::invalid_argument& e) {
        CHECK(std::string(e.what()).find("odd integer > 1") != std::string::npos);
    }

    // window_stats on a 3x3 ramp (proj/tests/test_adaptive_median.cpp:26-38): off-grid values, rank-coded
    {
        Image img = Image::from_pixels(3, 3, {0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9});
        WindowStats ws = window_stats(img, 3);
        CHECK(ws.k == 3);
        CHECK(ws.zmin.at(1, 1) == 0.1);
        CHECK(ws.zmed.at(1, 1) == 0.5);
        CHECK(ws.zmax.at(1, 1) == 0.9);
        CHECK(ws.zmin.at(0, 0) == 0.1);
        CHECK(ws.zmed.at(0, 0) == 0.2);
        CHECK(ws.zmax.at(0, 0) == 0.5);
    }
    // constants and invalid sizes (:40-48)
    {
        Image flat(6, 5, 0.25);
        WindowStats ws = window_stats(flat, 5);
        CHECK(ws.zmin == flat);
        CHECK(ws.zmed == flat);
        CHECK(ws.zmax == flat);
        CHECK_THROWS_AS(window_stats(flat, 4), std::invalid_argument);
        CHECK_THROWS_AS(window_stats(flat, 1), std::invalid_argument);
    }
    // ordering invariant on random data (:50-59), and the planes equal the oracle's
    {
        Image img = random_grid_image(21, 17, 99, 0.1);
        std::vector<uint8_t> in = to_u8(img);
        for (int k : {3, 5, 7, 9}) {
            WindowStats ws = window_stats(img, k);
            std::vector<uint8_t> o[3];
            for (auto& v : o) v.resize(img.size());
            hyb_oracle_window_stats_u8(in.data(), 17, 21, 17, k, o[0].data(), o[1].data(), o[2].data(), 17);
            for (std::size_t i = 0; i < img.size(); ++i) {
                CHECK(ws.zmin.pixels()[i] <= ws.zmed.pixels()[i]);
                CHECK(ws.zmed.pixels()[i] <= ws.zmax.pixels()[i]);
            }
            CHECK(ws.zmin == from_u8(o[0].data(), 21, 17));
            CHECK(ws.zmed == from_u8(o[1].data(), 21, 17));
            CHECK(ws.zmax == from_u8(o[2].data(), 21, 17));
        }
    }
    // constants are a fixed point (:61-65)
    {
        Image flat(9, 9, 0.7);
        CHECK(adaptive_median_serial(flat, 11) == flat);
        CHECK_THROWS_AS(adaptive_median_serial(flat, 4), std::invalid_argument);
    }
    // a lone impulse on a gradient is replaced by the window median (:67-78): off-grid values,
    // rank-coded by the host driver
    {
        Image img(5, 5);
        for (int r = 0; r < 5; ++r)
            for (int c = 0; c < 5; ++c) img.at(r, c) = 0.1 * (r + c) + 0.1;
        img.at(2, 2) = 1.0;
        Image out = adaptive_median_serial(img, 3);
        CHECK(std::fabs(out.at(2, 2) - 0.5) < 1e-12);
        CHECK(out.at(1, 2) == img.at(1, 2));
        CHECK(out.at(3, 1) == img.at(3, 1));
    }
    // oracle equivalence on random grid images (:80-96)
    for (int trial = 0; trial < 20; ++trial) {
        const int rows = 8 + trial % 25, cols = 8 + (trial * 7) % 25;
        Image img = random_grid_image(rows, cols, 1000 + trial, trial % 2 == 0 ? 0.2 : 0.0);
        for (int smax : {3, 5, 7, 11}) CHECK(adaptive_median_serial(img, smax) == oracle_amf(img, smax));
    }
    // finalized_at agrees across smax (:108-130)
    {
        Image img = random_grid_image(20, 20, 70, 0.25);
        Image small, big;
        std::vector<int> fs, fb;
        detail::adaptive_median_rows(img, 5, 0, 20, small, &fs);
        detail::adaptive_median_rows(img, 11, 0, 20, big, &fb);
        for (std::size_t i = 0; i < img.size(); ++i) {
            if (fs[i] != 0) {
                CHECK(fs[i] == 3 || fs[i] == 5);
                CHECK(fb[i] == fs[i]);
                CHECK(big.pixels()[i] == small.pixels()[i]);
            }
            if (fb[i] == 0) CHECK(big.pixels()[i] == img.pixels()[i]);
        }
    }
    // parallel: validate_config, parts > rows, every parts x workers == serial (test_parallel.cpp)
    {
        FilterConfig c;
        c.smax = 4;
        CHECK_THROWS_AS(validate_config(c), std::invalid_argument);
        c.smax = 3;
        c.parts = 0;
        CHECK_THROWS_AS(validate_config(c), std::invalid_argument);
        Image img = random_grid_image(8, 16, 1, 0.1);
        c.parts = 9;
        CHECK_THROWS_AS(adaptive_median_parallel(img, c), std::invalid_argument);
        Image big = random_grid_image(64, 64, 3, 0.1);
        for (int smax : {3, 11}) {
            const Image serial = adaptive_median_serial(big, smax);
            for (int parts : {2, 3, 4, 8})
                for (int workers : {1, 4}) {
                    FilterConfig cfg;
                    cfg.smax = smax;
                    cfg.parts = parts;
                    cfg.workers = workers;
                    CHECK(adaptive_median_parallel(big, cfg) == serial);
                }
        }
    }
    // hybrid: AMF + W1 equals the oracle, and parts do not change the output
    {
        const int rows = 300, cols = 260;
        std::vector<uint8_t> g((size_t)rows * cols), y(g.size()), work(g.size());
        hyb_make_phantom_u8(rows, cols, 8, 15.0, 0.2, 5, g.data(), cols);
        int64_t w = 0;
        hyb_oracle_hybrid_u8(g.data(), cols, rows, cols, 7, 3, work.data(), y.data(), cols, &w);
        const Image noisy = from_u8(g.data(), rows, cols);
        for (int parts : {1, 2, 5}) {
            FilterConfig cfg;
            cfg.smax = 7;
            cfg.parts = parts;
            cfg.wiener_window = 3;
            HybridResult r = hybrid_denoise(noisy, cfg);
            CHECK(r.noise_sum == w);
            CHECK(r.image == from_u8(y.data(), rows, cols));
            CHECK(r.sigma2 > 0);
        }
    }
    // multi-GPU behind the reference API: FilterConfig.device_ids / gpus (strips on several devices, or
    // several strips on one device where the box has one GPU) -- bit-identical to one device
    {
        const int rows = 517, cols = 389;
        std::vector<uint8_t> g((size_t)rows * cols), y(g.size()), work(g.size());
        hyb_make_phantom_u8(rows, cols, 10, 12.0, 0.3, 9, g.data(), cols);
        int64_t w = 0;
        hyb_oracle_hybrid_u8(g.data(), cols, rows, cols, 9, 5, work.data(), y.data(), cols, &w);
        const Image noisy = from_u8(g.data(), rows, cols);
        const Image expect = from_u8(y.data(), rows, cols);
        for (const std::vector<int>& ids : {std::vector<int>{0, 0}, std::vector<int>{0, 0, 0, 0, 0, 0, 0, 0}}) {
            FilterConfig cfg;
            cfg.smax = 9;
            cfg.wiener_window = 5;
            cfg.parts = 4;
            cfg.device_ids = ids;
            const HybridResult r = hybrid_denoise(noisy, cfg);
            CHECK(r.noise_sum == w);
            CHECK(r.image == expect);
        }
        FilterConfig bad;
        bad.gpus = 0;
        CHECK_THROWS_AS(hybrid_denoise(noisy, bad), std::invalid_argument);
    }
    // estimate_mode / reference / stretch_after_each (proj/include/denoise/pipeline.hpp:25-27,
    // proj/src/pipeline.cpp:25-53): the reference's call sites compile and behave
    {
        const int rows = 120, cols = 150;
        std::vector<uint8_t> g((size_t)rows * cols), f(g.size()), y(g.size()), fs(g.size());
        hyb_make_phantom_u8(rows, cols, 6, 10.0, 0.2, 4, g.data(), cols);
        const Image noisy = from_u8(g.data(), rows, cols);
        hyb_oracle_amf_u8(g.data(), cols, rows, cols, 0, rows, 7, f.data(), cols, nullptr, 0);
        FilterConfig cfg;
        cfg.smax = 7;
        cfg.wiener_window = 3;
        cfg.estimate_mode = EstimateMode::reference;
        CHECK_THROWS_AS(hybrid_denoise(noisy, cfg), std::invalid_argument);  // "reference mode requires ..."
        const Image small(10, 10, 0.5);
        CHECK_THROWS_AS(hybrid_denoise(noisy, cfg, &small), std::invalid_argument);
        Image clean(rows, cols);  // a reference image: the noiseless phantom stands in as a smooth ramp
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) clean.at(r, c) = (20.0 + 0.5 * c) / 255.0;
        const HybridResult hr = hybrid_denoise(noisy, cfg, &clean);
        double acc = 0.0;
        for (std::size_t i = 0; i < f.size(); ++i) {
            const double d = f[i] / 255.0 - clean.pixels()[i];
            acc += d * d;
        }
        const double sigma2 = acc / (double)f.size();
        CHECK(std::fabs(hr.sigma2 - sigma2) <= 1e-15 * std::max(1.0, sigma2));
        const long long Pn = (long long)rows * cols * 64;
        const int64_t Wn = std::llround(sigma2 * 255.0 * 255.0 * 81.0 * (double)Pn);
        hyb_oracle_wiener_gain_u8(f.data(), cols, rows, cols, 0, rows, 3, Wn, Pn, y.data(), cols);
        CHECK(hr.image == from_u8(y.data(), rows, cols));
        // stretch_after_each: AMF, stretch, W1 (robust); final_stretch: the closing stretch
        FilterConfig c2;
        c2.smax = 7;
        c2.wiener_window = 3;
        c2.final_stretch = true;
        const HybridResult h2 = hybrid_denoise(noisy, c2, nullptr, true);
        hyb_oracle_contrast_stretch_u8(f.data(), cols, rows, cols, fs.data(), cols);
        int64_t w2 = 0;
        hyb_oracle_wiener_stats_u8(fs.data(), cols, rows, cols, 0, rows, 3, &w2);
        hyb_oracle_wiener_gain_u8(fs.data(), cols, rows, cols, 0, rows, 3, w2, (int64_t)rows * cols, y.data(), cols);
        hyb_oracle_contrast_stretch_u8(y.data(), cols, rows, cols, y.data(), cols);
        CHECK(h2.noise_sum == w2);
        CHECK(h2.image == from_u8(y.data(), rows, cols));
        // final_stretch on the hot path: the stretch's range folded into the W1 gain (one device, and three
        // strips as a multi-device context on repeated ids)
        int64_t w3 = 0;
        hyb_oracle_wiener_stats_u8(f.data(), cols, rows, cols, 0, rows, 3, &w3);
        hyb_oracle_wiener_gain_u8(f.data(), cols, rows, cols, 0, rows, 3, w3, (int64_t)rows * cols, y.data(), cols);
        hyb_oracle_contrast_stretch_u8(y.data(), cols, rows, cols, y.data(), cols);
        for (int multi = 0; multi < 2; ++multi) {
            FilterConfig c3;
            c3.smax = 7;
            c3.wiener_window = 3;
            c3.final_stretch = true;
            if (multi) c3.device_ids = {0, 0, 0};
            const HybridResult h3 = hybrid_denoise(noisy, c3);
            CHECK(h3.noise_sum == w3);
            CHECK(h3.image == from_u8(y.data(), rows, cols));
        }
    }
    // the reference's pipeline tail (proj/tests/test_pipeline.cpp:29-57, test_wiener.cpp:110-160)
    {
        const Image kat = Image::from_pixels(2, 2, {0.2, 0.4, 0.6, 0.7});
        const Image st = contrast_stretch(kat);
        CHECK(st.at(0, 0) == 0.0 && st.at(1, 1) == 1.0);
        CHECK(std::fabs(st.at(0, 1) - 0.4) < 1e-14 && std::fabs(st.at(1, 0) - 0.8) < 1e-14);
        const Image flat(5, 5, 0.42);
        CHECK(contrast_stretch(flat) == flat);
        Image a(8, 8, 0.5), b(8, 8, 0.5);
        b.at(0, 0) = 0.9;
        const NoiseEstimate ref = estimate_noise_variance(a, &b);
        CHECK(ref.source == NoiseSource::reference && std::fabs(ref.sigma2 - 0.16 / 64.0) < 1e-15);
        CHECK(estimate_noise_variance(Image(32, 32, 0.3)).sigma2 == 0.0);
        const int n = 8;
        Image cosine(n, n);
        for (int r = 0; r < n; ++r)
            for (int c = 0; c < n; ++c) cosine.at(r, c) = std::cos(2.0 * M_PI * c / n);
        const Image w = wiener_filter(cosine, {0.01, NoiseSource::given}, false);
        double worst = 0.0;
        for (std::size_t i = 0; i < w.size(); ++i)
            worst = std::max(worst, std::fabs(w.pixels()[i] - 0.999375 * cosine.pixels()[i]));
        CHECK(worst < 1e-9);
        bool threw = false;
        try {
            wiener_filter(cosine, {-1e-9, NoiseSource::given});
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        // full pipeline: a constant image passes through untouched (test_pipeline.cpp:59-64)
        FilterConfig cfg;
        cfg.parts = 2;
        cfg.workers = 2;
        const Image flat6(32, 32, 0.6);
        const HybridResult hr = hybrid_denoise_reference(flat6, cfg);
        CHECK(hr.image == flat6 && hr.sigma2 == 0.0);
    }
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail;
}
