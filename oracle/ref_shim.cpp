// ref_shim.cpp -- extern "C" bridge onto the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY (see hyb_oracle.c).  oracle/Makefile compiles this
// file together with the reference's own sources where they lie under
// /root/reference/proj/src (image, tiling, noise, adaptive_median, parallel)
// into oracle/_ref/libref.so.  Nothing from the reference is copied into this
// repository; this file only converts uint8 <-> the reference's double Image
// and forwards calls.
//
// The uint8 <-> double map is k <-> k/255.0 (reference proj/src/pgm_io.cpp:73,88)
// and back with lround(p * 255) (proj/src/pgm_io.cpp:115).  The AMF only
// compares and selects, so it commutes with this strictly increasing map and
// the reference AMF on k/255 doubles equals the uint8 AMF bit-exactly.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "denoise/adaptive_median.hpp"
#include "denoise/image.hpp"
#include "denoise/noise.hpp"
#include "denoise/parallel.hpp"
#include "denoise/phantom.hpp"
#include "denoise/tiling.hpp"

extern "C" {
int hyb_oracle_wiener_stats_u8(const uint8_t*, size_t, int, int, int, int, int, int64_t*);
int hyb_oracle_wiener_gain_u8(const uint8_t*, size_t, int, int, int, int, int, int64_t, int64_t,
                              uint8_t*, size_t);
}

namespace {

thread_local std::string g_err;

denoise::Image to_image(const uint8_t* px, size_t pitch, int rows, int cols) {
    denoise::Image img(rows, cols);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) img.at(r, c) = px[(size_t)r * pitch + c] / 255.0;
    return img;
}

void from_image(const denoise::Image& img, uint8_t* px, size_t pitch) {
    for (int r = 0; r < img.rows(); ++r)
        for (int c = 0; c < img.cols(); ++c) {
            long q = std::lround(img.at(r, c) * 255.0);
            px[(size_t)r * pitch + c] = (uint8_t)(q < 0 ? 0 : (q > 255 ? 255 : q));
        }
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_validate_smax(int smax) {
    return guarded([&] { denoise::validate_smax(smax); });
}

// detail::adaptive_median_rows (reference proj/include/denoise/adaptive_median.hpp:47-48)
int ref_amf_rows_u8(const uint8_t* src, size_t pitch, int rows, int cols, int row_begin,
                    int row_end, int smax, uint8_t* dst, size_t dpitch, uint8_t* fin,
                    size_t fpitch) {
    return guarded([&] {
        denoise::Image in = to_image(src, pitch, rows, cols);
        denoise::Image out;
        std::vector<int> at;
        denoise::detail::adaptive_median_rows(in, smax, row_begin, row_end, out,
                                              fin ? &at : nullptr);
        from_image(out, dst, dpitch);
        if (fin)
            for (int r = 0; r < out.rows(); ++r)
                for (int c = 0; c < cols; ++c)
                    fin[(size_t)r * fpitch + c] = (uint8_t)at[(size_t)r * cols + c];
    });
}

// adaptive_median_parallel (reference proj/include/denoise/parallel.hpp:31).
// *seconds (nullable) receives the wall time of the reference call alone,
// measured like the reference's timed_run (parallel.hpp:36-49).
int ref_amf_parallel_u8(const uint8_t* src, size_t pitch, int rows, int cols, int smax,
                        int parts, int workers, int use_halo, uint8_t* dst, size_t dpitch,
                        double* seconds) {
    return guarded([&] {
        denoise::Image in = to_image(src, pitch, rows, cols);
        denoise::FilterConfig cfg;
        cfg.smax = smax;
        cfg.parts = parts;
        cfg.workers = workers;
        cfg.use_halo = use_halo != 0;
        auto [out, t] = denoise::timed_run([&] { return denoise::adaptive_median_parallel(in, cfg); });
        if (seconds) *seconds = t;
        from_image(out, dst, dpitch);
    });
}

// window_stats (reference proj/include/denoise/adaptive_median.hpp:24): zmin / zmed / zmax planes.
int ref_window_stats_u8(const uint8_t* src, size_t pitch, int rows, int cols, int k, uint8_t* zmin,
                        uint8_t* zmed, uint8_t* zmax, size_t opitch) {
    return guarded([&] {
        denoise::WindowStats ws = denoise::window_stats(to_image(src, pitch, rows, cols), k);
        from_image(ws.zmin, zmin, opitch);
        from_image(ws.zmed, zmed, opitch);
        from_image(ws.zmax, zmax, opitch);
    });
}

// split_bands geometry (reference proj/src/tiling.cpp:10-45): 4 ints per band.
int ref_split_bands(int rows, int cols, int parts, int halo, int* out) {
    return guarded([&] {
        denoise::Image img(rows, cols);
        auto tiles = denoise::split_bands(img, parts, halo);
        for (size_t i = 0; i < tiles.size(); ++i) {
            out[4 * i + 0] = tiles[i].core_start;
            out[4 * i + 1] = tiles[i].core_rows;
            out[4 * i + 2] = tiles[i].halo_above;
            out[4 * i + 3] = tiles[i].halo_below;
        }
    });
}

// Rng64 streams (reference proj/include/denoise/noise.hpp:24-40).
void ref_rng_uniform(uint64_t seed, int n, double* out) {
    denoise::Rng64 rng(seed);
    for (int i = 0; i < n; ++i) out[i] = rng.uniform01();
}
void ref_rng_normal(uint64_t seed, int n, double* out) {
    denoise::Rng64 rng(seed);
    for (int i = 0; i < n; ++i) out[i] = rng.normal();
}

void ref_rng_u64(uint64_t seed, int n, uint64_t* out) {
    denoise::Rng64 rng(seed);
    for (int i = 0; i < n; ++i) out[i] = rng.next_u64();
}

// oracles::random_image (reference proj/tests/support/oracles.hpp:18-23): Rng64(seed) uniforms,
// quantised to the k/255 grid with lround(p * 255); then, if density > 0, add_salt_pepper
// (proj/src/noise.cpp:40-57) at sp_seed (impulses are exactly 0 / 255).
int ref_random_image_u8(int rows, int cols, uint64_t seed, double density, uint64_t sp_seed, uint8_t* out) {
    return guarded([&] {
        denoise::Rng64 rng(seed);
        denoise::Image img(rows, cols);
        for (double& p : img.pixels()) p = std::lround(rng.uniform01() * 255.0) / 255.0;
        if (density > 0) img = denoise::add_salt_pepper(img, density, sp_seed);
        from_image(img, out, (size_t)cols);
    });
}

// degrade(make_phantom(rows, cols, seed), NoiseSpec{seed}) quantised to uint8 -- the
// noisy_phantom fixture of proj/tests/test_parallel.cpp:21-24.
int ref_noisy_phantom_u8(int rows, int cols, uint64_t seed, uint8_t* out) {
    return guarded([&] {
        denoise::NoiseSpec spec;
        spec.seed = seed;
        from_image(denoise::degrade(denoise::make_phantom(rows, cols, seed), spec), out, (size_t)cols);
    });
}

// add_salt_pepper (reference proj/src/noise.cpp:40-57) on a constant image;
// returns the number of corrupted pixels (the frozen-draw KAT of
// proj/tests/test_noise.cpp:109-124 expects 502 for 100x100, 0.05, seed 77).
int ref_salt_pepper_count(int rows, int cols, double value, double density, uint64_t seed) {
    denoise::Image img(rows, cols, value);
    denoise::Image hit = denoise::add_salt_pepper(img, density, seed);
    int n = 0;
    for (double p : hit.pixels()) n += (p == 0.0 || p == 1.0) && p != value;
    return n;
}

// CPU baseline of the whole hot path on the host cores: reference
// adaptive_median_parallel (parts = workers = threads), then the W1 oracle
// (the reference has no local Wiener) on `threads` row bands.  Conversions are
// outside both timed regions.  y must hold rows*cols bytes.
int ref_hybrid_baseline(const uint8_t* g, int rows, int cols, int smax, int win, int threads,
                        uint8_t* y, double* t_amf, double* t_wiener) {
    return guarded([&] {
        std::vector<uint8_t> f((size_t)rows * cols);
        denoise::Image in = to_image(g, (size_t)cols, rows, cols);
        denoise::FilterConfig cfg;
        cfg.smax = smax;
        cfg.parts = threads < rows ? threads : rows;
        cfg.workers = threads;
        auto [out, ta] = denoise::timed_run([&] { return denoise::adaptive_median_parallel(in, cfg); });
        from_image(out, f.data(), (size_t)cols);
        const int parts = cfg.parts;
        std::vector<int64_t> partial(parts, 0);
        const auto t0 = std::chrono::steady_clock::now();
        auto band = [&](int i, auto&& fn) {
            const int base = rows / parts, extra = rows % parts;
            const int start = i * base + (i < extra ? i : extra);
            fn(start, start + base + (i < extra ? 1 : 0));
        };
        {
            std::vector<std::thread> pool;
            for (int i = 0; i < parts; ++i)
                pool.emplace_back([&, i] {
                    band(i, [&](int b, int e) {
                        hyb_oracle_wiener_stats_u8(f.data(), cols, rows, cols, b, e, win, &partial[i]);
                    });
                });
            for (auto& t : pool) t.join();
        }
        int64_t w = 0;
        for (int64_t p : partial) w += p;
        {
            std::vector<std::thread> pool;
            for (int i = 0; i < parts; ++i)
                pool.emplace_back([&, i] {
                    band(i, [&](int b, int e) {
                        hyb_oracle_wiener_gain_u8(f.data(), cols, rows, cols, b, e, win, w,
                                                  (int64_t)rows * cols, y + (size_t)b * cols, cols);
                    });
                });
            for (auto& t : pool) t.join();
        }
        *t_amf = ta;
        *t_wiener = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

}  // extern "C"
