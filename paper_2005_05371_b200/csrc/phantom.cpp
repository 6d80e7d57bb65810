// phantom.cpp -- deterministic synthetic phantoms for BASELINE.json's configs (host side).
//
// Not on the timed path: it produces the input bytes shared by the CUDA path, the oracle and
// the CPU baseline.  Random streams follow the reference's Rng64 (proj/include/denoise/noise.hpp:
// 24-40): std::mt19937_64, uniforms from the top 53 bits, Marsaglia-polar normals
// (proj/src/noise.cpp:9-24); Gaussian noise on stream `seed`, impulses on stream `seed + 1`
// (proj/src/noise.cpp:59-62) with the threshold rule u < d/2 -> 0, u < d -> 255
// (proj/src/noise.cpp:47-55).  Choices BASELINE.json leaves open are fixed in DESIGN.md 3.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "../../include/hybrid_cuda.h"

namespace {

class Rng64 {
public:
    explicit Rng64(uint64_t seed) : gen_(seed) {}
    double uniform01() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
    double normal() {
        if (has_spare_) {
            has_spare_ = false;
            return spare_;
        }
        double u, v, s;
        do {
            u = 2.0 * uniform01() - 1.0;
            v = 2.0 * uniform01() - 1.0;
            s = u * u + v * v;
        } while (s >= 1.0 || s == 0.0);
        const double f = std::sqrt(-2.0 * std::log(s) / s);
        spare_ = v * f;
        has_spare_ = true;
        return u * f;
    }

private:
    std::mt19937_64 gen_;
    double spare_ = 0.0;
    bool has_spare_ = false;
};

constexpr uint64_t kGeometryStream = 0x9E3779B97F4A7C15ull;
constexpr double kPi = 3.14159265358979323846;

}  // namespace

extern "C" int hyb_make_phantom_u8(int rows, int cols, int n_ellipses, double sigma,
                                   double density, uint64_t seed, uint8_t* out, size_t pitch) {
    if (rows < 1 || cols < 1 || n_ellipses < 0 || !(sigma >= 0.0) || !(density >= 0.0) ||
        density > 1.0 || out == nullptr || pitch < static_cast<size_t>(cols))
        return HYB_EINVAL;
    std::vector<double> canvas(static_cast<size_t>(rows) * cols, 20.0);

    // ellipses in painter's order; axes are full lengths 20-200 px (semi-axes 10-100)
    Rng64 geo(seed ^ kGeometryStream);
    for (int e = 0; e < n_ellipses; ++e) {
        const double cx = geo.uniform01() * cols;
        const double cy = geo.uniform01() * rows;
        const double a = 0.5 * (20.0 + 180.0 * geo.uniform01());
        const double b = 0.5 * (20.0 + 180.0 * geo.uniform01());
        const double th = kPi * geo.uniform01();
        const double val = 40.0 + 180.0 * geo.uniform01();
        const double ct = std::cos(th), st = std::sin(th);
        const double ext = a > b ? a : b;
        const int r_lo = std::max(0, static_cast<int>(std::floor(cy - ext)));
        const int r_hi = std::min(rows - 1, static_cast<int>(std::ceil(cy + ext)));
        const int c_lo = std::max(0, static_cast<int>(std::floor(cx - ext)));
        const int c_hi = std::min(cols - 1, static_cast<int>(std::ceil(cx + ext)));
        for (int r = r_lo; r <= r_hi; ++r) {
            const double dy = r - cy;
            double* row = canvas.data() + static_cast<size_t>(r) * cols;
            for (int c = c_lo; c <= c_hi; ++c) {
                const double dx = c - cx;
                const double u = (dx * ct + dy * st) / a;
                const double v = (-dx * st + dy * ct) / b;
                if (u * u + v * v <= 1.0) row[c] = val;
            }
        }
    }

    // +-15 linear gradient along columns, Gaussian noise, round half away from zero, clip
    Rng64 gauss(seed);
    for (int r = 0; r < rows; ++r) {
        const double* row = canvas.data() + static_cast<size_t>(r) * cols;
        uint8_t* o = out + static_cast<size_t>(r) * pitch;
        for (int c = 0; c < cols; ++c) {
            const double grad = cols > 1 ? 15.0 * (2.0 * c / (cols - 1) - 1.0) : 0.0;
            const double x = row[c] + grad + sigma * gauss.normal();
            long q = std::lround(x);
            o[c] = static_cast<uint8_t>(q < 0 ? 0 : (q > 255 ? 255 : q));
        }
    }

    // salt & pepper, reference rule
    Rng64 imp(seed + 1);
    const double half = density / 2.0;
    for (int r = 0; r < rows; ++r) {
        uint8_t* o = out + static_cast<size_t>(r) * pitch;
        for (int c = 0; c < cols; ++c) {
            const double u = imp.uniform01();
            if (u < half)
                o[c] = 0;
            else if (u < density)
                o[c] = 255;
        }
    }
    return HYB_OK;
}
