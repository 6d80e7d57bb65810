// test_pgm.cpp -- the reference's PGM I/O unit tests (proj/tests/test_image_core.cpp:48-135)
// re-expressed against the host driver's load_pgm / save_pgm.  CPU only (no device calls).
// Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <random>
#include <stdexcept>
#include <string>

#include "../../paper_2005_05371_b200/host/denoise_cuda.hpp"

using namespace denoise_cuda;
namespace fs = std::filesystem;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                     \
    do {                                                                \
        ++g_checks;                                                     \
        if (!(cond)) {                                                  \
            ++g_fail;                                                   \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond); \
        }                                                               \
    } while (0)

template <class F>
static bool throws_runtime(F&& f, const char* needle) {
    try {
        f();
    } catch (const std::runtime_error& e) {
        return needle == nullptr || std::string(e.what()).find(needle) != std::string::npos;
    } catch (...) {
        return false;
    }
    return false;
}

static fs::path tmp(const std::string& name) { return fs::temp_directory_path() / ("hyb_pgm_test_" + name); }

static void write_bytes(const fs::path& p, const std::string& bytes) {
    std::ofstream out(p, std::ios::binary);
    out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
}

int main() {
    {  // P5 maxval 255
        const fs::path p = tmp("p5.pgm");
        write_bytes(p, std::string("P5\n2 2\n255\n") + '\x00' + '\x80' + '\xff' + '\x40');
        Image img = load_pgm(p);
        CHECK(img.rows() == 2 && img.cols() == 2);
        CHECK(img.at(0, 0) == 0.0);
        CHECK(std::fabs(img.at(0, 1) - 128.0 / 255.0) < 1e-12);
        CHECK(img.at(1, 0) == 1.0);
        CHECK(std::fabs(img.at(1, 1) - 64.0 / 255.0) < 1e-12);
        CHECK(to_u8(img) == (std::vector<uint8_t>{0, 128, 255, 64}));  // straight into the uint8 path
        fs::remove(p);
    }
    {  // ASCII P2, maxval -> 1
        const fs::path p = tmp("p2.pgm");
        write_bytes(p, "P2 1 1 255 255");
        Image img = load_pgm(p);
        CHECK(img.rows() == 1 && img.cols() == 1 && img.at(0, 0) == 1.0);
        fs::remove(p);
    }
    {  // comments and 16-bit big-endian samples
        const fs::path p = tmp("p5c.pgm");
        write_bytes(p, std::string("P5\n# a comment\n1 1\n65535\n") + '\xff' + '\xff');
        CHECK(load_pgm(p).at(0, 0) == 1.0);
        fs::remove(p);
    }
    {  // colour PPM rejected
        const fs::path p = tmp("p6.ppm");
        write_bytes(p, "P6\n1 1\n255\n\x01\x02\x03");
        CHECK(throws_runtime([&] { load_pgm(p); }, "unsupported magic"));
        fs::remove(p);
    }
    {  // truncated raster
        const fs::path p = tmp("trunc.pgm");
        write_bytes(p, std::string("P5\n2 2\n255\n") + '\x00' + '\x80');
        CHECK(throws_runtime([&] { load_pgm(p); }, "truncated"));
        fs::remove(p);
    }
    {  // sample above maxval, bad maxval, missing file
        const fs::path p = tmp("bad.pgm");
        write_bytes(p, "P2 2 1 10 3 11");
        CHECK(throws_runtime([&] { load_pgm(p); }, "exceeds maxval"));
        write_bytes(p, "P2 1 1 0 0");
        CHECK(throws_runtime([&] { load_pgm(p); }, "out of range"));
        fs::remove(p);
        CHECK(throws_runtime([&] { load_pgm(tmp("does_not_exist.pgm")); }, "cannot open"));
    }
    {  // writer: endpoints, halves away from zero
        const fs::path p = tmp("save.pgm");
        save_pgm(Image::from_pixels(1, 2, {0.0, 1.0}), p);
        std::ifstream in(p, std::ios::binary);
        const std::string content((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        CHECK(content == std::string("P5\n2 1\n255\n") + '\x00' + '\xff');
        save_pgm(Image(1, 1, 0.5), p);  // 127.5 -> 128
        CHECK(std::fabs(load_pgm(p).at(0, 0) - 128.0 / 255.0) < 1e-12);
        fs::remove(p);
    }
    CHECK(throws_runtime([] { save_pgm(Image(1, 1), "/nonexistent_dir/x.pgm"); }, nullptr));
    {  // round trip: error <= half a step; exact on the k/255 grid
        const fs::path p = tmp("rt.pgm");
        std::mt19937_64 gen(99);
        Image img(64, 64);
        for (double& v : img.pixels()) v = (gen() >> 11) * 0x1.0p-53;
        save_pgm(img, p);
        const Image back = load_pgm(p);
        double err = 0;
        for (std::size_t i = 0; i < img.size(); ++i) err = std::max(err, std::fabs(img.pixels()[i] - back.pixels()[i]));
        CHECK(err <= 1.0 / 510.0 + 1e-12);
        std::vector<double> px(256);
        for (int i = 0; i < 256; ++i) px[static_cast<std::size_t>(i)] = i / 255.0;
        const Image grid = Image::from_pixels(16, 16, px);
        save_pgm(grid, p);
        CHECK(load_pgm(p) == grid);
        fs::remove(p);
    }
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail;
}
