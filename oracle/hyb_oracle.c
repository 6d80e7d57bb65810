/*
 * hyb_oracle.c -- CPU restatement of the hybrid AMF + local Wiener path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path in paper_2005_05371_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it, and only
 * as the checker or the CPU baseline -- never as the product.
 *
 * Parity status:
 *   - AMF (hyb_oracle_amf_u8): PINNED.  Restates
 *     detail::adaptive_median_rows (reference proj/src/adaptive_median.cpp:123-215)
 *     on uint8 samples.  Checked against the reference itself, compiled here
 *     from /root/reference into oracle/_ref (tests/golden/make_golden.py and
 *     tests/test_oracle.py), and against the reference's own KATs
 *     (proj/tests/test_adaptive_median.cpp:26-78).
 *   - W1 local Wiener (hyb_oracle_wiener_*): the reference has NO such filter
 *     (SPEC.md:287 lists local-statistics Wiener as a non-goal), so this half
 *     is "parity unpinned" with respect to the reference; it follows the
 *     exact-integer W1 specification of SURVEY.md section 8(a) and is checked
 *     against an independent pure-Python Fraction implementation and
 *     hand-derived KATs (tests/golden/wiener_kat.json).
 *
 * Plain C99 + the gcc __int128 extension; no dependencies.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>

#define HYB_OK 0
#define HYB_EINVAL 1

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* validate_smax, reference proj/src/adaptive_median.cpp:11-16 */
int hyb_oracle_validate_smax(int smax) { return (smax <= 1 || smax % 2 == 0) ? HYB_EINVAL : HYB_OK; }

/*
 * window_stats, reference proj/src/adaptive_median.cpp:96-119: per pixel the min, the median
 * (sorted index (k*k-1)/2, :52-56 via median_of) and the max of the k x k window, coordinates
 * clamped (edge replication, :20-41).  k odd >= 3 (:97-100).  Outputs nullable; one pitch.
 * 256-bin counting per window, exact for uint8 samples.
 */
int hyb_oracle_window_stats_u8(const uint8_t* src, size_t spitch, int rows, int cols, int k,
                               uint8_t* zmin, uint8_t* zmed, uint8_t* zmax, size_t opitch) {
    if (k < 3 || k % 2 == 0 || rows < 1 || cols < 1) return HYB_EINVAL;
    const int rk = k / 2, m = (k * k - 1) / 2;
    uint32_t hist[256];
    for (int r = 0; r < rows; ++r) {
        for (int c = 0; c < cols; ++c) {
            for (int i = 0; i < 256; ++i) hist[i] = 0;
            for (int dr = -rk; dr <= rk; ++dr)
                for (int dc = -rk; dc <= rk; ++dc)
                    ++hist[src[(size_t)clampi(r + dr, 0, rows - 1) * spitch + (size_t)clampi(c + dc, 0, cols - 1)]];
            int lo = 0, hi = 255, md = -1, acc = 0;
            while (!hist[lo]) ++lo;
            while (!hist[hi]) --hi;
            for (int v = lo; v <= hi && md < 0; ++v) {
                acc += (int)hist[v];
                if (acc > m) md = v;
            }
            const size_t o = (size_t)r * opitch + (size_t)c;
            if (zmin) zmin[o] = (uint8_t)lo;
            if (zmed) zmed[o] = (uint8_t)md;
            if (zmax) zmax[o] = (uint8_t)hi;
        }
    }
    return HYB_OK;
}

/*
 * Adaptive median over rows [row_begin, row_end) of src (rows x cols, pitch
 * spitch).  Restates reference proj/src/adaptive_median.cpp:123-215:
 *   - windows k = 3, 5, ..., smax over the PRISTINE input (:40-50, stats never
 *     read partially written output),
 *   - coordinates clamped to src bounds = edge replication (:44-47),
 *   - zmed = element at sorted index (k*k-1)/2 (:52-56),
 *   - level A: zmin < zmed < zmax (strict, :175/:201); then level B keeps g
 *     when zmin < g < zmax, else zmed (:177/:203); record k (:180-182),
 *   - never finalized: output keeps the input value (copy at :134-137) and
 *     finalized_at stays 0 (:140).
 * The order statistics are taken with a 256-bin counting pass, which is exact
 * for uint8 samples (same multiset, same sorted order).
 */
int hyb_oracle_amf_u8(const uint8_t* src, size_t spitch, int rows, int cols, int row_begin,
                      int row_end, int smax, uint8_t* dst, size_t dpitch, uint8_t* fin,
                      size_t fpitch) {
    if (hyb_oracle_validate_smax(smax)) return HYB_EINVAL;
    if (rows < 1 || cols < 1) return HYB_EINVAL;
    if (row_begin < 0 || row_end > rows || row_begin >= row_end) return HYB_EINVAL;
    uint32_t hist[256];
    for (int r = row_begin; r < row_end; ++r) {
        for (int c = 0; c < cols; ++c) {
            const int g = src[(size_t)r * spitch + (size_t)c];
            int out = g, at = 0;
            for (int k = 3; k <= smax; k += 2) {
                const int rad = (k - 1) / 2;
                memset(hist, 0, sizeof hist);
                for (int dr = -rad; dr <= rad; ++dr) {
                    const uint8_t* row = src + (size_t)clampi(r + dr, 0, rows - 1) * spitch;
                    for (int dc = -rad; dc <= rad; ++dc) hist[row[clampi(c + dc, 0, cols - 1)]]++;
                }
                int zmin = 0, zmax = 255, zmed = -1;
                while (hist[zmin] == 0) ++zmin;
                while (hist[zmax] == 0) --zmax;
                const uint32_t want = (uint32_t)((k * k - 1) / 2); /* 0-based rank */
                uint32_t acc = 0;
                for (int v = zmin; v <= zmax; ++v) {
                    acc += hist[v];
                    if (acc > want) { zmed = v; break; }
                }
                if (zmin < zmed && zmed < zmax) {          /* level A */
                    out = (zmin < g && g < zmax) ? g : zmed; /* level B */
                    at = k;
                    break;
                }
            }
            dst[(size_t)(r - row_begin) * dpitch + (size_t)c] = (uint8_t)out;
            if (fin) fin[(size_t)(r - row_begin) * fpitch + (size_t)c] = (uint8_t)at;
        }
    }
    return HYB_OK;
}

/*
 * W1 local statistics at one pixel: S1 = sum f, S2 = sum f^2 over the win x win
 * window with coordinates clamped to f's bounds (edge replication, the same
 * border rule as the AMF above), and V = n*S2 - S1^2 (exact; n = win^2).
 */
static void local_stats(const uint8_t* f, size_t pitch, int rows, int cols, int r, int c, int win,
                        int64_t* s1, int64_t* v) {
    const int rad = (win - 1) / 2;
    int64_t a = 0, b = 0;
    for (int dr = -rad; dr <= rad; ++dr) {
        const uint8_t* row = f + (size_t)clampi(r + dr, 0, rows - 1) * pitch;
        for (int dc = -rad; dc <= rad; ++dc) {
            const int64_t x = row[clampi(c + dc, 0, cols - 1)];
            a += x;
            b += x * x;
        }
    }
    const int64_t n = (int64_t)win * win;
    *s1 = a;
    *v = n * b - a * a;
}

static int valid_win(int win) { return win >= 1 && (win % 2) == 1 && win <= 63; }

/*
 * W = sum over rows [row_begin, row_end) of V.  With the mean of the local
 * variances v = V/n^2 over all P pixels of the image, the noise estimate is
 * nu = W / (n^2 P)  (BASELINE.json north_star).
 * The sum is exact int64 and therefore independent of any partitioning.
 */
int hyb_oracle_wiener_stats_u8(const uint8_t* f, size_t pitch, int rows, int cols, int row_begin,
                               int row_end, int win, int64_t* noise_sum) {
    if (!valid_win(win) || rows < 1 || cols < 1) return HYB_EINVAL;
    if (row_begin < 0 || row_end > rows || row_begin >= row_end) return HYB_EINVAL;
    int64_t w = 0;
    for (int r = row_begin; r < row_end; ++r)
        for (int c = 0; c < cols; ++c) {
            int64_t s1, v;
            local_stats(f, pitch, rows, cols, r, c, win, &s1, &v);
            w += v;
        }
    *noise_sum += w;
    return HYB_OK;
}

/*
 * W1 gain, exact rational arithmetic:
 *   mu = S1/n, v = V/n^2, nu = W/(n^2 P)
 *   v <= nu  (V*P <= W):  y = mu
 *   otherwise:            y = mu + (v - nu)/v * (f - mu) = f - D*W/(n*V*P),  D = n*f - S1
 * quantised with round-half-away-from-zero (reference proj/src/pgm_io.cpp:115,
 * lround) and clamped to [0, 255].  y lies between mu and f, so y >= 0 and
 * "half away from zero" is "half up": y_q = floor((2*num + den) / (2*den)).
 */
int hyb_oracle_wiener_gain_u8(const uint8_t* f, size_t pitch, int rows, int cols, int row_begin,
                              int row_end, int win, int64_t noise_sum, int64_t pixel_count,
                              uint8_t* y, size_t ypitch) {
    if (!valid_win(win) || rows < 1 || cols < 1 || pixel_count < 1 || noise_sum < 0)
        return HYB_EINVAL;
    if (row_begin < 0 || row_end > rows || row_begin >= row_end) return HYB_EINVAL;
    const int64_t n = (int64_t)win * win;
    const int64_t P = pixel_count, W = noise_sum;
    for (int r = row_begin; r < row_end; ++r)
        for (int c = 0; c < cols; ++c) {
            int64_t s1, v;
            local_stats(f, pitch, rows, cols, r, c, win, &s1, &v);
            const int64_t fv = f[(size_t)r * pitch + (size_t)c];
            int64_t q;
            if ((__int128)v * P <= (__int128)W) {
                q = (2 * s1 + n) / (2 * n); /* round(S1/n), half up */
            } else {
                const __int128 den = (__int128)n * v * P;
                const __int128 num = (__int128)fv * den - (__int128)(n * fv - s1) * W;
                q = (int64_t)((2 * num + den) / (2 * den));
            }
            if (q < 0) q = 0;
            if (q > 255) q = 255;
            y[(size_t)(r - row_begin) * ypitch + (size_t)c] = (uint8_t)q;
        }
    return HYB_OK;
}

/*
 * Whole-image W1 (stats then gain) and the full hybrid: AMF over the whole
 * image, then W1 on the AMF output -- the stage order of hybrid_denoise
 * (reference proj/src/pipeline.cpp:35-53), with the Wiener stage replaced by
 * W1.  `work` must hold rows*cols bytes (the AMF output f, dense pitch = cols).
 */
int hyb_oracle_hybrid_u8(const uint8_t* g, size_t pitch, int rows, int cols, int smax, int win,
                         uint8_t* work, uint8_t* y, size_t ypitch, int64_t* noise_sum_out) {
    int st = hyb_oracle_amf_u8(g, pitch, rows, cols, 0, rows, smax, work, (size_t)cols, NULL, 0);
    if (st) return st;
    int64_t w = 0;
    st = hyb_oracle_wiener_stats_u8(work, (size_t)cols, rows, cols, 0, rows, win, &w);
    if (st) return st;
    if (noise_sum_out) *noise_sum_out = w;
    return hyb_oracle_wiener_gain_u8(work, (size_t)cols, rows, cols, 0, rows, win, w,
                                     (int64_t)rows * cols, y, ypitch);
}

/* contrast_stretch, reference proj/src/pipeline.cpp:10-21: out = (p - lo) / (hi - lo) over the
 * image's min / max, the image unchanged when hi == lo.  On k/255 inputs the reference's double
 * result is the exact rational (v - lo) / (hi - lo) up to one rounding; the uint8 form here is that
 * rational scaled to 0..255 and rounded half up: out = floor((510 (v - lo) + (hi - lo)) / (2 (hi - lo))),
 * so lo -> 0 and hi -> 255 exactly (the reference's endpoints 0.0 and 1.0, :16-19). */
int hyb_oracle_contrast_stretch_u8(const uint8_t* src, size_t pitch, int rows, int cols, uint8_t* dst,
                                   size_t dpitch) {
    if (rows < 1 || cols < 1) return 1;
    int lo = 255, hi = 0;
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            const int v = src[(size_t)r * pitch + c];
            if (v < lo) lo = v;
            if (v > hi) hi = v;
        }
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            const int v = src[(size_t)r * pitch + c];
            dst[(size_t)r * dpitch + c] =
                hi == lo ? (uint8_t)v : (uint8_t)((510 * (v - lo) + (hi - lo)) / (2 * (hi - lo)));
        }
    return 0;
}

