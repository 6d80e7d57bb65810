// capi.cu -- the extern "C" boundary of libhybrid_cuda (include/hybrid_cuda.h).
//
// Host orchestration only: argument validation with the reference's error texts, host/device
// pointer detection and staging, the strip partitioner (split_bands geometry, reference
// proj/src/tiling.cpp:23-32) and the exact noise reduction.  All pixel work is in amf.cu and
// wiener.cu; there is no CPU fallback -- a missing device or a failed launch is an error.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <map>
#include <tuple>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hybrid_cuda.h"
#include "hyb_internal.cuh"
#include "tma.cuh"

namespace hyb {
// Kernel-launch evidence: every launcher calls count_launch(), which adds to the counter of the
// context whose entry point is running on this thread (CtxScope below) -- per context, so several
// contexts (devices, host threads) do not mix their counts.
static thread_local long long* t_launch_counter = nullptr;
void count_launch() {
    if (t_launch_counter) ++*t_launch_counter;
}
}  // namespace hyb

namespace {

constexpr int kMaxSmax = 255;  // largest window the shared-memory tile supports
constexpr int kMaxWin = 63;

struct DevBuf {
    uint8_t* ptr = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t want) {
        if (want <= bytes) return cudaSuccess;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&ptr, want);
        if (e == cudaSuccess) bytes = want;
        return e;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
    }
};

struct Status {
    int code;
};

}  // namespace

struct hyb_ctx {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    std::string err;
    DevBuf in, out, fin, f, wsum;      // staging / scratch
    DevBuf sbar;                       // fused small-image kernel: grid-barrier words (zeroed once), stamps
    DevBuf mm, ys;                     // contrast stretch: min / max scratch, staged hybrid output
    DevBuf mmtot, mmparts;             // multi-device stretch: combined range, gathered partial ranges
    unsigned* stretch_mm = nullptr;    // hyb_hybrid_stretch_u8 in progress: the gains fold y's range here
    bool stretch_fused = false;        // ... and they did (else the stretch runs its own min / max pass)
    DevBuf fin64, fout64, fref64, fsc;  // frequency Wiener: staged doubles, scalar results
    hyb::FreqWork freq;
    bool small_used = false;           // the last hybrid call ran the fused kernel
    bool exclusive = false;            // hyb_set_exclusive: plain (non-cooperative) fused launches
    DevBuf amf_q[2], amf_cnt;          // AMF growth workspace (failure bitmap)
    std::vector<DevBuf> strip_g, strip_f;
    long long* host_w = nullptr;       // pinned readback of noise sums
    size_t host_w_n = 0;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaStream_t copy = nullptr;       // host<->device staging stream of the pipelined path
    cudaStream_t copy2 = nullptr;      // device->host stream of the pipelined batch path (PCIe duplex)
    // CUDA-graph cache of hyb_hybrid_u8 calls: a key seen once is captured on its second call and
    // replayed afterwards (one launch per step instead of ~10-30 API calls).
    using GraphKey = std::tuple<const void*, void*, size_t, size_t, int, int, int, int, int, cudaStream_t>;
    struct Graph {
        cudaGraphExec_t exec = nullptr;
        long long kernels = 0;
        std::vector<const void*> bufs;  // the scratch buffers the graph was captured over (buf_signature)
    };
    std::map<GraphKey, Graph> graphs;
    std::map<GraphKey, int> graph_seen;
    long long launches = 0;            // kernels this context launched (hyb_kernel_launches)
    // Multi-device context (hyb_create_multi): this context drives strip 0 on `device`; peers[i - 1]
    // drives strip i on its own device (ids may repeat).  peer_ok[i * n + j]: strip i's kernels can read
    // strip j's device memory (same device, or peer access enabled).
    std::vector<hyb_ctx*> peers;
    std::vector<char> peer_ok;
    DevBuf wparts, wtot, mg_in, mg_out;  // gathered partial W, total W, staged batch chunk
    // Asynchronous host-buffer calls (hyb_set_async): double-buffered staging, so call i + 1's upload
    // (copy stream) runs while call i's result downloads (copy2 stream) -- both PCIe directions busy.
    bool async_host = false;
    int async_parity = 0;
    DevBuf ain[2], aout[2];
    cudaEvent_t ev_in_free[2] = {}, ev_out_free[2] = {};
    cudaEvent_t ev_ah2d[2][16] = {}, ev_again[2][16] = {};
    cudaEvent_t ev_stats = nullptr, ev_done = nullptr, ev_start = nullptr, ev_gainx = nullptr;
    static constexpr int kMaxChunks = 16;
    cudaEvent_t ev_h2d[kMaxChunks] = {}, ev_gain[kMaxChunks] = {};
};

namespace {

// Routes count_launch() to ctx->launches for the duration of one entry point.
struct CtxScope {
    long long* prev;
    explicit CtxScope(hyb_ctx* ctx) : prev(hyb::t_launch_counter) { hyb::t_launch_counter = &ctx->launches; }
    ~CtxScope() { hyb::t_launch_counter = prev; }
};

// Every context-owned device buffer a captured CUDA graph may reference (pointer and size of each):
// DevBuf::ensure reallocates when a later call needs more room, so a graph captured before that
// would replay over freed memory.  A cached graph is replayed only while this signature is unchanged.
std::vector<const void*> buf_signature(const hyb_ctx* ctx) {
    std::vector<const void*> v;
    auto add = [&](const DevBuf& b) {
        v.push_back(b.ptr);
        v.push_back(reinterpret_cast<const void*>(b.bytes));
    };
    add(ctx->in);
    add(ctx->out);
    add(ctx->fin);
    add(ctx->f);
    add(ctx->wsum);
    add(ctx->sbar);
    add(ctx->amf_q[0]);
    for (const auto& b : ctx->strip_g) add(b);
    for (const auto& b : ctx->strip_f) add(b);
    return v;
}

int fail(hyb_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return code;
}

int cuda_fail(hyb_ctx* ctx, cudaError_t e, const char* where) {
    const int code = (e == cudaErrorMemoryAllocation) ? HYB_ENOMEM : HYB_ECUDA;
    return fail(ctx, code, std::string(where) + ": " + cudaGetErrorString(e));
}

#define HYB_CHECK(expr)                                         \
    do {                                                        \
        cudaError_t e_ = (expr);                                \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #expr); \
    } while (0)
#define HYB_CHECK_C(c, expr)                                    \
    do {                                                        \
        cudaError_t e_ = (expr);                                \
        if (e_ != cudaSuccess) return cuda_fail((c), e_, #expr); \
    } while (0)

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

std::string str_smax(int smax) { return "smax must be an odd integer > 1, got " + std::to_string(smax); }

int check_smax(hyb_ctx* ctx, int smax) {
    if (smax <= 1 || smax % 2 == 0) return fail(ctx, HYB_EINVAL, str_smax(smax));
    if (smax > kMaxSmax)
        return fail(ctx, HYB_EINVAL, "smax " + std::to_string(smax) +
                                         " exceeds the largest supported window " +
                                         std::to_string(kMaxSmax));
    return HYB_OK;
}

int check_dims(hyb_ctx* ctx, int rows, int cols) {
    if (rows < 1 || cols < 1)
        return fail(ctx, HYB_EINVAL, "image dimensions must be at least 1x1, got " +
                                         std::to_string(rows) + "x" + std::to_string(cols));
    return HYB_OK;
}

int check_range(hyb_ctx* ctx, int rows, int b, int e) {
    if (b < 0 || e > rows || b >= e)
        return fail(ctx, HYB_EINVAL, "bad row range [" + std::to_string(b) + ", " + std::to_string(e) +
                                         ") for " + std::to_string(rows) + " rows");
    return HYB_OK;
}

int check_win(hyb_ctx* ctx, int win) {
    if (win < 1 || win % 2 == 0 || win > kMaxWin)
        return fail(ctx, HYB_EINVAL, "wiener window must be an odd integer in [1, " +
                                         std::to_string(kMaxWin) + "], got " + std::to_string(win));
    return HYB_OK;
}

int check_pitch(hyb_ctx* ctx, size_t pitch, int cols, const char* what) {
    if (pitch < (size_t)cols)
        return fail(ctx, HYB_EINVAL, std::string(what) + " pitch " + std::to_string(pitch) +
                                         " is smaller than cols " + std::to_string(cols));
    return HYB_OK;
}

// Pitch of context buffers: 16-byte multiple (TMA), so images with cols % 16 == 0 stay contiguous
// and host<->device staging is a single linear copy.
size_t round_pitch(int cols) { return ((size_t)cols + 15) & ~(size_t)15; }

int ensure_host_w(hyb_ctx* ctx, size_t n) {
    if (ctx->host_w_n >= n) return HYB_OK;
    if (ctx->host_w) cudaFreeHost(ctx->host_w);
    ctx->host_w = nullptr;
    ctx->host_w_n = 0;
    HYB_CHECK(cudaMallocHost(&ctx->host_w, n * sizeof(long long)));
    ctx->host_w_n = n;
    return HYB_OK;
}

// Copies rows x cols bytes between two pitched buffers (any direction) on the ctx stream.
cudaError_t copy2d(hyb_ctx* ctx, void* dst, size_t dp, const void* src, size_t sp, int cols, int rows) {
    if (dp == (size_t)cols && sp == (size_t)cols)  // both contiguous: one linear DMA
        return cudaMemcpyAsync(dst, src, (size_t)cols * rows, cudaMemcpyDefault, ctx->stream);
    return cudaMemcpy2DAsync(dst, dp, src, sp, (size_t)cols, (size_t)rows, cudaMemcpyDefault, ctx->stream);
}

// AMF launch with the context's growth workspace.
// AMF growth workspace (bitmaps, records, counters): the counters are zeroed when (re)allocated and
// every launch leaves them zero.
cudaError_t ensure_amf_work(hyb_ctx* ctx, const hyb::Plane& p) {
    const size_t need = hyb::amf_work_bytes(p);
    if (need <= ctx->amf_q[0].bytes) return cudaSuccess;
    cudaError_t e = ctx->amf_q[0].ensure(need);
    if (e == cudaSuccess) e = cudaMemsetAsync(ctx->amf_q[0].ptr, 0, 64, ctx->stream);
    return e;
}

cudaError_t run_amf(hyb_ctx* ctx, const hyb::Plane& p, int smax, uint8_t* fin, size_t fpitch, size_t fslice) {
    cudaError_t e;
    if ((e = ensure_amf_work(ctx, p)) != cudaSuccess) return e;
    return hyb::launch_amf(p, smax, fin, fpitch, fslice, hyb::amf_work(ctx->amf_q[0].ptr, p), ctx->stream);
}

// The fused single-kernel step (small.cu) when the image qualifies (g TMA-compatible on the device).
// Timed calls record ev[0] / ev[1] = ev[2] around it and read back the kernel's own stamps (AMF /
// Wiener split) into host_w[1..3].  Returns false when not taken.
bool try_small(hyb_ctx* ctx, const uint8_t* g, size_t pitch, int rows, int cols, int smax, int win, uint8_t* y,
               size_t ypitch, bool timed, int* status) {
    *status = HYB_OK;
    if (!hyb::tma_compatible(g, pitch, 0)) return false;
    const hyb::SmallPlan pl = hyb::plan_small(rows, cols, smax, win);
    if (!pl.ok) return false;
    const size_t fp = round_pitch(cols);
    cudaError_t e;
    if ((e = ctx->f.ensure(fp * rows)) != cudaSuccess || (e = ctx->wsum.ensure(sizeof(long long))) != cudaSuccess) {
        *status = cuda_fail(ctx, e, "try_small: allocation");
        return true;
    }
    if (!ctx->sbar.ptr) {
        if ((e = ctx->sbar.ensure(64)) != cudaSuccess || (e = cudaMemset(ctx->sbar.ptr, 0, 64)) != cudaSuccess) {
            *status = cuda_fail(ctx, e, "try_small: barrier words");
            return true;
        }
    }
    if (timed && ((*status = ensure_host_w(ctx, 4)) || (e = cudaEventRecord(ctx->ev[0], ctx->stream)) != cudaSuccess)) {
        if (!*status) *status = cuda_fail(ctx, e, "try_small: event");
        return true;
    }
    const hyb::SmallBufs bufs{g, pitch, ctx->f.ptr, fp, y, ypitch, reinterpret_cast<unsigned long long*>(ctx->wsum.ptr),
                              reinterpret_cast<unsigned*>(ctx->sbar.ptr)};
    e = hyb::launch_small(pl, bufs, rows, cols, smax, win, !ctx->exclusive, ctx->stream);
    if (e == cudaErrorCooperativeLaunchTooLarge) {
        // the grid no longer fits co-resident (another context holds SMs): the separate kernels
        cudaGetLastError();
        return false;
    }
    if (e != cudaSuccess) {
        *status = cuda_fail(ctx, e, "launch_small");
        return true;
    }
    ctx->small_used = true;
    if (timed) {
        if ((e = cudaEventRecord(ctx->ev[1], ctx->stream)) != cudaSuccess ||
            (e = cudaEventRecord(ctx->ev[2], ctx->stream)) != cudaSuccess ||
            (e = cudaMemcpyAsync(ctx->host_w + 1, ctx->sbar.ptr + 8, 3 * sizeof(long long), cudaMemcpyDeviceToHost,
                                 ctx->stream)) != cudaSuccess)
            *status = cuda_fail(ctx, e, "try_small: stamps");
    }
    return true;
}

// Core of hyb_hybrid_u8 on device-resident buffers.
int hybrid_device(hyb_ctx* ctx, const uint8_t* g, size_t pitch, int rows, int cols, int smax,
                  int win, int parts, uint8_t* y, size_t ypitch, bool timed) {
    const int rA = (smax - 1) / 2, rW = (win - 1) / 2;
    HYB_CHECK(ctx->wsum.ensure(sizeof(long long)));
    unsigned long long* W = reinterpret_cast<unsigned long long*>(ctx->wsum.ptr);
    const long long P = (long long)rows * cols;
    if (parts == 1) {
        int st;
        if (try_small(ctx, g, pitch, rows, cols, smax, win, y, ypitch, timed, &st)) return st;
    }
    if (timed) HYB_CHECK(cudaEventRecord(ctx->ev[0], ctx->stream));
    if (parts == 1) {
        const size_t fp = round_pitch(cols);
        HYB_CHECK(ctx->f.ensure(fp * rows));
        hyb::Plane a{g, pitch, 0, ctx->f.ptr, fp, 0, rows, cols, 0, rows, 1};
        HYB_CHECK(cudaMemsetAsync(W, 0, sizeof(long long), ctx->stream));  // first: kernels chain by PDL
        HYB_CHECK(run_amf(ctx, a, smax, nullptr, 0, 0));
        if (timed) HYB_CHECK(cudaEventRecord(ctx->ev[1], ctx->stream));
        hyb::Plane w{ctx->f.ptr, fp, 0, y, ypitch, 0, rows, cols, 0, rows, 1};
        HYB_CHECK(hyb::launch_wiener_stats(w, win, W, ctx->stream));
        HYB_CHECK(hyb::launch_wiener_gain(w, win, reinterpret_cast<const long long*>(W), P, ctx->stream,
                                          ctx->stretch_mm));
        ctx->stretch_fused = ctx->stretch_mm != nullptr;
    } else {
        // split_bands geometry (reference proj/src/tiling.cpp:23-32) with halo rA + rW
        const int h = rA + rW;
        // grow only: dropping DevBufs would leak their device memory (DevBuf frees in release())
        if ((int)ctx->strip_g.size() < parts) ctx->strip_g.resize(parts);
        if ((int)ctx->strip_f.size() < parts) ctx->strip_f.resize(parts);
        struct S { int start, core, hA, hB, fa, fb; };
        std::vector<S> s(parts);
        const int base = rows / parts, extra = rows % parts;
        int start = 0;
        for (int i = 0; i < parts; ++i) {
            S& t = s[i];
            t.start = start;
            t.core = base + (i < extra ? 1 : 0);
            t.hA = std::min(h, start);
            t.hB = std::min(h, rows - start - t.core);
            t.fa = std::min(rW, start);
            t.fb = std::min(rW, rows - start - t.core);
            start += t.core;
        }
        const size_t sp = round_pitch(cols);
        for (int i = 0; i < parts; ++i) {
            const S& t = s[i];
            const int grows = t.hA + t.core + t.hB, frows = t.fa + t.core + t.fb;
            HYB_CHECK(ctx->strip_g[i].ensure(sp * grows));
            HYB_CHECK(ctx->strip_f[i].ensure(sp * frows));
            // the strip's own copy of g: core rows plus clamped halo (a real halo copy)
            HYB_CHECK(copy2d(ctx, ctx->strip_g[i].ptr, sp, g + (size_t)(t.start - t.hA) * pitch, pitch,
                             cols, grows));
            hyb::Plane a{ctx->strip_g[i].ptr, sp, 0, ctx->strip_f[i].ptr, sp, 0, grows, cols,
                         t.hA - t.fa, t.hA + t.core + t.fb, 1};
            HYB_CHECK(run_amf(ctx, a, smax, nullptr, 0, 0));
        }
        if (timed) HYB_CHECK(cudaEventRecord(ctx->ev[1], ctx->stream));
        HYB_CHECK(cudaMemsetAsync(W, 0, sizeof(long long), ctx->stream));
        for (int i = 0; i < parts; ++i) {
            const S& t = s[i];
            hyb::Plane w{ctx->strip_f[i].ptr, sp, 0, nullptr, 0, 0, t.fa + t.core + t.fb, cols, t.fa,
                         t.fa + t.core, 1};
            HYB_CHECK(hyb::launch_wiener_stats(w, win, W, ctx->stream));
        }
        for (int i = 0; i < parts; ++i) {
            const S& t = s[i];
            hyb::Plane w{ctx->strip_f[i].ptr, sp, 0, y + (size_t)t.start * ypitch, ypitch, 0,
                         t.fa + t.core + t.fb, cols, t.fa, t.fa + t.core, 1};
            HYB_CHECK(hyb::launch_wiener_gain(w, win, reinterpret_cast<const long long*>(W), P,
                                              ctx->stream, ctx->stretch_mm));
        }
        ctx->stretch_fused = ctx->stretch_mm != nullptr;
    }
    if (timed) HYB_CHECK(cudaEventRecord(ctx->ev[2], ctx->stream));
    return HYB_OK;
}

// Host buffers, one GPU, parts == 1: the image moves in row chunks so the PCIe transfers overlap
// the kernels.  Copy stream: H2D chunk k -> ev_h2d[k].  Compute stream: AMF of chunk k once the
// chunks holding its rows + rA halo have landed, statistics of chunk k-1 (its f halo rows are now
// final); after the single noise reduction, gain of chunk k -> ev_gain[k] while the copy stream
// brings chunk k-1 back.  The W dependence keeps every gain after every statistic, so the
// critical path is H2D + last AMF/stats + first gain + D2H instead of H2D + all kernels + D2H.
int hybrid_host_pipelined(hyb_ctx* ctx, const uint8_t* g, size_t pitch, int rows, int cols, int smax, int win,
                          uint8_t* y, size_t y_pitch, bool timed) {
    const int rA = (smax - 1) / 2, rW = (win - 1) / 2;
    // Chunking pays only when the copies dominate: each chunk adds the fixed latency of its kernels,
    // so images below ~8 MB move in one piece.
    const long long bytes = (long long)rows * cols;
    const int want = bytes < (8ll << 20) ? 1 : 4;
    const int K = std::max(1, std::min(want, rows / std::max(64, 2 * (rA + rW) + 1)));
    const size_t pp = round_pitch(cols);
    HYB_CHECK(ctx->in.ensure(pp * rows));
    HYB_CHECK(ctx->f.ensure(pp * rows));
    HYB_CHECK(ctx->out.ensure(pp * rows));
    if (K == 1 && hyb::plan_small(rows, cols, smax, win).ok) {
        // one piece: upload, the fused kernel, download, all on the compute stream
        if (timed) HYB_CHECK(cudaEventRecord(ctx->ev[3], ctx->stream));
        HYB_CHECK(copy2d(ctx, ctx->in.ptr, pp, g, pitch, cols, rows));
        int st;
        if (!try_small(ctx, ctx->in.ptr, pp, rows, cols, smax, win, ctx->out.ptr, pp, timed, &st))
            st = hybrid_device(ctx, ctx->in.ptr, pp, rows, cols, smax, win, 1, ctx->out.ptr, pp, timed);
        if (st) return st;
        HYB_CHECK(copy2d(ctx, y, y_pitch, ctx->out.ptr, pp, cols, rows));
        return HYB_OK;
    }
    HYB_CHECK(ctx->wsum.ensure(sizeof(long long)));
    unsigned long long* W = reinterpret_cast<unsigned long long*>(ctx->wsum.ptr);
    std::vector<int> a(K + 1);
    for (int k = 0; k <= K; ++k) a[k] = (int)((long long)rows * k / K);
    cudaStream_t cs = ctx->stream, xs = ctx->copy;
    auto cp = [&](void* dst, size_t dp, const void* src, size_t sp, int nrows) {
        if (dp == (size_t)cols && sp == (size_t)cols)
            return cudaMemcpyAsync(dst, src, (size_t)cols * nrows, cudaMemcpyDefault, xs);
        return cudaMemcpy2DAsync(dst, dp, src, sp, (size_t)cols, (size_t)nrows, cudaMemcpyDefault, xs);
    };
    if (timed) HYB_CHECK(cudaEventRecord(ctx->ev[3], cs));
    HYB_CHECK(cudaEventRecord(ctx->ev_gain[0], cs));  // copy stream starts after earlier compute-stream work
    HYB_CHECK(cudaStreamWaitEvent(xs, ctx->ev_gain[0], 0));
    for (int k = 0; k < K; ++k) {
        HYB_CHECK(cp(ctx->in.ptr + (size_t)a[k] * pp, pp, g + (size_t)a[k] * pitch, pitch, a[k + 1] - a[k]));
        HYB_CHECK(cudaEventRecord(ctx->ev_h2d[k], xs));
    }
    HYB_CHECK(cudaMemsetAsync(W, 0, sizeof(long long), cs));
    if (timed) HYB_CHECK(cudaEventRecord(ctx->ev[0], cs));
    auto stats = [&](int k) -> cudaError_t {
        hyb::Plane w{ctx->f.ptr, pp, 0, nullptr, 0, 0, rows, cols, a[k], a[k + 1], 1};
        return hyb::launch_wiener_stats(w, win, W, cs);
    };
    for (int k = 0; k < K; ++k) {
        int need = k;  // last chunk holding input rows < a[k+1] + rA
        while (need + 1 < K && a[need + 1] < std::min(rows, a[k + 1] + rA)) ++need;
        HYB_CHECK(cudaStreamWaitEvent(cs, ctx->ev_h2d[need], 0));
        hyb::Plane am{ctx->in.ptr, pp, 0, ctx->f.ptr + (size_t)a[k] * pp, pp, 0, rows, cols, a[k], a[k + 1], 1};
        HYB_CHECK(run_amf(ctx, am, smax, nullptr, 0, 0));
        if (k >= 1 && a[k + 1] - a[k] >= rW) HYB_CHECK(stats(k - 1));
        else if (k >= 1) return fail(ctx, HYB_EINVAL, "chunk thinner than the Wiener halo");
    }
    HYB_CHECK(stats(K - 1));
    if (timed) HYB_CHECK(cudaEventRecord(ctx->ev[1], cs));
    for (int k = 0; k < K; ++k) {
        hyb::Plane w{ctx->f.ptr, pp, 0, ctx->out.ptr + (size_t)a[k] * pp, pp, 0, rows, cols, a[k], a[k + 1], 1};
        HYB_CHECK(hyb::launch_wiener_gain(w, win, reinterpret_cast<const long long*>(W), (long long)rows * cols, cs));
        HYB_CHECK(cudaEventRecord(ctx->ev_gain[k], cs));
        HYB_CHECK(cudaStreamWaitEvent(xs, ctx->ev_gain[k], 0));
        HYB_CHECK(cp(y + (size_t)a[k] * y_pitch, y_pitch, ctx->out.ptr + (size_t)a[k] * pp, pp, a[k + 1] - a[k]));
    }
    if (timed) HYB_CHECK(cudaEventRecord(ctx->ev[2], cs));
    HYB_CHECK(cudaEventRecord(ctx->ev_h2d[0], xs));  // compute stream resumes after the last D2H
    HYB_CHECK(cudaStreamWaitEvent(cs, ctx->ev_h2d[0], 0));
    return HYB_OK;
}

// Device holding p (-1: host memory, pinned or pageable).
int ptr_device(const void* p) {
    cudaPointerAttributes a;
    if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) ? a.device : -1;
}

// Multi-device hybrid (hyb_create_multi): one strip per device in one process -- the paper's
// parts = workers partition (reference proj/src/parallel.cpp:27-70, split_bands geometry
// proj/src/tiling.cpp:23-32) with one GPU per band.  Per strip i on its device (own stream, all strips
// concurrent):
//   1. its rows of g plus a halo of rA + rW rows, straight from the caller's buffer (H2D from host
//      memory, a peer copy over NVLink from another device, or a local copy);
//   2. the AMF on its core rows +- rW (so the W1 statistics of its core rows need no second exchange),
//      then the statistics of its core rows into its partial W;
//   3. after every strip's statistics (cross-device events), the exact total W by one reduction kernel
//      per device reading the other devices' partials over NVLink (peer access) -- every device gets the
//      identical int64 W, so the output is bit-identical to one GPU;
//   4. the gain of its core rows, written straight into y when y is device memory this device can
//      store to (its own, or a peer's over NVLink), else staged and copied out.
// The caller's stream (ctx->stream, strip 0) orders the call: every strip starts after the work already
// on it, and it waits for every strip's end.
//   5. (stretch: hyb_hybrid_stretch_u8, reference proj/src/pipeline.cpp:55-57) every gain also folds the
//      range of its rows into its device's partial (min, 255 - max); after all gains each device combines
//      the partials over NVLink the same way and maps its own rows with the global range -- the contrast
//      stretch's min / max fused into the gain plus one exchange.
int hybrid_multi(hyb_ctx* ctx, const uint8_t* g, size_t pitch, int rows, int cols, int smax, int win, int parts,
                 uint8_t* y, size_t ypitch, hyb_stats* stats, bool stretch = false) {
    int st;
    if ((st = check_smax(ctx, smax)) || (st = check_win(ctx, win)) || (st = check_dims(ctx, rows, cols)) ||
        (st = check_pitch(ctx, pitch, cols, "g")) || (st = check_pitch(ctx, ypitch, cols, "y")))
        return st;
    if (parts < 1) return fail(ctx, HYB_EINVAL, "parts must be >= 1, got " + std::to_string(parts));
    const int n = 1 + (int)ctx->peers.size();
    if (std::max(parts, n) > rows)
        return fail(ctx, HYB_EINVAL, "parts " + std::to_string(std::max(parts, n)) + " exceeds image rows " +
                                         std::to_string(rows));
    if (!g || !y) return fail(ctx, HYB_EINVAL, "null image pointer");
    std::vector<hyb_ctx*> sub(n);
    sub[0] = ctx;
    for (int i = 1; i < n; ++i) sub[i] = ctx->peers[i - 1];
    const int rA = (smax - 1) / 2, rW = (win - 1) / 2, h = rA + rW;
    const int ydev = ptr_device(y);
    const bool timed = stats != nullptr;
    struct S { int start, core, hA, hB, fa, fb; };
    std::vector<S> s(n);
    {
        const int base = rows / n, extra = rows % n;
        int start = 0;
        for (int i = 0; i < n; ++i) {
            S& t = s[i];
            t.start = start;
            t.core = base + (i < extra ? 1 : 0);
            t.hA = std::min(h, start);
            t.hB = std::min(h, rows - start - t.core);
            t.fa = std::min(rW, start);
            t.fb = std::min(rW, rows - start - t.core);
            start += t.core;
        }
    }
    const size_t sp = round_pitch(cols);
    const long long P = (long long)rows * cols;
    HYB_CHECK(cudaSetDevice(ctx->device));
    if (timed) HYB_CHECK(cudaEventRecord(ctx->ev[3], ctx->stream));
    HYB_CHECK(cudaEventRecord(ctx->ev_start, ctx->stream));
    // 1-2: halo rows + AMF + statistics per strip
    for (int i = 0; i < n; ++i) {
        hyb_ctx* c = sub[i];
        const S& t = s[i];
        CtxScope scope(c);
        if (cudaSetDevice(c->device) != cudaSuccess) return cuda_fail(ctx, cudaGetLastError(), "cudaSetDevice");
        auto chk = [&](cudaError_t e, const char* what) { return e == cudaSuccess ? HYB_OK : cuda_fail(ctx, e, what); };
        if (i && (st = chk(cudaStreamWaitEvent(c->stream, ctx->ev_start, 0), "wait start"))) return st;
        if (c->strip_g.empty()) c->strip_g.resize(1);
        if (c->strip_f.empty()) c->strip_f.resize(1);
        const int grows = t.hA + t.core + t.hB, frows = t.fa + t.core + t.fb;
        if ((st = chk(c->strip_g[0].ensure(sp * grows), "strip alloc")) ||
            (st = chk(c->strip_f[0].ensure(sp * frows), "strip alloc")) ||
            (st = chk(c->wsum.ensure(sizeof(long long)), "alloc")) ||
            (st = chk(c->wtot.ensure(sizeof(long long)), "alloc")) ||
            (st = chk(c->wparts.ensure(sizeof(long long) * n), "alloc")))
            return st;
        if (stretch &&
            ((st = chk(c->mm.ensure(2 * sizeof(unsigned)), "alloc")) ||
             (st = chk(c->mmtot.ensure(2 * sizeof(unsigned)), "alloc")) ||
             (st = chk(c->mmparts.ensure(2 * sizeof(unsigned) * n), "alloc")) ||
             (st = chk(cudaMemsetAsync(c->mm.ptr, 0xFF, 2 * sizeof(unsigned), c->stream), "memset"))))
            return st;
        if ((st = chk(copy2d(c, c->strip_g[0].ptr, sp, g + (size_t)(t.start - t.hA) * pitch, pitch, cols, grows),
                      "strip halo copy")))
            return st;
        if ((st = chk(cudaMemsetAsync(c->wsum.ptr, 0, sizeof(long long), c->stream), "memset")))
            return st;
        hyb::Plane a{c->strip_g[0].ptr, sp, 0, c->strip_f[0].ptr, sp, 0, grows, cols, t.hA - t.fa,
                     t.hA + t.core + t.fb, 1};
        if ((st = chk(run_amf(c, a, smax, nullptr, 0, 0), "strip AMF"))) return st;
        hyb::Plane w{c->strip_f[0].ptr, sp, 0, nullptr, 0, 0, frows, cols, t.fa, t.fa + t.core, 1};
        if ((st = chk(hyb::launch_wiener_stats(w, win, reinterpret_cast<unsigned long long*>(c->wsum.ptr), c->stream),
                      "strip statistics")))
            return st;
        if ((st = chk(cudaEventRecord(c->ev_stats, c->stream), "event"))) return st;
    }
    if (timed) {
        HYB_CHECK(cudaSetDevice(ctx->device));
        HYB_CHECK(cudaEventRecord(ctx->ev[1], ctx->stream));
    }
    // 3-4: exact total W on every device, then the gain of its core rows
    std::vector<uint8_t*> ydst(n);
    std::vector<size_t> ydp(n);
    std::vector<char> ydirect(n);
    for (int i = 0; i < n; ++i) {
        hyb_ctx* c = sub[i];
        const S& t = s[i];
        CtxScope scope(c);
        if (cudaSetDevice(c->device) != cudaSuccess) return cuda_fail(ctx, cudaGetLastError(), "cudaSetDevice");
        auto chk = [&](cudaError_t e, const char* what) { return e == cudaSuccess ? HYB_OK : cuda_fail(ctx, e, what); };
        hyb::Partials parts_w{};
        parts_w.n = n;
        for (int j = 0; j < n; ++j) {
            if (j != i && (st = chk(cudaStreamWaitEvent(c->stream, sub[j]->ev_stats, 0), "wait statistics")))
                return st;
            if (ctx->peer_ok[(size_t)i * n + j]) {
                parts_w.p[j] = reinterpret_cast<const long long*>(sub[j]->wsum.ptr);
            } else {
                long long* dst = reinterpret_cast<long long*>(c->wparts.ptr) + j;
                if ((st = chk(cudaMemcpyPeerAsync(dst, c->device, sub[j]->wsum.ptr, sub[j]->device, sizeof(long long),
                                                  c->stream),
                              "partial W copy")))
                    return st;
                parts_w.p[j] = dst;
            }
        }
        long long* Wt = reinterpret_cast<long long*>(c->wtot.ptr);
        if ((st = chk(hyb::launch_sum_partials(parts_w, Wt, c->stream), "W reduction"))) return st;
        // output rows: straight into y when this device can store there (y on this device, or on a strip's
        // device with peer access enabled), else staged + copied out
        bool direct = ydev >= 0 && ydev == c->device;
        for (int j = 0; j < n && ydev >= 0 && !direct; ++j)
            direct = sub[j]->device == ydev && ctx->peer_ok[(size_t)i * n + j];
        uint8_t* yd = y + (size_t)t.start * ypitch;
        size_t yp = ypitch;
        if (!direct) {
            if ((st = chk(c->out.ensure(sp * t.core), "alloc"))) return st;
            yd = c->out.ptr;
            yp = sp;
        }
        hyb::Plane w{c->strip_f[0].ptr, sp, 0, yd, yp, 0, t.fa + t.core + t.fb, cols, t.fa, t.fa + t.core, 1};
        if ((st = chk(hyb::launch_wiener_gain(w, win, Wt, P, c->stream,
                                              stretch ? reinterpret_cast<unsigned*>(c->mm.ptr) : nullptr),
                      "strip gain")))
            return st;
        ydst[i] = yd;
        ydp[i] = yp;
        ydirect[i] = direct;
        if (stretch) {
            if ((st = chk(cudaEventRecord(c->ev_gainx, c->stream), "event"))) return st;
            continue;  // the map (step 5) comes first
        }
        if (!direct &&
            (st = chk(copy2d(c, y + (size_t)t.start * ypitch, ypitch, yd, yp, cols, t.core), "strip output copy")))
            return st;
        if ((st = chk(cudaEventRecord(c->ev_done, c->stream), "event"))) return st;
    }
    // 5: the global range from every strip's partial on every device, then the map of its own rows
    for (int i = 0; i < n && stretch; ++i) {
        hyb_ctx* c = sub[i];
        const S& t = s[i];
        CtxScope scope(c);
        if (cudaSetDevice(c->device) != cudaSuccess) return cuda_fail(ctx, cudaGetLastError(), "cudaSetDevice");
        auto chk = [&](cudaError_t e, const char* what) { return e == cudaSuccess ? HYB_OK : cuda_fail(ctx, e, what); };
        hyb::MmPartials pm{};
        pm.n = n;
        for (int j = 0; j < n; ++j) {
            if (j != i && (st = chk(cudaStreamWaitEvent(c->stream, sub[j]->ev_gainx, 0), "wait gain"))) return st;
            if (ctx->peer_ok[(size_t)i * n + j]) {
                pm.p[j] = reinterpret_cast<const unsigned*>(sub[j]->mm.ptr);
            } else {
                unsigned* dst = reinterpret_cast<unsigned*>(c->mmparts.ptr) + 2 * j;
                if ((st = chk(cudaMemcpyPeerAsync(dst, c->device, sub[j]->mm.ptr, sub[j]->device, 2 * sizeof(unsigned),
                                                  c->stream),
                              "partial range copy")))
                    return st;
                pm.p[j] = dst;
            }
        }
        unsigned* mt = reinterpret_cast<unsigned*>(c->mmtot.ptr);
        if ((st = chk(hyb::launch_min_partials(pm, mt, c->stream), "range reduction")) ||
            (st = chk(hyb::launch_stretch_map(ydst[i], ydp[i], t.core, cols, ydst[i], ydp[i], mt, c->stream),
                      "strip stretch")))
            return st;
        if (!ydirect[i] && (st = chk(copy2d(c, y + (size_t)t.start * ypitch, ypitch, ydst[i], ydp[i], cols, t.core),
                                     "strip output copy")))
            return st;
        if ((st = chk(cudaEventRecord(c->ev_done, c->stream), "event"))) return st;
    }
    HYB_CHECK(cudaSetDevice(ctx->device));
    for (int i = 1; i < n; ++i) HYB_CHECK(cudaStreamWaitEvent(ctx->stream, sub[i]->ev_done, 0));
    if (timed) {
        HYB_CHECK(cudaEventRecord(ctx->ev[2], ctx->stream));
        if ((st = ensure_host_w(ctx, 1))) return st;
        HYB_CHECK(cudaMemcpyAsync(ctx->host_w, ctx->wtot.ptr, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (timed || ydev < 0 || ptr_device(g) < 0) HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    if (timed) {
        float a = 0, w = 0, t = 0;
        HYB_CHECK(cudaEventElapsedTime(&a, ctx->ev[3], ctx->ev[1]));
        HYB_CHECK(cudaEventElapsedTime(&w, ctx->ev[1], ctx->ev[2]));
        HYB_CHECK(cudaEventElapsedTime(&t, ctx->ev[3], ctx->ev[2]));
        const double nn = (double)win * win;
        stats->noise_sum = ctx->host_w[0];
        stats->pixel_count = P;
        stats->sigma2 = (double)stats->noise_sum / (nn * nn * (double)P) / (255.0 * 255.0);
        stats->t_adaptive = a * 1e-3;  // strip 0's stream: halo copies, AMF and statistics enqueued for every strip
        stats->t_wiener = w * 1e-3;
        stats->t_total = t * 1e-3;
    }
    return HYB_OK;
}

// Asynchronous host-buffer hybrid (hyb_set_async, pinned host buffers, one device): the same chunked
// pipeline as hybrid_host_pipelined, but with double-buffered device staging (call parity b) and the
// download on its own stream, and no host synchronisation: call i + 1's H2D (copy stream) overlaps call
// i's D2H (copy2 stream), so a sequence of images keeps both PCIe directions busy.  Cross-call hazards
// are events: in[b] is refilled after call i - 2's last AMF read (ev_in_free), out[b] rewritten after
// call i - 2's download (ev_out_free); f and W are used on the compute stream only (serialised).
int hybrid_host_async(hyb_ctx* ctx, const uint8_t* g, size_t pitch, int rows, int cols, int smax, int win, uint8_t* y,
                      size_t y_pitch) {
    const int b = ctx->async_parity;
    const int rA = (smax - 1) / 2, rW = (win - 1) / 2;
    const long long bytes = (long long)rows * cols;
    const int want = bytes < (8ll << 20) ? 1 : 4;
    const int K = std::max(1, std::min(want, rows / std::max(64, 2 * (rA + rW) + 1)));
    const size_t pp = round_pitch(cols);
    if (!ctx->ev_in_free[b]) {
        for (int i = 0; i < 2; ++i) {
            HYB_CHECK(cudaEventCreateWithFlags(&ctx->ev_in_free[i], cudaEventDisableTiming));
            HYB_CHECK(cudaEventCreateWithFlags(&ctx->ev_out_free[i], cudaEventDisableTiming));
            for (int k = 0; k < hyb_ctx::kMaxChunks; ++k) {
                HYB_CHECK(cudaEventCreateWithFlags(&ctx->ev_ah2d[i][k], cudaEventDisableTiming));
                HYB_CHECK(cudaEventCreateWithFlags(&ctx->ev_again[i][k], cudaEventDisableTiming));
            }
        }
    }
    HYB_CHECK(ctx->ain[b].ensure(pp * rows));
    HYB_CHECK(ctx->aout[b].ensure(pp * rows));
    HYB_CHECK(ctx->f.ensure(pp * rows));
    HYB_CHECK(ctx->wsum.ensure(sizeof(long long)));
    unsigned long long* W = reinterpret_cast<unsigned long long*>(ctx->wsum.ptr);
    uint8_t* in = ctx->ain[b].ptr;
    uint8_t* out = ctx->aout[b].ptr;
    cudaStream_t cs = ctx->stream, xs = ctx->copy, ys = ctx->copy2;
    std::vector<int> a(K + 1);
    for (int k = 0; k <= K; ++k) a[k] = (int)((long long)rows * k / K);
    auto cp = [&](void* dst, size_t dp, const void* src, size_t sp, int nrows, cudaStream_t st) {
        if (dp == (size_t)cols && sp == (size_t)cols)
            return cudaMemcpyAsync(dst, src, (size_t)cols * nrows, cudaMemcpyDefault, st);
        return cudaMemcpy2DAsync(dst, dp, src, sp, (size_t)cols, (size_t)nrows, cudaMemcpyDefault, st);
    };
    // upload (copy stream), once call i - 2 is done reading in[b]
    HYB_CHECK(cudaStreamWaitEvent(xs, ctx->ev_in_free[b], 0));
    for (int k = 0; k < K; ++k) {
        HYB_CHECK(cp(in + (size_t)a[k] * pp, pp, g + (size_t)a[k] * pitch, pitch, a[k + 1] - a[k], xs));
        HYB_CHECK(cudaEventRecord(ctx->ev_ah2d[b][k], xs));
    }
    // compute stream: AMF + statistics per chunk as the rows land, then the gains
    if (K == 1 && hyb::plan_small(rows, cols, smax, win).ok) {
        HYB_CHECK(cudaStreamWaitEvent(cs, ctx->ev_ah2d[b][0], 0));
        HYB_CHECK(cudaStreamWaitEvent(cs, ctx->ev_out_free[b], 0));
        int st;
        if (!try_small(ctx, in, pp, rows, cols, smax, win, out, pp, false, &st))
            st = hybrid_device(ctx, in, pp, rows, cols, smax, win, 1, out, pp, false);
        if (st) return st;
        HYB_CHECK(cudaEventRecord(ctx->ev_in_free[b], cs));
        HYB_CHECK(cudaEventRecord(ctx->ev_again[b][0], cs));
    } else {
        HYB_CHECK(cudaMemsetAsync(W, 0, sizeof(long long), cs));
        auto stats = [&](int k) -> cudaError_t {
            hyb::Plane w{ctx->f.ptr, pp, 0, nullptr, 0, 0, rows, cols, a[k], a[k + 1], 1};
            return hyb::launch_wiener_stats(w, win, W, cs);
        };
        for (int k = 0; k < K; ++k) {
            int need = k;  // last chunk holding input rows < a[k+1] + rA
            while (need + 1 < K && a[need + 1] < std::min(rows, a[k + 1] + rA)) ++need;
            HYB_CHECK(cudaStreamWaitEvent(cs, ctx->ev_ah2d[b][need], 0));
            hyb::Plane am{in, pp, 0, ctx->f.ptr + (size_t)a[k] * pp, pp, 0, rows, cols, a[k], a[k + 1], 1};
            HYB_CHECK(run_amf(ctx, am, smax, nullptr, 0, 0));
            if (k >= 1 && a[k + 1] - a[k] >= rW) HYB_CHECK(stats(k - 1));
            else if (k >= 1) return fail(ctx, HYB_EINVAL, "chunk thinner than the Wiener halo");
        }
        HYB_CHECK(stats(K - 1));
        HYB_CHECK(cudaEventRecord(ctx->ev_in_free[b], cs));
        HYB_CHECK(cudaStreamWaitEvent(cs, ctx->ev_out_free[b], 0));
        for (int k = 0; k < K; ++k) {
            hyb::Plane w{ctx->f.ptr, pp, 0, out + (size_t)a[k] * pp, pp, 0, rows, cols, a[k], a[k + 1], 1};
            HYB_CHECK(hyb::launch_wiener_gain(w, win, reinterpret_cast<const long long*>(W), bytes, cs));
            HYB_CHECK(cudaEventRecord(ctx->ev_again[b][k], cs));
        }
    }
    // download (copy2 stream) chunk by chunk as the gains finish
    const int Kd = (K == 1 && hyb::plan_small(rows, cols, smax, win).ok) ? 1 : K;
    for (int k = 0; k < Kd; ++k) {
        HYB_CHECK(cudaStreamWaitEvent(ys, ctx->ev_again[b][k], 0));
        HYB_CHECK(cp(y + (size_t)a[k] * y_pitch, y_pitch, out + (size_t)a[k] * pp, pp, a[k + 1] - a[k], ys));
    }
    HYB_CHECK(cudaEventRecord(ctx->ev_out_free[b], ys));
    ctx->async_parity ^= 1;
    return HYB_OK;
}

}  // namespace

extern "C" {

hyb_ctx* hyb_create(int device, int* status) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || device < 0 || device >= n) {
        if (status) *status = HYB_ECUDA;
        cudaGetLastError();
        return nullptr;
    }
    hyb_ctx* ctx = new hyb_ctx;
    ctx->device = device;
    e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking);
    for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaEventCreate(&ctx->ev[i]);
    if (e != cudaSuccess) {
        if (status) *status = HYB_ECUDA;
        delete ctx;
        return nullptr;
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->copy2, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_stats, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_done, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_gainx, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_start, cudaEventDisableTiming);
    for (int i = 0; i < hyb_ctx::kMaxChunks && e == cudaSuccess; ++i) {
        e = cudaEventCreateWithFlags(&ctx->ev_h2d[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_gain[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        if (status) *status = HYB_ECUDA;
        delete ctx;
        return nullptr;
    }
    ctx->stream = ctx->own;
    if (status) *status = HYB_OK;
    return ctx;
}

int hyb_destroy(hyb_ctx* ctx) {
    if (!ctx) return HYB_OK;
    for (hyb_ctx* p : ctx->peers) hyb_destroy(p);
    ctx->peers.clear();
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->in.release();
    ctx->out.release();
    ctx->fin.release();
    ctx->f.release();
    ctx->wsum.release();
    ctx->sbar.release();
    ctx->mm.release();
    ctx->ys.release();
    ctx->fin64.release();
    ctx->fout64.release();
    ctx->fref64.release();
    ctx->fsc.release();
    ctx->freq.release();
    for (auto& b : ctx->amf_q) b.release();
    ctx->amf_cnt.release();
    for (auto& b : ctx->strip_g) b.release();
    for (auto& b : ctx->strip_f) b.release();
    ctx->wparts.release();
    ctx->wtot.release();
    for (int b = 0; b < 2; ++b) {
        ctx->ain[b].release();
        ctx->aout[b].release();
        for (cudaEvent_t ev : {ctx->ev_in_free[b], ctx->ev_out_free[b]})
            if (ev) cudaEventDestroy(ev);
        for (int k = 0; k < hyb_ctx::kMaxChunks; ++k) {
            if (ctx->ev_ah2d[b][k]) cudaEventDestroy(ctx->ev_ah2d[b][k]);
            if (ctx->ev_again[b][k]) cudaEventDestroy(ctx->ev_again[b][k]);
        }
    }
    ctx->mg_in.release();
    ctx->mg_out.release();
    if (ctx->host_w) cudaFreeHost(ctx->host_w);
    for (cudaEvent_t ev : {ctx->ev_stats, ctx->ev_done, ctx->ev_start, ctx->ev_gainx})
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : ctx->ev)
        if (ev) cudaEventDestroy(ev);
    for (auto& kv : ctx->graphs)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    for (auto& ev : ctx->ev_h2d)
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : ctx->ev_gain)
        if (ev) cudaEventDestroy(ev);
    if (ctx->copy) cudaStreamDestroy(ctx->copy);
    if (ctx->copy2) cudaStreamDestroy(ctx->copy2);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    delete ctx;
    return HYB_OK;
}

int hyb_set_stream(hyb_ctx* ctx, void* stream) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
    return HYB_OK;
}

int hyb_set_async(hyb_ctx* ctx, int async_host) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    if (ctx->async_host && !async_host) {  // leaving async mode: complete the pending calls
        const int st = hyb_synchronize(ctx);
        if (st) return st;
    }
    ctx->async_host = async_host != 0;
    return HYB_OK;
}

int hyb_synchronize(hyb_ctx* ctx) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    HYB_CHECK(cudaSetDevice(ctx->device));
    // join the copy streams into the context stream first, so work the caller enqueues on that stream
    // afterwards (or an event recorded there) is ordered after every pending call
    HYB_CHECK(cudaEventRecord(ctx->ev_h2d[hyb_ctx::kMaxChunks - 1], ctx->copy));
    HYB_CHECK(cudaStreamWaitEvent(ctx->stream, ctx->ev_h2d[hyb_ctx::kMaxChunks - 1], 0));
    HYB_CHECK(cudaEventRecord(ctx->ev_gain[hyb_ctx::kMaxChunks - 1], ctx->copy2));
    HYB_CHECK(cudaStreamWaitEvent(ctx->stream, ctx->ev_gain[hyb_ctx::kMaxChunks - 1], 0));
    HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    for (hyb_ctx* p : ctx->peers) {
        const int st = hyb_synchronize(p);
        if (st) return fail(ctx, st, p->err);
    }
    return HYB_OK;
}

int hyb_set_exclusive(hyb_ctx* ctx, int exclusive) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    ctx->exclusive = exclusive != 0;
    return HYB_OK;
}

const char* hyb_last_error(const hyb_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t hyb_kernel_launches(const hyb_ctx* ctx) {
    if (!ctx) return 0;
    long long n = ctx->launches;
    for (const hyb_ctx* p : ctx->peers) n += p->launches;
    return n;
}

hyb_ctx* hyb_create_multi(int n_devices, const int* device_ids, int* status) {
    if (n_devices < 1 || n_devices > hyb::kMaxDevices || !device_ids) {
        if (status) *status = HYB_EINVAL;
        return nullptr;
    }
    hyb_ctx* ctx = hyb_create(device_ids[0], status);
    if (!ctx) return nullptr;
    for (int i = 1; i < n_devices; ++i) {
        hyb_ctx* p = hyb_create(device_ids[i], status);
        if (!p) {
            hyb_destroy(ctx);
            return nullptr;
        }
        ctx->peers.push_back(p);
    }
    // all-pairs peer access (NVLink on B200 boxes); pairs without it exchange through copies
    ctx->peer_ok.assign((size_t)n_devices * n_devices, 0);
    for (int i = 0; i < n_devices; ++i)
        for (int j = 0; j < n_devices; ++j) {
            const int di = device_ids[i], dj = device_ids[j];
            int can = di == dj;
            if (!can && cudaDeviceCanAccessPeer(&can, di, dj) == cudaSuccess && can) {
                cudaSetDevice(di);
                const cudaError_t e = cudaDeviceEnablePeerAccess(dj, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) can = 0;
                cudaGetLastError();
            }
            ctx->peer_ok[(size_t)i * n_devices + j] = (char)(can != 0);
        }
    cudaSetDevice(device_ids[0]);
    if (status) *status = HYB_OK;
    return ctx;
}

int hyb_context_devices(const hyb_ctx* ctx, int* device_ids) {
    if (!ctx) return 0;
    if (device_ids) {
        device_ids[0] = ctx->device;
        for (size_t i = 0; i < ctx->peers.size(); ++i) device_ids[i + 1] = ctx->peers[i]->device;
    }
    return 1 + (int)ctx->peers.size();
}

int hyb_validate_smax(int smax) { return (smax <= 1 || smax % 2 == 0) ? HYB_EINVAL : HYB_OK; }

int hyb_validate_config(int smax, int parts, int workers) {
    if (hyb_validate_smax(smax)) return HYB_EINVAL;
    if (parts < 1 || workers < 1) return HYB_EINVAL;
    return HYB_OK;
}

int hyb_amf_u8(hyb_ctx* ctx, const uint8_t* src, size_t src_pitch, int rows, int cols,
               int row_begin, int row_end, int smax, uint8_t* dst, size_t dst_pitch,
               uint8_t* finalized_at, size_t fin_pitch) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    int st;
    if ((st = check_smax(ctx, smax)) || (st = check_dims(ctx, rows, cols)) ||
        (st = check_range(ctx, rows, row_begin, row_end)) ||
        (st = check_pitch(ctx, src_pitch, cols, "src")) || (st = check_pitch(ctx, dst_pitch, cols, "dst")))
        return st;
    if (!src || !dst) return fail(ctx, HYB_EINVAL, "null image pointer");
    if (finalized_at && (st = check_pitch(ctx, fin_pitch, cols, "finalized_at"))) return st;
    HYB_CHECK(cudaSetDevice(ctx->device));
    const int orows = row_end - row_begin;
    // device buffers are used in place when TMA can address them (16-byte aligned base and pitch)
    const bool dsrc = is_device_ptr(src) && hyb::tma_compatible(src, src_pitch, 0);
    const bool ddst = is_device_ptr(dst) && hyb::tma_compatible(dst, dst_pitch, 0);
    const bool dfin = finalized_at && is_device_ptr(finalized_at) && hyb::tma_compatible(finalized_at, fin_pitch, 0);
    const size_t pp = round_pitch(cols);
    const uint8_t* s = src;
    size_t sp = src_pitch;
    if (!dsrc) {
        HYB_CHECK(ctx->in.ensure(pp * rows));
        HYB_CHECK(copy2d(ctx, ctx->in.ptr, pp, src, src_pitch, cols, rows));
        s = ctx->in.ptr;
        sp = pp;
    }
    uint8_t* d = dst;
    size_t dp = dst_pitch;
    if (!ddst) {
        HYB_CHECK(ctx->out.ensure(pp * orows));
        d = ctx->out.ptr;
        dp = pp;
    }
    uint8_t* fz = finalized_at;
    size_t fp = fin_pitch;
    if (finalized_at && !dfin) {
        HYB_CHECK(ctx->fin.ensure(pp * orows));
        fz = ctx->fin.ptr;
        fp = pp;
    }
    hyb::Plane p{s, sp, 0, d, dp, 0, rows, cols, row_begin, row_end, 1};
    HYB_CHECK(run_amf(ctx, p, smax, fz, fp, 0));
    if (!ddst) HYB_CHECK(copy2d(ctx, dst, dst_pitch, d, dp, cols, orows));
    if (finalized_at && !dfin) HYB_CHECK(copy2d(ctx, finalized_at, fin_pitch, fz, fp, cols, orows));
    if (!dsrc || !ddst || (finalized_at && !dfin)) HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    return HYB_OK;
}

int hyb_amf_batch_u8(hyb_ctx* ctx, const uint8_t* src, size_t src_pitch, size_t src_slice_stride,
                     int n_slices, int rows, int cols, int smax, uint8_t* dst, size_t dst_pitch,
                     size_t dst_slice_stride) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    int st;
    if ((st = check_smax(ctx, smax)) || (st = check_dims(ctx, rows, cols)) ||
        (st = check_pitch(ctx, src_pitch, cols, "src")) || (st = check_pitch(ctx, dst_pitch, cols, "dst")))
        return st;
    if (n_slices < 1) return fail(ctx, HYB_EINVAL, "n_slices must be >= 1, got " + std::to_string(n_slices));
    if (!is_device_ptr(src) || !is_device_ptr(dst))
        return fail(ctx, HYB_EINVAL, "hyb_amf_batch_u8 takes device buffers");
    if (!hyb::tma_compatible(src, src_pitch, src_slice_stride) || !hyb::tma_compatible(dst, dst_pitch, dst_slice_stride))
        return fail(ctx, HYB_EINVAL, "batch buffers need 16-byte aligned bases, pitches and slice strides");
    HYB_CHECK(cudaSetDevice(ctx->device));
    hyb::Plane p{src, src_pitch, src_slice_stride, dst, dst_pitch, dst_slice_stride, rows, cols, 0, rows,
                 n_slices};
    HYB_CHECK(run_amf(ctx, p, smax, nullptr, 0, 0));
    return HYB_OK;
}

int hyb_wiener_stats_u8(hyb_ctx* ctx, const uint8_t* f, size_t pitch, int rows, int cols,
                        int row_begin, int row_end, int win, int64_t* noise_sum) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    int st;
    if ((st = check_win(ctx, win)) || (st = check_dims(ctx, rows, cols)) ||
        (st = check_range(ctx, rows, row_begin, row_end)) || (st = check_pitch(ctx, pitch, cols, "f")))
        return st;
    if (!f || !noise_sum) return fail(ctx, HYB_EINVAL, "null pointer");
    HYB_CHECK(cudaSetDevice(ctx->device));
    const uint8_t* s = f;
    size_t sp = pitch;
    const bool df = is_device_ptr(f);
    if (!df) {
        sp = round_pitch(cols);
        HYB_CHECK(ctx->in.ensure(sp * rows));
        HYB_CHECK(copy2d(ctx, ctx->in.ptr, sp, f, pitch, cols, rows));
        s = ctx->in.ptr;
    }
    hyb::Plane p{s, sp, 0, nullptr, 0, 0, rows, cols, row_begin, row_end, 1};
    if (is_device_ptr(noise_sum)) {
        HYB_CHECK(hyb::launch_wiener_stats(p, win, reinterpret_cast<unsigned long long*>(noise_sum),
                                           ctx->stream));
        if (!df) HYB_CHECK(cudaStreamSynchronize(ctx->stream));
        return HYB_OK;
    }
    HYB_CHECK(ctx->wsum.ensure(sizeof(long long)));
    if ((st = ensure_host_w(ctx, 1))) return st;
    HYB_CHECK(cudaMemsetAsync(ctx->wsum.ptr, 0, sizeof(long long), ctx->stream));
    HYB_CHECK(hyb::launch_wiener_stats(p, win, reinterpret_cast<unsigned long long*>(ctx->wsum.ptr),
                                       ctx->stream));
    HYB_CHECK(cudaMemcpyAsync(ctx->host_w, ctx->wsum.ptr, sizeof(long long), cudaMemcpyDeviceToHost,
                              ctx->stream));
    HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    *noise_sum += ctx->host_w[0];
    return HYB_OK;
}

int hyb_wiener_gain_u8(hyb_ctx* ctx, const uint8_t* f, size_t pitch, int rows, int cols,
                       int row_begin, int row_end, int win, const int64_t* noise_sum,
                       int64_t pixel_count, uint8_t* y, size_t y_pitch) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    int st;
    if ((st = check_win(ctx, win)) || (st = check_dims(ctx, rows, cols)) ||
        (st = check_range(ctx, rows, row_begin, row_end)) || (st = check_pitch(ctx, pitch, cols, "f")) ||
        (st = check_pitch(ctx, y_pitch, cols, "y")))
        return st;
    if (!f || !y || !noise_sum) return fail(ctx, HYB_EINVAL, "null pointer");
    if (pixel_count < 1) return fail(ctx, HYB_EINVAL, "pixel_count must be >= 1");
    HYB_CHECK(cudaSetDevice(ctx->device));
    const bool df = is_device_ptr(f), dy = is_device_ptr(y);
    const size_t pp = round_pitch(cols);
    const int orows = row_end - row_begin;
    const uint8_t* s = f;
    size_t sp = pitch;
    if (!df) {
        HYB_CHECK(ctx->in.ensure(pp * rows));
        HYB_CHECK(copy2d(ctx, ctx->in.ptr, pp, f, pitch, cols, rows));
        s = ctx->in.ptr;
        sp = pp;
    }
    uint8_t* d = y;
    size_t dp = y_pitch;
    if (!dy) {
        HYB_CHECK(ctx->out.ensure(pp * orows));
        d = ctx->out.ptr;
        dp = pp;
    }
    const long long* W = reinterpret_cast<const long long*>(noise_sum);
    if (!is_device_ptr(noise_sum)) {
        if (*noise_sum < 0) return fail(ctx, HYB_EINVAL, "noise sum must be nonnegative");
        HYB_CHECK(ctx->wsum.ensure(sizeof(long long)));
        if ((st = ensure_host_w(ctx, 1))) return st;
        ctx->host_w[0] = *noise_sum;
        HYB_CHECK(cudaMemcpyAsync(ctx->wsum.ptr, ctx->host_w, sizeof(long long), cudaMemcpyHostToDevice,
                                  ctx->stream));
        W = reinterpret_cast<const long long*>(ctx->wsum.ptr);
    }
    hyb::Plane p{s, sp, 0, d, dp, 0, rows, cols, row_begin, row_end, 1};
    HYB_CHECK(hyb::launch_wiener_gain(p, win, W, pixel_count, ctx->stream));
    if (!dy) HYB_CHECK(copy2d(ctx, y, y_pitch, d, dp, cols, orows));
    if (!df || !dy || W != reinterpret_cast<const long long*>(noise_sum))
        HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    return HYB_OK;
}

int hyb_wiener_u8(hyb_ctx* ctx, const uint8_t* f, size_t pitch, int rows, int cols, int win,
                  uint8_t* y, size_t y_pitch, int64_t* noise_sum_out) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    int st;
    if ((st = check_win(ctx, win)) || (st = check_dims(ctx, rows, cols)) ||
        (st = check_pitch(ctx, pitch, cols, "f")) || (st = check_pitch(ctx, y_pitch, cols, "y")))
        return st;
    if (!f || !y) return fail(ctx, HYB_EINVAL, "null image pointer");
    HYB_CHECK(cudaSetDevice(ctx->device));
    const bool df = is_device_ptr(f), dy = is_device_ptr(y);
    const size_t pp = round_pitch(cols);
    const uint8_t* s = f;
    size_t sp = pitch;
    if (!df) {
        HYB_CHECK(ctx->in.ensure(pp * rows));
        HYB_CHECK(copy2d(ctx, ctx->in.ptr, pp, f, pitch, cols, rows));
        s = ctx->in.ptr;
        sp = pp;
    }
    uint8_t* d = y;
    size_t dp = y_pitch;
    if (!dy) {
        HYB_CHECK(ctx->out.ensure(pp * rows));
        d = ctx->out.ptr;
        dp = pp;
    }
    HYB_CHECK(ctx->wsum.ensure(sizeof(long long)));
    unsigned long long* W = reinterpret_cast<unsigned long long*>(ctx->wsum.ptr);
    HYB_CHECK(cudaMemsetAsync(W, 0, sizeof(long long), ctx->stream));
    hyb::Plane p{s, sp, 0, d, dp, 0, rows, cols, 0, rows, 1};
    HYB_CHECK(hyb::launch_wiener_stats(p, win, W, ctx->stream));
    HYB_CHECK(hyb::launch_wiener_gain(p, win, reinterpret_cast<const long long*>(W), (long long)rows * cols,
                                      ctx->stream));
    if (!dy) HYB_CHECK(copy2d(ctx, y, y_pitch, d, dp, cols, rows));
    if (noise_sum_out) {
        if ((st = ensure_host_w(ctx, 1))) return st;
        HYB_CHECK(cudaMemcpyAsync(ctx->host_w, W, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (!df || !dy || noise_sum_out) HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    if (noise_sum_out) *noise_sum_out = ctx->host_w[0];
    return HYB_OK;
}

static int hybrid_u8_impl(hyb_ctx* ctx, const uint8_t* g, size_t pitch, int rows, int cols, int smax,
                          int win, int parts, uint8_t* y, size_t y_pitch, hyb_stats* stats, bool capturing);

int hyb_hybrid_u8(hyb_ctx* ctx, const uint8_t* g, size_t pitch, int rows, int cols, int smax,
                  int win, int parts, uint8_t* y, size_t y_pitch, hyb_stats* stats) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    if (!ctx->peers.empty()) return hybrid_multi(ctx, g, pitch, rows, cols, smax, win, parts, y, y_pitch, stats);
    if (ctx->async_host && !stats && parts == 1) {
        cudaPointerAttributes pa{}, pb{};
        const bool pinned = g && y && cudaPointerGetAttributes(&pa, g) == cudaSuccess &&
                            cudaPointerGetAttributes(&pb, y) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
                            pb.type == cudaMemoryTypeHost;
        cudaGetLastError();
        int st;
        if (pinned && !(st = check_smax(ctx, smax)) && !(st = check_win(ctx, win)) && !(st = check_dims(ctx, rows, cols)) &&
            !(st = check_pitch(ctx, pitch, cols, "g")) && !(st = check_pitch(ctx, y_pitch, cols, "y"))) {
            HYB_CHECK(cudaSetDevice(ctx->device));
            return hybrid_host_async(ctx, g, pitch, rows, cols, smax, win, y, y_pitch);
        }
        if (pinned) return st;
    }
    // Untimed calls on device buffers or pinned host buffers replay a cached CUDA graph.
    cudaPointerAttributes ga{}, ya{};
    const bool gok = g && cudaPointerGetAttributes(&ga, g) == cudaSuccess;
    const bool yok = y && cudaPointerGetAttributes(&ya, y) == cudaSuccess;
    cudaGetLastError();
    // Cooperative launches (the fused small-image kernel without exclusive mode) are cheaper as
    // direct launches than as graph nodes, so those calls are not captured.
    const bool coop_small = !ctx->exclusive && parts == 1 && hyb::plan_small(rows, cols, smax, win).ok;
    const bool graphable = !coop_small && !stats && gok && yok && ga.type != cudaMemoryTypeUnregistered &&
                           ya.type != cudaMemoryTypeUnregistered && ctx->stream != nullptr &&
                           ctx->stream != cudaStreamLegacy && ctx->stream != cudaStreamPerThread;  // not capturable
    if (!graphable) return hybrid_u8_impl(ctx, g, pitch, rows, cols, smax, win, parts, y, y_pitch, stats, false);
    const hyb_ctx::GraphKey key{g, y, pitch, y_pitch, rows, cols, smax, win, parts, ctx->stream};
    auto it = ctx->graphs.find(key);
    if (it != ctx->graphs.end() && it->second.bufs != buf_signature(ctx)) {
        // scratch reallocated since the capture (a larger image, a batch, more strips): drop the graph,
        // run plainly now (re-allocating what this call needs) and re-capture on the next call
        HYB_CHECK(cudaSetDevice(ctx->device));
        cudaGraphExecDestroy(it->second.exec);
        ctx->graphs.erase(it);
        ctx->graph_seen[key] = 1;
        return hybrid_u8_impl(ctx, g, pitch, rows, cols, smax, win, parts, y, y_pitch, nullptr, false);
    }
    if (it == ctx->graphs.end()) {
        int& seen = ctx->graph_seen[key];
        if (seen++ == 0)  // first use: plain run (allocates every buffer the sequence needs)
            return hybrid_u8_impl(ctx, g, pitch, rows, cols, smax, win, parts, y, y_pitch, nullptr, false);
        HYB_CHECK(cudaSetDevice(ctx->device));
        HYB_CHECK(cudaStreamSynchronize(ctx->stream));
        const long long k0 = ctx->launches;
        const std::vector<const void*> sig = buf_signature(ctx);
        HYB_CHECK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        int st = hybrid_u8_impl(ctx, g, pitch, rows, cols, smax, win, parts, y, y_pitch, nullptr, true);
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
        if (st) {
            if (graph) cudaGraphDestroy(graph);
            return st;
        }
        if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamEndCapture");
        if (buf_signature(ctx) != sig) {
            // the captured call allocated (it cannot: the plain run before it did) -- do not keep it
            cudaGraphDestroy(graph);
            return fail(ctx, HYB_ECUDA, "scratch reallocated during graph capture");
        }
        hyb_ctx::Graph gr;
        e = cudaGraphInstantiate(&gr.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaGraphInstantiate");
        gr.kernels = ctx->launches - k0;
        gr.bufs = sig;
        ctx->launches = k0;  // counted at each replay instead
        if (ctx->graphs.size() >= 4096) {
            for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second.exec);
            ctx->graphs.clear();
        }
        it = ctx->graphs.emplace(key, gr).first;
    }
    HYB_CHECK(cudaGraphLaunch(it->second.exec, ctx->stream));
    ctx->launches += it->second.kernels;
    if (ga.type != cudaMemoryTypeDevice || ya.type != cudaMemoryTypeDevice)
        HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    return HYB_OK;
}

// Fused-kernel runs report the kernel's own AMF / Wiener split (globaltimer stamps, host_w[1..3]).
static void small_times(hyb_ctx* ctx, hyb_stats* stats) {
    if (!ctx->small_used) return;
    const unsigned long long t0 = ctx->host_w[1], t1 = ctx->host_w[2], t2 = ctx->host_w[3];
    stats->t_adaptive = (double)(t1 - t0) * 1e-9;  // k = 3..smax (to the grid barrier)
    stats->t_wiener = (double)(t2 - t1) * 1e-9;    // statistics + gain
}

static int hybrid_u8_impl(hyb_ctx* ctx, const uint8_t* g, size_t pitch, int rows, int cols, int smax,
                          int win, int parts, uint8_t* y, size_t y_pitch, hyb_stats* stats, bool capturing) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    ctx->small_used = false;
    int st;
    if ((st = check_smax(ctx, smax)) || (st = check_win(ctx, win)) || (st = check_dims(ctx, rows, cols)) ||
        (st = check_pitch(ctx, pitch, cols, "g")) || (st = check_pitch(ctx, y_pitch, cols, "y")))
        return st;
    if (parts < 1) return fail(ctx, HYB_EINVAL, "parts must be >= 1, got " + std::to_string(parts));
    if (parts > rows)
        return fail(ctx, HYB_EINVAL, "parts " + std::to_string(parts) + " exceeds image rows " +
                                         std::to_string(rows));
    if (!g || !y) return fail(ctx, HYB_EINVAL, "null image pointer");
    HYB_CHECK(cudaSetDevice(ctx->device));
    const bool dg = is_device_ptr(g) && hyb::tma_compatible(g, pitch, 0), dy = is_device_ptr(y);
    const size_t pp = round_pitch(cols);
    const bool timed = stats != nullptr;
    if (!dg && !dy && !is_device_ptr(g) && parts == 1) {
        if ((st = hybrid_host_pipelined(ctx, g, pitch, rows, cols, smax, win, y, y_pitch, timed))) return st;
        if (timed) {
            if ((st = ensure_host_w(ctx, 1))) return st;
            HYB_CHECK(cudaMemcpyAsync(ctx->host_w, ctx->wsum.ptr, sizeof(long long), cudaMemcpyDeviceToHost,
                                      ctx->stream));
        }
        if (!capturing) HYB_CHECK(cudaStreamSynchronize(ctx->stream));
        if (timed) {
            float am = 0, w = 0, t = 0;
            HYB_CHECK(cudaEventElapsedTime(&am, ctx->ev[0], ctx->ev[1]));
            HYB_CHECK(cudaEventElapsedTime(&w, ctx->ev[1], ctx->ev[2]));
            HYB_CHECK(cudaEventElapsedTime(&t, ctx->ev[3], ctx->ev[2]));
            const double n = (double)win * win;
            stats->noise_sum = ctx->host_w[0];
            stats->pixel_count = (int64_t)rows * cols;
            stats->sigma2 = (double)stats->noise_sum / (n * n * (double)stats->pixel_count) / (255.0 * 255.0);
            stats->t_adaptive = am * 1e-3;  // AMF + statistics (interleaved with the upload)
            stats->t_wiener = w * 1e-3;     // gains (interleaved with the download)
            stats->t_total = t * 1e-3;
            small_times(ctx, stats);
        }
        return HYB_OK;
    }
    if (timed) HYB_CHECK(cudaEventRecord(ctx->ev[3], ctx->stream));
    const uint8_t* s = g;
    size_t sp = pitch;
    if (!dg) {
        HYB_CHECK(ctx->in.ensure(pp * rows));
        HYB_CHECK(copy2d(ctx, ctx->in.ptr, pp, g, pitch, cols, rows));
        s = ctx->in.ptr;
        sp = pp;
    }
    uint8_t* d = y;
    size_t dp = y_pitch;
    if (!dy) {
        HYB_CHECK(ctx->out.ensure(pp * rows));
        d = ctx->out.ptr;
        dp = pp;
    }
    if ((st = hybrid_device(ctx, s, sp, rows, cols, smax, win, parts, d, dp, timed))) return st;
    if (!dy) HYB_CHECK(copy2d(ctx, y, y_pitch, d, dp, cols, rows));
    if (timed) {
        if ((st = ensure_host_w(ctx, 1))) return st;
        HYB_CHECK(cudaMemcpyAsync(ctx->host_w, ctx->wsum.ptr, sizeof(long long), cudaMemcpyDeviceToHost,
                                  ctx->stream));
    }
    if ((!dg || !dy || timed) && !capturing) HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    if (timed) {
        float a = 0, w = 0, t = 0;
        HYB_CHECK(cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]));
        HYB_CHECK(cudaEventElapsedTime(&w, ctx->ev[1], ctx->ev[2]));
        HYB_CHECK(cudaEventElapsedTime(&t, ctx->ev[3], ctx->ev[2]));
        const double n = (double)win * win;
        stats->noise_sum = ctx->host_w[0];
        stats->pixel_count = (int64_t)rows * cols;
        stats->sigma2 = (double)stats->noise_sum / (n * n * (double)stats->pixel_count) / (255.0 * 255.0);
        stats->t_adaptive = a * 1e-3;
        stats->t_wiener = w * 1e-3;
        stats->t_total = t * 1e-3;
        small_times(ctx, stats);
    }
    return HYB_OK;
}

int hyb_contrast_stretch_u8(hyb_ctx* ctx, const uint8_t* src, size_t pitch, int rows, int cols, uint8_t* dst,
                            size_t dst_pitch) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    int st;
    if ((st = check_dims(ctx, rows, cols)) || (st = check_pitch(ctx, pitch, cols, "src")) ||
        (st = check_pitch(ctx, dst_pitch, cols, "dst")))
        return st;
    if (!src || !dst) return fail(ctx, HYB_EINVAL, "null image pointer");
    HYB_CHECK(cudaSetDevice(ctx->device));
    const bool ds = is_device_ptr(src), dd = is_device_ptr(dst);
    const size_t pp = round_pitch(cols);
    const uint8_t* s = src;
    size_t sp = pitch;
    if (!ds) {
        HYB_CHECK(ctx->in.ensure(pp * rows));
        HYB_CHECK(copy2d(ctx, ctx->in.ptr, pp, src, pitch, cols, rows));
        s = ctx->in.ptr;
        sp = pp;
    }
    uint8_t* d = dst;
    size_t dp = dst_pitch;
    if (!dd) {
        HYB_CHECK(ctx->out.ensure(pp * rows));
        d = ctx->out.ptr;
        dp = pp;
    }
    HYB_CHECK(ctx->mm.ensure(2 * sizeof(unsigned)));
    HYB_CHECK(hyb::launch_contrast_stretch(s, sp, rows, cols, d, dp, reinterpret_cast<unsigned*>(ctx->mm.ptr),
                                           ctx->stream));
    if (!dd) HYB_CHECK(copy2d(ctx, dst, dst_pitch, d, dp, cols, rows));
    if (!ds || !dd) HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    return HYB_OK;
}

int hyb_window_stats_u8(hyb_ctx* ctx, const uint8_t* src, size_t pitch, int rows, int cols, int k, uint8_t* zmin,
                        uint8_t* zmed, uint8_t* zmax, size_t out_pitch) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    int st;
    if (k < 3 || k % 2 == 0)  // proj/src/adaptive_median.cpp:97-100
        return fail(ctx, HYB_EINVAL, "window size must be an odd integer >= 3, got " + std::to_string(k));
    if ((st = check_dims(ctx, rows, cols)) || (st = check_pitch(ctx, pitch, cols, "src")) ||
        (st = check_pitch(ctx, out_pitch, cols, "out")))
        return st;
    if (!src) return fail(ctx, HYB_EINVAL, "null image pointer");
    HYB_CHECK(cudaSetDevice(ctx->device));
    const size_t pp = round_pitch(cols);
    const uint8_t* s = src;
    size_t sp = pitch;
    if (!is_device_ptr(src)) {
        HYB_CHECK(ctx->in.ensure(pp * rows));
        HYB_CHECK(copy2d(ctx, ctx->in.ptr, pp, src, pitch, cols, rows));
        s = ctx->in.ptr;
        sp = pp;
    }
    // device outputs are written in place; host ones go through three planes of ctx->out (pitch pp)
    uint8_t* outs[3] = {zmin, zmed, zmax};
    bool staged[3] = {false, false, false};
    bool any_staged = false;
    for (int i = 0; i < 3; ++i) staged[i] = outs[i] && !is_device_ptr(outs[i]), any_staged |= staged[i];
    if (any_staged) HYB_CHECK(ctx->out.ensure(3 * pp * rows));
    uint8_t* d[3];
    size_t dp = out_pitch;
    if (any_staged) dp = pp;
    for (int i = 0; i < 3; ++i) d[i] = staged[i] ? ctx->out.ptr + (size_t)i * pp * rows : outs[i];
    if (any_staged && dp != out_pitch) {
        // one pitch per launch: with mixed host / device outputs, stage the device ones too
        for (int i = 0; i < 3; ++i)
            if (outs[i] && !staged[i]) staged[i] = true, d[i] = ctx->out.ptr + (size_t)i * pp * rows;
    }
    HYB_CHECK(hyb::launch_window_stats(s, sp, rows, cols, k, d[0], d[1], d[2], dp, ctx->stream));
    for (int i = 0; i < 3; ++i)
        if (staged[i]) HYB_CHECK(copy2d(ctx, outs[i], out_pitch, d[i], dp, cols, rows));
    if (any_staged || s != src) HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    return HYB_OK;
}

int hyb_hybrid_stretch_u8(hyb_ctx* ctx, const uint8_t* g, size_t pitch, int rows, int cols, int smax, int win,
                          int parts, uint8_t* y, size_t y_pitch, hyb_stats* stats) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    int st;
    if ((st = check_dims(ctx, rows, cols)) || (st = check_pitch(ctx, y_pitch, cols, "y"))) return st;
    if (!y) return fail(ctx, HYB_EINVAL, "null image pointer");
    // multi-device: per-strip ranges fused into the gains, one exchange, per-strip maps (hybrid_multi 5.)
    if (!ctx->peers.empty()) return hybrid_multi(ctx, g, pitch, rows, cols, smax, win, parts, y, y_pitch, stats, true);
    HYB_CHECK(cudaSetDevice(ctx->device));
    // stages 1-2 into a device buffer, then the final stretch (in place when y is on the device).  The
    // separate-kernel gains fold y's range into mm as they write it, leaving only the map; the fused
    // small-image kernel does not, and then the stretch runs its own min / max pass first.
    const bool dy = is_device_ptr(y);
    const size_t pp = round_pitch(cols);
    uint8_t* d = y;
    size_t dp = y_pitch;
    if (!dy) {
        HYB_CHECK(ctx->ys.ensure(pp * rows));
        d = ctx->ys.ptr;
        dp = pp;
    }
    HYB_CHECK(ctx->mm.ensure(2 * sizeof(unsigned)));
    unsigned* mm = reinterpret_cast<unsigned*>(ctx->mm.ptr);
    HYB_CHECK(cudaMemsetAsync(mm, 0xFF, 2 * sizeof(unsigned), ctx->stream));
    ctx->stretch_mm = mm;
    ctx->stretch_fused = false;
    st = hybrid_u8_impl(ctx, g, pitch, rows, cols, smax, win, parts, d, dp, stats, false);  // no graph replay
    ctx->stretch_mm = nullptr;
    if (st) return st;
    if (ctx->stretch_fused)
        HYB_CHECK(hyb::launch_stretch_map(d, dp, rows, cols, d, dp, mm, ctx->stream));
    else
        HYB_CHECK(hyb::launch_contrast_stretch(d, dp, rows, cols, d, dp, mm, ctx->stream));
    if (!dy) {
        HYB_CHECK(copy2d(ctx, y, y_pitch, d, dp, cols, rows));
        HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    }
    return HYB_OK;
}

// Stages a double image (host or device, pitch in elements) on the device; returns the device view.
static int stage_f64(hyb_ctx* ctx, DevBuf& buf, const double* src, size_t pitch, int rows, int cols,
                     const double** dev, size_t* dpitch) {
    if (is_device_ptr(src)) {
        *dev = src;
        *dpitch = pitch;
        return HYB_OK;
    }
    HYB_CHECK(buf.ensure((size_t)rows * cols * sizeof(double)));
    HYB_CHECK(cudaMemcpy2DAsync(buf.ptr, (size_t)cols * sizeof(double), src, pitch * sizeof(double),
                                (size_t)cols * sizeof(double), (size_t)rows, cudaMemcpyDefault, ctx->stream));
    *dev = reinterpret_cast<const double*>(buf.ptr);
    *dpitch = (size_t)cols;
    return HYB_OK;
}

int hyb_wiener_freq_f64(hyb_ctx* ctx, const double* f, size_t pitch, int rows, int cols, double sigma2, int clamp,
                        double* out, size_t out_pitch) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    int st;
    if ((st = check_dims(ctx, rows, cols))) return st;
    if (pitch < (size_t)cols || out_pitch < (size_t)cols) return fail(ctx, HYB_EINVAL, "pitch smaller than cols");
    if (!f || !out) return fail(ctx, HYB_EINVAL, "null image pointer");
    if (!(sigma2 >= 0.0)) return fail(ctx, HYB_EINVAL, "noise variance must be nonnegative");
    HYB_CHECK(cudaSetDevice(ctx->device));
    const double* s = nullptr;
    size_t sp = 0;
    if ((st = stage_f64(ctx, ctx->fin64, f, pitch, rows, cols, &s, &sp))) return st;
    const bool dout = is_device_ptr(out);
    double* d = out;
    size_t dp = out_pitch;
    if (!dout) {
        HYB_CHECK(ctx->fout64.ensure((size_t)rows * cols * sizeof(double)));
        d = reinterpret_cast<double*>(ctx->fout64.ptr);
        dp = (size_t)cols;
    }
    int cst = 0;
    HYB_CHECK(hyb::launch_wiener_freq(s, sp, rows, cols, sigma2, clamp != 0, d, dp, ctx->freq, ctx->stream, &cst));
    if (cst) return fail(ctx, HYB_ECUDA, "cuFFT error " + std::to_string(cst));
    if (!dout)
        HYB_CHECK(cudaMemcpy2DAsync(out, out_pitch * sizeof(double), d, dp * sizeof(double),
                                    (size_t)cols * sizeof(double), (size_t)rows, cudaMemcpyDefault, ctx->stream));
    if (!dout || !is_device_ptr(f)) HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    return HYB_OK;
}

int hyb_contrast_stretch_f64(hyb_ctx* ctx, const double* src, size_t pitch, int rows, int cols, double* dst,
                             size_t dst_pitch) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    int st;
    if ((st = check_dims(ctx, rows, cols))) return st;
    if (pitch < (size_t)cols || dst_pitch < (size_t)cols) return fail(ctx, HYB_EINVAL, "pitch smaller than cols");
    if (!src || !dst) return fail(ctx, HYB_EINVAL, "null image pointer");
    HYB_CHECK(cudaSetDevice(ctx->device));
    const double* s = nullptr;
    size_t sp = 0;
    if ((st = stage_f64(ctx, ctx->fin64, src, pitch, rows, cols, &s, &sp))) return st;
    const bool dd = is_device_ptr(dst);
    double* d = dst;
    size_t dp = dst_pitch;
    if (!dd) {
        HYB_CHECK(ctx->fout64.ensure((size_t)rows * cols * sizeof(double)));
        d = reinterpret_cast<double*>(ctx->fout64.ptr);
        dp = (size_t)cols;
    }
    HYB_CHECK(hyb::launch_contrast_stretch_f64(s, sp, rows, cols, d, dp, ctx->freq, ctx->stream));
    if (!dd)
        HYB_CHECK(cudaMemcpy2DAsync(dst, dst_pitch * sizeof(double), d, dp * sizeof(double),
                                    (size_t)cols * sizeof(double), (size_t)rows, cudaMemcpyDefault, ctx->stream));
    if (!dd || !is_device_ptr(src)) HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    return HYB_OK;
}

int hyb_noise_robust_f64(hyb_ctx* ctx, const double* f, size_t pitch, int rows, int cols, double* sigma2) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    int st;
    if ((st = check_dims(ctx, rows, cols))) return st;
    if (pitch < (size_t)cols) return fail(ctx, HYB_EINVAL, "pitch smaller than cols");
    if (!f || !sigma2) return fail(ctx, HYB_EINVAL, "null pointer");
    HYB_CHECK(cudaSetDevice(ctx->device));
    const double* s = nullptr;
    size_t sp = 0;
    if ((st = stage_f64(ctx, ctx->fin64, f, pitch, rows, cols, &s, &sp))) return st;
    HYB_CHECK(ctx->fsc.ensure(sizeof(double)));
    double* dm = reinterpret_cast<double*>(ctx->fsc.ptr);
    HYB_CHECK(hyb::launch_noise_robust(s, sp, rows, cols, ctx->freq, dm, ctx->stream));
    double med = 0.0;
    HYB_CHECK(cudaMemcpyAsync(&med, dm, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    const double sigma = med / 0.6745;
    *sigma2 = sigma * sigma;
    return HYB_OK;
}

int hyb_noise_reference_f64(hyb_ctx* ctx, const double* f, size_t pitch, const double* ref, size_t ref_pitch,
                            int rows, int cols, double* sigma2) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    int st;
    if ((st = check_dims(ctx, rows, cols))) return st;
    if (pitch < (size_t)cols || ref_pitch < (size_t)cols) return fail(ctx, HYB_EINVAL, "pitch smaller than cols");
    if (!f || !ref || !sigma2) return fail(ctx, HYB_EINVAL, "null pointer");
    HYB_CHECK(cudaSetDevice(ctx->device));
    const double *a = nullptr, *b = nullptr;
    size_t ap = 0, bp = 0;
    if ((st = stage_f64(ctx, ctx->fin64, f, pitch, rows, cols, &a, &ap))) return st;
    if ((st = stage_f64(ctx, ctx->fref64, ref, ref_pitch, rows, cols, &b, &bp))) return st;
    HYB_CHECK(ctx->fsc.ensure(sizeof(double)));
    double* acc = reinterpret_cast<double*>(ctx->fsc.ptr);
    HYB_CHECK(hyb::launch_noise_reference(a, ap, b, bp, rows, cols, acc, ctx->stream));
    double sum = 0.0;
    HYB_CHECK(cudaMemcpyAsync(&sum, acc, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    *sigma2 = sum / ((double)rows * cols);
    return HYB_OK;
}

}  // extern "C"

namespace {

// Host-buffer stacks: slices move in chunks of ~8 MB through three streams so the two PCIe
// directions and the kernels overlap -- copy stream: H2D of chunk k; compute stream: the hybrid
// of chunk k (slices are independent, each with its own noise sum); copy2 stream: D2H of chunk k.
// Returns false (nothing enqueued) when the layout does not fit.
bool batch_host_pipelined(hyb_ctx* ctx, const uint8_t* g, size_t pitch, size_t slice_stride, int n_slices,
                          int rows, int cols, int smax, int win, uint8_t* y, size_t y_pitch, size_t y_slice_stride,
                          unsigned long long* W, int* status) {
    *status = HYB_OK;
    const size_t pp = round_pitch(cols), ps = pp * rows;
    const size_t slice_bytes = (size_t)cols * rows;
    if (slice_stride != pitch * rows || y_slice_stride != y_pitch * rows) return false;
    int per = (int)std::max<size_t>(1, ((size_t)8 << 20) / slice_bytes);
    int K = (n_slices + per - 1) / per;
    if (K < 2) return false;
    if (K > hyb_ctx::kMaxChunks) {
        K = hyb_ctx::kMaxChunks;
        per = (n_slices + K - 1) / K;
        K = (n_slices + per - 1) / per;
    }
    cudaStream_t cs = ctx->stream, xs = ctx->copy, ys = ctx->copy2;
    auto run = [&]() -> cudaError_t {
        cudaError_t e;
        auto cp = [&](void* dst, size_t dp, const void* src, size_t sp, int nrows, cudaStream_t st) {
            if (dp == (size_t)cols && sp == (size_t)cols)
                return cudaMemcpyAsync(dst, src, (size_t)cols * nrows, cudaMemcpyDefault, st);
            return cudaMemcpy2DAsync(dst, dp, src, sp, (size_t)cols, (size_t)nrows, cudaMemcpyDefault, st);
        };
        // both copy streams start after earlier compute-stream work
        if ((e = cudaEventRecord(ctx->ev_gain[0], cs)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(xs, ctx->ev_gain[0], 0)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(ys, ctx->ev_gain[0], 0)) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(W, 0, sizeof(long long) * n_slices, cs)) != cudaSuccess) return e;
        for (int k = 0; k < K; ++k) {
            const int z0 = k * per, nz = std::min(per, n_slices - z0);
            if ((e = cp(ctx->in.ptr + ps * z0, pp, g + slice_stride * z0, pitch, rows * nz, xs)) != cudaSuccess)
                return e;
            if ((e = cudaEventRecord(ctx->ev_h2d[k], xs)) != cudaSuccess) return e;
        }
        for (int k = 0; k < K; ++k) {
            const int z0 = k * per, nz = std::min(per, n_slices - z0);
            if ((e = cudaStreamWaitEvent(cs, ctx->ev_h2d[k], 0)) != cudaSuccess) return e;
            hyb::Plane a{ctx->in.ptr + ps * z0, pp, ps, ctx->f.ptr + ps * z0, pp, ps, rows, cols, 0, rows, nz};
            if ((e = run_amf(ctx, a, smax, nullptr, 0, 0)) != cudaSuccess) return e;
            hyb::Plane w{ctx->f.ptr + ps * z0, pp, ps, ctx->out.ptr + ps * z0, pp, ps, rows, cols, 0, rows, nz};
            if ((e = hyb::launch_wiener_stats(w, win, W + z0, cs)) != cudaSuccess) return e;
            if ((e = hyb::launch_wiener_gain(w, win, reinterpret_cast<const long long*>(W + z0),
                                             (long long)rows * cols, cs)) != cudaSuccess)
                return e;
            if ((e = cudaEventRecord(ctx->ev_gain[k], cs)) != cudaSuccess) return e;
            if ((e = cudaStreamWaitEvent(ys, ctx->ev_gain[k], 0)) != cudaSuccess) return e;
            if ((e = cp(y + y_slice_stride * z0, y_pitch, ctx->out.ptr + ps * z0, pp, rows * nz, ys)) != cudaSuccess)
                return e;
        }
        // the compute stream resumes after the last download and the last upload
        if ((e = cudaEventRecord(ctx->ev_h2d[0], ys)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(cs, ctx->ev_h2d[0], 0)) != cudaSuccess) return e;
        if ((e = cudaEventRecord(ctx->ev_h2d[1], xs)) != cudaSuccess) return e;
        return cudaStreamWaitEvent(cs, ctx->ev_h2d[1], 0);
    };
    const cudaError_t e = run();
    if (e != cudaSuccess) *status = cuda_fail(ctx, e, "batch pipeline");
    return true;
}

// Core of hyb_hybrid_batch_u8 on one device (arguments validated).
int batch_single(hyb_ctx* ctx, const uint8_t* g, size_t pitch, size_t slice_stride, int n_slices, int rows, int cols,
                 int smax, int win, uint8_t* y, size_t y_pitch, size_t y_slice_stride, int64_t* noise_sums) {
    int st;
    HYB_CHECK(cudaSetDevice(ctx->device));
    const bool dg = is_device_ptr(g) && hyb::tma_compatible(g, pitch, slice_stride), dy = is_device_ptr(y);
    const size_t pp = round_pitch(cols), ps = pp * rows;
    if (!dg && !dy && !is_device_ptr(g)) {
        HYB_CHECK(ctx->in.ensure(ps * n_slices));
        HYB_CHECK(ctx->out.ensure(ps * n_slices));
        HYB_CHECK(ctx->f.ensure(ps * n_slices));
        HYB_CHECK(ctx->wsum.ensure(sizeof(long long) * n_slices));
        unsigned long long* W = reinterpret_cast<unsigned long long*>(ctx->wsum.ptr);
        if (batch_host_pipelined(ctx, g, pitch, slice_stride, n_slices, rows, cols, smax, win, y, y_pitch,
                                 y_slice_stride, W, &st)) {
            if (st) return st;
            if (noise_sums) {
                if ((st = ensure_host_w(ctx, n_slices))) return st;
                HYB_CHECK(cudaMemcpyAsync(ctx->host_w, W, sizeof(long long) * n_slices, cudaMemcpyDeviceToHost,
                                          ctx->stream));
            }
            HYB_CHECK(cudaStreamSynchronize(ctx->stream));
            if (noise_sums)
                for (int z = 0; z < n_slices; ++z) noise_sums[z] = ctx->host_w[z];
            return HYB_OK;
        }
    }
    const uint8_t* s = g;
    size_t sp = pitch, ss = slice_stride;
    if (!dg) {
        HYB_CHECK(ctx->in.ensure(ps * n_slices));
        if (slice_stride == pitch * rows) {
            HYB_CHECK(copy2d(ctx, ctx->in.ptr, pp, g, pitch, cols, rows * n_slices));
        } else {
            for (int z = 0; z < n_slices; ++z)
                HYB_CHECK(copy2d(ctx, ctx->in.ptr + ps * z, pp, g + slice_stride * z, pitch, cols, rows));
        }
        s = ctx->in.ptr;
        sp = pp;
        ss = ps;
    }
    uint8_t* d = y;
    size_t dp = y_pitch, ds = y_slice_stride;
    if (!dy) {
        HYB_CHECK(ctx->out.ensure(ps * n_slices));
        d = ctx->out.ptr;
        dp = pp;
        ds = ps;
    }
    HYB_CHECK(ctx->f.ensure(ps * n_slices));
    HYB_CHECK(ctx->wsum.ensure(sizeof(long long) * n_slices));
    unsigned long long* W = reinterpret_cast<unsigned long long*>(ctx->wsum.ptr);
    hyb::Plane a{s, sp, ss, ctx->f.ptr, pp, ps, rows, cols, 0, rows, n_slices};
    HYB_CHECK(cudaMemsetAsync(W, 0, sizeof(long long) * n_slices, ctx->stream));
    HYB_CHECK(run_amf(ctx, a, smax, nullptr, 0, 0));
    hyb::Plane w{ctx->f.ptr, pp, ps, d, dp, ds, rows, cols, 0, rows, n_slices};
    HYB_CHECK(hyb::launch_wiener_stats(w, win, W, ctx->stream));
    HYB_CHECK(hyb::launch_wiener_gain(w, win, reinterpret_cast<const long long*>(W), (long long)rows * cols,
                                      ctx->stream));
    if (!dy) {
        if (y_slice_stride == y_pitch * rows) {
            HYB_CHECK(copy2d(ctx, y, y_pitch, d, dp, cols, rows * n_slices));
        } else {
            for (int z = 0; z < n_slices; ++z)
                HYB_CHECK(copy2d(ctx, y + y_slice_stride * z, y_pitch, d + ds * z, dp, cols, rows));
        }
    }
    if (noise_sums) {
        if ((st = ensure_host_w(ctx, n_slices))) return st;
        HYB_CHECK(cudaMemcpyAsync(ctx->host_w, W, sizeof(long long) * n_slices, cudaMemcpyDeviceToHost,
                                  ctx->stream));
    }
    if (!dg || !dy || noise_sums) HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    if (noise_sums)
        for (int z = 0; z < n_slices; ++z) noise_sums[z] = ctx->host_w[z];
    return HYB_OK;
}

// Multi-device CT stack (hyb_create_multi): slices sharded by contiguous chunks, one chunk per device,
// each an independent batch on its own device (no cross-slice reduction: every slice has its own noise
// sum).  One host thread per device enqueues (and, for host buffers, pipelines) its
// chunk; chunks whose input / output live on another device move through NVLink peer copies.
int batch_multi(hyb_ctx* ctx, const uint8_t* g, size_t pitch, size_t slice_stride, int n_slices, int rows, int cols,
                int smax, int win, uint8_t* y, size_t y_pitch, size_t y_slice_stride, int64_t* noise_sums) {
    const int n = 1 + (int)ctx->peers.size();
    std::vector<hyb_ctx*> sub(n);
    sub[0] = ctx;
    for (int i = 1; i < n; ++i) sub[i] = ctx->peers[i - 1];
    const int gdev = ptr_device(g), ydev = ptr_device(y);
    HYB_CHECK(cudaSetDevice(ctx->device));
    HYB_CHECK(cudaEventRecord(ctx->ev_start, ctx->stream));
    std::vector<int64_t> ws(noise_sums ? n_slices : 0);
    std::vector<int> status(n, HYB_OK);
    std::vector<std::string> errs(n);
    const size_t pp = round_pitch(cols), ps = pp * rows;
    auto work = [&](int i) {
        hyb_ctx* c = sub[i];
        const int z0 = (int)((long long)n_slices * i / n), z1 = (int)((long long)n_slices * (i + 1) / n), nz = z1 - z0;
        CtxScope scope(c);
        auto run = [&]() -> int {
            if (cudaSetDevice(c->device) != cudaSuccess) return cuda_fail(c, cudaGetLastError(), "cudaSetDevice");
            if (i) HYB_CHECK_C(c, cudaStreamWaitEvent(c->stream, ctx->ev_start, 0));
            if (nz > 0) {
                const uint8_t* gi = g + slice_stride * z0;
                size_t gp = pitch, gs = slice_stride;
                uint8_t* yi = y + y_slice_stride * z0;
                size_t yp = y_pitch, ys = y_slice_stride;
                const bool remote_g = gdev >= 0 && gdev != c->device, remote_y = ydev >= 0 && ydev != c->device;
                if (remote_g) {  // peer copy of the chunk into this device
                    HYB_CHECK_C(c, c->mg_in.ensure(ps * nz));
                    for (int z = 0; z < nz; ++z)
                        HYB_CHECK_C(c, copy2d(c, c->mg_in.ptr + ps * z, pp, gi + slice_stride * z, pitch, cols, rows));
                    gi = c->mg_in.ptr;
                    gp = pp;
                    gs = ps;
                }
                if (remote_y) {
                    HYB_CHECK_C(c, c->mg_out.ensure(ps * nz));
                    yi = c->mg_out.ptr;
                    yp = pp;
                    ys = ps;
                }
                int st = batch_single(c, gi, gp, gs, nz, rows, cols, smax, win, yi, yp, ys,
                                      noise_sums ? ws.data() + z0 : nullptr);
                if (st) return st;
                if (remote_y)
                    for (int z = 0; z < nz; ++z)
                        HYB_CHECK_C(c, copy2d(c, y + y_slice_stride * (z0 + z), y_pitch, yi + ys * z, yp, cols, rows));
            }
            HYB_CHECK_C(c, cudaEventRecord(c->ev_done, c->stream));
            return HYB_OK;
        };
        status[i] = run();
        if (status[i]) errs[i] = c->err;
    };
    std::vector<std::thread> pool;
    for (int i = 1; i < n; ++i) pool.emplace_back(work, i);
    work(0);
    for (auto& t : pool) t.join();
    for (int i = 0; i < n; ++i)  // the first error, like the reference's band pool (proj/src/parallel.cpp:67)
        if (status[i]) return fail(ctx, status[i], errs[i]);
    HYB_CHECK(cudaSetDevice(ctx->device));
    for (int i = 1; i < n; ++i) HYB_CHECK(cudaStreamWaitEvent(ctx->stream, sub[i]->ev_done, 0));
    if (gdev < 0 || ydev < 0 || noise_sums) HYB_CHECK(cudaStreamSynchronize(ctx->stream));
    if (noise_sums)
        for (int z = 0; z < n_slices; ++z) noise_sums[z] = ws[z];
    return HYB_OK;
}

}  // namespace

extern "C" {

int hyb_hybrid_batch_u8(hyb_ctx* ctx, const uint8_t* g, size_t pitch, size_t slice_stride,
                        int n_slices, int rows, int cols, int smax, int win, uint8_t* y,
                        size_t y_pitch, size_t y_slice_stride, int64_t* noise_sums) {
    if (!ctx) return HYB_EINVAL;
    CtxScope scope_(ctx);
    int st;
    if ((st = check_smax(ctx, smax)) || (st = check_win(ctx, win)) || (st = check_dims(ctx, rows, cols)) ||
        (st = check_pitch(ctx, pitch, cols, "g")) || (st = check_pitch(ctx, y_pitch, cols, "y")))
        return st;
    if (n_slices < 1) return fail(ctx, HYB_EINVAL, "n_slices must be >= 1, got " + std::to_string(n_slices));
    if (!g || !y) return fail(ctx, HYB_EINVAL, "null image pointer");
    if (slice_stride < pitch * rows || y_slice_stride < y_pitch * rows)
        return fail(ctx, HYB_EINVAL, "slice stride smaller than one slice");
    if (!ctx->peers.empty())
        return batch_multi(ctx, g, pitch, slice_stride, n_slices, rows, cols, smax, win, y, y_pitch, y_slice_stride,
                           noise_sums);
    return batch_single(ctx, g, pitch, slice_stride, n_slices, rows, cols, smax, win, y, y_pitch, y_slice_stride,
                        noise_sums);
}

}  // extern "C"
