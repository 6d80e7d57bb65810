// zc_probe.cu -- can the kernels move their own PCIe traffic?  Times copy-engine H2D/D2H of one
// config-1 image against SM loads/stores on mapped pinned host memory (zero-copy), and checks
// whether a TMA tensor map may point at host memory.
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../../paper_2005_05371_b200/csrc/tma.cuh"
using namespace hyb;

__global__ void zc_read(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

__global__ void zc_tma(const __grid_constant__ CUtensorMap m, int bytes, uint8_t* out, int n) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    uint8_t* tile = smem + 1024;
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(bar, bytes);
        tma_load_3d(tile, &m, bar, 0, blockIdx.x * 32, 0);
    }
    mbar_wait(bar, 0);
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[(size_t)blockIdx.x * n + i] = tile[i];
}

static float ev_ms(cudaEvent_t a, cudaEvent_t b) { float m; cudaEventElapsedTime(&m, a, b); return m; }

int main() {
    const size_t bytes = 1600 * 1600;
    uint8_t *h_in, *h_out, *d_a, *d_b, *d_h_in, *d_h_out;
    cudaHostAlloc(&h_in, bytes, cudaHostAllocMapped);
    cudaHostAlloc(&h_out, bytes, cudaHostAllocMapped);
    cudaHostGetDevicePointer((void**)&d_h_in, h_in, 0);
    cudaHostGetDevicePointer((void**)&d_h_out, h_out, 0);
    printf("host ptr %p device view %p (same=%d)\n", h_in, d_h_in, h_in == d_h_in);
    cudaMalloc(&d_a, bytes);
    cudaMalloc(&d_b, bytes);
    for (size_t i = 0; i < bytes; ++i) h_in[i] = (uint8_t)(i * 7 + 3);
    cudaStream_t s, s2;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t e0, e1, e2, e3;
    cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2); cudaEventCreate(&e3);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t n16 = bytes / 16;
    auto rep = [&](const char* name, auto fn) {
        std::vector<float> v;
        for (int r = 0; r < 30; ++r) {
            cudaEventRecord(e0, s); fn(); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
            v.push_back(ev_ms(e0, e1) * 1e3f);
        }
        std::sort(v.begin(), v.end());
        printf("%-44s min %7.1f  med %7.1f  max %7.1f us   (%.1f GB/s at median)\n", name, v[0], v[15], v[29],
               bytes / (v[15] * 1e-6) / 1e9);
    };
    rep("memcpy H2D (copy engine)", [&] { cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s); });
    rep("memcpy D2H (copy engine)", [&] { cudaMemcpyAsync(h_out, d_a, bytes, cudaMemcpyDeviceToHost, s); });
    for (int per : {1, 2, 4, 8}) {
        for (int thr : {256, 512, 1024}) {
            char nm[96];
            snprintf(nm, sizeof nm, "SM read host -> dev  grid %dx%d thr %d", sms, per, thr);
            rep(nm, [&] { zc_read<<<sms * per, thr, 0, s>>>((const uint4*)d_h_in, (uint4*)d_a, n16); });
        }
    }
    for (int per : {1, 4}) {
        char nm[96];
        snprintf(nm, sizeof nm, "SM write dev -> host grid %dx%d", sms, per);
        rep(nm, [&] { zc_read<<<sms * per, 512, 0, s>>>((const uint4*)d_a, (uint4*)d_h_out, n16); });
    }
    rep("duplex: SM read + SM write (one kernel each)", [&] {
        cudaEventRecord(e2, s);
        cudaStreamWaitEvent(s2, e2, 0);
        zc_read<<<sms * 2, 512, 0, s>>>((const uint4*)d_h_in, (uint4*)d_a, n16);
        zc_read<<<sms * 2, 512, 0, s2>>>((const uint4*)d_b, (uint4*)d_h_out, n16);
        cudaEventRecord(e3, s2);
        cudaStreamWaitEvent(s, e3, 0);
    });
    rep("duplex: memcpy H2D + memcpy D2H", [&] {
        cudaEventRecord(e2, s);
        cudaStreamWaitEvent(s2, e2, 0);
        cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s2);
        cudaEventRecord(e3, s2);
        cudaStreamWaitEvent(s, e3, 0);
    });
    cudaMemset(d_a, 0, bytes);
    zc_read<<<sms * 2, 512, 0, s>>>((const uint4*)d_h_in, (uint4*)d_a, n16);
    cudaStreamSynchronize(s);
    std::vector<uint8_t> chk(bytes);
    cudaMemcpy(chk.data(), d_a, bytes, cudaMemcpyDeviceToHost);
    printf("zero-copy read correct: %d\n", (int)std::equal(chk.begin(), chk.end(), h_in));

    // TMA with a tensor map over the mapped host buffer
    extern cudaError_t make_tmap_u8(CUtensorMap*, const void*, int, int, int, size_t, size_t, int, int);
    CUtensorMap m;
    cudaError_t te = hyb::make_tmap_u8(&m, d_h_in, 1600, 1600, 1, 1600, 0, 128, 32);
    printf("tmap over host memory: %s\n", cudaGetErrorString(te));
    if (te == cudaSuccess) {
        cudaMemset(d_b, 0, bytes);
        zc_tma<<<50, 256, 1024 + 128 * 32, s>>>(m, 128 * 32, d_b, 128 * 32);
        cudaError_t e = cudaStreamSynchronize(s);
        printf("TMA from host memory: %s\n", cudaGetErrorString(e));
        if (e == cudaSuccess) {
            cudaMemcpy(chk.data(), d_b, 50 * 128 * 32, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int b = 0; b < 50; ++b)
                for (int r = 0; r < 32; ++r)
                    for (int c = 0; c < 128; ++c)
                        bad += chk[(size_t)b * 4096 + r * 128 + c] != h_in[(size_t)(b * 32 + r) * 1600 + c];
            printf("TMA from host memory mismatches: %d\n", bad);
            rep("TMA host tiles 50 CTAs x 128x32", [&] { zc_tma<<<50, 256, 1024 + 128 * 32, s>>>(m, 128 * 32, d_b, 128 * 32); });
        }
    }
    return 0;
}
