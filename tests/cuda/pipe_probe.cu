// pipe_probe.cu -- which pipe executes the min/max forms a compare-exchange network can use on
// sm_100a: VIMNMX.U16x2 (__vminu2), HMNMX2 (__hmin2 on half2), FMNMX (fminf), and mixes.
// Prints warp-instructions per clock per SM for each form (two independent pipes => a 50/50 mix
// runs ~2x the single-form rate).
#include <cuda_fp16.h>
#include <cstdio>

constexpr int ITERS = 2048;

template <int MODE>
__global__ void probe(unsigned* out, unsigned seed) {
    unsigned u[8];
    __half2 h[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        u[i] = (seed * (threadIdx.x + 7 * i + 1)) & 0x00FF00FFu;
        h[i] = __halves2half2(__ushort2half_rn(u[i] & 0xFF), __ushort2half_rn(u[i] >> 16));
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int a = s, b = (s + 1 + (it & 3)) & 7;  // rotating partner
            if (MODE == 0 || (MODE == 2 && (s & 1) == 0)) {
                const unsigned lo = __vminu2(u[a], u[b]), hi = __vmaxu2(u[a], u[b]);
                u[a] = lo;
                u[(a + 4) & 7] = hi;
            } else {
                const __half2 lo = __hmin2(h[a], h[b]), hi = __hmax2(h[a], h[b]);
                h[a] = lo;
                h[(a + 4) & 7] = hi;
            }
        }
    }
    unsigned acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= u[i] ^ *reinterpret_cast<unsigned*>(&h[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
float run(unsigned* out, int blocks) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe<MODE><<<blocks, 256>>>(out, 3);
    cudaEventRecord(e0);
    probe<MODE><<<blocks, 256>>>(out, 5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8;
    unsigned* out;
    cudaMalloc(&out, blocks * 256 * 4);
    const double warp_ops = (double)blocks * 8 * ITERS * 4 * 2;  // warps * iters * CEs * 2 ops
    const char* names[3] = {"vimnmx.u16x2", "hmnmx2", "50/50 mix"};
    float t[3] = {run<0>(out, blocks), run<1>(out, blocks), run<2>(out, blocks)};
    for (int m = 0; m < 3; ++m)
        printf("%-14s %8.3f ms  %.2f warp-op/clk/SM\n", names[m], t[m],
               warp_ops / (t[m] * 1e-3) / (clk * 1e3) / sms);
    return 0;
}
