// imad_probe.cu -- throughput of the integer forms a compare-exchange can be built from on sm_100a:
// VIMNMX.U16x2 (ALU), IMAD as an add with a register multiplier (constant memory, FMA pipe), IMAD with an
// immediate multiplier, and mixes (a CE as min + max, or as min + a + b - min on the FMA pipe).
// Prints warp-instructions per clock per SM (SASS checked with cuobjdump).
#include <cstdio>

constexpr int ITERS = 2048;
__constant__ unsigned kOne[2] = {1u, 0xFFFFFFFFu};

__device__ __forceinline__ unsigned mad_reg(unsigned a, unsigned b) {
    unsigned r;
    asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(kOne[0]), "r"(b));
    return r;
}
__device__ __forceinline__ unsigned mad_imm(unsigned a, unsigned b) {
    unsigned r;
    asm volatile("mad.lo.u32 %0, %1, 3, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

template <int MODE>
__global__ void probe(unsigned* out, unsigned seed) {
    unsigned u[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) u[i] = (seed * (threadIdx.x + 7 * i + 1)) & 0x00FF00FFu;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int a = s, b = (s + 1 + (it & 3)) & 7;
            if (MODE == 0) {  // 2 VIMNMX
                const unsigned lo = __vminu2(u[a], u[b]), hi = __vmaxu2(u[a], u[b]);
                u[a] = lo;
                u[(a + 4) & 7] = hi;
            } else if (MODE == 1) {  // 2 IMAD (register multiplier)
                u[a] = mad_reg(u[a], u[b]);
                u[(a + 4) & 7] = mad_reg(u[(a + 4) & 7], u[b]);
            } else if (MODE == 2) {  // 2 IMAD (immediate multiplier)
                u[a] = mad_imm(u[a], u[b]);
                u[(a + 4) & 7] = mad_imm(u[(a + 4) & 7], u[b]);
            } else if (MODE == 3) {  // CE as min + (a + b - min): 1 VIMNMX + 2 IMAD
                const unsigned s2 = mad_reg(u[a], u[b]);
                const unsigned lo = __vminu2(u[a], u[b]);
                u[a] = lo;
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(u[(a + 4) & 7]) : "r"(lo), "r"(kOne[1]), "r"(s2));
            } else if (MODE == 4) {  // 1 VIMNMX + 1 IMAD
                u[a] = __vminu2(u[a], u[b]);
                u[(a + 4) & 7] = mad_reg(u[(a + 4) & 7], u[b]);
            }
        }
    }
    unsigned acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= u[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
float run(unsigned* out, int blocks) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe<MODE><<<blocks, 256>>>(out, 3);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) probe<MODE><<<blocks, 256>>>(out, 5 + r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz
    const int blocks = sms * 8;
    unsigned* out;
    cudaMalloc(&out, (size_t)blocks * 256 * 4);
    const char* names[] = {"2 VIMNMX", "2 IMAD reg", "2 IMAD imm", "CE vimnmx+2imad", "VIMNMX+IMAD"};
    float t[5] = {run<0>(out, blocks), run<1>(out, blocks), run<2>(out, blocks), run<3>(out, blocks), run<4>(out, blocks)};
    const int per_iter[5] = {8, 8, 8, 12, 8};  // warp instructions per inner iteration (4 steps)
    for (int m = 0; m < 5; ++m) {
        const double winstr = (double)blocks * 8 * ITERS * per_iter[m];
        const double clk_s = t[m] * 1e-3 * clk * 1e3;
        printf("%-18s %8.3f ms  %.2f warp-instr/clk/SM\n", names[m], t[m], winstr / clk_s / sms);
    }
    return 0;
}
