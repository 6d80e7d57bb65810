// tma_probe2.cu -- which TMA coordinates / data types work on this stack.
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2005_05371_b200/csrc/tma.cuh"
using namespace hyb;

__global__ void k2(const __grid_constant__ CUtensorMap m, int x, int y, int bytes, unsigned* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    uint8_t* tile = smem + 1024;
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(bar, bytes);
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     ::"r"(smem_u32(tile)), "l"(&m), "r"(smem_u32(bar)), "r"(x), "r"(y) : "memory");
    }
    mbar_wait(bar, 0);
    if (threadIdx.x == 0) { out[0] = tile[0]; out[1] = tile[1]; out[2] = smem_u32(tile); }
}

int main(int argc, char** argv) {
    const int dt = atoi(argv[1]), bw = atoi(argv[2]), bh = atoi(argv[3]), x = atoi(argv[4]), y = atoi(argv[5]);
    const int esz = dt == 0 ? 1 : (dt == 1 ? 2 : 4);
    const int rows = 64, pitch = 512, cols = pitch / esz;
    uint8_t* in; unsigned* out;
    cudaMalloc(&in, pitch * rows); cudaMalloc(&out, 16);
    std::vector<uint8_t> h(pitch * rows);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (uint8_t)(i * 13 + 1);
    cudaMemcpy(in, h.data(), h.size(), cudaMemcpyHostToDevice);
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t str[1] = {(cuuint64_t)pitch};
    const cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh}, es[2] = {1, 1};
    CUtensorMapDataType t = dt == 0 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : (dt == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_UINT32);
    CUresult r = cuTensorMapEncodeTiled(&m, t, 2, in, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k2<<<1, 32, 1024 + bw * bh * esz>>>(m, x, y, bw * bh * esz, out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned ho[3] = {0, 0, 0};
    cudaMemcpy(ho, out, 12, cudaMemcpyDeviceToHost);
    const int want = h[(size_t)y * pitch + (size_t)x * esz];
    printf("dt=%d box=%dx%d at (%d,%d): enc=%d %s got=%u want=%d smem=%u\n", dt, bw, bh, x, y, (int)r,
           cudaGetErrorString(e), ho[0], want, ho[2]);
    return 0;
}
