// tma_probe.cu -- bisects the TMA / mbarrier helpers of tma.cuh on a real device.
// usage: tma_probe <variant>; prints OK or the CUDA error.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../paper_2005_05371_b200/csrc/tma.cuh"

using namespace hyb;

__global__ void probe(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, int variant,
                      unsigned* flag, const CUtensorMap* gdesc, const __grid_constant__ CUtensorMap t2d) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    uint8_t* tile = smem + 128;
    if (threadIdx.x == 0) {
        if (variant & 1) prefetch_tmap(&tin);
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (variant & 8) {  // mbarrier only: arrive with zero tx, then wait
        if (threadIdx.x == 0) mbar_expect_tx(bar, 0);
        mbar_wait(bar, 0);
    }
    if (variant & 16) {  // arrive only, no wait
        if (threadIdx.x == 0) mbar_expect_tx(bar, 0);
    }
    if (variant & 32) {  // TMA issue only (coords 0,0), no wait
        if (threadIdx.x == 0) {
            mbar_expect_tx(bar, 64 * 32);
            tma_load_3d(tile, &tin, bar, 0, 0, 0);
        }
    }
    if (variant & 64) {  // TMA 2-D form, positive coords, then wait
        if (threadIdx.x == 0) {
            mbar_expect_tx(bar, 64 * 32);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                ::"r"(smem_u32(tile)), "l"(&tin), "r"(smem_u32(bar)), "r"(0), "r"(0) : "memory");
        }
        mbar_wait(bar, 0);
    }
    if (variant & 256) {  // 2-D map encoded by libcuda directly, CUTLASS-style 2-D instruction
        const int cx = (variant & 2048) ? -3 : ((variant & 8192) ? 50 : 0), cy = (variant & 2048) ? -2 : ((variant & 8192) ? 20 : 0);
        if (threadIdx.x == 0) {
            mbar_expect_tx(bar, 64 * 32);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                ::"r"(smem_u32(tile)), "l"(&t2d), "r"(smem_u32(bar)), "r"((variant & 16384) ? 8 : cx), "r"((variant & 16384) ? 4 : cy) : "memory");
        }
        mbar_wait(bar, 0);
    }
    if (variant >= 1024) {  // 3-D instruction forms: bit 1024 = .tile keyword, 2048 = negative coords
        const int cx = (variant & 2048) ? -3 : ((variant & 8192) ? 50 : ((variant & 16384) ? 8 : 0)), cy = (variant & 2048) ? -2 : ((variant & 8192) ? 20 : ((variant & 16384) ? 4 : 0));
        if (threadIdx.x == 0) {
            mbar_expect_tx(bar, 64 * 32);
            if (variant & 4096)
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                    ::"r"(smem_u32(tile)), "l"(&tin), "r"(smem_u32(bar)), "r"(cx), "r"(cy), "r"(0) : "memory");
            else
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                    ::"r"(smem_u32(tile)), "l"(&tin), "r"(smem_u32(bar)), "r"(cx), "r"(cy), "r"(0) : "memory");
        }
        mbar_wait(bar, 0);
    }
    if (variant & 128) {  // descriptor in global memory
        if (threadIdx.x == 0) {
            mbar_expect_tx(bar, 64 * 32);
            tma_load_3d(tile, gdesc, bar, (variant & 16384) ? 8 : 0, (variant & 16384) ? 4 : 0, 0);
        }
        mbar_wait(bar, 0);
    }
    if (variant & 2) {
        if (threadIdx.x == 0) {
            mbar_expect_tx(bar, 64 * 32);
            tma_load_3d(tile, &tin, bar, -3, -2, 0);
        }
        mbar_wait(bar, 0);
    }
    if (variant & 4) {
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            tma_store_3d(&tout, tile, (variant & 32768) ? 8 : 0, (variant & 32768) ? 4 : 0, 0);
            tma_store_commit();
            tma_store_wait_all();
        }
    }
    if (threadIdx.x == 0) *flag = 1234u;
}

int main(int argc, char** argv) {
    const int variant = argc > 1 ? atoi(argv[1]) : 7;
    const int rows = 40, cols = 100;
    const size_t pitch = 128;
    uint8_t *in, *out;
    unsigned* flag;
    cudaMalloc(&in, pitch * rows);
    cudaMalloc(&out, pitch * rows);
    cudaMalloc(&flag, 4);
    std::vector<uint8_t> h(pitch * rows);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (uint8_t)(i * 7);
    cudaMemcpy(in, h.data(), h.size(), cudaMemcpyHostToDevice);
    cudaMemset(out, 0, pitch * rows);
    CUtensorMap tin, tout;
    cudaError_t e1 = make_tmap_u8(&tin, in, cols, rows, 1, pitch, 0, 64, 32);
    cudaError_t e2 = make_tmap_u8(&tout, out, cols, rows, 1, pitch, 0, 64, 32);
    if (e1 || e2) {
        printf("encode failed %d %d\n", e1, e2);
        return 1;
    }
    CUtensorMap t2d;
    {
        const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
        const cuuint64_t str[1] = {pitch};
        const cuuint32_t box[2] = {64, 32}, es[2] = {1, 1};
        CUresult r = cuTensorMapEncodeTiled(&t2d, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, in, dims, str, box, es,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("direct encode 2d: %d\n", (int)r);
        CUtensorMap t3;
        const cuuint64_t d3[3] = {(cuuint64_t)cols, (cuuint64_t)rows, 1};
        const cuuint64_t s3[2] = {pitch, pitch * rows};
        const cuuint32_t b3[3] = {64, 32, 1}, e3[3] = {1, 1, 1};
        r = cuTensorMapEncodeTiled(&t3, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, in, d3, s3, b3, e3,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("direct encode 3d: %d same=%d\n", (int)r, memcmp(&t3, &tin, sizeof t3) == 0);
        const unsigned* a = (const unsigned*)&t3; const unsigned* b = (const unsigned*)&tin;
        for (int i = 0; i < 8; ++i) printf("%08x/%08x ", a[i], b[i]);
        printf("\n");
    }
    CUtensorMap* gdesc;
    cudaMalloc(&gdesc, sizeof(CUtensorMap));
    cudaMemcpy(gdesc, &tin, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    printf("sizeof %zu align %zu\n", sizeof(CUtensorMap), alignof(CUtensorMap));
    probe<<<1, 128, 128 + 64 * 32>>>(tin, tout, variant, flag, gdesc, t2d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned hf = 0;
    cudaMemcpy(&hf, flag, 4, cudaMemcpyDeviceToHost);
    std::vector<uint8_t> o(pitch * rows);
    cudaMemcpy(o.data(), out, o.size(), cudaMemcpyDeviceToHost);
    int bad = 0;
    if ((variant & 6) == 6)
        for (int r = 0; r < 32; ++r)
            for (int c = 0; c < 64; ++c) {
                const int sr = r - 2, sc = c - 3;
                const uint8_t want = (sr < 0 || sc < 0) ? 0 : h[sr * pitch + sc];
                bad += o[r * pitch + c] != want;
            }
    printf("variant %d: %s flag=%u bad=%d first=%d %d\n", variant, cudaGetErrorString(e), hf, bad, (int)o[0], (int)o[1]);
    return e != cudaSuccess;
}
