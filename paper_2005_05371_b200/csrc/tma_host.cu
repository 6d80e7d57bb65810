// tma_host.cu -- host-side tensor-map encoding (cuTensorMapEncodeTiled via the runtime's driver
// entry point, so the library needs no direct libcuda link).
#include <cuda.h>
#include <cuda_runtime.h>

#include "tma.cuh"

namespace hyb {
namespace {

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
    // resolved once (thread-safe static initialisation); the entry point is device independent
    static const EncodeTiled fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<EncodeTiled>(p);
        return (EncodeTiled) nullptr;
    }();
    return fn;
}

}  // namespace

cudaError_t make_tmap_u8(CUtensorMap* map, const void* base, int cols, int rows, int slices, size_t pitch,
                         size_t slice_stride, int box_w, int box_h) {
    EncodeTiled enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    if (slices <= 1) slice_stride = (pitch * (size_t)rows + 15) & ~(size_t)15;
    const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)(slices < 1 ? 1 : slices)};
    const cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)slice_stride};
    const cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace hyb
