// multi.cu -- the exchange step of the multi-device hybrid (one process, one strip per device;
// capi.cu hybrid_multi): the exact noise sum W of the whole image from the per-strip partial sums.
// Each device runs this reduction itself, reading the other devices' partials straight from their
// memory over NVLink when peer access is enabled (else from local copies), so every device applies
// the gain with the same W -- the single-process analogue of the one int64 all-reduce of
// partition.py.  Integer sums: the result is identical for every strip split.
#include "hyb_internal.cuh"

namespace hyb {
namespace {

__global__ void sum_partials_kernel(const Partials parts, long long* out) {
    if (threadIdx.x == 0) {
        long long s = 0;
        for (int i = 0; i < parts.n; ++i) s += *(volatile const long long*)parts.p[i];
        *out = s;
    }
}

__global__ void min_partials_kernel(const MmPartials parts, unsigned* out) {
    if (threadIdx.x < 2) {
        unsigned v = 0xFFFFFFFFu;
        for (int i = 0; i < parts.n; ++i) v = min(v, ((volatile const unsigned*)parts.p[i])[threadIdx.x]);
        out[threadIdx.x] = v;
    }
}

}  // namespace

// contrast_stretch over the strips: every device combines the per-strip ranges its gains folded
// (mm[0] = min, mm[1] = 255 - max) the same way, so every strip maps with the same global range.
cudaError_t launch_min_partials(const MmPartials& parts, unsigned* out, cudaStream_t stream) {
    min_partials_kernel<<<1, 32, 0, stream>>>(parts, out);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_sum_partials(const Partials& parts, long long* out, cudaStream_t stream) {
    sum_partials_kernel<<<1, 32, 0, stream>>>(parts, out);
    count_launch();
    return cudaGetLastError();
}

}  // namespace hyb
