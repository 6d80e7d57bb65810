// hyb_internal.cuh -- shared declarations of libhybrid_cuda (kernels + launchers).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace hyb {

// Geometry of one filtering launch: `n_slices` images of rows x cols with byte
// pitches and slice strides.  Output row i corresponds to input row row_begin + i.
struct Plane {
    const uint8_t* src;
    size_t spitch;
    size_t sslice;
    uint8_t* dst;
    size_t dpitch;
    size_t dslice;
    int rows, cols;
    int row_begin, row_end;
    int n_slices;
};

// Device workspace of the AMF growth stage: the per-tile level-A failure bitmap written by the
// k = 3 kernel (amf_bitmap_bytes(p) bytes, 512 per 128 x 32 tile).
struct AmfWork {
    uint8_t* bitmap;
};
size_t amf_bitmap_bytes(const Plane& p);

// AMF launch (amf.cu): k = 3 tile kernel + one tile-wise growth kernel (k = 5..smax).  fin may be null.
cudaError_t launch_amf(const Plane& p, int smax, uint8_t* fin, size_t fpitch, size_t fslice,
                       const AmfWork& work, cudaStream_t stream);

// W1 statistics launch (wiener.cu): adds sum of V over the rows into noise_sum[slice].
cudaError_t launch_wiener_stats(const Plane& p, int win, unsigned long long* noise_sum,
                                cudaStream_t stream);
// W1 gain launch: noise_sum[slice] read on the device; pixel_count per slice.
cudaError_t launch_wiener_gain(const Plane& p, int win, const long long* noise_sum,
                               long long pixel_count, cudaStream_t stream);

// Kernel-launch counter (bench evidence), incremented by every launcher.
void count_launch();

}  // namespace hyb
