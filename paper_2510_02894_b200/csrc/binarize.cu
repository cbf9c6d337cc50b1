// Device-side mask loading: typed NPY payload -> uint8 0/1
// mask in C order (x fastest), on the GPU.
//
// Mirrors reference load_npy binarization (pkg/src/shapecore/volume.py:140-184):
// supported descrs |b1 |u1 <i2 <i4 <i8 <f4 <f8 (volume.py:34-42); Fortran-order
// payloads are transposed into the canonical order (volume.py:171-172); with a
// label, voxels equal to dtype(label) are foreground, otherwise any nonzero
// voxel is (volume.py:173-176).  The host parses the header and converts the
// label to the payload dtype exactly as numpy would.
#include "sc_device.cuh"

namespace sc {

template <typename T>
__global__ void __launch_bounds__(256) binarize_kernel(const T* __restrict__ src, long long s0,
                                                       long long s1, long long s2, int fortran,
                                                       int has_label, T label,
                                                       uint8_t* __restrict__ dst) {
  const long long n = s0 * s1 * s2;
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < n;
       o += (long long)gridDim.x * blockDim.x) {
    long long si = o;
    if (fortran) {  // output (i, j, k) in C order <- input offset i + s0*(j + s1*k)
      const long long k = o % s2, ij = o / s2;
      const long long j = ij % s1, i = ij / s1;
      si = i + s0 * (j + s1 * k);
    }
    const T v = src[si];
    dst[o] = has_label ? (uint8_t)(v == label) : (uint8_t)(v != (T)0);
  }
}

// dtype codes: 0 |b1, 1 |u1, 2 <i2, 3 <i4, 4 <i8, 5 <f4, 6 <f8
int launch_binarize(const void* src, int dtype, const long long shape[3], int fortran,
                    int has_label, long long label_i, double label_f, uint8_t* dst, int grid,
                    cudaStream_t s) {
  const long long a = shape[0], b = shape[1], c = shape[2];
  switch (dtype) {
    case 0:
    case 1:
      binarize_kernel<uint8_t><<<grid, 256, 0, s>>>((const uint8_t*)src, a, b, c, fortran,
                                                     has_label, (uint8_t)label_i, dst);
      break;
    case 2:
      binarize_kernel<int16_t><<<grid, 256, 0, s>>>((const int16_t*)src, a, b, c, fortran,
                                                     has_label, (int16_t)label_i, dst);
      break;
    case 3:
      binarize_kernel<int32_t><<<grid, 256, 0, s>>>((const int32_t*)src, a, b, c, fortran,
                                                     has_label, (int32_t)label_i, dst);
      break;
    case 4:
      binarize_kernel<long long><<<grid, 256, 0, s>>>((const long long*)src, a, b, c, fortran,
                                                       has_label, (long long)label_i, dst);
      break;
    case 5:
      binarize_kernel<float><<<grid, 256, 0, s>>>((const float*)src, a, b, c, fortran, has_label,
                                                   (float)label_f, dst);
      break;
    case 6:
      binarize_kernel<double><<<grid, 256, 0, s>>>((const double*)src, a, b, c, fortran,
                                                    has_label, label_f, dst);
      break;
    default:
      return -1;
  }
  return 0;
}

}  // namespace sc
