// Device-side mask loading: typed NPY payload -> uint8 0/1
// mask in C order (x fastest), on the GPU.
//
// Mirrors reference load_npy binarization (pkg/src/shapecore/volume.py:140-184):
// supported descrs |b1 |u1 <i2 <i4 <i8 <f4 <f8 (volume.py:34-42); Fortran-order
// payloads are transposed into the canonical order (volume.py:171-172); with a
// label, voxels equal to dtype(label) are foreground, otherwise any nonzero
// voxel is (volume.py:173-176).  The host parses the header and converts the
// label to the payload dtype exactly as numpy would.
//
// The host stages the payload's occupied slab in chunks of whole planes (C
// order: z slices of rows of x; Fortran order: x slices of rows of z), and one
// kernel per chunk binarizes it while the next chunk crosses PCIe:
//   binarize_c -- C order: elementwise, 16 output bytes per thread step.
//   binarize_f -- Fortran order: a 32 x 32 shared-memory tile transpose per
//                 (row y, z block, x block): reads coalesced along z (the
//                 payload's fastest axis), writes coalesced along x.
#include "sc_device.cuh"

namespace sc {

template <typename T>
__device__ __forceinline__ uint8_t occ(T v, int has_label, T label) {
  return has_label ? (uint8_t)(v == label) : (uint8_t)(v != (T)0);
}

template <typename T>
__global__ void __launch_bounds__(256) binarize_c(const T* __restrict__ src, long long n,
                                                  int has_label, T label,
                                                  uint8_t* __restrict__ dst) {
  // chunks start at arbitrary byte offsets: a scalar head up to the first
  // 16-byte boundary of dst, then 16 output bytes per thread step, then a tail
  const long long head = min(n, (long long)((16 - ((uintptr_t)dst & 15)) & 15));
  const long long n16 = (n - head) / 16;
  const T* s = src + head;
  uint4* d = reinterpret_cast<uint4*>(dst + head);
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n16;
       q += (long long)gridDim.x * blockDim.x) {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      uint32_t v = 0;
#pragma unroll
      for (int b = 0; b < 4; b++)
        v |= (uint32_t)occ<T>(s[16 * q + 4 * k + b], has_label, label) << (8 * b);
      w[k] = v;
    }
    d[q] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  if (blockIdx.x == 0) {
    for (long long i = threadIdx.x; i < head; i += blockDim.x)
      dst[i] = occ<T>(src[i], has_label, label);
    for (long long i = head + 16 * n16 + threadIdx.x; i < n; i += blockDim.x)
      dst[i] = occ<T>(src[i], has_label, label);
  }
}

// src: xs x-slices [x][y][z] (cy rows of nz elements each) of x in [xa, xa + xs)
// dst: the slab mask [z][y][x], rows of cx bytes; writes columns xa .. xa + xs.
template <typename T>
__global__ void __launch_bounds__(256) binarize_f(const T* __restrict__ src, int xs, int cy,
                                                  int nz, int cx, int xa, int has_label, T label,
                                                  uint8_t* __restrict__ dst) {
  __shared__ uint8_t tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int z0 = blockIdx.x * 32, x0 = blockIdx.y * 32;
  for (int y = blockIdx.z; y < cy; y += gridDim.z) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int x = x0 + ty + 8 * i, z = z0 + tx;
      uint8_t v = 0;
      if (x < xs && z < nz) v = occ<T>(src[((long long)x * cy + y) * nz + z], has_label, label);
      tile[ty + 8 * i][tx] = v;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int z = z0 + ty + 8 * i, x = x0 + tx;
      if (x < xs && z < nz) dst[((long long)z * cy + y) * cx + xa + x] = tile[tx][ty + 8 * i];
    }
    __syncthreads();
  }
}

template <typename T>
void launch_t(const void* src, int fortran, long long planes, long long rows, long long row_elems,
              int cx, int xa, int has_label, T label, uint8_t* dst, int grid, cudaStream_t s) {
  const T* p = static_cast<const T*>(src);
  if (!fortran) {
    binarize_c<T><<<grid, 256, 0, s>>>(p, planes * rows * row_elems, has_label, label, dst);
  } else {
    dim3 g((unsigned)((row_elems + 31) / 32), (unsigned)((planes + 31) / 32),
           (unsigned)std::min<long long>(rows, 1024));
    binarize_f<T><<<g, 256, 0, s>>>(p, (int)planes, (int)rows, (int)row_elems, cx, xa, has_label,
                                    label, dst);
  }
}

// One staged chunk of `planes` planes x `rows` rows x `row_elems` elements.
// C order: the chunk's mask bytes go to dst (contiguous, same order).
// Fortran: planes are x slices; dst is the whole slab mask [z][y][cx] and the
// chunk fills columns [xa, xa + planes).
// dtype codes: 0 |b1, 1 |u1, 2 <i2, 3 <i4, 4 <i8, 5 <f4, 6 <f8
int launch_binarize(const void* src, int dtype, int fortran, long long planes, long long rows,
                    long long row_elems, int cx, int xa, int has_label, long long label_i,
                    double label_f, uint8_t* dst, int grid, cudaStream_t s) {
  switch (dtype) {
    case 0:
    case 1:
      launch_t<uint8_t>(src, fortran, planes, rows, row_elems, cx, xa, has_label,
                        (uint8_t)label_i, dst, grid, s);
      break;
    case 2:
      launch_t<int16_t>(src, fortran, planes, rows, row_elems, cx, xa, has_label,
                        (int16_t)label_i, dst, grid, s);
      break;
    case 3:
      launch_t<int32_t>(src, fortran, planes, rows, row_elems, cx, xa, has_label,
                        (int32_t)label_i, dst, grid, s);
      break;
    case 4:
      launch_t<long long>(src, fortran, planes, rows, row_elems, cx, xa, has_label,
                          (long long)label_i, dst, grid, s);
      break;
    case 5:
      launch_t<float>(src, fortran, planes, rows, row_elems, cx, xa, has_label, (float)label_f,
                      dst, grid, s);
      break;
    case 6:
      launch_t<double>(src, fortran, planes, rows, row_elems, cx, xa, has_label, label_f, dst,
                       grid, s);
      break;
    default:
      return -1;
  }
  return 0;
}

}  // namespace sc
