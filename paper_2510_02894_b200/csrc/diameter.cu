// Generic diameters API and the FP32 peak probe (sm_100a).
//
//  * cloud_diameters -- diameters(xs, ys, zs) (reference features.py:195-221)
//    on arbitrary fp64 points with the reference's in-loop bit-equality tests.
//  * fp32_probe      -- FFMA / FFMA2 throughput probe (the measured FP32 peak
//    the pass-1 roofline is quoted against).
//
// The shape-coefficient diameter search itself lives in pass_bodies.cuh /
// passes.cu.
#include "sc_device.cuh"

namespace sc {

__global__ void empty_kernel() {}


// ---- generic fp64 cloud (diameters API) ------------------------------------
constexpr int kCloudTile = 256;

// Grid-stride over the 64-bit tile-pair index (T(T+1)/2 pairs of 256-point
// tiles): any n the ABI accepts is covered whatever the grid size.
__global__ void __launch_bounds__(kCloudTile) cloud_diameters(const double* __restrict__ xs,
                                                              const double* __restrict__ ys,
                                                              const double* __restrict__ zs,
                                                              long long n, long long T,
                                                              unsigned long long* __restrict__ out4) {
  __shared__ double sx[kCloudTile], sy[kCloudTile], sz[kCloudTile];
  double m3 = 0.0, mxy = 0.0, mxz = 0.0, myz = 0.0;
  const long long units = T * (T + 1) / 2;
  for (long long u = blockIdx.x; u < units; u += gridDim.x) {
    int I, J;
    tile_pair(u, T, I, J);
    const long long i = (long long)I * kCloudTile + threadIdx.x;
    const long long j = (long long)J * kCloudTile + threadIdx.x;
    const long long jc = j < n ? j : n - 1;
    __syncthreads();  // previous unit's tile fully read
    sx[threadIdx.x] = xs[jc]; sy[threadIdx.x] = ys[jc]; sz[threadIdx.x] = zs[jc];
    __syncthreads();
    if (i < n) {
      const double xi = xs[i], yi = ys[i], zi = zs[i];
      const int jn = (int)min((long long)kCloudTile, n - (long long)J * kCloudTile);
      for (int t = 0; t < jn; t++) {
        const double d = ref_sq_dist(xi, yi, zi, sx[t], sy[t], sz[t]);
        m3 = fmax(m3, d);
        if (sz[t] == zi) mxy = fmax(mxy, d);
        if (sy[t] == yi) mxz = fmax(mxz, d);
        if (sx[t] == xi) myz = fmax(myz, d);
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    m3 = fmax(m3, __shfl_xor_sync(0xffffffffu, m3, o));
    mxy = fmax(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
    mxz = fmax(mxz, __shfl_xor_sync(0xffffffffu, mxz, o));
    myz = fmax(myz, __shfl_xor_sync(0xffffffffu, myz, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomic_max_pos_f64(&out4[0], m3);
    atomic_max_pos_f64(&out4[1], mxy);
    atomic_max_pos_f64(&out4[2], mxz);
    atomic_max_pos_f64(&out4[3], myz);
  }
}

// ---- FP32 CUDA-core throughput probe (the diameter roofline's denominator) --
// 16 independent chains per thread.  MODE 0: FFMA2 with all-register operands
// (as in diam3d_pass1); 1: FFMA, all registers; 2: FFMA2 with uniform
// operands; 3: FFMA with an immediate operand (the fastest scalar form).
template <int MODE>
__global__ void __launch_bounds__(256) fp32_probe(float* out, int iters, float b, float c) {
  float r = 0.f;
  const float tb = (MODE == 0 || MODE == 1) ? b + threadIdx.x * 1e-9f : b;
  const float tc = (MODE == 0 || MODE == 1) ? c - threadIdx.x * 1e-9f : c;
  if (MODE == 0 || MODE == 2) {
    float2 acc[16];
#pragma unroll
    for (int k = 0; k < 16; k++) acc[k] = make_float2(threadIdx.x * 1e-3f + k, k * 0.5f);
    const float2 bb = make_float2(tb, tb), cc = make_float2(tc, -tc);
    for (int i = 0; i < iters; i++) {
#pragma unroll
      for (int k = 0; k < 16; k++) acc[k] = __ffma2_rn(acc[k], bb, cc);
    }
#pragma unroll
    for (int k = 0; k < 16; k++) r += acc[k].x + acc[k].y;
  } else {
    float acc[16];
#pragma unroll
    for (int k = 0; k < 16; k++) acc[k] = threadIdx.x * 1e-3f + k;
    for (int i = 0; i < iters; i++) {
#pragma unroll
      for (int k = 0; k < 16; k++) acc[k] = MODE == 3 ? fmaf(acc[k], 1.0001f, 0.5f) : fmaf(acc[k], tb, tc);
    }
#pragma unroll
    for (int k = 0; k < 16; k++) r += acc[k];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template __global__ void fp32_probe<0>(float*, int, float, float);
template __global__ void fp32_probe<1>(float*, int, float, float);
template __global__ void fp32_probe<2>(float*, int, float, float);
template __global__ void fp32_probe<3>(float*, int, float, float);

}  // namespace sc
