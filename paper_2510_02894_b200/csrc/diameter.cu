// Diameter stage of the shape-coefficient path (sm_100a).
//
// Replaces reference _diameters_sq_seq / _diameters_sq_par
// (pkg/src/shapecore/features.py:121-192): the maximum over all vertex pairs
// of the squared distance, and the maxima over pairs sharing z (XY), y (XZ)
// and x (YZ) bit for bit (features.py:145-147).
//
//  * diam3d_pass1<R>  -- the O(V^2) hot loop.  Triangular grid of square tile
//    pairs (I <= J); the J tile is staged in shared memory as duplicated
//    (x,x,y,y),(z,z) so every pair-of-pairs is three FADD2 + FMUL2 + two FFMA2
//    on the packed fp32 pipe plus one 3-input FMNMX3.  Coordinates are fp32 in
//    a bbox-centred frame.  Each tile pair's maximum is kept (item_max) and the
//    global maximum is an integer atomicMax on the fp32 bit pattern.
//  * diam3d_refine    -- exactness: every tile pair whose pass-1 maximum lies
//    within kRefineRel of the global pass-1 maximum is re-evaluated in fp64
//    with the reference's own arithmetic on the reference's own coordinates,
//    so the final 3-D diameter is the reference's value bit for bit.  Tile
//    pairs below the threshold provably cannot hold the maximum (the pass-1
//    error is < 17 * 2^-24 relative).
//  * plane_*          -- keyed planar pass: counting-sort vertices by the
//    doubled lattice key of z / y / x (bit-equal fp64 coordinate <=> equal
//    key), then an fp64 reference-arithmetic pair max inside every plane.
//  * cloud_diameters  -- the generic diameters(xs, ys, zs) API on arbitrary
//    fp64 points with the reference's in-loop bit-equality tests.
#include "sc_device.cuh"

namespace sc {

constexpr int kDiamThreads = 256;

__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// Upper-triangle tile-pair index -> (I, J), I <= J, row-major over I.
__device__ __forceinline__ void tile_pair(long long t, int T, int& I, int& J) {
  // off(I) = I*T - I*(I-1)/2 ; solve off(I) <= t < off(I+1)
  double b = 2.0 * T + 1.0;
  int i = (int)((b - sqrt(b * b - 8.0 * (double)t)) * 0.5);
  if (i < 0) i = 0;
  if (i > T - 1) i = T - 1;
  auto off = [T](long long r) { return r * T - r * (r - 1) / 2; };
  while (i > 0 && off(i) > t) i--;
  while (i < T - 1 && off(i + 1) <= t) i++;
  I = i;
  J = (int)(i + (t - off(i)));
}

__device__ __forceinline__ float3 frame_coord(int4 k, const Frame& f) {
  return make_float3((float)(k.x - f.cx2) * f.hx, (float)(k.y - f.cy2) * f.hy,
                     (float)(k.z - f.cz2) * f.hz);
}

template <int R>
__global__ void __launch_bounds__(kDiamThreads) diam3d_pass1(const int4* __restrict__ keys,
                                                             long long n, int T, long long item0,
                                                             long long n_items, Frame f,
                                                             float* __restrict__ item_max,
                                                             Stats* __restrict__ st) {
  constexpr int TS = kDiamThreads * R;
  extern __shared__ float4 smem4[];
  float4* sA = smem4;                                    // (x, x, y, y)
  float2* sB = reinterpret_cast<float2*>(smem4 + TS);    // (z, z)
  const long long item = item0 + blockIdx.x;
  if (item >= item0 + n_items) return;
  int I, J;
  tile_pair(item, T, I, J);

  // Stage the J tile (indices past n repeat the last vertex: harmless for a max).
  for (int t = threadIdx.x; t < TS; t += kDiamThreads) {
    long long j = (long long)J * TS + t;
    if (j >= n) j = n - 1;
    float3 c = frame_coord(keys[j], f);
    sA[t] = make_float4(c.x, c.x, c.y, c.y);
    sB[t] = make_float2(c.z, c.z);
  }
  // Register-block R i vertices as R/2 packed pairs, negated for FADD2.
  float2 nx2[R / 2], ny2[R / 2], nz2[R / 2];
#pragma unroll
  for (int p = 0; p < R / 2; p++) {
    long long i0 = (long long)I * TS + (2 * p) * kDiamThreads + threadIdx.x;
    long long i1 = i0 + kDiamThreads;
    float3 a = frame_coord(keys[i0 < n ? i0 : n - 1], f);
    float3 b = frame_coord(keys[i1 < n ? i1 : n - 1], f);
    nx2[p] = make_float2(-a.x, -b.x);
    ny2[p] = make_float2(-a.y, -b.y);
    nz2[p] = make_float2(-a.z, -b.z);
  }
  __syncthreads();

  float m0 = 0.f, m1 = 0.f;
#pragma unroll 2
  for (int j = 0; j < TS; j++) {
    const float4 a = sA[j];
    const float2 zz = sB[j];
    const float2 xx = make_float2(a.x, a.y), yy = make_float2(a.z, a.w);
#pragma unroll
    for (int p = 0; p < R / 2; p++) {
      float2 dx = __fadd2_rn(xx, nx2[p]);
      float2 dy = __fadd2_rn(yy, ny2[p]);
      float2 dz = __fadd2_rn(zz, nz2[p]);
      float2 d = __fmul2_rn(dx, dx);
      d = __ffma2_rn(dy, dy, d);
      d = __ffma2_rn(dz, dz, d);
      if (p & 1) m1 = fmax3f(m1, d.x, d.y);
      else m0 = fmax3f(m0, d.x, d.y);
    }
  }
  float m = fmaxf(m0, m1);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float s_red[kDiamThreads / 32];
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kDiamThreads / 32; w++) m = fmaxf(m, s_red[w]);
    item_max[blockIdx.x] = m;
    atomic_max_pos_f32(&st->d3_f32, m);
  }
}

// Relative margin of the pass-1 re-check threshold.  The fp32 frame error is
// bounded by 17*2^-24 ~ 1.0e-6 of D^2; tile pairs whose pass-1
// maximum is below M*(1 - kRefineRel) cannot contain the exact maximum.
constexpr float kRefineRel = 8e-6f;

template <int R>
__global__ void __launch_bounds__(kDiamThreads) diam3d_refine(const int4* __restrict__ keys,
                                                              long long n, int T,
                                                              long long item0, long long n_items,
                                                              Frame f,
                                                              const float* __restrict__ item_max,
                                                              Stats* __restrict__ st) {
  constexpr int TS = kDiamThreads * R;
  const long long item = item0 + blockIdx.x;
  if (item >= item0 + n_items) return;
  const float tau = __uint_as_float(st->d3_f32) * (1.f - kRefineRel);
  if (item_max[blockIdx.x] < tau) return;
  int I, J;
  tile_pair(item, T, I, J);
  __shared__ double sx[kDiamThreads], sy[kDiamThreads], sz[kDiamThreads];
  double best = 0.0;
  for (int r = 0; r < R; r++) {
    long long i = (long long)I * TS + r * kDiamThreads + threadIdx.x;
    const bool iv = i < n;
    int4 ki = keys[iv ? i : n - 1];
    double xi = ref_coord(ki.x, f.sx), yi = ref_coord(ki.y, f.sy), zi = ref_coord(ki.z, f.sz);
    for (int c = 0; c < TS; c += kDiamThreads) {
      __syncthreads();
      long long j = (long long)J * TS + c + threadIdx.x;
      int4 kj = keys[j < n ? j : n - 1];
      sx[threadIdx.x] = ref_coord(kj.x, f.sx);
      sy[threadIdx.x] = ref_coord(kj.y, f.sy);
      sz[threadIdx.x] = ref_coord(kj.z, f.sz);
      __syncthreads();
      if (iv)
        for (int t = 0; t < kDiamThreads; t++)
          best = fmax(best, ref_sq_dist(xi, yi, zi, sx[t], sy[t], sz[t]));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) atomic_max_pos_f64(&st->sq[0], best);
  if (threadIdx.x == 0) atomicAdd(&st->n_refined, 1ull);
}

// ---- planar pass -----------------------------------------------------------
// Plane index space: [0, nZ) XY planes keyed by Z2, [nZ, nZ+nY) XZ by Y2,
// [nZ+nY, P) YZ by X2, where key ranges come from the occupied bbox.
__device__ __forceinline__ void plane_ids(int4 k, const PlaneSpace& ps, int out[3]) {
  out[0] = k.z - ps.lo[0];
  out[1] = ps.cnt[0] + (k.y - ps.lo[1]);
  out[2] = ps.cnt[0] + ps.cnt[1] + (k.x - ps.lo[2]);
}

__global__ void plane_hist(const int4* __restrict__ keys, long long n, PlaneSpace ps,
                           unsigned int* __restrict__ counts) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    int id[3];
    plane_ids(keys[v], ps, id);
    atomicAdd(&counts[id[0]], 1u);
    atomicAdd(&counts[id[1]], 1u);
    atomicAdd(&counts[id[2]], 1u);
  }
}

// Exclusive scan of P counts (P <= a few 10^4) in one block of 1024 threads.
__global__ void __launch_bounds__(1024) plane_scan(const unsigned int* __restrict__ counts, int P,
                                                   unsigned int* __restrict__ start,
                                                   unsigned int* __restrict__ cursor) {
  __shared__ unsigned int s[1024];
  __shared__ unsigned int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < P; base += 1024) {
    int i = base + threadIdx.x;
    unsigned int v = i < P ? counts[i] : 0u;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      unsigned int t = threadIdx.x >= o ? s[threadIdx.x - o] : 0u;
      __syncthreads();
      s[threadIdx.x] += t;
      __syncthreads();
    }
    unsigned int excl = carry + s[threadIdx.x] - v;
    if (i < P) { start[i] = excl; cursor[i] = excl; }
    __syncthreads();
    if (threadIdx.x == 1023) carry += s[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) start[P] = carry;
}

__global__ void plane_scatter(const int4* __restrict__ keys, long long n, PlaneSpace ps,
                              unsigned int* __restrict__ cursor, int2* __restrict__ sorted) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    int4 k = keys[v];
    int id[3];
    plane_ids(k, ps, id);
    sorted[atomicAdd(&cursor[id[0]], 1u)] = make_int2(k.x, k.y);  // XY: (X, Y)
    sorted[atomicAdd(&cursor[id[1]], 1u)] = make_int2(k.x, k.z);  // XZ: (X, Z)
    sorted[atomicAdd(&cursor[id[2]], 1u)] = make_int2(k.y, k.z);  // YZ: (Y, Z)
  }
}

constexpr int kPlaneChunk = 2048;

// One block per plane (grid-strided over planes [p0, p1)): exact fp64 max over
// the plane's vertex pairs with the reference formula (the out-of-plane delta
// is exactly 0, so dx*dx + dy*dy + 0 == the reference's 3-term sum).
__global__ void __launch_bounds__(256) plane_pairs(const int2* __restrict__ sorted,
                                                   const unsigned int* __restrict__ start,
                                                   int p0, int p1, PlaneSpace ps, Frame f,
                                                   Stats* __restrict__ st) {
  __shared__ double sa[kPlaneChunk], sb[kPlaneChunk];
  __shared__ double s_red[8];
  for (int p = p0 + blockIdx.x; p < p1; p += gridDim.x) {
    const int axis = p < ps.cnt[0] ? 0 : (p < ps.cnt[0] + ps.cnt[1] ? 1 : 2);
    const unsigned int b = start[p], e = start[p + 1];
    const int np = (int)(e - b);
    if (np < 2) continue;  // block-uniform
    const double s_a = axis == 2 ? f.sy : f.sx;
    const double s_b = axis == 0 ? f.sy : f.sz;
    double best = 0.0;
    for (int c0 = 0; c0 < np; c0 += kPlaneChunk) {
      const int c1 = min(np, c0 + kPlaneChunk);
      __syncthreads();
      for (int t = c0 + threadIdx.x; t < c1; t += blockDim.x) {
        int2 k = sorted[b + t];
        sa[t - c0] = ref_coord(k.x, s_a);
        sb[t - c0] = ref_coord(k.y, s_b);
      }
      __syncthreads();
      for (int i = threadIdx.x; i < c1 - 1; i += blockDim.x) {
        int2 k = sorted[b + i];
        const double ai = ref_coord(k.x, s_a), bi = ref_coord(k.y, s_b);
        for (int j = max(i + 1, c0); j < c1; j++) {
          double da = __dsub_rn(sa[j - c0], ai), db = __dsub_rn(sb[j - c0], bi);
          best = fmax(best, __dadd_rn(__dmul_rn(da, da), __dmul_rn(db, db)));
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < (int)(blockDim.x >> 5); w++) best = fmax(best, s_red[w]);
      atomic_max_pos_f64(&st->sq[1 + axis], best);
    }
    __syncthreads();
  }
}

// ---- generic fp64 cloud (diameters API) ------------------------------------
constexpr int kCloudTile = 256;

__global__ void __launch_bounds__(kCloudTile) cloud_diameters(const double* __restrict__ xs,
                                                              const double* __restrict__ ys,
                                                              const double* __restrict__ zs,
                                                              long long n, int T,
                                                              unsigned long long* __restrict__ out4) {
  __shared__ double sx[kCloudTile], sy[kCloudTile], sz[kCloudTile];
  int I, J;
  tile_pair(blockIdx.x, T, I, J);
  long long i = (long long)I * kCloudTile + threadIdx.x;
  long long j = (long long)J * kCloudTile + threadIdx.x;
  long long jc = j < n ? j : n - 1;
  sx[threadIdx.x] = xs[jc]; sy[threadIdx.x] = ys[jc]; sz[threadIdx.x] = zs[jc];
  __syncthreads();
  double m3 = 0.0, mxy = 0.0, mxz = 0.0, myz = 0.0;
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

// Explicit instantiations used by the engine.
template __global__ void diam3d_pass1<2>(const int4*, long long, int, long long, long long, Frame,
                                         float*, Stats*);
template __global__ void diam3d_pass1<4>(const int4*, long long, int, long long, long long, Frame,
                                         float*, Stats*);
template __global__ void diam3d_pass1<8>(const int4*, long long, int, long long, long long, Frame,
                                         float*, Stats*);
template __global__ void diam3d_refine<2>(const int4*, long long, int, long long, long long, Frame,
                                          const float*, Stats*);
template __global__ void diam3d_refine<4>(const int4*, long long, int, long long, long long, Frame,
                                          const float*, Stats*);
template __global__ void diam3d_refine<8>(const int4*, long long, int, long long, long long, Frame,
                                          const float*, Stats*);

}  // namespace sc
