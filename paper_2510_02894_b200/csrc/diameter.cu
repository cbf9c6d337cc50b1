// Diameter stage of the shape-coefficient path (sm_100a).
//
// Replaces reference _diameters_sq_seq / _diameters_sq_par
// (pkg/src/shapecore/features.py:121-192): the maximum over all vertex pairs
// of the squared distance, and the maxima over pairs sharing z (XY), y (XZ)
// and x (YZ) bit for bit (features.py:145-147).
//
// Every kernel here is device-driven: the vertex count, bounding box and plane
// layout are read from the Stats the marching-cubes stage wrote, so a whole
// ROI is enqueued without a host round trip (and can be graph-captured).
//
//  * diam3d_pass1   -- the O(V^2) hot loop over the surviving chunk pairs
//    listed by unit_filter (prune.cu).  A warp evaluates one 128 x 128 unit:
//    the J chunk is staged in the warp's shared memory as (x, y, z, |p|^2),
//    each lane register-blocks 4 i vertices, so a pair costs 1.5 FFMA2 plus
//    half an FMNMX3 on the fp32 CUDA cores (dot form |pj|^2 - 2 pi.pj in a
//    bbox-centred frame).  One maximum per unit is kept.
//  * diam3d_refine  -- exactness: every unit whose pass-1 maximum lies within
//    kRefineRel of the pass-1 maximum is re-evaluated in fp64 with the
//    reference's own arithmetic on the reference's own coordinates, so the 3-D
//    diameter is the reference's value bit for bit.  Units below the threshold
//    provably cannot hold the maximum (pass-1 error < ~1e-6 of D^2).
//    The planar pass (planar.cu) has the same two steps per plane family.
//  * cloud_diameters -- the generic diameters(xs, ys, zs) API on arbitrary
//    fp64 points with the reference's in-loop bit-equality tests.
#include "sc_device.cuh"

namespace sc {

constexpr int kDiamThreads = 256;
constexpr int kWarps = kDiamThreads / 32;
constexpr int kChunk = kChunk3;                // vertices per chunk (pair unit = chunk x chunk)
constexpr int kR = kChunk / 32;                // 4 i vertices per lane

// Pass 1 (see header).  Work unit = one surviving chunk pair (I <= J, 256 x
// 256 vertex pairs, listed by unit_filter); every WARP is an independent
// worker with its own shared-memory copy of the J chunk, so load balance is
// per unit and no block barrier is involved.  Error of the dot form: in the
// bbox-centred frame |p| <= D*sqrt(3)/2, so the absolute error is
// < ~12 * 2^-24 * D^2.
//
// PACKED: two i vertices share one FFMA2 (the j coordinate is the broadcast
// scalar operand), so 4 pairs cost 6 FFMA2 + 2 FMNMX3 = 2 issue slots per
// pair instead of 3.5 for scalar FFMA.
template <bool PACKED>
__global__ void __launch_bounds__(kDiamThreads, 4) diam3d_pass1(const int4* __restrict__ keys,
                                                                long long cap, const RoiParams* __restrict__ rp,
                                                                const uint2* __restrict__ work,
                                                                float* __restrict__ umax,
                                                                Stats* __restrict__ st) {
  // Re-run pending: too many vertices (scan_all) or surviving units (unit_filter).
  if (st->ovf || (long long)st->n_work > rp->wcap) return;
  Frame f = rp->f;
  __shared__ float4 sj_all[kWarps][kChunk];  // (x, y, z, |p|^2) per warp
  const long long n = n_vertices(st, cap);
  if (n == 0) return;
  frame_centre(st, f);
  const long long n_work = (long long)st->n_work;
  long long w0, w1;
  w0 = 0;
  w1 = n_work;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* sj = sj_all[warp];
  // Each warp takes a contiguous run of units, so consecutive units usually
  // share the I chunk (always, without pruning) and its registers are reused.
  const long long gwarps = (long long)gridDim.x * kWarps;
  const long long gw = (long long)blockIdx.x * kWarps + warp;
  const long long per = (w1 - w0 + gwarps - 1) / gwarps;
  const long long wb = w0 + gw * per, we = min(w1, wb + per);
  float run = 0.f;
  int prevI = -1;
  float a[kR], b[kR], c[kR], ni[kR];
  for (long long w = wb; w < we; w++) {
    const uint2 ij = work[w];
    const int I = (int)ij.x, J = (int)ij.y;
    float m[kR];
    __syncwarp();  // previous unit is done with sj
#pragma unroll
    for (int r = 0; r < kR; r++) {
      if (I != prevI) {
        const long long i = (long long)I * kChunk + r * 32 + lane;
        const float3 p = frame_coord(keys[i < n ? i : n - 1], f);
        a[r] = -2.f * p.x;
        b[r] = -2.f * p.y;
        c[r] = -2.f * p.z;
        ni[r] = fmaf(p.x, p.x, fmaf(p.y, p.y, p.z * p.z));
      }
      m[r] = -3.0e38f;
      long long j = (long long)J * kChunk + r * 32 + lane;
      if (j >= n) j = n - 1;  // repeats of a real vertex are harmless for a max
      const float3 q = frame_coord(keys[j], f);
      sj[r * 32 + lane] = make_float4(q.x, q.y, q.z, fmaf(q.x, q.x, fmaf(q.y, q.y, q.z * q.z)));
    }
    prevI = I;
    __syncwarp();
    if (PACKED) {
      float2 a2[kR / 2], b2[kR / 2], c2[kR / 2];
#pragma unroll
      for (int r = 0; r < kR / 2; r++) {
        a2[r] = make_float2(a[2 * r], a[2 * r + 1]);
        b2[r] = make_float2(b[2 * r], b[2 * r + 1]);
        c2[r] = make_float2(c[2 * r], c[2 * r + 1]);
      }
#pragma unroll 2
      for (int j = 0; j < kChunk; j += 2) {
        const float4 q0 = sj[j], q1 = sj[j + 1];
#pragma unroll
        for (int r = 0; r < kR / 2; r++) {
          float2 t0 = __ffma2_rn(a2[r], make_float2(q0.x, q0.x), make_float2(q0.w, q0.w));
          float2 t1 = __ffma2_rn(a2[r], make_float2(q1.x, q1.x), make_float2(q1.w, q1.w));
          t0 = __ffma2_rn(b2[r], make_float2(q0.y, q0.y), t0);
          t1 = __ffma2_rn(b2[r], make_float2(q1.y, q1.y), t1);
          t0 = __ffma2_rn(c2[r], make_float2(q0.z, q0.z), t0);
          t1 = __ffma2_rn(c2[r], make_float2(q1.z, q1.z), t1);
          m[2 * r] = fmax3f(m[2 * r], t0.x, t1.x);
          m[2 * r + 1] = fmax3f(m[2 * r + 1], t0.y, t1.y);
        }
      }
    } else {
#pragma unroll 2
      for (int j = 0; j < kChunk; j += 2) {
        const float4 q0 = sj[j], q1 = sj[j + 1];
#pragma unroll
        for (int r = 0; r < kR; r++) {
          float t0 = fmaf(q0.x, a[r], q0.w);
          float t1 = fmaf(q1.x, a[r], q1.w);
          t0 = fmaf(q0.y, b[r], t0);
          t1 = fmaf(q1.y, b[r], t1);
          t0 = fmaf(q0.z, c[r], t0);
          t1 = fmaf(q1.z, c[r], t1);
          m[r] = fmax3f(m[r], t0, t1);
        }
      }
    }
    float best = 0.f;
#pragma unroll
    for (int r = 0; r < kR; r++) best = fmaxf(best, m[r] + ni[r]);
#pragma unroll
    for (int o = 16; o; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) umax[w] = best;
    run = fmaxf(run, best);
  }
  if (lane == 0) atomic_max_pos_f32(&st->d3_f32, run);
}
template __global__ void diam3d_pass1<true>(const int4*, long long, const RoiParams*,
                                            const uint2*, float*, Stats*);
template __global__ void diam3d_pass1<false>(const int4*, long long, const RoiParams*,
                                             const uint2*, float*, Stats*);

// Exact re-check.  Every block sweeps 256 work entries at a time: the units
// whose pass-1 maximum lies within kRefineRel of the (now complete) pass-1
// maximum are listed in shared memory and each is re-evaluated, 128 x 128 in
// fp64 with the reference arithmetic on the reference coordinates (thread =
// one i vertex x half of the j chunk).  Selection is fully parallel: no
// serial scan of the unit maxima anywhere.
__global__ void __launch_bounds__(kDiamThreads) diam3d_refine(const int4* __restrict__ keys,
                                                              long long cap, const RoiParams* __restrict__ rp,
                                                              const uint2* __restrict__ work,
                                                              const float* __restrict__ umax,
                                                              Stats* __restrict__ st) {
  if (st->ovf || (long long)st->n_work > rp->wcap) return;  // re-run pending
  static_assert(kDiamThreads % kChunk == 0, "refine splits j across kDiamThreads / kChunk groups");
  constexpr int kSplit = kDiamThreads / kChunk, kJ = kChunk / kSplit;
  Frame f = rp->f;
  __shared__ double sx[kChunk], sy[kChunk], sz[kChunk];
  __shared__ unsigned int s_list[kDiamThreads];
  __shared__ int s_n;
  const long long n = n_vertices(st, cap);
  long long w0, w1;
  w0 = 0;
  w1 = (long long)st->n_work;
  const float tau = __uint_as_float(st->d3_f32) * (1.f - kRefineRel);
  const int ti = threadIdx.x % kChunk, tj = (threadIdx.x / kChunk) * kJ;
  double best = 0.0;
  // Block b sweeps entries w0 + b, w0 + b + G, ... (G = grid size), 256 at a
  // time, so candidates (adjacent in the work list) spread over the blocks.
  const long long G = gridDim.x;
  for (long long sweep = 0; w0 + sweep * kDiamThreads * G < w1; sweep++) {
    __syncthreads();  // previous sweep is done with s_list / s_n
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const long long w = w0 + (sweep * kDiamThreads + threadIdx.x) * G + blockIdx.x;
    if (w < w1 && umax[w] >= tau) s_list[atomicAdd(&s_n, 1)] = (unsigned int)w;
    __syncthreads();
    const int cnt = s_n;
    if (threadIdx.x == 0 && cnt) atomicAdd(&st->n_cand, (unsigned long long)cnt);
    for (int q = 0; q < cnt; q++) {
      const uint2 ij = work[s_list[q]];
      const int I = (int)ij.x, J = (int)ij.y;
      __syncthreads();  // previous candidate is done with sx/sy/sz
      if (threadIdx.x < kChunk) {
        const long long j = (long long)J * kChunk + threadIdx.x;
        const int4 kj = keys[j < n ? j : n - 1];
        sx[threadIdx.x] = ref_coord(kj.x, f.sx);
        sy[threadIdx.x] = ref_coord(kj.y, f.sy);
        sz[threadIdx.x] = ref_coord(kj.z, f.sz);
      }
      __syncthreads();
      const long long i = (long long)I * kChunk + ti;
      if (i < n) {
        const int4 ki = keys[i];
        const double xi = ref_coord(ki.x, f.sx), yi = ref_coord(ki.y, f.sy), zi = ref_coord(ki.z, f.sz);
#pragma unroll 4
        for (int t = tj; t < tj + kJ; t++)
          best = fmax(best, ref_sq_dist(xi, yi, zi, sx[t], sy[t], sz[t]));
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best > 0.0) atomic_max_pos_f64(&st->sq[0], best);
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

}  // namespace sc
