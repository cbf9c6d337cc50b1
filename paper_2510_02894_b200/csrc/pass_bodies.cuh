// Pass-1 and exact re-check bodies of the 3-D and planar diameter searches
// (sm_100a), fused into one pass-1 kernel and one re-check kernel by
// passes.cu.  Replaces reference _diameters_sq_seq / _diameters_sq_par
// (pkg/src/shapecore/features.py:121-192).
//
//  * pass1_3d     -- the O(V^2) hot loop over the surviving 3-D chunk pairs
//    listed by unit_filter (prune.cu).  A warp evaluates one 128 x 128 unit:
//    the J chunk is staged in the warp's shared memory as (x, y, z, |p|^2),
//    each lane register-blocks 4 i vertices, so a pair costs 1.5 FFMA2 plus
//    half an FMNMX3 on the fp32 CUDA cores (dot form |pj|^2 - 2 pi.pj in a
//    bbox-centred frame).  One maximum per unit is kept.
//  * pass1_planar -- the same over the surviving in-plane chunk pairs listed by
//    plane_filter (planar.cu), 2-D (1 FFMA2 + 0.5 FMNMX3 per pair).
//  * refine_3d / refine_planar -- exactness: every unit whose pass-1 maximum
//    reaches its family's threshold tau (refine_tau: an absolute margin of
//    96 u R^2 below the family's pass-1 maximum) is re-evaluated in
//    fp64 with the reference's own arithmetic on the reference's own
//    coordinates, so every diameter is the reference's value bit for bit.
//    Units below the threshold provably cannot hold the maximum (pass-1 error
//    <= 35 u R^2; sc_device.cuh refine_tau).
#pragma once
#include "sc_device.cuh"

namespace sc {

constexpr int kDiamThreads = 256;
constexpr int kWarps = kDiamThreads / 32;
constexpr int kChunk = kChunk3;  // vertices per 3-D chunk (pair unit = chunk x chunk)
constexpr int kR = kChunk / 32;  // 4 i vertices per lane
constexpr int kPlaneThreads = kDiamThreads;
constexpr int kPlaneWarps = kPlaneThreads / 32;
constexpr int kPC = kPlaneChunk;  // in-plane chunk edge (pair unit = chunk x chunk)
constexpr int kPR = kPC / 32;     // 4 i entries per lane
static_assert(kPC == kChunk, "the fused pass-1 kernel shares one smem chunk per warp");

// Pass 1 (see header).  Work unit = one surviving chunk pair (I <= J, 128 x
// 128 vertex pairs, listed by unit_filter / unit_expand with the mask of its
// 64 x 64 sub-pairs to evaluate); every WARP is an independent
// worker with its own shared-memory copy of the J chunk, so load balance is
// per unit and no block barrier is involved.  Error of the dot form: in the
// bbox-centred frame |p| <= D*sqrt(3)/2, so the absolute error is
// < ~12 * 2^-24 * D^2.
//
// PACKED: two i vertices share one FFMA2 (the j coordinate is the broadcast
// scalar operand), so 4 pairs cost 6 FFMA2 + 2 FMNMX3 = 2 issue slots per
// pair instead of 3.5 for scalar FFMA.
template <bool PACKED>
__device__ __forceinline__ void pass1_3d(const int4* __restrict__ keys, long long cap,
                                         const RoiParams* __restrict__ rp,
                                         const uint2* __restrict__ work, float* __restrict__ umax,
                                         Stats* __restrict__ st, float4* __restrict__ sj) {
  Frame f = rp->f;
  const long long n = n_vertices(st, cap);
  if (n == 0) return;
  frame_centre(st, f);
  const long long n_work = (long long)st->n_work;
  long long w0, w1;
  w0 = 0;
  w1 = n_work;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
    const int I = (int)ij.x, J = (int)(ij.y & kIdxMask);
    const unsigned int sub = ij.y >> kSubShift;  // 64 x 64 sub-pairs to evaluate
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
      if (sub == 0xFu) {
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
        // Only the listed 64 x 64 sub-pairs: i half a = packed pair a (i = a*64
        // + {0, 32} + lane), j half b.  a, b are compile-time in each body.
#pragma unroll
        for (int a = 0; a < 2; a++)
#pragma unroll
          for (int b = 0; b < 2; b++) {
            if (!(sub & (1u << (2 * a + b)))) continue;
#pragma unroll 2
            for (int j = 64 * b; j < 64 * b + 64; j += 2) {
              const float4 q0 = sj[j], q1 = sj[j + 1];
              float2 t0 = __ffma2_rn(a2[a], make_float2(q0.x, q0.x), make_float2(q0.w, q0.w));
              float2 t1 = __ffma2_rn(a2[a], make_float2(q1.x, q1.x), make_float2(q1.w, q1.w));
              t0 = __ffma2_rn(b2[a], make_float2(q0.y, q0.y), t0);
              t1 = __ffma2_rn(b2[a], make_float2(q1.y, q1.y), t1);
              t0 = __ffma2_rn(c2[a], make_float2(q0.z, q0.z), t0);
              t1 = __ffma2_rn(c2[a], make_float2(q1.z, q1.z), t1);
              m[2 * a] = fmax3f(m[2 * a], t0.x, t1.x);
              m[2 * a + 1] = fmax3f(m[2 * a + 1], t0.y, t1.y);
            }
          }
      }
    } else {
#pragma unroll
      for (int ha = 0; ha < 2; ha++)
#pragma unroll
        for (int hb = 0; hb < 2; hb++) {
          if (!(sub & (1u << (2 * ha + hb)))) continue;
#pragma unroll 2
          for (int j = 64 * hb; j < 64 * hb + 64; j += 2) {
            const float4 q0 = sj[j], q1 = sj[j + 1];
#pragma unroll
            for (int r = 2 * ha; r < 2 * ha + 2; r++) {
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

// Exact re-check.  Every block sweeps 256 work entries at a time: the units
// whose pass-1 maximum reaches refine_tau of the (now complete) pass-1
// maximum are listed in shared memory and each is re-evaluated, 128 x 128 in
// fp64 with the reference arithmetic on the reference coordinates (thread =
// one i vertex x half of the j chunk).  Selection is fully parallel: no
// serial scan of the unit maxima anywhere.
__device__ __forceinline__ void refine_3d(const int4* __restrict__ keys, long long cap,
                                          const RoiParams* __restrict__ rp,
                                          const uint2* __restrict__ work,
                                          const float* __restrict__ umax, Stats* __restrict__ st,
                                          double* sx, double* sy, double* sz,
                                          unsigned int* s_list, int& s_n) {
  static_assert(kDiamThreads % kChunk == 0, "refine splits j across kDiamThreads / kChunk groups");
  constexpr int kSplit = kDiamThreads / kChunk, kJ = kChunk / kSplit;
  Frame f = rp->f;
  const long long n = n_vertices(st, cap);
  long long w0, w1;
  w0 = 0;
  w1 = (long long)st->n_work;
  const int* bb = st->bbox;
  const double R2 = half_extent_sq(bb[0], bb[3], f.sx) + half_extent_sq(bb[1], bb[4], f.sy) +
                    half_extent_sq(bb[2], bb[5], f.sz);
  const float tau = refine_tau(__uint_as_float(st->d3_f32), R2);
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
      const int I = (int)ij.x, J = (int)(ij.y & kIdxMask);
      __syncthreads();  // previous candidate is done with sx/sy/sz
      if (threadIdx.x < kChunk) {
        const long long j = (long long)J * kChunk + threadIdx.x;
        const int4 kj = keys[j < n ? j : n - 1];
        sx[threadIdx.x] = ref_coord(kj.x + f.ox2, f.sx);
        sy[threadIdx.x] = ref_coord(kj.y + f.oy2, f.sy);
        sz[threadIdx.x] = ref_coord(kj.z + f.oz2, f.sz);
      }
      __syncthreads();
      const long long i = (long long)I * kChunk + ti;
      if (i < n) {
        const int4 ki = keys[i];
        const double xi = ref_coord(ki.x + f.ox2, f.sx), yi = ref_coord(ki.y + f.oy2, f.sy), zi = ref_coord(ki.z + f.oz2, f.sz);
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

__device__ __forceinline__ float2 plane_point(int2 k, const PlaneAxes& ax) {
  return make_float2((float)(k.x - ax.ca) * ax.ha, (float)(k.y - ax.cb) * ax.hb);
}

// Planar pass 1: fp32 dot form over every surviving in-plane chunk pair
// (128 x 128).  Every warp is an independent worker (own shared-memory copy
// of the J chunk as (a, b, |p|^2)); each lane register-blocks 4 i entries and
// evaluates two of them per FFMA2, so a pair costs one FFMA2 + half an FMNMX3.
// One maximum per work entry; per-family maxima in st->pl_f32[axis].  The
// refine kernel selects the re-check candidates from the unit maxima.
__device__ __forceinline__ void pass1_planar(const int2* __restrict__ sorted,
                                             const unsigned int* __restrict__ start,
                                             const uint2* __restrict__ pwork,
                                             const RoiParams* __restrict__ rp,
                                             float* __restrict__ umax, Stats* __restrict__ st,
                                             float4* __restrict__ sj) {
  Frame f = rp->f;
  const PlaneSpace ps = plane_space(st);
  const long long w0 = 0, w1 = (long long)st->n_pwork;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long gwarps = (long long)gridDim.x * kPlaneWarps;
  // Rotated by the 3-D list's warp count: when both lists are short (fewer
  // units than warps), the planar units go to the warps the 3-D list left
  // idle instead of queueing behind 3-D units on the same warps.
  const long long busy3 = min((long long)st->n_work, gwarps);
  const long long gw = ((long long)blockIdx.x * kPlaneWarps + warp + gwarps - busy3) % gwarps;
  const long long per = (w1 - w0 + gwarps - 1) / gwarps;
  const long long wb = w0 + gw * per, we = min(w1, wb + per);
  float run0 = 0.f, run1 = 0.f, run2 = 0.f;  // per-family maxima
  unsigned int prev_p = 0xffffffffu, prev_i = 0xffffffffu;
  float2 a2[kPR / 2], b2[kPR / 2];
  float ni[kPR];
  int axis = 0;
  for (long long w = wb; w < we; w++) {
    const uint2 u = pwork[w];
    const unsigned int p = u.x & kIdxMask, I = u.y >> 16, J = u.y & 0xffffu;
    const unsigned int sub = u.x >> kSubShift;  // 64 x 64 sub-pairs to evaluate
    const unsigned int b0 = start[p], np = start[p + 1] - b0;
    axis = plane_axis((int)p, ps);
    const PlaneAxes ax = plane_axes(axis, st, f);
    __syncwarp();  // previous unit is done with sj
    if (p != prev_p || I != prev_i) {
#pragma unroll
      for (int r = 0; r < kPR / 2; r++) {
        unsigned int i0 = I * kPC + (2 * r) * 32 + lane, i1 = i0 + 32;
        const float2 q0 = plane_point(sorted[b0 + min(i0, np - 1)], ax);
        const float2 q1 = plane_point(sorted[b0 + min(i1, np - 1)], ax);
        a2[r] = make_float2(-2.f * q0.x, -2.f * q1.x);
        b2[r] = make_float2(-2.f * q0.y, -2.f * q1.y);
        ni[2 * r] = fmaf(q0.x, q0.x, q0.y * q0.y);
        ni[2 * r + 1] = fmaf(q1.x, q1.x, q1.y * q1.y);
      }
      prev_p = p;
      prev_i = I;
    }
#pragma unroll
    for (int r = 0; r < kPR; r++) {
      const unsigned int j = J * kPC + r * 32 + lane;
      const float2 q = plane_point(sorted[b0 + min(j, np - 1)], ax);  // repeats are harmless
      sj[r * 32 + lane] = make_float4(q.x, q.y, fmaf(q.x, q.x, q.y * q.y), 0.f);
    }
    __syncwarp();
    float m[kPR];
#pragma unroll
    for (int r = 0; r < kPR; r++) m[r] = -3.0e38f;
    if (sub == 0xFu) {
#pragma unroll 2
      for (int j = 0; j < kPC; j += 2) {
        const float4 q0 = sj[j], q1 = sj[j + 1];
#pragma unroll
        for (int r = 0; r < kPR / 2; r++) {
          float2 t0 = __ffma2_rn(a2[r], make_float2(q0.x, q0.x), make_float2(q0.z, q0.z));
          float2 t1 = __ffma2_rn(a2[r], make_float2(q1.x, q1.x), make_float2(q1.z, q1.z));
          t0 = __ffma2_rn(b2[r], make_float2(q0.y, q0.y), t0);
          t1 = __ffma2_rn(b2[r], make_float2(q1.y, q1.y), t1);
          m[2 * r] = fmax3f(m[2 * r], t0.x, t1.x);
          m[2 * r + 1] = fmax3f(m[2 * r + 1], t0.y, t1.y);
        }
      }
    } else {
      // Only the listed 64 x 64 sub-pairs (i half a = packed pair a).
#pragma unroll
      for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 2; b++) {
          if (!(sub & (1u << (2 * a + b)))) continue;
#pragma unroll 2
          for (int j = 64 * b; j < 64 * b + 64; j += 2) {
            const float4 q0 = sj[j], q1 = sj[j + 1];
            float2 t0 = __ffma2_rn(a2[a], make_float2(q0.x, q0.x), make_float2(q0.z, q0.z));
            float2 t1 = __ffma2_rn(a2[a], make_float2(q1.x, q1.x), make_float2(q1.z, q1.z));
            t0 = __ffma2_rn(b2[a], make_float2(q0.y, q0.y), t0);
            t1 = __ffma2_rn(b2[a], make_float2(q1.y, q1.y), t1);
            m[2 * a] = fmax3f(m[2 * a], t0.x, t1.x);
            m[2 * a + 1] = fmax3f(m[2 * a + 1], t0.y, t1.y);
          }
        }
    }
    float best = 0.f;
#pragma unroll
    for (int r = 0; r < kPR; r++) best = fmaxf(best, m[r] + ni[r]);
#pragma unroll
    for (int o = 16; o; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) umax[w] = best;
    if (axis == 0) run0 = fmaxf(run0, best);
    else if (axis == 1) run1 = fmaxf(run1, best);
    else run2 = fmaxf(run2, best);
  }
  if (lane == 0) {
    if (run0 > 0.f) atomic_max_pos_f32(&st->pl_f32[0], run0);
    if (run1 > 0.f) atomic_max_pos_f32(&st->pl_f32[1], run1);
    if (run2 > 0.f) atomic_max_pos_f32(&st->pl_f32[2], run2);
  }
}

// Exact planar re-check (fp64, reference arithmetic: the out-of-plane delta
// is exactly 0, so da*da + db*db is the reference's 3-term sum bit for bit).
// Every block sweeps 256 work entries at a time, lists those within
// their family threshold (refine_tau) in shared memory and re-checks
// each: 128 i entries x two halves of the j chunk.
__device__ __forceinline__ void refine_planar(const int2* __restrict__ sorted,
                                              const unsigned int* __restrict__ start,
                                              const uint2* __restrict__ pwork,
                                              const RoiParams* __restrict__ rp,
                                              const float* __restrict__ umax,
                                              Stats* __restrict__ st, double* sa, double* sb,
                                              double* s_red, unsigned int* s_list, int& s_n) {
  Frame f = rp->f;
  constexpr int kSplit = kPlaneThreads / kPC, kJ = kPC / kSplit;
  const PlaneSpace ps = plane_space(st);
  const long long w0 = 0, w1 = (long long)st->n_pwork;
  float tau[3];
  {
    const int* bb = st->bbox;
    const double ex = half_extent_sq(bb[0], bb[3], f.sx), ey = half_extent_sq(bb[1], bb[4], f.sy),
                 ez = half_extent_sq(bb[2], bb[5], f.sz);
    const double R2[3] = {ex + ey, ex + ez, ey + ez};  // XY, XZ, YZ frames (plane_axes)
#pragma unroll
    for (int a = 0; a < 3; a++) tau[a] = refine_tau(__uint_as_float(st->pl_f32[a]), R2[a]);
  }
  const int ti = threadIdx.x % kPC, tj = (threadIdx.x / kPC) * kJ;
  // Block b sweeps entries w0 + b, w0 + b + G, ... (G = grid size), 256 at a
  // time, so candidates (adjacent in the work list) spread over the blocks.
  const long long G = gridDim.x;
  for (long long sweep = 0; w0 + sweep * kPlaneThreads * G < w1; sweep++) {
    __syncthreads();  // previous sweep is done with s_list / s_n
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const long long w = w0 + (sweep * kPlaneThreads + threadIdx.x) * G + blockIdx.x;
    if (w < w1) {
      const int a = plane_axis((int)(pwork[w].x & kIdxMask), ps);
      if (umax[w] >= (a == 0 ? tau[0] : (a == 1 ? tau[1] : tau[2])))
        s_list[atomicAdd(&s_n, 1)] = (unsigned int)w;
    }
    __syncthreads();
    const int cnt = s_n;
    if (threadIdx.x == 0 && cnt) atomicAdd(&st->n_pcand, (unsigned long long)cnt);
    for (int q = 0; q < cnt; q++) {
      const uint2 u = pwork[s_list[q]];
      const unsigned int p = u.x & kIdxMask, I = u.y >> 16, J = u.y & 0xffffu;
      const int axis = plane_axis((int)p, ps);
      const PlaneAxes ax = plane_axes(axis, st, f);
      const unsigned int b0 = start[p], np = start[p + 1] - b0;
      const unsigned int i = I * kPC + ti;
      const unsigned int jn = min((unsigned int)kPC, np - J * kPC);
      __syncthreads();  // previous candidate is done with sa/sb/s_red
      if (threadIdx.x < kPC && J * kPC + threadIdx.x < np) {
        const int2 k = sorted[b0 + J * kPC + threadIdx.x];
        sa[threadIdx.x] = ref_coord(k.x + ax.oa, ax.sa);
        sb[threadIdx.x] = ref_coord(k.y + ax.ob, ax.sb);
      }
      __syncthreads();
      double best = 0.0;
      if (i < np) {
        const int2 k = sorted[b0 + i];
        const double ai = ref_coord(k.x + ax.oa, ax.sa), bi = ref_coord(k.y + ax.ob, ax.sb);
        const unsigned int te = min(jn, (unsigned int)(tj + kJ));
        for (unsigned int t = tj; t < te; t++) {
          const double da = __dsub_rn(sa[t], ai), db = __dsub_rn(sb[t], bi);
          best = fmax(best, __dadd_rn(__dmul_rn(da, da), __dmul_rn(db, db)));
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
      if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = best;
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int wi = 1; wi < kPlaneThreads / 32; wi++) best = fmax(best, s_red[wi]);
        if (best > 0.0) atomic_max_pos_f64(&st->sq[1 + axis], best);
      }
    }
  }
}

}  // namespace sc
