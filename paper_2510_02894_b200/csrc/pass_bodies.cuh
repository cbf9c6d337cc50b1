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

// Vertex-level reach filter of pass 1.  A vertex p of chunk I can only be
// an end of a pair of unit (I, J) reaching LB if its squared max distance to
// J's box reaches LB: reach(p, box J) >= |p - q| for every q in J, and the
// maximum pair has |p* - q*|^2 = D^2 >= LB.  reach is formed in fp32 on the
// same frame coordinates as pass 1: a frame coordinate is off by <= 2u|t|
// (the int -> float is exact, one rounding each for h and the product), a
// box-side difference by <= 6u R_a, its square by <= 28u R_a^2, the FMA sum
// adds <= 8u R^2: |error| <= 36 u R^2 < kReachMargin R^2.  Dropping only
// vertices below LB - kReachMargin R^2 keeps both ends of the maximum pair,
// so the unit holding it still reaches refine_tau and is re-checked in fp64
// (the re-check itself always evaluates the full unit).
constexpr double kReachMargin = 64.0 / 16777216.0;

struct FBox {  // chunk (or half-chunk) box in pass-1 frame coordinates
  float lx, ly, lz, hx, hy, hz;
};

__device__ __forceinline__ FBox frame_box(int4 lo, int4 hi, const Frame& f) {
  FBox b;
  b.lx = (float)(lo.x - f.cx2) * f.hx; b.hx = (float)(hi.x - f.cx2) * f.hx;
  b.ly = (float)(lo.y - f.cy2) * f.hy; b.hy = (float)(hi.y - f.cy2) * f.hy;
  b.lz = (float)(lo.z - f.cz2) * f.hz; b.hz = (float)(hi.z - f.cz2) * f.hz;
  return b;
}

__device__ __forceinline__ float reach_sq(float3 p, const FBox& b) {
  const float dx = fmaxf(p.x - b.lx, b.hx - p.x), dy = fmaxf(p.y - b.ly, b.hy - p.y),
              dz = fmaxf(p.z - b.lz, b.hz - p.z);
  return fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}

// Box of chunk c restricted to its 64-vertex halves selected by `halves`
// (bit h = half h; 3 = the whole chunk).
__device__ __forceinline__ FBox half_box(const int4* __restrict__ boxes,
                                         const int4* __restrict__ hboxes, int c,
                                         unsigned int halves, const Frame& f) {
  if (halves == 3u) return frame_box(boxes[2 * c], boxes[2 * c + 1], f);
  const int h = halves == 2u ? 1 : 0;
  return frame_box(hboxes[4 * c + 2 * h], hboxes[4 * c + 2 * h + 1], f);
}

// Stream-compact this lane's candidate into buf (warp-uniform count n).
__device__ __forceinline__ void warp_append(float4* buf, int& n, bool keep, float4 v) {
  const unsigned int bal = __ballot_sync(0xffffffffu, keep);
  if (keep) buf[n + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u))] = v;
  n += __popc(bal);
}

// Max over i entries si[i0 .. i0 + 64 P) (clamped to ni: repeats are
// harmless) x the j list sj[0, nj2) of the dot-form pass-1 value; lane
// holds P packed i pairs (i0 + 64 p + {0, 32} + lane).
template <int P>
__device__ __forceinline__ float eval_rows(const float4* __restrict__ si,
                                           const float4* __restrict__ sj, int i0, int ni,
                                           int nj2) {
  const int lane = threadIdx.x & 31;
  float2 a2[P], b2[P], c2[P];
  float n0[P], n1[P], m0[P], m1[P];
#pragma unroll
  for (int p = 0; p < P; p++) {
    const float4 e0 = si[min(i0 + 64 * p + lane, ni - 1)];
    const float4 e1 = si[min(i0 + 64 * p + 32 + lane, ni - 1)];
    a2[p] = make_float2(-2.f * e0.x, -2.f * e1.x);
    b2[p] = make_float2(-2.f * e0.y, -2.f * e1.y);
    c2[p] = make_float2(-2.f * e0.z, -2.f * e1.z);
    n0[p] = e0.w;
    n1[p] = e1.w;
    m0[p] = m1[p] = -3.0e38f;
  }
#pragma unroll 4
  for (int j = 0; j < nj2; j += 2) {
    const float4 q0 = sj[j], q1 = sj[j + 1];
#pragma unroll
    for (int p = 0; p < P; p++) {
      float2 t0 = __ffma2_rn(a2[p], make_float2(q0.x, q0.x), make_float2(q0.w, q0.w));
      float2 t1 = __ffma2_rn(a2[p], make_float2(q1.x, q1.x), make_float2(q1.w, q1.w));
      t0 = __ffma2_rn(b2[p], make_float2(q0.y, q0.y), t0);
      t1 = __ffma2_rn(b2[p], make_float2(q1.y, q1.y), t1);
      t0 = __ffma2_rn(c2[p], make_float2(q0.z, q0.z), t0);
      t1 = __ffma2_rn(c2[p], make_float2(q1.z, q1.z), t1);
      m0[p] = fmax3f(m0[p], t0.x, t1.x);
      m1[p] = fmax3f(m1[p], t0.y, t1.y);
    }
  }
  float best = 0.f;
#pragma unroll
  for (int p = 0; p < P; p++) best = fmaxf(best, fmaxf(m0[p] + n0[p], m1[p] + n1[p]));
  return best;
}

// Pass 1 (see header).  Work unit = one surviving chunk pair (I <= J, 128 x
// 128 vertex pairs, listed by unit_filter / unit_expand with the mask of its
// 64 x 64 sub-pairs that can reach LB); every WARP is an independent worker,
// so load balance is per unit and no block barrier is involved.  Error of the
// dot form: in the bbox-centred frame |p| <= R, absolute error <= 35 u R^2.
//
// FILTER (the product path): the warp first keeps only the vertices of each
// side whose reach to the other side's (sub-pair-selected) box can attain LB
// (kReachMargin), stream-compacted into two shared-memory lists (si, sj) as
// (x, y, z, |p|^2); then every lane takes 2 (or 4) i entries and loops over
// the j list, two i per FFMA2 (4 pairs = 6 FFMA2 + 2 FMNMX3).  Only the
// compacted cross product is evaluated.
// !FILTER (option pass1_packed=0): every listed 64 x 64 sub-pair, scalar FFMA
// (the unfiltered baseline).
template <bool FILTER>
__device__ __forceinline__ void pass1_3d(const int4* __restrict__ keys,
                                         const float4* __restrict__ fkeys, long long cap,
                                         const RoiParams* __restrict__ rp,
                                         const uint2* __restrict__ work, float* __restrict__ umax,
                                         Stats* __restrict__ st, float4* __restrict__ sj,
                                         float4* __restrict__ si,
                                         const int4* __restrict__ boxes,
                                         const int4* __restrict__ hboxes, int vfilter) {
  Frame f = rp->f;
  const long long n = n_vertices(st, cap);
  if (n == 0) return;
  frame_centre(st, f);
  const long long n_work = (long long)st->n_work;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Each warp takes a contiguous run of units.
  // (32-bit split: a work list never exceeds 2^32 entries -- it is capped by
  // wcap -- and a 64-bit division per warp was ~3 % of the kernel)
  const unsigned int gwarps = gridDim.x * kWarps;
  const unsigned int gw = blockIdx.x * kWarps + warp;
  const unsigned int per = ((unsigned int)n_work + gwarps - 1) / gwarps;
  const long long wb = (long long)gw * per, we = min(n_work, wb + per);
  if (wb >= we) return;
  float run = 0.f;
  if (FILTER) {
    const int* bb = st->bbox;
    const double R2 = half_extent_sq(bb[0], bb[3], f.sx) + half_extent_sq(bb[1], bb[4], f.sy) +
                      half_extent_sq(bb[2], bb[5], f.sz);
    const double lb = __longlong_as_double((long long)st->lb);
    // (no filtering when pruning is off: every pair is evaluated)
    const float thr = vfilter ? __double2float_rd(lb - kReachMargin * R2) : -3.0e38f;
    unsigned long long evals = 0;  // pair slots evaluated (diagnostics)
    uint2 ij_next = work[wb];
    for (long long w = wb; w < we; w++) {
      const uint2 ij = ij_next;
      if (w + 1 < we) ij_next = work[w + 1];  // next unit's entry in flight during this one
      const int I = (int)ij.x, J = (int)(ij.y & kIdxMask);
      const unsigned int sub = ij.y >> kSubShift;  // bit 2a + b: i half a x j half b
      // i half a meets the j halves (sub >> 2a) & 3; j half b the i halves
      // bit b | bit (2 + b) << 1.
      const unsigned int ja0 = sub & 3u, ja1 = (sub >> 2) & 3u;
      const unsigned int ib0 = (sub & 1u) | ((sub >> 1) & 2u), ib1 = ((sub >> 1) & 1u) | ((sub >> 2) & 2u);
      __syncwarp();  // the previous unit is done with si / sj
      // j side first; the i side only when some j survives (most units keep
      // no vertex on at least one side once the reach filter applies).
      int ni = 0, nj = 0;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const unsigned int ih = h ? ib1 : ib0;
        const FBox bi = half_box(boxes, hboxes, I, ih ? ih : 3u, f);  // reach target of j half h
#pragma unroll
        for (int r = 2 * h; r < 2 * h + 2; r++) {
          const long long j = (long long)J * kChunk + r * 32 + lane;
          const float4 q = fkeys[j < n ? j : n - 1];
          warp_append(sj, nj, j < n && ih && reach_sq(make_float3(q.x, q.y, q.z), bi) >= thr, q);
        }
      }
      if (nj > 0) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const unsigned int jh = h ? ja1 : ja0;
          const FBox bj = half_box(boxes, hboxes, J, jh ? jh : 3u, f);  // reach target of i half h
#pragma unroll
          for (int r = 2 * h; r < 2 * h + 2; r++) {
            const long long i = (long long)I * kChunk + r * 32 + lane;
            const float4 p = fkeys[i < n ? i : n - 1];
            warp_append(si, ni, i < n && jh && reach_sq(make_float3(p.x, p.y, p.z), bj) >= thr, p);
          }
        }
      }
      __syncwarp();
      float best = 0.f;
      if (ni > 0 && nj > 0) {
        if ((nj & 1) && lane == 0) sj[nj] = sj[nj - 1];  // even trip count (a repeat is harmless)
        __syncwarp();
        const int nj2 = (nj + 1) & ~1;
        // 4 i entries per lane (two FFMA2 pairs) while more than 64 remain, else 2.
        int i0 = 0;
        for (; ni - i0 > 64; i0 += 128) {
          best = fmaxf(best, eval_rows<2>(si, sj, i0, ni, nj2));
          evals += 128ull * (unsigned long long)nj2;
        }
        if (i0 < ni) {
          best = fmaxf(best, eval_rows<1>(si, sj, i0, ni, nj2));
          evals += 64ull * (unsigned long long)nj2;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (lane == 0) umax[w] = best;
      run = fmaxf(run, best);
    }
    if (lane == 0) {
      atomic_max_pos_f32(&st->d3_f32, run);
      if (evals) atomicAdd(&st->n_eval, evals);
    }
    return;
  }
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

// In-plane box of a chunk (or of its halves selected by `halves`, bit h =
// half h; 3 = whole chunk) in the planar pass-1 frame: (lo.a, lo.b, hi.a, hi.b).
__device__ __forceinline__ float4 plane_half_box(const int4* __restrict__ pboxes,
                                                 const int4* __restrict__ hpboxes, unsigned int c,
                                                 unsigned int halves, const PlaneAxes& ax) {
  const int4 b = halves == 3u ? pboxes[c] : hpboxes[2 * c + (halves == 2u ? 1 : 0)];
  return make_float4((float)(b.x - ax.ca) * ax.ha, (float)(b.y - ax.cb) * ax.hb,
                     (float)(b.z - ax.ca) * ax.ha, (float)(b.w - ax.cb) * ax.hb);
}

__device__ __forceinline__ float reach_sq2(float2 p, float4 b) {
  const float da = fmaxf(p.x - b.x, b.z - p.x), db = fmaxf(p.y - b.y, b.w - p.y);
  return fmaf(da, da, db * db);
}

// 2-D counterpart of eval_rows: entries (a, b, |p|^2, -).
template <int P>
__device__ __forceinline__ float eval_rows2(const float4* __restrict__ si,
                                            const float4* __restrict__ sj, int i0, int ni,
                                            int nj2) {
  const int lane = threadIdx.x & 31;
  float2 a2[P], b2[P];
  float n0[P], n1[P], m0[P], m1[P];
#pragma unroll
  for (int p = 0; p < P; p++) {
    const float4 e0 = si[min(i0 + 64 * p + lane, ni - 1)];
    const float4 e1 = si[min(i0 + 64 * p + 32 + lane, ni - 1)];
    a2[p] = make_float2(-2.f * e0.x, -2.f * e1.x);
    b2[p] = make_float2(-2.f * e0.y, -2.f * e1.y);
    n0[p] = e0.z;
    n1[p] = e1.z;
    m0[p] = m1[p] = -3.0e38f;
  }
#pragma unroll 4
  for (int j = 0; j < nj2; j += 2) {
    const float4 q0 = sj[j], q1 = sj[j + 1];
#pragma unroll
    for (int p = 0; p < P; p++) {
      float2 t0 = __ffma2_rn(a2[p], make_float2(q0.x, q0.x), make_float2(q0.z, q0.z));
      float2 t1 = __ffma2_rn(a2[p], make_float2(q1.x, q1.x), make_float2(q1.z, q1.z));
      t0 = __ffma2_rn(b2[p], make_float2(q0.y, q0.y), t0);
      t1 = __ffma2_rn(b2[p], make_float2(q1.y, q1.y), t1);
      m0[p] = fmax3f(m0[p], t0.x, t1.x);
      m1[p] = fmax3f(m1[p], t0.y, t1.y);
    }
  }
  float best = 0.f;
#pragma unroll
  for (int p = 0; p < P; p++) best = fmaxf(best, fmaxf(m0[p] + n0[p], m1[p] + n1[p]));
  return best;
}

__device__ __forceinline__ float2 plane_point(int2 k, const PlaneAxes& ax) {
  return make_float2((float)(k.x - ax.ca) * ax.ha, (float)(k.y - ax.cb) * ax.hb);
}

// Planar pass 1: the same scheme as pass1_3d over every surviving in-plane
// chunk pair (128 x 128 entries of one plane): per side, the entries whose
// in-plane reach to the other side's (sub-pair-selected) box can attain the
// family's lower bound plb (margin kReachMargin R_family^2, the 2-D case of
// the 3-D argument), stream-compacted into si / sj as (a, b, |p|^2); then the
// compacted cross product in the fp32 dot form, two i per FFMA2 (4 pairs = 4
// FFMA2 + 2 FMNMX3).  One maximum per work entry; per-family maxima in
// st->pl_f32[axis].  The refine kernel selects the re-check candidates.
__device__ __forceinline__ void pass1_planar(const int2* __restrict__ sorted,
                                             const unsigned int* __restrict__ start,
                                             const uint2* __restrict__ pwork,
                                             const RoiParams* __restrict__ rp,
                                             float* __restrict__ umax, Stats* __restrict__ st,
                                             float4* __restrict__ sj, float4* __restrict__ si,
                                             const unsigned int* __restrict__ cstart,
                                             const int4* __restrict__ pboxes,
                                             const int4* __restrict__ hpboxes, int vfilter) {
  Frame f = rp->f;
  const PlaneSpace ps = plane_space(st);
  const long long w0 = 0, w1 = (long long)st->n_pwork;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned int gwarps = gridDim.x * kPlaneWarps;
  // Rotated by the 3-D list's warp count: when both lists are short (fewer
  // units than warps), the planar units go to the warps the 3-D list left
  // idle instead of queueing behind 3-D units on the same warps.
  const unsigned int busy3 = (unsigned int)min((unsigned long long)st->n_work, (unsigned long long)gwarps);
  const unsigned int gw = (blockIdx.x * kPlaneWarps + warp + gwarps - busy3) % gwarps;
  const unsigned int per = ((unsigned int)(w1 - w0) + gwarps - 1) / gwarps;
  const long long wb = w0 + (long long)gw * per, we = min(w1, wb + per);
  if (wb >= we) return;
  float thr[3];
  {
    const int* bb = st->bbox;
    const double ex = half_extent_sq(bb[0], bb[3], f.sx), ey = half_extent_sq(bb[1], bb[4], f.sy),
                 ez = half_extent_sq(bb[2], bb[5], f.sz);
    const double R2[3] = {ex + ey, ex + ez, ey + ez};  // XY, XZ, YZ frames (plane_axes)
#pragma unroll
    for (int a = 0; a < 3; a++)
      thr[a] = vfilter ? __double2float_rd(__longlong_as_double((long long)st->plb[a]) -
                                           kReachMargin * R2[a])
                       : -3.0e38f;
  }
  float run0 = 0.f, run1 = 0.f, run2 = 0.f;  // per-family maxima
  unsigned long long evals = 0;
  uint2 u_next = pwork[wb];
  for (long long w = wb; w < we; w++) {
    const uint2 u = u_next;
    if (w + 1 < we) u_next = pwork[w + 1];  // next unit's entry in flight during this one
    const unsigned int p = u.x & kIdxMask, I = u.y >> 16, J = u.y & 0xffffu;
    const unsigned int sub = u.x >> kSubShift;  // bit 2a + b: i half a x j half b
    const unsigned int b0 = start[p], np = start[p + 1] - b0, c0 = cstart[p];
    const int axis = plane_axis((int)p, ps);
    const PlaneAxes ax = plane_axes(axis, st, f);
    const float th = axis == 0 ? thr[0] : (axis == 1 ? thr[1] : thr[2]);
    const unsigned int ja0 = sub & 3u, ja1 = (sub >> 2) & 3u;
    const unsigned int ib0 = (sub & 1u) | ((sub >> 1) & 2u), ib1 = ((sub >> 1) & 1u) | ((sub >> 2) & 2u);
    __syncwarp();  // previous unit is done with si / sj
    int ni = 0, nj = 0;  // j side first, the i side only if some j survives
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const unsigned int ih = h ? ib1 : ib0;
      const float4 bi = plane_half_box(pboxes, hpboxes, c0 + I, ih ? ih : 3u, ax);
#pragma unroll
      for (int r = 2 * h; r < 2 * h + 2; r++) {
        const unsigned int j = J * kPC + r * 32 + lane;
        const float2 qj = plane_point(sorted[b0 + min(j, np - 1)], ax);
        warp_append(sj, nj, j < np && ih && reach_sq2(qj, bi) >= th,
                    make_float4(qj.x, qj.y, fmaf(qj.x, qj.x, qj.y * qj.y), 0.f));
      }
    }
    if (nj > 0) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const unsigned int jh = h ? ja1 : ja0;
        const float4 bj = plane_half_box(pboxes, hpboxes, c0 + J, jh ? jh : 3u, ax);
#pragma unroll
        for (int r = 2 * h; r < 2 * h + 2; r++) {
          const unsigned int i = I * kPC + r * 32 + lane;
          const float2 pi = plane_point(sorted[b0 + min(i, np - 1)], ax);
          warp_append(si, ni, i < np && jh && reach_sq2(pi, bj) >= th,
                      make_float4(pi.x, pi.y, fmaf(pi.x, pi.x, pi.y * pi.y), 0.f));
        }
      }
    }
    __syncwarp();
    float best = 0.f;
    if (ni > 0 && nj > 0) {
      if ((nj & 1) && lane == 0) sj[nj] = sj[nj - 1];  // even trip count (repeat is harmless)
      __syncwarp();
      const int nj2 = (nj + 1) & ~1;
      int i0 = 0;
      for (; ni - i0 > 64; i0 += 128) {
        best = fmaxf(best, eval_rows2<2>(si, sj, i0, ni, nj2));
        evals += 128ull * (unsigned long long)nj2;
      }
      if (i0 < ni) {
        best = fmaxf(best, eval_rows2<1>(si, sj, i0, ni, nj2));
        evals += 64ull * (unsigned long long)nj2;
      }
    }
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
    if (evals) atomicAdd(&st->n_peval, evals);
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
