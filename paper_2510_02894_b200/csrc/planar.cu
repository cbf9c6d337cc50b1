// Planar maximum diameters (sm_100a): maxima over vertex pairs sharing z
// (XY), y (XZ) or x (YZ), bit-exact with reference features.py:145-147.
//
// Every vertex belongs to three planes, keyed by its doubled lattice
// coordinate (bit-equal fp64 coordinate <=> equal key).  mc_cells histograms
// (plane, in-plane Morton brick) bins, so the counting sort below leaves every
// plane's list spatially compact; then the same three steps as the 3-D pass:
//
//   plane_bins_scan  -- per plane: in-plane bin offsets, plane population
//   (scan_all)       -- plane / tile-pair / chunk offsets, unit and chunk maps
//   (scatter_all)    -- plane lists in brick order
//   plane_boxes      -- box of every 256-entry in-plane chunk + 8 extremes
//   plane_lb         -- exact per-family lower bound from the extremes
//   plane_filter     -- keep in-plane chunk pairs whose box distance reaches it
//   plane_pass1      -- fp32 dot-form max per surviving unit (+ selection)
//   plane_refine     -- fp64 reference-arithmetic re-check of the candidates
#include <climits>

#include "sc_device.cuh"

namespace sc {

constexpr int kPT = 256;  // in-plane tile / chunk edge

// One warp per plane: exclusive offsets of its 256 brick bins (into
// pbin_cursor, plane-relative), its population (plane_counts), and reset of
// its bins and extremes for the next ROI.
__global__ void plane_bins_scan(unsigned int* __restrict__ pbin_counts,
                                unsigned int* __restrict__ pbin_cursor,
                                unsigned int* __restrict__ plane_counts,
                                unsigned long long* __restrict__ pext,
                                const Stats* __restrict__ st) {
  if (st->bbox[3] < 0) return;
  const PlaneSpace ps = plane_space(st);
  const int P = ps.cnt[0] + ps.cnt[1] + ps.cnt[2];
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < P; p += warps) {
    unsigned int* cnt = pbin_counts + (long long)p * kPlaneBins + lane * 8;
    unsigned int v[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      v[k] = cnt[k];
      sum += v[k];
      cnt[k] = 0u;
    }
    unsigned int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    unsigned int run = incl - sum;
    unsigned int* cur = pbin_cursor + (long long)p * kPlaneBins + lane * 8;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      cur[k] = run;
      run += v[k];
    }
    if (lane == 31) plane_counts[p] = incl;
    if (lane < 8) pext[(long long)p * 8 + lane] = 0ull;
  }
}

__device__ __forceinline__ unsigned long long pack_pext(float v, unsigned int idx) {
  unsigned int b = __float_as_uint(v);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);  // order-preserving
  return ((unsigned long long)b << 32) | idx;
}

// One warp per in-plane chunk c (cmap[c] = plane): its 2-D integer box
// (lo.a, lo.b, hi.a, hi.b) and the plane's 8 arg-extremes (+-a, +-b,
// +-(a+b), +-(a-b) in the mm frame), index = plane-relative entry.
__global__ void plane_boxes(const int2* __restrict__ sorted,
                            const unsigned int* __restrict__ start,
                            const unsigned int* __restrict__ cstart,
                            const unsigned int* __restrict__ cmap, const RoiParams* __restrict__ rp,
                            const Stats* __restrict__ st, int4* __restrict__ pboxes,
                            unsigned long long* __restrict__ pext) {
  if (st->ovf) return;  // re-run pending (scan_all)
  Frame f = rp->f;
  if (st->bbox[3] < 0) return;
  const PlaneSpace ps = plane_space(st);
  const long long chunks = (long long)st->plane_chunks;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long c = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < chunks;
       c += warps) {
    const int p = (int)cmap[c];
    const PlaneAxes ax = plane_axes(plane_axis(p, ps), st, f);
    const unsigned int b0 = start[p], np = start[p + 1] - b0;
    const unsigned int e0 = (unsigned int)(c - cstart[p]) * kPT;
    const unsigned int e1 = min(np, e0 + kPT);
    int la = INT_MAX, lb = INT_MAX, ha = INT_MIN, hb = INT_MIN;
    unsigned long long ext[8];
#pragma unroll
    for (int d = 0; d < 8; d++) ext[d] = 0ull;
    for (unsigned int e = e0 + lane; e < e1; e += 32) {
      const int2 k = sorted[b0 + e];
      la = min(la, k.x); lb = min(lb, k.y); ha = max(ha, k.x); hb = max(hb, k.y);
      const float a = (float)k.x * ax.ha, b = (float)k.y * ax.hb;
      const float pr[4] = {a, b, a + b, a - b};
#pragma unroll
      for (int d = 0; d < 4; d++) {
        const unsigned long long hi = pack_pext(pr[d], e), lo = pack_pext(-pr[d], e);
        ext[2 * d] = hi > ext[2 * d] ? hi : ext[2 * d];
        ext[2 * d + 1] = lo > ext[2 * d + 1] ? lo : ext[2 * d + 1];
      }
    }
    la = __reduce_min_sync(0xffffffffu, la); lb = __reduce_min_sync(0xffffffffu, lb);
    ha = __reduce_max_sync(0xffffffffu, ha); hb = __reduce_max_sync(0xffffffffu, hb);
    if (lane == 0) pboxes[c] = make_int4(la, lb, ha, hb);
#pragma unroll
    for (int d = 0; d < 8; d++) {
      unsigned long long x = ext[d];
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, x, o);
        x = t > x ? t : x;
      }
      if (lane == 0 && x) atomicMax(&pext[(long long)p * 8 + d], x);
    }
  }
}

// One warp per plane: the exact (reference arithmetic) max over the 28 pairs
// of its 8 extreme entries -- a real pair, so it bounds that family's maximum
// from below and seeds it.
__global__ void plane_lb(const int2* __restrict__ sorted, const unsigned int* __restrict__ start,
                         const unsigned long long* __restrict__ pext, const RoiParams* __restrict__ rp,
                         Stats* __restrict__ st) {
  if (st->ovf) return;  // re-run pending (scan_all)
  Frame f = rp->f;
  if (st->bbox[3] < 0) return;
  const PlaneSpace ps = plane_space(st);
  const int P = ps.cnt[0] + ps.cnt[1] + ps.cnt[2];
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < P; p += warps) {
    const unsigned int b0 = start[p], np = start[p + 1] - b0;
    if (np < 2) continue;  // warp-uniform
    const int axis = plane_axis(p, ps);
    const PlaneAxes ax = plane_axes(axis, st, f);
    double best = 0.0;
    if (lane < 28) {
      int i = 0, j = lane;  // lane -> pair (i < j) of 8
      while (j >= 7 - i) { j -= 7 - i; i++; }
      j += i + 1;
      const int2 ki = sorted[b0 + (unsigned int)(pext[(long long)p * 8 + i] & 0xffffffffu)];
      const int2 kj = sorted[b0 + (unsigned int)(pext[(long long)p * 8 + j] & 0xffffffffu)];
      const double da = __dsub_rn(ref_coord(kj.x, ax.sa), ref_coord(ki.x, ax.sa));
      const double db = __dsub_rn(ref_coord(kj.y, ax.sb), ref_coord(ki.y, ax.sb));
      best = __dadd_rn(__dmul_rn(da, da), __dmul_rn(db, db));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0 && best > 0.0) {
      atomic_max_pos_f64(&st->plb[axis], best);
      atomic_max_pos_f64(&st->sq[1 + axis], best);
    }
  }
}

__device__ __forceinline__ double reach2(int loA, int hiA, int loB, int hiB, double h) {
  const double d = (double)max(hiA - loB, hiB - loA) * h;
  return d * d;
}

// Keep in-plane chunk pairs whose box distance can reach the family's lower
// bound (margin 1e-9 covers fp64 rounding of both sides); compact into pwork.
__global__ void plane_filter(const unsigned int* __restrict__ start,
                             const unsigned int* __restrict__ tstart,
                             const unsigned int* __restrict__ cstart,
                             const unsigned int* __restrict__ umap,
                             const int4* __restrict__ pboxes, const RoiParams* __restrict__ rp, int prune, long long ucap,
                             Stats* __restrict__ st, unsigned int* __restrict__ pwork) {
  if (st->ovf) return;  // re-run pending (scan_all)
  Frame f = rp->f;
  const long long units = (long long)st->plane_units;
  if (st->bbox[3] < 0 || units > ucap) return;  // host re-runs with room
  const PlaneSpace ps = plane_space(st);
  double thr[3];
#pragma unroll
  for (int a = 0; a < 3; a++)
    thr[a] = __longlong_as_double((long long)st->plb[a]) * (1.0 - 1e-9);
  const int lane = threadIdx.x & 31;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < units;
       base += (long long)gridDim.x * blockDim.x) {
    const long long u = base + threadIdx.x;
    bool keep = false;
    if (u < units) {
      if (!prune) {
        keep = true;
      } else {
        const int p = (int)umap[u];
        const int axis = plane_axis(p, ps);
        const PlaneAxes ax = plane_axes(axis, st, f);
        const unsigned int np = start[p + 1] - start[p];
        int I, J;
        tile_pair(u - tstart[p], (np + kPT - 1) / kPT, I, J);
        const int4 bi = pboxes[cstart[p] + I], bj = pboxes[cstart[p] + J];
        const double ub = reach2(bi.x, bi.z, bj.x, bj.z, 0.5 * ax.sa) +
                          reach2(bi.y, bi.w, bj.y, bj.w, 0.5 * ax.sb);
        keep = ub >= (axis == 0 ? thr[0] : (axis == 1 ? thr[1] : thr[2]));
      }
    }
    const unsigned int mask = __ballot_sync(0xffffffffu, keep);
    if (!mask) continue;
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(&st->n_pwork, (unsigned long long)__popc(mask));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (keep) pwork[pos + __popc(mask & ((1u << lane) - 1))] = (unsigned int)u;
  }
}

// Planar pass 1: fp32 dot form over every surviving in-plane tile pair
// (kPT x kPT); one maximum per work entry; per-family maxima in
// st->pl_f32[axis].  The last block compacts the re-check candidates.
__global__ void __launch_bounds__(kPT) plane_pass1(const int2* __restrict__ sorted,
                                                   const unsigned int* __restrict__ start,
                                                   const unsigned int* __restrict__ tstart,
                                                   const unsigned int* __restrict__ umap,
                                                   const unsigned int* __restrict__ pwork,
                                                   const RoiParams* __restrict__ rp, int shard, int nshards,
                                                   long long ucap, float* __restrict__ umax,
                                                   unsigned int* __restrict__ cand,
                                                   Stats* __restrict__ st) {
  if (st->ovf) return;  // re-run pending (scan_all)
  Frame f = rp->f;
  __shared__ float4 sj[kPT];  // (a, b, |p|^2, -)
  __shared__ float s_red[kPT / 32];
  if (st->bbox[3] < 0 || (long long)st->plane_units > ucap) return;
  const PlaneSpace ps = plane_space(st);
  long long w0, w1;
  shard_span((long long)st->n_pwork, shard, nshards, w0, w1);
  float run0 = 0.f, run1 = 0.f, run2 = 0.f;  // per-family maxima (registers)
  for (long long w = w0 + blockIdx.x; w < w1; w += gridDim.x) {
    const unsigned int u = pwork[w];
    const int p = (int)umap[u];
    const int axis = plane_axis(p, ps);
    const PlaneAxes ax = plane_axes(axis, st, f);
    const unsigned int b0 = start[p], np = start[p + 1] - b0;
    int I, J;
    tile_pair(u - tstart[p], (np + kPT - 1) / kPT, I, J);
    const unsigned int i = I * kPT + threadIdx.x, j = J * kPT + threadIdx.x;
    const unsigned int jn = min((unsigned int)kPT, np - J * kPT);
    __syncthreads();
    if (j < np) {
      const int2 k = sorted[b0 + j];
      const float pa = (float)(k.x - ax.ca) * ax.ha, pb = (float)(k.y - ax.cb) * ax.hb;
      sj[threadIdx.x] = make_float4(pa, pb, fmaf(pa, pa, pb * pb), 0.f);
    }
    __syncthreads();
    float best = 0.f;
    if (i < np) {
      const int2 k = sorted[b0 + i];
      const float pa = (float)(k.x - ax.ca) * ax.ha, pb = (float)(k.y - ax.cb) * ax.hb;
      const float a2 = -2.f * pa, b2 = -2.f * pb;
      float m = -3.0e38f;
      unsigned int t = 0;
      for (; t + 1 < jn; t += 2) {
        const float4 q0 = sj[t], q1 = sj[t + 1];
        m = fmax3f(m, fmaf(q0.y, b2, fmaf(q0.x, a2, q0.z)), fmaf(q1.y, b2, fmaf(q1.x, a2, q1.z)));
      }
      if (t < jn) m = fmaxf(m, fmaf(sj[t].y, b2, fmaf(sj[t].x, a2, sj[t].z)));
      best = fmaxf(0.f, m + fmaf(pa, pa, pb * pb));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int wi = 1; wi < kPT / 32; wi++) best = fmaxf(best, s_red[wi]);
      umax[w] = best;
      if (axis == 0) run0 = fmaxf(run0, best);
      else if (axis == 1) run1 = fmaxf(run1, best);
      else run2 = fmaxf(run2, best);
    }
  }
  if (threadIdx.x == 0) {
    if (run0 > 0.f) atomic_max_pos_f32(&st->pl_f32[0], run0);
    if (run1 > 0.f) atomic_max_pos_f32(&st->pl_f32[1], run1);
    if (run2 > 0.f) atomic_max_pos_f32(&st->pl_f32[2], run2);
  }
  if (!last_block(&st->done2)) return;
  // Last block: work entries within kRefineRel of their family maximum.
  const float tau0 = __uint_as_float(__ldcg(&st->pl_f32[0])) * (1.f - kRefineRel);
  const float tau1 = __uint_as_float(__ldcg(&st->pl_f32[1])) * (1.f - kRefineRel);
  const float tau2 = __uint_as_float(__ldcg(&st->pl_f32[2])) * (1.f - kRefineRel);
  const int lane = threadIdx.x & 31;
  for (long long base = w0; base < w1; base += blockDim.x) {
    const long long w = base + threadIdx.x;
    bool hit = false;
    if (w < w1) {
      const int a = plane_axis((int)umap[pwork[w]], ps);
      hit = __ldcg(umax + w) >= (a == 0 ? tau0 : (a == 1 ? tau1 : tau2));
    }
    const unsigned int mask = __ballot_sync(0xffffffffu, hit);
    if (!mask) continue;
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(&st->n_pcand, (unsigned long long)__popc(mask));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (hit) cand[pos + __popc(mask & ((1u << lane) - 1))] = (unsigned int)w;
  }
}

// Exact planar re-check of the selected in-plane tile pairs (fp64, reference
// arithmetic: the out-of-plane delta is exactly 0, so da*da + db*db is the
// reference's 3-term sum bit for bit).
__global__ void __launch_bounds__(kPT) plane_refine(const int2* __restrict__ sorted,
                                                    const unsigned int* __restrict__ start,
                                                    const unsigned int* __restrict__ tstart,
                                                    const unsigned int* __restrict__ umap,
                                                    const unsigned int* __restrict__ pwork,
                                                    const RoiParams* __restrict__ rp, const unsigned int* __restrict__ cand,
                                                    Stats* __restrict__ st) {
  if (st->ovf) return;  // re-run pending (scan_all)
  Frame f = rp->f;
  __shared__ double sa[kPT], sb[kPT];
  __shared__ double s_red[kPT / 32];
  if (st->bbox[3] < 0) return;
  const PlaneSpace ps = plane_space(st);
  const long long nc = (long long)st->n_pcand;
  for (long long c = blockIdx.x; c < nc; c += gridDim.x) {
    const unsigned int u = pwork[cand[c]];
    const int p = (int)umap[u];
    const int axis = plane_axis(p, ps);
    const PlaneAxes ax = plane_axes(axis, st, f);
    const unsigned int b0 = start[p], np = start[p + 1] - b0;
    int I, J;
    tile_pair(u - tstart[p], (np + kPT - 1) / kPT, I, J);
    const unsigned int i = I * kPT + threadIdx.x, j = J * kPT + threadIdx.x;
    const unsigned int jn = min((unsigned int)kPT, np - J * kPT);
    __syncthreads();
    if (j < np) {
      const int2 k = sorted[b0 + j];
      sa[threadIdx.x] = ref_coord(k.x, ax.sa);
      sb[threadIdx.x] = ref_coord(k.y, ax.sb);
    }
    __syncthreads();
    double best = 0.0;
    if (i < np) {
      const int2 k = sorted[b0 + i];
      const double ai = ref_coord(k.x, ax.sa), bi = ref_coord(k.y, ax.sb);
      for (unsigned int t = 0; t < jn; t++) {
        const double da = __dsub_rn(sa[t], ai), db = __dsub_rn(sb[t], bi);
        best = fmax(best, __dadd_rn(__dmul_rn(da, da), __dmul_rn(db, db)));
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int wi = 1; wi < kPT / 32; wi++) best = fmax(best, s_red[wi]);
      if (best > 0.0) atomic_max_pos_f64(&st->sq[1 + axis], best);
    }
  }
}

}  // namespace sc
