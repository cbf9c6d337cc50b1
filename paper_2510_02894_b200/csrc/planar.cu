// Planar maximum diameters (sm_100a): maxima over vertex pairs sharing z
// (XY), y (XZ) or x (YZ), bit-exact with reference features.py:145-147.
//
// Every vertex belongs to three planes, keyed by its doubled lattice
// coordinate (bit-equal fp64 coordinate <=> equal key).  mc_cells histograms
// (plane, in-plane Morton brick) bins, so the counting sort below leaves every
// plane's list spatially compact; then the same three steps as the 3-D pass:
//
//   plane_bins_scan  -- per plane: in-plane bin offsets, plane population
//   (scan_all)       -- per-plane offsets: entries, 256-entry tile pairs,
//                       128-entry chunks
//   (scatter_all)    -- plane lists in brick order
//   plane_boxes      -- box of every 128-entry in-plane chunk + 8 extremes
//   plane_lb         -- exact per-family lower bound from the extremes
//   plane_filter     -- keep in-plane chunk pairs whose box distance reaches it
//                       (tile pairs first, then their 2 x 2 chunk pairs)
//   plane_pass1      -- fp32 dot-form max per surviving unit (+ selection)
//   plane_refine     -- fp64 reference-arithmetic re-check of the candidates
//
// A unit (work entry) is one in-plane chunk pair: uint2 {plane, I << 16 | J}.
// The owning plane of a tile pair / chunk is found by binary search over the
// per-plane offsets, so no per-unit maps are materialised.
#include <climits>

#include "sc_device.cuh"

namespace sc {

constexpr int kPT = kPlaneTile;      // in-plane tile edge (first filter level)
constexpr int kPC = kPlaneChunk;     // in-plane chunk edge (pair unit = chunk x chunk)
constexpr int kPR = kPC / 32;        // 4 i entries per lane in plane_pass1
constexpr int kPlaneThreads = 256;
constexpr int kPlaneWarps = kPlaneThreads / 32;

// Largest p in [0, P) with off[p] <= x (off non-decreasing, off[0] = 0): the
// plane owning global tile pair / chunk x.
__device__ __forceinline__ int find_plane(const unsigned int* __restrict__ off, int P,
                                          unsigned long long x) {
  int lo = 0, hi = P - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((unsigned long long)off[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Per-plane offsets staged in shared memory for the binary searches (volumes
// up to ~2700 voxels per axis summed; larger ones search global memory).
constexpr int kOffSmem = 8192;

__device__ __forceinline__ const unsigned int* stage_offsets(const unsigned int* __restrict__ off,
                                                             int P, unsigned int* s_off) {
  if (P + 1 > kOffSmem) return off;
  for (int i = threadIdx.x; i <= P; i += blockDim.x) s_off[i] = off[i];
  __syncthreads();
  return s_off;
}

__device__ __forceinline__ unsigned int plane_nchunks(unsigned int np) {
  return np >= 2 ? (np + kPC - 1) / kPC : 0u;
}

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

// One warp per in-plane chunk c: its 2-D integer box (lo.a, lo.b, hi.a,
// hi.b) and the plane's 8 arg-extremes (+-a, +-b, +-(a+b), +-(a-b) in the mm
// frame), index = plane-relative entry.
__global__ void plane_boxes(const int2* __restrict__ sorted,
                            const unsigned int* __restrict__ start,
                            const unsigned int* __restrict__ cstart,
                            const RoiParams* __restrict__ rp,
                            const Stats* __restrict__ st, int4* __restrict__ pboxes,
                            unsigned long long* __restrict__ pext) {
  if (st->ovf) return;  // re-run pending (scan_all)
  Frame f = rp->f;
  if (st->bbox[3] < 0) return;
  const PlaneSpace ps = plane_space(st);
  const int P = ps.cnt[0] + ps.cnt[1] + ps.cnt[2];
  const long long chunks = (long long)st->plane_chunks;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  if ((long long)blockIdx.x * (blockDim.x >> 5) >= chunks) return;  // block-uniform
  __shared__ unsigned int s_off[kOffSmem];
  const unsigned int* coff = stage_offsets(cstart, P, s_off);
  for (long long c = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < chunks;
       c += warps) {
    const int p = find_plane(coff, P, (unsigned long long)c);
    const PlaneAxes ax = plane_axes(plane_axis(p, ps), st, f);
    const unsigned int b0 = start[p], np = start[p + 1] - b0;
    const unsigned int e0 = (unsigned int)(c - coff[p]) * kPC;
    const unsigned int e1 = min(np, e0 + kPC);
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

__device__ __forceinline__ int4 box_union(int4 a, int4 b) {
  return make_int4(min(a.x, b.x), min(a.y, b.y), max(a.z, b.z), max(a.w, b.w));
}

// Two levels, like unit_filter: a 256-entry tile pair of a plane (boxes =
// union of its two chunk boxes) is tested against the family's lower bound
// (margin 1e-9 covers fp64 rounding of both sides); only if it can reach it
// are its 2 x 2 chunk pairs tested and listed in pwork.
__global__ void plane_filter(const unsigned int* __restrict__ start,
                             const unsigned int* __restrict__ tstart,
                             const unsigned int* __restrict__ cstart,
                             const int4* __restrict__ pboxes, const RoiParams* __restrict__ rp,
                             int prune, int shard, int nshards, long long wcap,
                             Stats* __restrict__ st, uint2* __restrict__ pwork) {
  if (st->ovf) return;  // re-run pending (scan_all)
  Frame f = rp->f;
  const long long units = (long long)st->plane_units;
  if (st->bbox[3] < 0) return;
  const PlaneSpace ps = plane_space(st);
  const int P = ps.cnt[0] + ps.cnt[1] + ps.cnt[2];
  double thr[3];
#pragma unroll
  for (int a = 0; a < 3; a++)
    thr[a] = __longlong_as_double((long long)st->plb[a]) * (1.0 - 1e-9);
  const int lane = threadIdx.x & 31;
  if ((long long)blockIdx.x * blockDim.x >= units) return;  // block-uniform
  __shared__ unsigned int s_off[kOffSmem];
  const unsigned int* toff = stage_offsets(tstart, P, s_off);
  for (long long base = (long long)blockIdx.x * blockDim.x; base < units;
       base += (long long)gridDim.x * blockDim.x) {
    const long long u = base + threadIdx.x;
    bool coarse = false;
    int p = 0, I = 0, J = 0, nc = 0;
    unsigned int c0 = 0;
    double th = 0.0, hA = 0.0, hB = 0.0;
    if (u < units) {
      p = find_plane(toff, P, (unsigned long long)u);
      const int axis = plane_axis(p, ps);
      const PlaneAxes ax = plane_axes(axis, st, f);
      hA = 0.5 * ax.sa;
      hB = 0.5 * ax.sb;
      th = axis == 0 ? thr[0] : (axis == 1 ? thr[1] : thr[2]);
      const unsigned int np = start[p + 1] - start[p];
      nc = (int)plane_nchunks(np);
      c0 = cstart[p];
      tile_pair(u - toff[p], (np + kPT - 1) / kPT, I, J);
      coarse = true;
      if (prune) {
        int4 bi = pboxes[c0 + 2 * I], bj = pboxes[c0 + 2 * J];
        if (2 * I + 1 < nc) bi = box_union(bi, pboxes[c0 + 2 * I + 1]);
        if (2 * J + 1 < nc) bj = box_union(bj, pboxes[c0 + 2 * J + 1]);
        coarse = reach2(bi.x, bi.z, bj.x, bj.z, hA) + reach2(bi.y, bi.w, bj.y, bj.w, hB) >= th;
      }
    }
    if (!__any_sync(0xffffffffu, coarse)) continue;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int i = 2 * I + h, j0 = 2 * J, j1 = 2 * J + 1;
      bool k0 = false, k1 = false;
      if (coarse && i < nc) {
        // Shards own chunk pairs by identity (coarse unit u, sub-pair), so the
        // split is the same whatever order the lists come out in.
        k0 = j0 >= i && j0 < nc && (u * 4 + 2 * h) % nshards == shard;
        k1 = j1 < nc && (u * 4 + 2 * h + 1) % nshards == shard;  // j1 = 2J + 1 >= i always
        if (prune && (k0 || k1)) {
          const int4 bi = pboxes[c0 + i];
          if (k0) {
            const int4 bj = pboxes[c0 + j0];
            k0 = reach2(bi.x, bi.z, bj.x, bj.z, hA) + reach2(bi.y, bi.w, bj.y, bj.w, hB) >= th;
          }
          if (k1) {
            const int4 bj = pboxes[c0 + j1];
            k1 = reach2(bi.x, bi.z, bj.x, bj.z, hA) + reach2(bi.y, bi.w, bj.y, bj.w, hB) >= th;
          }
        }
      }
      const unsigned int m0 = __ballot_sync(0xffffffffu, k0);
      const unsigned int m1 = __ballot_sync(0xffffffffu, k1);
      if (!(m0 | m1)) continue;
      unsigned long long pos = 0;
      if (lane == 0) pos = atomicAdd(&st->n_pwork, (unsigned long long)(__popc(m0) + __popc(m1)));
      pos = __shfl_sync(0xffffffffu, pos, 0);
      const unsigned int lt = (1u << lane) - 1;
      long long o = (long long)pos + __popc(m0 & lt) + __popc(m1 & lt);
      if (k0) {
        if (o < wcap) pwork[o] = make_uint2((unsigned int)p, ((unsigned int)i << 16) | (unsigned int)j0);
        o++;
      }
      if (k1 && o < wcap)
        pwork[o] = make_uint2((unsigned int)p, ((unsigned int)i << 16) | (unsigned int)j1);
    }
  }
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
__global__ void __launch_bounds__(kPlaneThreads, 4) plane_pass1(
    const int2* __restrict__ sorted, const unsigned int* __restrict__ start,
    const uint2* __restrict__ pwork, const RoiParams* __restrict__ rp,
    long long wcap, float* __restrict__ umax, Stats* __restrict__ st) {
  if (st->ovf) return;  // re-run pending (scan_all)
  Frame f = rp->f;
  __shared__ float4 sj_all[kPlaneWarps][kPC];
  if (st->bbox[3] < 0 || (long long)st->n_pwork > wcap) return;  // host re-runs with room
  const PlaneSpace ps = plane_space(st);
  const long long w0 = 0, w1 = (long long)st->n_pwork;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* sj = sj_all[warp];
  const long long gwarps = (long long)gridDim.x * kPlaneWarps;
  const long long gw = (long long)blockIdx.x * kPlaneWarps + warp;
  const long long per = (w1 - w0 + gwarps - 1) / gwarps;
  const long long wb = w0 + gw * per, we = min(w1, wb + per);
  float run0 = 0.f, run1 = 0.f, run2 = 0.f;  // per-family maxima
  unsigned int prev_p = 0xffffffffu, prev_i = 0xffffffffu;
  float2 a2[kPR / 2], b2[kPR / 2];
  float ni[kPR];
  int axis = 0;
  for (long long w = wb; w < we; w++) {
    const uint2 u = pwork[w];
    const unsigned int p = u.x, I = u.y >> 16, J = u.y & 0xffffu;
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
// kRefineRel of their family's pass-1 maximum in shared memory and re-checks
// each: 128 i entries x two halves of the j chunk.
__global__ void __launch_bounds__(kPlaneThreads) plane_refine(
    const int2* __restrict__ sorted, const unsigned int* __restrict__ start,
    const uint2* __restrict__ pwork, const RoiParams* __restrict__ rp,
    const float* __restrict__ umax, long long wcap, Stats* __restrict__ st) {
  if (st->ovf) return;  // re-run pending (scan_all)
  Frame f = rp->f;
  constexpr int kSplit = kPlaneThreads / kPC, kJ = kPC / kSplit;
  __shared__ double sa[kPC], sb[kPC];
  __shared__ double s_red[kPlaneThreads / 32];
  __shared__ unsigned int s_list[kPlaneThreads];
  __shared__ int s_n;
  if (st->bbox[3] < 0 || (long long)st->n_pwork > wcap) return;
  const PlaneSpace ps = plane_space(st);
  const long long w0 = 0, w1 = (long long)st->n_pwork;
  float tau[3];
#pragma unroll
  for (int a = 0; a < 3; a++) tau[a] = __uint_as_float(st->pl_f32[a]) * (1.f - kRefineRel);
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
      const int a = plane_axis((int)pwork[w].x, ps);
      if (umax[w] >= (a == 0 ? tau[0] : (a == 1 ? tau[1] : tau[2])))
        s_list[atomicAdd(&s_n, 1)] = (unsigned int)w;
    }
    __syncthreads();
    const int cnt = s_n;
    if (threadIdx.x == 0 && cnt) atomicAdd(&st->n_pcand, (unsigned long long)cnt);
    for (int q = 0; q < cnt; q++) {
      const uint2 u = pwork[s_list[q]];
      const unsigned int p = u.x, I = u.y >> 16, J = u.y & 0xffffu;
      const int axis = plane_axis((int)p, ps);
      const PlaneAxes ax = plane_axes(axis, st, f);
      const unsigned int b0 = start[p], np = start[p + 1] - b0;
      const unsigned int i = I * kPC + ti;
      const unsigned int jn = min((unsigned int)kPC, np - J * kPC);
      __syncthreads();  // previous candidate is done with sa/sb/s_red
      if (threadIdx.x < kPC && J * kPC + threadIdx.x < np) {
        const int2 k = sorted[b0 + J * kPC + threadIdx.x];
        sa[threadIdx.x] = ref_coord(k.x, ax.sa);
        sb[threadIdx.x] = ref_coord(k.y, ax.sb);
      }
      __syncthreads();
      double best = 0.0;
      if (i < np) {
        const int2 k = sorted[b0 + i];
        const double ai = ref_coord(k.x, ax.sa), bi = ref_coord(k.y, ax.sb);
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
