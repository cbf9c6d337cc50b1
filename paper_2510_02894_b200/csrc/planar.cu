// Planar maximum diameters (sm_100a): maxima over vertex pairs sharing z
// (XY), y (XZ) or x (YZ), bit-exact with reference features.py:145-147.
//
// Every vertex belongs to three planes, keyed by its doubled lattice
// coordinate (bit-equal fp64 coordinate <=> equal key).  mc_cells histograms
// (plane, in-plane Morton brick) bins, so the counting sort below leaves every
// plane's list spatially compact; then the same three steps as the 3-D pass:
//
//   (scan_all)       -- per plane: in-plane bin offsets and population, then
//                       per-plane offsets: entries, 256-entry tile pairs,
//                       128-entry chunks
//   (scatter_all)    -- plane lists in brick order
//   plane_boxes      -- box of every 128-entry in-plane chunk + 8 extremes
//   plane_lb         -- exact per-family lower bound from the extremes
//   plane_filter     -- keep in-plane chunk pairs whose box distance reaches it
//                       (tile pairs first, then their 2 x 2 chunk pairs)
//   (pass1_planar / refine_planar in pass_bodies.cuh, run inside the fused
//    pass-1 and re-check kernels of passes.cu)
//
// A unit (work entry) is one in-plane chunk pair: uint2 {plane, I << 16 | J}.
// The owning plane of a chunk comes from scatter_all's chunk -> plane map; that
// of a tile pair (plane_filter) by binary search over the per-plane offsets.
#include <climits>

#include "sc_device.cuh"

namespace sc {

constexpr int kPT = kPlaneTile;      // in-plane tile edge (first filter level)
constexpr int kPC = kPlaneChunk;     // in-plane chunk edge (pair unit = chunk x chunk)

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

__device__ __forceinline__ unsigned int order_key32(float v) {  // order-preserving
  const unsigned int b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}


// One warp per in-plane chunk c: its 2-D integer box (lo.a, lo.b, hi.a,
// hi.b) and the plane's 8 arg-extremes (+-a, +-b, +-(a+b), +-(a-b) in the mm
// frame), index = plane-relative entry.
__global__ void plane_boxes(const int2* __restrict__ sorted,
                            const unsigned int* __restrict__ start,
                            const unsigned int* __restrict__ cstart,
                            const RoiParams* __restrict__ rp,
                            const Stats* __restrict__ st, int4* __restrict__ pboxes,
                            unsigned long long* __restrict__ pext, int4* __restrict__ hpboxes,
                            const unsigned int* __restrict__ cmap) {
  pdl_enter();
  KTrace kt_(st, kTrPlaneBoxes);
  if (st->ovf) return;  // re-run pending (scan_all)
  Frame f = rp->f;
  if (st->bbox[3] < 0) return;
  const PlaneSpace ps = plane_space(st);
  const long long chunks = (long long)st->plane_chunks;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  if ((long long)blockIdx.x * (blockDim.x >> 5) >= chunks) return;  // block-uniform
  const unsigned int* coff = cstart;
  for (long long c = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < chunks;
       c += warps) {
    const int p = (int)cmap[c];  // (scatter_all's chunk -> plane map)
    const PlaneAxes ax = plane_axes(plane_axis(p, ps), st, f);
    const unsigned int b0 = start[p], np = start[p + 1] - b0;
    const unsigned int e0 = (unsigned int)(c - coff[p]) * kPC;
    const unsigned int e1 = min(np, e0 + kPC);
    // Boxes of the two 64-entry halves (entries past the end clamp to the
    // last one, as pass 1 does) and their union.
    int la[2] = {INT_MAX, INT_MAX}, lb[2] = {INT_MAX, INT_MAX};
    int ha[2] = {INT_MIN, INT_MIN}, hb[2] = {INT_MIN, INT_MIN};
    unsigned int ek[8], ei[8];  // per lane: best order key and its entry, per extreme
#pragma unroll
    for (int d = 0; d < 8; d++) { ek[d] = 0u; ei[d] = 0u; }
#pragma unroll
    for (int t = 0; t < kPC / 32; t++) {
      const unsigned int e = min(e0 + t * 32 + lane, e1 - 1);
      const int hh = t / (kPC / 64);
      const int2 k = sorted[b0 + e];
      la[hh] = min(la[hh], k.x); lb[hh] = min(lb[hh], k.y);
      ha[hh] = max(ha[hh], k.x); hb[hh] = max(hb[hh], k.y);
      const float a = (float)k.x * ax.ha, b = (float)k.y * ax.hb;
      const float pr[4] = {a, b, a + b, a - b};
#pragma unroll
      for (int d = 0; d < 4; d++) {
        const unsigned int hi = order_key32(pr[d]), lo = order_key32(-pr[d]);
        if (hi > ek[2 * d]) { ek[2 * d] = hi; ei[2 * d] = e; }
        if (lo > ek[2 * d + 1]) { ek[2 * d + 1] = lo; ei[2 * d + 1] = e; }
      }
    }
#pragma unroll
    for (int hh = 0; hh < 2; hh++) {
      la[hh] = __reduce_min_sync(0xffffffffu, la[hh]); lb[hh] = __reduce_min_sync(0xffffffffu, lb[hh]);
      ha[hh] = __reduce_max_sync(0xffffffffu, ha[hh]); hb[hh] = __reduce_max_sync(0xffffffffu, hb[hh]);
    }
    if (lane == 0) {
      pboxes[c] = make_int4(min(la[0], la[1]), min(lb[0], lb[1]), max(ha[0], ha[1]),
                            max(hb[0], hb[1]));
      hpboxes[2 * c] = make_int4(la[0], lb[0], ha[0], hb[0]);
      hpboxes[2 * c + 1] = make_int4(la[1], lb[1], ha[1], hb[1]);
    }
    // warp arg-max per extreme: hardware u32 max-reduce, the owner by ballot
#pragma unroll
    for (int d = 0; d < 8; d++) {
      const unsigned int m = __reduce_max_sync(0xffffffffu, ek[d]);
      const int owner = __ffs(__ballot_sync(0xffffffffu, ek[d] == m)) - 1;
      const unsigned int idx = __shfl_sync(0xffffffffu, ei[d], owner);
      if (lane == 0 && m)
        atomicMax(&pext[(long long)p * 8 + d], ((unsigned long long)m << 32) | idx);
    }
  }
}

// One warp per plane: the exact (reference arithmetic) max over the 28 pairs
// of its 8 extreme entries -- a real pair, so it bounds that family's maximum
// from below and seeds it.
__global__ void plane_lb(const int2* __restrict__ sorted, const unsigned int* __restrict__ start,
                         const unsigned long long* __restrict__ pext, const RoiParams* __restrict__ rp,
                         Stats* __restrict__ st) {
  pdl_enter();
  KTrace kt_(st, kTrPlaneLb);
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
      const double da = __dsub_rn(ref_coord(kj.x + ax.oa, ax.sa), ref_coord(ki.x + ax.oa, ax.sa));
      const double db = __dsub_rn(ref_coord(kj.y + ax.ob, ax.sb), ref_coord(ki.y + ax.ob, ax.sb));
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
__global__ void __launch_bounds__(256, 4) plane_filter(const unsigned int* __restrict__ start,
                             const unsigned int* __restrict__ tstart,
                             const unsigned int* __restrict__ cstart,
                             const int4* __restrict__ pboxes, const RoiParams* __restrict__ rp,
                             int prune, int shard, int nshards, long long wcap,
                             Stats* __restrict__ st, uint2* __restrict__ pwork,
                             const int4* __restrict__ hpboxes) {
  pdl_enter();
  KTrace kt_(st, kTrPlaneFilter);
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
        // Shards own whole planes (plane index mod N): every pair of a plane
        // is evaluated by one shard, so the split is exact whatever order the
        // plane's entries come out in on each GPU (no canonical planar order).
        const bool own = p % nshards == shard;
        k0 = own && j0 >= i && j0 < nc;
        k1 = own && j1 < nc;  // j1 = 2J + 1 >= i always
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
      // 64 x 64 sub-pairs that can reach the bound (bit 2a + b; for i == j
      // the mirrored (1, 0) repeats (0, 1)); 0xF = whole unit without pruning.
      unsigned int s0 = 0xFu, s1 = 0xFu;
      if (prune && (k0 || k1)) {
        auto subs = [&](int ci, int cj) {
          unsigned int m = 0u;
#pragma unroll
          for (int a = 0; a < 2; a++)
#pragma unroll
            for (int b = 0; b < 2; b++) {
              if (ci == cj && a == 1 && b == 0) continue;
              const int4 bi = hpboxes[2 * (c0 + ci) + a], bj = hpboxes[2 * (c0 + cj) + b];
              if (reach2(bi.x, bi.z, bj.x, bj.z, hA) + reach2(bi.y, bi.w, bj.y, bj.w, hB) >= th)
                m |= 1u << (2 * a + b);
            }
          return m;
        };
        if (k0) { s0 = subs(i, j0); k0 = s0 != 0u; }
        if (k1) { s1 = subs(i, j1); k1 = s1 != 0u; }
      }
      const unsigned int m0 = __ballot_sync(0xffffffffu, k0);
      const unsigned int m1 = __ballot_sync(0xffffffffu, k1);
      if (!(m0 | m1)) continue;
      const unsigned int nsub =
          __reduce_add_sync(0xffffffffu, (k0 ? __popc(s0) : 0u) + (k1 ? __popc(s1) : 0u));
      unsigned long long pos = 0;
      if (lane == 0) {
        pos = atomicAdd(&st->n_pwork, (unsigned long long)(__popc(m0) + __popc(m1)));
        atomicAdd(&st->n_psub, (unsigned long long)nsub);
      }
      pos = __shfl_sync(0xffffffffu, pos, 0);
      const unsigned int lt = (1u << lane) - 1;
      long long o = (long long)pos + __popc(m0 & lt) + __popc(m1 & lt);
      if (k0) {
        if (o < wcap)
          pwork[o] = make_uint2((unsigned int)p | (s0 << kSubShift),
                                ((unsigned int)i << 16) | (unsigned int)j0);
        o++;
      }
      if (k1 && o < wcap)
        pwork[o] = make_uint2((unsigned int)p | (s1 << kSubShift),
                              ((unsigned int)i << 16) | (unsigned int)j1);
    }
  }
}

}  // namespace sc
