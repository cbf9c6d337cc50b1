// Vertex ordering and exact work pruning for the diameter stage (sm_100a).
//
// The maximum pair distance D^2 is at least LB = the largest exact pair value
// among a few extreme vertices (13 directions, both ends).  After a Morton
// brick ordering of the vertices, every 128-vertex chunk is spatially compact,
// so most chunk pairs have an upper bound UB^2 = max distance^2 between their
// boxes below LB: they cannot hold the maximum pair and are not evaluated.  Surviving units run through
// diam3d_pass1 and the fp64 re-check keeps the result bit-identical to the
// reference's all-pairs loop (features.py:121-192).
//
//   scan_all        -- block 0: brick offsets; block 1: plane offsets, in-plane
//                      tile-pair offsets and the unit -> plane map
//   scatter_all     -- counting-sort scatter: keys by brick, plane coordinates
//                      by plane (histograms were built by mc_cells)
//   boxes_extremes  -- integer box of every 256-chunk + 13-direction extremes
//   unit_filter     -- exact LB, compact the surviving chunk pairs
#include <climits>

#include "sc_device.cuh"

namespace sc {

constexpr int kChunkV = kChunk3;
constexpr int kPerLane = kChunkV / 32;
constexpr int kSuper = 8;  // super-chunk = 8 chunks (1024 vertices): first level of unit_filter
// kSingleLevelMax (sc_device.cuh): chunk pairs tested directly (one level) up
// to this many; above it the super-chunk level goes first.  Two levels pay off
// from ~300 chunks on (C2 batch 42.5 -> 41.8 us/ROI, C5 30.9 -> 27.8 moving the
// switch from 2^22 to 2^16 pairs): fewer warp-slot microseconds per ROI.
constexpr int kNDir = 13;

__device__ __forceinline__ long long n_verts(const Stats* st, long long cap) {
  long long n = (long long)st->n_vert;
  return n < cap ? n : cap;
}

__device__ __forceinline__ unsigned int plane_tiles(unsigned int np, int pt) {
  if (np < 2) return 0u;
  const unsigned int t = (np + pt - 1) / pt;
  return t * (t + 1) / 2;
}

// kScanBlocks brick blocks + plane blocks, kScanThreads threads each.  Brick
// blocks: kScanSlices 1024-bin slices each (16 bins per thread, 128-bit loads)
// of the exclusive scan of the brick counts -> sort cursor (and zero the
// counts for the next ROI), plus empty super-chunk boxes.  Plane blocks: one
// warp per plane scans its in-plane bins; the last plane block to finish turns
// the plane populations into offsets: entries -> start, 256-entry tile pairs
// -> tstart, 128-entry chunks -> cstart.
__global__ void __launch_bounds__(kScanThreads) scan_all(unsigned int* __restrict__ sort_counts,
                                                         unsigned int* __restrict__ sort_cursor,
                                                         unsigned int* __restrict__ plane_counts,
                                                         unsigned int* __restrict__ start,
                                                         unsigned int* __restrict__ tstart,
                                                         unsigned int* __restrict__ cstart,
                                                         long long dcap, Stats* __restrict__ st,
                                                         int4* __restrict__ sboxes,
                                                         unsigned int* __restrict__ pbin_counts,
                                                         unsigned int* __restrict__ pbin_cursor,
                                                         unsigned long long* __restrict__ pext,
                                                         int full_cursor) {
  pdl_enter();
  KTrace kt_(st, kTrScan);
  if (blockIdx.x == 0 && threadIdx.x == 0) st->t_mesh = global_ns();  // marching cubes done
  int bb[6];
#pragma unroll
  for (int i = 0; i < 6; i++) bb[i] = st->bbox[i];
  if (bb[3] < 0) return;
  const bool brick_block = blockIdx.x < kScanBlocks;
  if (!brick_block) {
    // Plane blocks: one warp per plane -- exclusive offsets of its in-plane
    // bins (pbin_cursor, plane-relative), its population (plane_counts), reset
    // of its bins and extremes for the next ROI; then the last plane block to
    // finish derives the per-plane offsets (start / tstart / cstart).
    const PlaneSpace ps = plane_space(bb);
    const int P = ps.cnt[0] + ps.cnt[1] + ps.cnt[2];
    const int lane = threadIdx.x & 31;
    const int nwarps = (int)(gridDim.x - kScanBlocks) * (blockDim.x >> 5);
    for (int p = (int)(blockIdx.x - kScanBlocks) * (blockDim.x >> 5) + (threadIdx.x >> 5); p < P;
         p += nwarps) {
      // 8 bins per lane as two 16-byte accesses (scalar 4-byte accesses
      // strided by 32 B across the warp cost 8x the L2 sector requests)
      uint4* cnt4 = reinterpret_cast<uint4*>(pbin_counts + (long long)p * kPlaneBins + lane * 8);
      const uint4 c0 = cnt4[0], c1 = cnt4[1];
      const unsigned int v[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      unsigned int sum = 0;
#pragma unroll
      for (int k = 0; k < 8; k++) sum += v[k];
      cnt4[0] = make_uint4(0u, 0u, 0u, 0u);
      cnt4[1] = make_uint4(0u, 0u, 0u, 0u);
      unsigned int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      unsigned int run = incl - sum;
      unsigned int o[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        o[k] = run;
        run += v[k];
      }
      uint4* cur4 = reinterpret_cast<uint4*>(pbin_cursor + (long long)p * kPlaneBins + lane * 8);
      cur4[0] = make_uint4(o[0], o[1], o[2], o[3]);
      cur4[1] = make_uint4(o[4], o[5], o[6], o[7]);
      if (lane == 31) {
        plane_counts[p] = incl;
        // planar work entries index a plane's 128-entry chunks with 16 bits:
        // a larger plane stops the ROI (the host reports it as an input error)
        if ((long long)incl > kPlaneMaxEntries) {
          st->plane_ovf = 1u;
          st->ovf = 1u;
        }
      }
      if (lane < 8) pext[(long long)p * 8 + lane] = 0ull;
    }
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(&st->done1, 1u) == gridDim.x - kScanBlocks - 1;
    }
    __syncthreads();
    if (!s_last || (long long)st->n_vert > dcap) return;  // overflow: later kernels stand down
    __threadfence();
  }
  constexpr int kPerThread = (kScanSlices << kSortSliceBits) / kScanThreads;  // 16 bins
  static_assert(kPerThread % 4 == 0, "bins are moved as uint4");
  uint4* cnt4 = reinterpret_cast<uint4*>(
      sort_counts + (long long)blockIdx.x * (kScanSlices << kSortSliceBits) + threadIdx.x * kPerThread);
  // More vertices than the diameter-side buffers hold: every later kernel
  // stands down (positions from the full histograms would overflow) and the
  // host re-runs the ROI with exact sizes.
  if (brick_block && (long long)st->n_vert > dcap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) st->ovf = 1u;
    // still leave the brick histogram zeroed for the next ROI
#pragma unroll
    for (int k = 0; k < kPerThread / 4; k++) cnt4[k] = make_uint4(0u, 0u, 0u, 0u);
    return;
  }
  if (brick_block) {
    {  // empty super-chunk boxes, filled by boxes_extremes with atomics
      const long long n = (long long)st->n_vert;
      const long long CT = ((n + kChunkV - 1) / kChunkV + kSuper - 1) / kSuper;
      for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < CT;
           t += (long long)kScanBlocks * blockDim.x) {  // (brick blocks only)
        sboxes[2 * t] = make_int4(INT_MAX, INT_MAX, INT_MAX, 0);
        sboxes[2 * t + 1] = make_int4(INT_MIN, INT_MIN, INT_MIN, 0);
      }
    }
    // Block base = super-bin prefix of its first slice; within the block one
    // scan over its kScanSlices slices (the super bins are their sums).
    const unsigned int* sup = sort_counts + kSortBins;
    // No vertex in this block's slices (block-uniform): its counts are still
    // zero and no vertex will look up its cursors -- nothing to write.  (Most
    // slices of a small or thin-shelled ROI's Morton range.)
    bool any = false;
#pragma unroll
    for (int i = 0; i < kScanSlices; i++) any |= sup[kScanSlices * blockIdx.x + i] != 0u;
    // (the shard entry's canonical order reads every bin's cursor: write them all)
    if (!any && !full_cursor) return;
    unsigned int base;
    block_exscan(threadIdx.x < kScanSlices * blockIdx.x ? sup[threadIdx.x] : 0u, &base);
    uint4 v[kPerThread / 4];
    unsigned int sum = 0;
#pragma unroll
    for (int k = 0; k < kPerThread / 4; k++) {
      v[k] = cnt4[k];
      sum += v[k].x + v[k].y + v[k].z + v[k].w;
    }
    unsigned int total;
    unsigned int run = base + block_exscan(sum, &total);
    uint4* cur4 = reinterpret_cast<uint4*>(
        sort_cursor + (long long)blockIdx.x * (kScanSlices << kSortSliceBits) + threadIdx.x * kPerThread);
#pragma unroll
    for (int k = 0; k < kPerThread / 4; k++) {
      uint4 o;
      o.x = run; run += v[k].x;
      o.y = run; run += v[k].y;
      o.z = run; run += v[k].z;
      o.w = run; run += v[k].w;
      cur4[k] = o;
      cnt4[k] = make_uint4(0u, 0u, 0u, 0u);
    }
    return;
  }
  const PlaneSpace ps = plane_space(bb);
  const int P = ps.cnt[0] + ps.cnt[1] + ps.cnt[2];
  const int per = (P + kScanThreads - 1) / kScanThreads;
  const int b = threadIdx.x * per, e = min(P, b + per);
  unsigned int s1 = 0, s2 = 0, s3 = 0;
  for (int i = b; i < e; i++) {
    const unsigned int v = plane_counts[i];
    s1 += v;
    s2 += plane_tiles(v, kPlaneTile);
    s3 += v >= 2 ? (v + kPlaneChunk - 1) / kPlaneChunk : 0u;
  }
  unsigned int t1, t2, t3;
  unsigned int r1 = block_exscan(s1, &t1);
  unsigned int r2 = block_exscan(s2, &t2);
  unsigned int r3 = block_exscan(s3, &t3);
  for (int i = b; i < e; i++) {
    const unsigned int v = plane_counts[i];
    const unsigned int nch = v >= 2 ? (v + kPlaneChunk - 1) / kPlaneChunk : 0u;
    start[i] = r1;
    tstart[i] = r2;
    cstart[i] = r3;
    r1 += v;
    r2 += plane_tiles(v, kPlaneTile);
    r3 += nch;
  }
  if (threadIdx.x == 0) {
    start[P] = t1;
    tstart[P] = t2;
    cstart[P] = t3;
    st->plane_units = t2;
    st->plane_chunks = t3;
  }
}

// Counting-sort scatter: keys into Morton-brick order (keys_sorted), and the
// in-plane coordinates of every vertex into its three plane lists, each in
// in-plane brick order: XY -> (X, Y), XZ -> (X, Z), YZ -> (Y, Z).
__global__ void scatter_all(const int4* __restrict__ keys, long long cap,
                            const Stats* __restrict__ st, unsigned int* __restrict__ sort_cursor,
                            int4* __restrict__ keys_sorted,
                            const unsigned int* __restrict__ plane_start,
                            unsigned int* __restrict__ pbin_cursor,
                            int2* __restrict__ plane_sorted,
                            unsigned int* __restrict__ sort_supers,
                            const unsigned int* __restrict__ cstart,
                            unsigned int* __restrict__ cmap) {
  pdl_enter();
  KTrace kt_(st, kTrScatter);
  // scan_all has consumed the super-bin counts: leave them zeroed for the next ROI.
  if (blockIdx.x == 0) sort_supers[threadIdx.x] = 0u;
  if (st->ovf) return;  // re-run pending (scan_all)
  const long long n = n_verts(st, cap);
  int bb[6];
#pragma unroll
  for (int i = 0; i < 6; i++) bb[i] = st->bbox[i];
  const int s = brick_shift(bb);
  const PlaneSpace ps = plane_space(bb);
  const PlaneBricks pbk = plane_bricks(bb);
  {  // in-plane chunk -> plane map for plane_boxes (one search per chunk here
     // instead of one per chunk-warp there)
    const int P = ps.cnt[0] + ps.cnt[1] + ps.cnt[2];
    const long long nch = (long long)st->plane_chunks;
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < nch;
         c += (long long)gridDim.x * blockDim.x)
      cmap[c] = (unsigned int)find_plane(cstart, P, (unsigned long long)c);
  }
  // Two vertices per thread per step (the second one grid-stride away), so
  // the key loads, cursor atomics and start loads of both are in flight
  // together: the loop is a chain of dependent memory round trips.
  constexpr int kU = 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < n; base += kU * stride) {
    bool ok[kU];
    int4 k[kU];
    int id[kU][3];
    unsigned int pb[kU][3], bin[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
      const long long v = base + u * stride + threadIdx.x;
      ok[u] = v < n;
      k[u] = ok[u] ? keys[v] : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kU; u++) {
      bin[u] = brick_bin(k[u].x, k[u].y, k[u].z, bb, s);
      plane_ids(k[u].x, k[u].y, k[u].z, ps, id[u]);
      plane_bins(k[u].x, k[u].y, k[u].z, pbk, pb[u]);
    }
    unsigned int pk[kU], pos[kU][3];
#pragma unroll
    for (int u = 0; u < kU; u++) {
      pk[u] = seg_add(sort_cursor, bin[u], ok[u]);
#pragma unroll
      for (int a = 0; a < 3; a++)
        pos[u][a] = seg_add(pbin_cursor, (unsigned int)id[u][a] * kPlaneBins + pb[u][a], ok[u]) +
                    (ok[u] ? plane_start[id[u][a]] : 0u);
    }
#pragma unroll
    for (int u = 0; u < kU; u++)
      if (ok[u]) {
        keys_sorted[pk[u]] = k[u];
        plane_sorted[pos[u][0]] = make_int2(k[u].x, k[u].y);
        plane_sorted[pos[u][1]] = make_int2(k[u].x, k[u].z);
        plane_sorted[pos[u][2]] = make_int2(k[u].y, k[u].z);
      }
  }
}

// 13 directions; projections in the (un-centred) mm frame.  Arg-extremes are
// reduced as packed (order-preserving value bits, vertex index).
// The components are -1 / 0 / 1 and the direction loop is unrolled, so every
// projection compiles to at most two adds.
__device__ __forceinline__ float dir_proj(int d, float x, float y, float z) {
  constexpr int kDir[kNDir][3] = {{1, 0, 0},  {0, 1, 0},  {0, 0, 1},  {1, 1, 0},  {1, -1, 0},
                                  {1, 0, 1},  {1, 0, -1}, {0, 1, 1},  {0, 1, -1}, {1, 1, 1},
                                  {1, 1, -1}, {1, -1, 1}, {-1, 1, 1}};
  float p = 0.f;
  if (kDir[d][0]) p += kDir[d][0] > 0 ? x : -x;
  if (kDir[d][1]) p += kDir[d][1] > 0 ? y : -y;
  if (kDir[d][2]) p += kDir[d][2] > 0 ? z : -z;
  return p;
}

__device__ __forceinline__ unsigned int order_key(float v) {  // order-preserving, never 0 for finite v
  const unsigned int b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// One warp per 256-chunk of the sorted keys: its integer box (boxes[2c] = lo,
// boxes[2c+1] = hi) and its contribution to the 26 arg-extremes.
__global__ void __launch_bounds__(256) boxes_extremes(const int4* __restrict__ keys,
                                                      long long cap, const RoiParams* __restrict__ rp,
                                                      Stats* __restrict__ st,
                                                      int4* __restrict__ boxes,
                                                      int4* __restrict__ sboxes,
                                                      int4* __restrict__ hboxes,
                                                      float4* __restrict__ fkeys) {
  pdl_enter();
  KTrace kt_(st, kTrBoxes);
  if (st->ovf) return;  // re-run pending (scan_all)
  Frame f = rp->f;
  Frame fc = f;  // pass 1's bbox-centred frame
  frame_centre(st, fc);
  __shared__ unsigned long long s_ext[2 * kNDir];
  if (threadIdx.x < 2 * kNDir) s_ext[threadIdx.x] = 0ull;
  __syncthreads();
  const long long n = n_verts(st, cap);
  const long long chunks = (n + kChunkV - 1) / kChunkV;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long c = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < chunks;
       c += warps) {
    // Boxes of the two 64-vertex halves (t = 0,1 and t = 2,3), and their union.
    int l[2][3], u[2][3];
    float px[kPerLane], py[kPerLane], pz[kPerLane];
    unsigned int idx[kPerLane];
#pragma unroll
    for (int hh = 0; hh < 2; hh++)
#pragma unroll
      for (int a = 0; a < 3; a++) { l[hh][a] = INT_MAX; u[hh][a] = INT_MIN; }
#pragma unroll
    for (int t = 0; t < kPerLane; t++) {
      long long v = c * kChunkV + t * 32 + lane;
      const bool real = v < n;
      if (v >= n) v = n - 1;  // pass 1 clamps the same way
      const int4 k = keys[v];
      if (real) {  // pass-1 operand (x, y, z, |p|^2), formed once per vertex
        const float3 q = frame_coord(k, fc);
        fkeys[v] = make_float4(q.x, q.y, q.z, fmaf(q.x, q.x, fmaf(q.y, q.y, q.z * q.z)));
      }
      const int hh = t / (kPerLane / 2);
      l[hh][0] = min(l[hh][0], k.x); l[hh][1] = min(l[hh][1], k.y); l[hh][2] = min(l[hh][2], k.z);
      u[hh][0] = max(u[hh][0], k.x); u[hh][1] = max(u[hh][1], k.y); u[hh][2] = max(u[hh][2], k.z);
      px[t] = (float)k.x * f.hx; py[t] = (float)k.y * f.hy; pz[t] = (float)k.z * f.hz;
      idx[t] = (unsigned int)v;
    }
#pragma unroll
    for (int hh = 0; hh < 2; hh++)
#pragma unroll
      for (int a = 0; a < 3; a++) {
        l[hh][a] = __reduce_min_sync(0xffffffffu, l[hh][a]);
        u[hh][a] = __reduce_max_sync(0xffffffffu, u[hh][a]);
      }
    const int lx = min(l[0][0], l[1][0]), ly = min(l[0][1], l[1][1]), lz = min(l[0][2], l[1][2]);
    const int hx = max(u[0][0], u[1][0]), hy = max(u[0][1], u[1][1]), hz = max(u[0][2], u[1][2]);
    if (lane == 0) {
      boxes[2 * c] = make_int4(lx, ly, lz, 0);
      boxes[2 * c + 1] = make_int4(hx, hy, hz, 0);
      hboxes[4 * c] = make_int4(l[0][0], l[0][1], l[0][2], 0);
      hboxes[4 * c + 1] = make_int4(u[0][0], u[0][1], u[0][2], 0);
      hboxes[4 * c + 2] = make_int4(l[1][0], l[1][1], l[1][2], 0);
      hboxes[4 * c + 3] = make_int4(u[1][0], u[1][1], u[1][2], 0);
      int* slo = reinterpret_cast<int*>(sboxes + 2 * (c / kSuper));
      int* shi = reinterpret_cast<int*>(sboxes + 2 * (c / kSuper) + 1);
      atomicMin(slo, lx); atomicMin(slo + 1, ly); atomicMin(slo + 2, lz);
      atomicMax(shi, hx); atomicMax(shi + 1, hy); atomicMax(shi + 2, hz);
    }
#pragma unroll
    for (int d = 0; d < kNDir; d++) {
      // Per lane: largest and smallest projection (and their vertices);
      // warp: hardware u32 max-reduce of order-preserving keys, the owning lane
      // found by ballot.
      float phi = -3.0e38f, plo = 3.0e38f;
      unsigned int ihi = 0u, ilo = 0u;
#pragma unroll
      for (int t = 0; t < kPerLane; t++) {
        const float p = dir_proj(d, px[t], py[t], pz[t]);
        if (p > phi) { phi = p; ihi = idx[t]; }
        if (p < plo) { plo = p; ilo = idx[t]; }
      }
      const unsigned int khi = order_key(phi), klo = order_key(-plo);
      const unsigned int mhi = __reduce_max_sync(0xffffffffu, khi);
      const unsigned int mlo = __reduce_max_sync(0xffffffffu, klo);
      const int shi = __ffs(__ballot_sync(0xffffffffu, khi == mhi)) - 1;
      const int slo = __ffs(__ballot_sync(0xffffffffu, klo == mlo)) - 1;
      ihi = __shfl_sync(0xffffffffu, ihi, shi);
      ilo = __shfl_sync(0xffffffffu, ilo, slo);
      if (lane == 0) {
        atomicMax(&s_ext[2 * d], ((unsigned long long)mhi << 32) | ihi);
        atomicMax(&s_ext[2 * d + 1], ((unsigned long long)mlo << 32) | ilo);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * kNDir && s_ext[threadIdx.x])
    atomicMax(&st->ext[threadIdx.x], s_ext[threadIdx.x]);
  // The last block to finish turns the 26 extremes into the exact lower bound
  // LB = max exact (reference fp64 arithmetic) squared distance among them --
  // a real pair, so LB <= D^2; it also seeds the exact 3-D maximum.  (Once
  // here instead of in every unit_filter block.)
  if (!last_block(&st->done3) || n == 0) return;
  __shared__ double qx[2 * kNDir], qy[2 * kNDir], qz[2 * kNDir];
  __shared__ double s_lb[32];
  if (threadIdx.x < 2 * kNDir) {
    const unsigned int ix = (unsigned int)(__ldcg(&st->ext[threadIdx.x]) & 0xffffffffu);
    const int4 k = keys[ix < n ? ix : n - 1];
    qx[threadIdx.x] = ref_coord(k.x + f.ox2, f.sx);
    qy[threadIdx.x] = ref_coord(k.y + f.oy2, f.sy);
    qz[threadIdx.x] = ref_coord(k.z + f.oz2, f.sz);
  }
  __syncthreads();
  double lb = 0.0;
  for (int p = threadIdx.x; p < 4 * kNDir * kNDir; p += blockDim.x) {
    const int i = p / (2 * kNDir), j = p % (2 * kNDir);
    lb = fmax(lb, ref_sq_dist(qx[i], qy[i], qz[i], qx[j], qy[j], qz[j]));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) lb = fmax(lb, __shfl_xor_sync(0xffffffffu, lb, o));
  if (lane == 0) s_lb[threadIdx.x >> 5] = lb;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++) lb = fmax(lb, s_lb[w]);
    if (lb > 0.0) {
      atomic_max_pos_f64(&st->lb, lb);
      atomic_max_pos_f64(&st->sq[0], lb);
    }
  }
}

__device__ __forceinline__ double axis_reach(int loA, int hiA, int loB, int hiB, double h) {
  const double d = (double)max(hiA - loB, hiB - loA) * h;
  return d * d;
}

// Per-launch constants of the chunk-pair test (unit_filter / unit_expand).
struct PairTest {
  const int4* boxes;
  const int4* hboxes;
  Stats* st;
  uint2* work;
  double h3[3];
  double thr;
  long long C, wcap;
  int prune, shard, nshards;
};

__device__ __forceinline__ double box_reach(const PairTest& F, int4 alo, int4 ahi, int4 blo,
                                            int4 bhi) {
  return axis_reach(alo.x, ahi.x, blo.x, bhi.x, F.h3[0]) +
         axis_reach(alo.y, ahi.y, blo.y, bhi.y, F.h3[1]) +
         axis_reach(alo.z, ahi.z, blo.z, bhi.z, F.h3[2]);
}

// Which 64 x 64 sub-pairs of a kept chunk pair (i, j) can reach LB (bit
// 2a + b, half a of i, half b of j; for i == j the mirrored (1, 0) is the same
// pairs as (0, 1)).
__device__ __forceinline__ unsigned int sub_mask(const PairTest& F, int i, int j) {
  unsigned int m = 0u;
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int b = 0; b < 2; b++)
      if (!(i == j && a == 1 && b == 0) &&
          box_reach(F, F.hboxes[4 * i + 2 * a], F.hboxes[4 * i + 2 * a + 1],
                    F.hboxes[4 * j + 2 * b], F.hboxes[4 * j + 2 * b + 1]) >= F.thr)
        m |= 1u << (2 * a + b);
  return m;
}

// One chunk pair per lane (all 32 lanes call): shard ownership by the pair's
// identity (its tile_pair index, so the split is the same whatever order the
// lists come out in), the box test, the sub-pair mask, and a warp-aggregated
// append of the kept units.
__device__ __forceinline__ void test_chunk_pair(const PairTest& F, bool valid, int i, int j) {
  const int lane = threadIdx.x & 31;
  bool keep = valid && i < F.C && j < F.C && j >= i &&
              ((long long)i * F.C - (long long)i * (i - 1) / 2 + (j - i)) % F.nshards == F.shard;
  if (keep && F.prune)
    keep = box_reach(F, F.boxes[2 * i], F.boxes[2 * i + 1], F.boxes[2 * j], F.boxes[2 * j + 1]) >=
           F.thr;
  unsigned int sub = 0xFu;
  if (keep && F.prune) {
    sub = sub_mask(F, i, j);
    keep = sub != 0u;
  }
  const unsigned int mask = __ballot_sync(0xffffffffu, keep);
  if (!mask) return;
  const unsigned int nsub = __reduce_add_sync(0xffffffffu, keep ? __popc(sub) : 0u);
  unsigned long long pos = 0;
  if (lane == 0) {
    pos = atomicAdd(&F.st->n_work, (unsigned long long)__popc(mask));
    atomicAdd(&F.st->n_sub, (unsigned long long)nsub);
  }
  pos = __shfl_sync(0xffffffffu, pos, 0);
  const long long o = (long long)pos + __popc(mask & ((1u << lane) - 1));
  if (keep && o < F.wcap)
    F.work[o] = make_uint2((unsigned int)i, (unsigned int)j | (sub << kSubShift));
}

// Every chunk pair (I <= J) is kept iff the max distance between the two
// chunk boxes can reach LB (from boxes_extremes); survivors are compacted
// into `work` (pair index t over the C x C upper triangle).
__global__ void __launch_bounds__(256) unit_filter(const int4* __restrict__ keys,
                                                   const int4* __restrict__ boxes, long long cap,
                                                   const RoiParams* __restrict__ rp, int prune,
                                                   int shard, int nshards, Stats* __restrict__ st,
                                                   uint2* __restrict__ work,
                                                   const int4* __restrict__ sboxes,
                                                   const int4* __restrict__ hboxes,
                                                   uint2* __restrict__ slist, long long scap) {
  pdl_enter();
  KTrace kt_(st, kTrUnitFilter);
  if (st->ovf) return;  // re-run pending (scan_all)
  Frame f = rp->f;
  const long long n = n_verts(st, cap);
  if (n == 0) return;
  const double lb = __longlong_as_double((long long)st->lb);  // boxes_extremes' last block
  const double thr = lb * (1.0 - 1e-9);  // UB and LB are exact up to fp64 rounding
  // Two levels: a pair of super-chunks (8 chunks = 1024 vertices, boxes from
  // boxes_extremes) is tested first; only if it can reach LB are its (up to
  // 64) chunk pairs tested -- by unit_expand, one thread per chunk pair.
  const long long C = (n + kChunkV - 1) / kChunkV;
  const long long CT = (C + kSuper - 1) / kSuper;
  const long long units = CT * (CT + 1) / 2;
  PairTest F{boxes, hboxes, st, work, {0.5 * f.sx, 0.5 * f.sy, 0.5 * f.sz}, thr, C, rp->wcap,
             prune, shard, nshards};
  const int lane = threadIdx.x & 31;
  const long long fine_units = C * (C + 1) / 2;
  if (fine_units <= kSingleLevelMax) {
    // Small ROI: every chunk pair tested directly, listed in tile_pair order.
    for (long long base = (long long)blockIdx.x * blockDim.x; base < fine_units;
         base += (long long)gridDim.x * blockDim.x) {
      const long long u = base + threadIdx.x;
      int i = 0, j = 0;
      if (u < fine_units) tile_pair(u, C, i, j);
      test_chunk_pair(F, u < fine_units, i, j);
    }
    return;
  }
  // Large ROI: list the surviving super pairs (warp-aggregated append).
  for (long long base = (long long)blockIdx.x * blockDim.x; base < units;
       base += (long long)gridDim.x * blockDim.x) {
    const long long u = base + threadIdx.x;
    bool coarse = false;
    int IT = 0, JT = 0;
    if (u < units) {
      tile_pair(u, CT, IT, JT);
      coarse = !prune || box_reach(F, sboxes[2 * IT], sboxes[2 * IT + 1], sboxes[2 * JT],
                                   sboxes[2 * JT + 1]) >= thr;
    }
    const unsigned int cm = __ballot_sync(0xffffffffu, coarse);
    if (!cm) continue;
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(&st->n_super, (unsigned long long)__popc(cm));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    const long long o = (long long)pos + __popc(cm & ((1u << lane) - 1));
    if (coarse && o < scap) slist[o] = make_uint2((unsigned int)IT, (unsigned int)JT);
  }
}

// Second level of the large-ROI filter: every chunk pair of every listed super
// pair, one per thread (lanes 0-31 of a warp = 32 of one super pair's 64), so
// no warp walks a serial chain of survivors.
__global__ void __launch_bounds__(256) unit_expand(const int4* __restrict__ boxes, long long cap,
                                                   const RoiParams* __restrict__ rp, int prune,
                                                   int shard, int nshards, Stats* __restrict__ st,
                                                   uint2* __restrict__ work,
                                                   const int4* __restrict__ hboxes,
                                                   const uint2* __restrict__ slist,
                                                   long long scap) {
  pdl_enter();
  KTrace kt_(st, kTrUnitExpand);
  if (st->ovf) return;
  const long long ns = min((long long)st->n_super, scap);
  if (ns == 0) return;  // small ROI: unit_filter listed everything itself
  const Frame f = rp->f;
  const long long n = n_verts(st, cap);
  const long long C = (n + kChunkV - 1) / kChunkV;
  const double lb = __longlong_as_double((long long)st->lb);
  PairTest F{boxes, hboxes, st, work, {0.5 * f.sx, 0.5 * f.sy, 0.5 * f.sz}, lb * (1.0 - 1e-9),
             C, rp->wcap, prune, shard, nshards};
  const long long total = ns * (kSuper * kSuper);
  for (long long base = (long long)blockIdx.x * blockDim.x; base < total;
       base += (long long)gridDim.x * blockDim.x) {
    const long long t = base + threadIdx.x;
    const bool valid = t < total;
    int i = 0, j = 0;
    if (valid) {
      const uint2 sp = slist[t >> 6];
      const int r = (int)(t & 63);
      i = kSuper * (int)sp.x + (r >> 3);
      j = kSuper * (int)sp.y + (r & 7);
    }
    test_chunk_pair(F, valid, i, j);
  }
}

}  // namespace sc

namespace sc {

// ---- canonical vertex order (shard entry only) ------------------------------
// scatter_all places the vertices of one brick bin (and the entries of one
// in-plane bin) in atomic-arrival order, which differs run to run.  The pair-
// grid shards of one ROI run on different GPUs (or one after another), and a
// shard owns chunk pairs by their IDENTITY (prune.cu test_chunk_pair,
// planar.cu plane_filter): that partition covers every vertex pair exactly
// once only if every shard sees the same vertex -> chunk assignment.  These
// kernels sort each bin's segment by the vertex key (a total order), so the
// order after them is a function of the mask alone.  Segment bounds are found
// from the data itself: bins are contiguous and ascending after the scatter.

__device__ __forceinline__ bool key_less(int4 a, int4 b) {
  if (a.z != b.z) return a.z < b.z;
  if (a.y != b.y) return a.y < b.y;
  return a.x < b.x;
}

// Warp-stable LSD radix sort of one segment [lo, hi) by a W-bit local key
// (the element's coordinates inside its bin; distinct within the bin), 5 bits
// per pass: per pass a digit histogram (match_any peers, leader adds), a
// 32-way exclusive scan, and a stable scatter (rank among equal-digit peers
// of the 32-element step + running digit offset).  O(B) per pass, so large
// bins cost linear, not quadratic, time.  Ping-pongs between `a` (input and
// final output) and `t` (scratch of the same layout).  s_run: 32 ints per warp.
template <typename T, typename LocalKey>
__device__ __forceinline__ void canon_segment(T* __restrict__ a, T* __restrict__ t,
                                              unsigned int lo, unsigned int hi, int W,
                                              int* s_run, LocalKey lkey) {
  const int lane = threadIdx.x & 31;
  const unsigned int lt = (1u << lane) - 1u;
  if (hi - lo <= 1) return;
  T* src = a;
  T* dst = t;
  const int passes = (W + 4) / 5;
  for (int pz = 0; pz < passes; pz++) {
    const int sh = 5 * pz;
    __syncwarp();
    s_run[lane] = 0;  // digit histogram (one leader per distinct digit per step)
    __syncwarp();
    for (unsigned int i0 = lo; i0 < hi; i0 += 32) {
      const unsigned int i = i0 + lane;
      const unsigned int d = i < hi ? (lkey(src[i]) >> sh) & 31u : 32u;
      const unsigned int peers = __match_any_sync(0xffffffffu, d);
      if (d < 32u && !(peers & lt)) s_run[d] += __popc(peers);
      __syncwarp();
    }
    const unsigned int cnt = (unsigned int)s_run[lane];
    unsigned int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    __syncwarp();
    s_run[lane] = (int)(incl - cnt);
    __syncwarp();
    for (unsigned int i0 = lo; i0 < hi; i0 += 32) {
      const unsigned int i = i0 + lane;
      const bool ok = i < hi;
      T e{};
      if (ok) e = src[i];
      const unsigned int d = ok ? (lkey(e) >> sh) & 31u : 32u;
      const unsigned int peers = __match_any_sync(0xffffffffu, d);
      const unsigned int r = __popc(peers & lt);
      const int base = ok ? s_run[d] : 0;
      __syncwarp();
      if (ok) {
        dst[lo + (unsigned int)base + r] = e;
        if (r == 0) s_run[d] = base + __popc(peers);
      }
      __syncwarp();
    }
    T* x = src; src = dst; dst = x;
  }
  if (src != a)  // odd pass count: the sorted segment is in the scratch
    for (unsigned int i = lo + lane; i < hi; i += 32) a[i] = src[i];
}

// One warp per segment: every element ranked through a warp-private bitmap of
// the bin's local key space (keys are distinct within a bin, so a key's rank
// is the number of set bits below it): set bits, per-word prefix popcounts
// (16-bit: a bin holds < 2^16 entries), place each element at lo + rank in
// the scratch, copy back.  O(B / 32 + 2^W / 1024) steps per warp and one warp
// per bin, so thousands of bins are in flight at once.  W <= kCanonBitsMax.
constexpr int kCanonBitsMax = 15;  // 1024 bitmap words per warp
constexpr int kCanonWarps = 4;     // warps per block (shared memory: 6 KB per warp)

template <typename T, typename LocalKey>
__device__ __forceinline__ void canon_warp_bitmap(T* __restrict__ a, T* __restrict__ t,
                                                  unsigned int lo, unsigned int hi, int W,
                                                  unsigned int* bits, unsigned short* pre,
                                                  LocalKey lkey) {
  const int lane = threadIdx.x & 31;
  const int nwords = 1 << (W > 5 ? W - 5 : 0);
  for (int w = lane; w < nwords; w += 32) bits[w] = 0u;
  __syncwarp();
  // (8 elements per lane in flight per step: the longest segment bounds the
  // kernel, so its steps must not each pay a full memory latency)
  constexpr int U = 4;
  for (unsigned int b0 = lo; b0 < hi; b0 += 32 * U) {
    T e[U];
#pragma unroll
    for (int q = 0; q < U; q++)
      if (b0 + 32 * q + lane < hi) e[q] = a[b0 + 32 * q + lane];
#pragma unroll
    for (int q = 0; q < U; q++)
      if (b0 + 32 * q + lane < hi) {
        const unsigned int L = lkey(e[q]);
        atomicOr(&bits[L >> 5], 1u << (L & 31u));
      }
  }
  __syncwarp();
  const int per = (nwords + 31) >> 5, w0 = lane * per;
  unsigned int v = 0;
  for (int k = 0; k < per; k++)
    if (w0 + k < nwords) v += __popc(bits[w0 + k]);
  unsigned int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  unsigned int run = incl - v;
  for (int k = 0; k < per; k++)
    if (w0 + k < nwords) {
      pre[w0 + k] = (unsigned short)run;
      run += __popc(bits[w0 + k]);
    }
  __syncwarp();
  for (unsigned int b0 = lo; b0 < hi; b0 += 32 * U) {
    T e[U];
#pragma unroll
    for (int q = 0; q < U; q++)
      if (b0 + 32 * q + lane < hi) e[q] = a[b0 + 32 * q + lane];
#pragma unroll
    for (int q = 0; q < U; q++)
      if (b0 + 32 * q + lane < hi) {
        const unsigned int L = lkey(e[q]);
        t[lo + pre[L >> 5] + __popc(bits[L >> 5] & ((1u << (L & 31u)) - 1u))] = e[q];
      }
  }
  __syncwarp();
  for (unsigned int b0 = lo; b0 < hi; b0 += 32 * U) {
    T e[U];
#pragma unroll
    for (int q = 0; q < U; q++)
      if (b0 + 32 * q + lane < hi) e[q] = t[b0 + 32 * q + lane];
#pragma unroll
    for (int q = 0; q < U; q++)
      if (b0 + 32 * q + lane < hi) a[b0 + 32 * q + lane] = e[q];
  }
  __syncwarp();
}

template <typename T, typename LocalKey>
__device__ __forceinline__ void canon_one(T* __restrict__ a, T* __restrict__ t, unsigned int lo,
                                          unsigned int hi, int W, LocalKey lkey) {
  __shared__ unsigned int s_bits[kCanonWarps][1 << (kCanonBitsMax - 5)];
  __shared__ unsigned short s_pre[kCanonWarps][1 << (kCanonBitsMax - 5)];
  __shared__ int s_run[kCanonWarps][32];
  const int w = threadIdx.x >> 5;
  if (hi <= lo + 1) return;
  if (hi - lo <= 32) {  // small segment: one element per lane, ranked by shuffles
    const int lane = threadIdx.x & 31;
    const bool ok = lo + lane < hi;
    T e{};
    unsigned int k = 0xffffffffu;  // (never below a real key: local keys have < 32 bits)
    if (ok) {
      e = a[lo + lane];
      k = lkey(e);
    }
    unsigned int r = 0;
#pragma unroll
    for (int j = 0; j < 32; j++) r += __shfl_sync(0xffffffffu, k, j) < k ? 1u : 0u;
    __syncwarp();  // every element is in registers: sort in place
    if (ok) a[lo + r] = e;
    __syncwarp();
    return;
  }
  if (W <= kCanonBitsMax)
    canon_warp_bitmap(a, t, lo, hi, W, s_bits[w], s_pre[w], lkey);
  else  // very large grids: the linear radix passes
    canon_segment(a, t, lo, hi, W, s_run[w], lkey);
}

// Canonical order of the brick bins: one warp per bin, its segment
// [cursor[b - 1], cursor[b]) (scatter_all advanced every cursor from the bin's
// start to its end; scan_all wrote every cursor, full_cursor = 1) sorted in
// place by the vertex's coordinates inside its brick (z major).
__global__ void __launch_bounds__(32 * kCanonWarps) canon_keys(int4* __restrict__ keys,
                                                               int4* __restrict__ tmp,
                                                               const unsigned int* __restrict__ cursor,
                                                               const Stats* __restrict__ st) {
  if (st->ovf) return;
  int bb[6];
#pragma unroll
  for (int i = 0; i < 6; i++) bb[i] = st->bbox[i];
  if (bb[3] < 0) return;
  const int sft = brick_shift(bb);
  const int x0 = 2 * bb[0] - 1, y0 = 2 * bb[1] - 1, z0 = 2 * bb[2] - 1;
  const unsigned int m = (1u << sft) - 1u;
  auto lkey = [=](int4 k) {
    return ((((unsigned int)(k.z - z0) & m) << (2 * sft)) |
            (((unsigned int)(k.y - y0) & m) << sft) | ((unsigned int)(k.x - x0) & m));
  };
  const int nw = (int)(gridDim.x * kCanonWarps);
  for (int b = (int)(blockIdx.x * kCanonWarps + (threadIdx.x >> 5)); b < kSortBins; b += nw) {
    const unsigned int hi = cursor[b], lo = b ? cursor[b - 1] : 0u;
    canon_one(keys, tmp, lo, hi, 3 * sft, lkey);
  }
}

}  // namespace sc
