// Exact work pruning for the O(V^2) diameter pass (sm_100a).
//
// The maximum pair distance D^2 is at least LB = the largest exact pair value
// among a few extreme vertices (13 directions, both ends).  After a Morton
// brick ordering of the vertices, every 2048-vertex tile and every 256-vertex
// chunk is spatially compact, so most (tile, chunk) work units have an upper
// bound UB^2 = max distance^2 between their boxes below LB: they cannot hold
// the maximum pair and are not evaluated.  Surviving units run through
// diam3d_pass1 exactly as before and the fp64 re-check keeps the result
// bit-identical to the reference's all-pairs loop (features.py:121-192).
//
//   sort_hist / sort_scan / sort_scatter -- counting sort by 15-bit Morton brick
//   chunk_boxes                          -- integer bbox of every 256-chunk
//   extremes / lower_bound               -- LB from 26 extreme vertices (fp64 exact)
//   unit_filter                          -- compacted list of surviving units
#include <climits>

#include "sc_device.cuh"

namespace sc {

constexpr int kSortBits = 15;  // 5 bits per axis
constexpr int kSortBins = 1 << kSortBits;
constexpr int kChunkV = 256;   // == diameter.cu kChunk
constexpr int kTileV = 2048;   // == diameter.cu kTile
constexpr int kNDir = 13;

__device__ __forceinline__ long long n_verts(const Stats* st, long long cap) {
  long long n = (long long)st->n_vert;
  return n < cap ? n : cap;
}

__device__ __forceinline__ unsigned int spread5(unsigned int v) {  // 5 bits -> every 3rd bit
  v &= 31u;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

// Brick shift (in doubled units) so that the bbox spans <= 32 bricks per axis.
__device__ __forceinline__ int brick_shift(const Stats* st) {
  const int* bb = st->bbox;
  int ext = max(bb[3] - bb[0], max(bb[4] - bb[1], bb[5] - bb[2])) * 2 + 3;
  int s = 5;  // >= 16-voxel bricks
  while ((ext >> s) >= 32) s++;
  return s;
}

__device__ __forceinline__ unsigned int brick_bin(int4 k, const Stats* st, int s) {
  const int* bb = st->bbox;
  const unsigned int bx = (unsigned int)(k.x - (2 * bb[0] - 1)) >> s;
  const unsigned int by = (unsigned int)(k.y - (2 * bb[1] - 1)) >> s;
  const unsigned int bz = (unsigned int)(k.z - (2 * bb[2] - 1)) >> s;
  return spread5(bx) | (spread5(by) << 1) | (spread5(bz) << 2);
}

__device__ __forceinline__ unsigned int group_add_u(unsigned int* base, unsigned int id, bool ok) {
  const int lane = threadIdx.x & 31;
  const unsigned int peers = __match_any_sync(0xffffffffu, ok ? id : 0x80000000u + lane);
  const int leader = __ffs(peers) - 1;
  unsigned int pos = 0;
  if (ok && lane == leader) pos = atomicAdd(base + id, (unsigned int)__popc(peers));
  pos = __shfl_sync(0xffffffffu, pos, leader);
  return pos + __popc(peers & ((1u << lane) - 1));
}

__global__ void sort_hist(const int4* __restrict__ keys, long long cap,
                          const Stats* __restrict__ st, unsigned int* __restrict__ counts) {
  const long long n = n_verts(st, cap);
  const int s = brick_shift(st);
  for (long long base = (long long)blockIdx.x * blockDim.x; base < n;
       base += (long long)gridDim.x * blockDim.x) {
    const long long v = base + threadIdx.x;
    const bool ok = v < n;
    group_add_u(counts, ok ? brick_bin(keys[v], st, s) : 0u, ok);
  }
}

// 32768 bins, 1024 threads x 32 consecutive bins each: one pass.
__global__ void __launch_bounds__(1024) sort_scan(unsigned int* __restrict__ counts,
                                                  unsigned int* __restrict__ cursor) {
  uint4* c4 = reinterpret_cast<uint4*>(counts) + threadIdx.x * 8;
  uint4* o4 = reinterpret_cast<uint4*>(cursor) + threadIdx.x * 8;
  uint4 v[8];
  unsigned int sum = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) {
    v[k] = c4[k];
    sum += v[k].x + v[k].y + v[k].z + v[k].w;
  }
  unsigned int total;
  unsigned int run = block_exscan_1024(sum, &total);
#pragma unroll
  for (int k = 0; k < 8; k++) {
    uint4 o;
    o.x = run; run += v[k].x;
    o.y = run; run += v[k].y;
    o.z = run; run += v[k].z;
    o.w = run; run += v[k].w;
    o4[k] = o;
    c4[k] = make_uint4(0, 0, 0, 0);  // leave the histogram zeroed for the next ROI
  }
}

__global__ void sort_scatter(const int4* __restrict__ keys, long long cap,
                             const Stats* __restrict__ st, unsigned int* __restrict__ cursor,
                             int4* __restrict__ out) {
  const long long n = n_verts(st, cap);
  const int s = brick_shift(st);
  for (long long base = (long long)blockIdx.x * blockDim.x; base < n;
       base += (long long)gridDim.x * blockDim.x) {
    const long long v = base + threadIdx.x;
    const bool ok = v < n;
    const int4 k = ok ? keys[v] : make_int4(0, 0, 0, 0);
    const unsigned int pos = group_add_u(cursor, ok ? brick_bin(k, st, s) : 0u, ok);
    if (ok) out[pos] = k;
  }
}

// Integer box of each 256-vertex chunk of the sorted keys: boxes[2c] = lo,
// boxes[2c+1] = hi (doubled units).  One warp per chunk.
__global__ void chunk_boxes(const int4* __restrict__ keys, long long cap,
                            const Stats* __restrict__ st, int4* __restrict__ boxes) {
  const long long n = n_verts(st, cap);
  const long long chunks = (n + kChunkV - 1) / kChunkV;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long c = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < chunks;
       c += warps) {
    int lx = INT_MAX, ly = INT_MAX, lz = INT_MAX, hx = INT_MIN, hy = INT_MIN, hz = INT_MIN;
    for (int t = lane; t < kChunkV; t += 32) {
      long long v = c * kChunkV + t;
      if (v >= n) v = n - 1;  // pass 1 clamps the same way
      const int4 k = keys[v];
      lx = min(lx, k.x); ly = min(ly, k.y); lz = min(lz, k.z);
      hx = max(hx, k.x); hy = max(hy, k.y); hz = max(hz, k.z);
    }
    lx = __reduce_min_sync(0xffffffffu, lx); ly = __reduce_min_sync(0xffffffffu, ly);
    lz = __reduce_min_sync(0xffffffffu, lz); hx = __reduce_max_sync(0xffffffffu, hx);
    hy = __reduce_max_sync(0xffffffffu, hy); hz = __reduce_max_sync(0xffffffffu, hz);
    if (lane == 0) {
      boxes[2 * c] = make_int4(lx, ly, lz, 0);
      boxes[2 * c + 1] = make_int4(hx, hy, hz, 0);
    }
  }
}

// 13 directions (integer), projections in the mm frame (doubled key * half
// spacing).  The arg-extremes are reduced as packed (orderable value, index).
__constant__ int c_dir[kNDir][3] = {{1, 0, 0},  {0, 1, 0},  {0, 0, 1},  {1, 1, 0},  {1, -1, 0},
                                    {1, 0, 1},  {1, 0, -1}, {0, 1, 1},  {0, 1, -1}, {1, 1, 1},
                                    {1, 1, -1}, {1, -1, 1}, {-1, 1, 1}};

__device__ __forceinline__ unsigned long long pack_ext(float v, unsigned int idx) {
  unsigned int b = __float_as_uint(v);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);  // order-preserving
  return ((unsigned long long)b << 32) | idx;
}

__global__ void __launch_bounds__(256) extremes(const int4* __restrict__ keys, long long cap,
                                                Frame f, Stats* __restrict__ st) {
  __shared__ unsigned long long s_ext[2 * kNDir];
  if (threadIdx.x < 2 * kNDir) s_ext[threadIdx.x] = 0ull;
  __syncthreads();
  const long long n = n_verts(st, cap);
  unsigned long long best[2 * kNDir];
#pragma unroll
  for (int d = 0; d < 2 * kNDir; d++) best[d] = 0ull;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    const int4 k = keys[v];
    const float x = (float)k.x * f.hx, y = (float)k.y * f.hy, z = (float)k.z * f.hz;
#pragma unroll
    for (int d = 0; d < kNDir; d++) {
      const float p = c_dir[d][0] * x + c_dir[d][1] * y + c_dir[d][2] * z;
      const unsigned long long hi = pack_ext(p, (unsigned int)v);
      const unsigned long long lo = pack_ext(-p, (unsigned int)v);
      best[2 * d] = hi > best[2 * d] ? hi : best[2 * d];
      best[2 * d + 1] = lo > best[2 * d + 1] ? lo : best[2 * d + 1];
    }
  }
#pragma unroll
  for (int d = 0; d < 2 * kNDir; d++) {
    unsigned long long b = best[d];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const unsigned long long t = __shfl_xor_sync(0xffffffffu, b, o);
      b = t > b ? t : b;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(&s_ext[d], b);
  }
  __syncthreads();
  if (threadIdx.x < 2 * kNDir) atomicMax(&st->ext[threadIdx.x], s_ext[threadIdx.x]);
}

// LB = max exact (reference fp64 arithmetic) squared distance among the 26
// extreme vertices; also seeds the exact 3-D maximum (it is a real pair).
__global__ void lower_bound(const int4* __restrict__ keys, Frame f, Stats* __restrict__ st) {
  __shared__ double px[2 * kNDir], py[2 * kNDir], pz[2 * kNDir];
  if (st->bbox[3] < 0) return;
  if (threadIdx.x < 2 * kNDir) {
    const unsigned int idx = (unsigned int)(st->ext[threadIdx.x] & 0xffffffffu);
    const int4 k = keys[idx];
    px[threadIdx.x] = ref_coord(k.x, f.sx);
    py[threadIdx.x] = ref_coord(k.y, f.sy);
    pz[threadIdx.x] = ref_coord(k.z, f.sz);
  }
  __syncthreads();
  double best = 0.0;
  for (int p = threadIdx.x; p < 4 * kNDir * kNDir; p += blockDim.x) {
    const int i = p / (2 * kNDir), j = p % (2 * kNDir);
    best = fmax(best, ref_sq_dist(px[i], py[i], pz[i], px[j], py[j], pz[j]));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) {
    atomic_max_pos_f64(&st->lb, best);
    atomic_max_pos_f64(&st->sq[0], best);
  }
}

// Work units of the 3-D pass: (tile pair item, j chunk q), item over the
// upper triangle of T x T tiles.  Keep a unit iff the max distance between the
// I tile's box and the chunk's box can reach LB.
__device__ __forceinline__ void tile_pair_p(long long t, long long T, int& I, int& J) {
  double b = 2.0 * T + 1.0;
  long long i = (long long)((b - sqrt(b * b - 8.0 * (double)t)) * 0.5);
  if (i < 0) i = 0;
  if (i > T - 1) i = T - 1;
  auto off = [T](long long r) { return r * T - r * (r - 1) / 2; };
  while (i > 0 && off(i) > t) i--;
  while (i < T - 1 && off(i + 1) <= t) i++;
  I = (int)i;
  J = (int)(i + (t - off(i)));
}

__device__ __forceinline__ double axis_reach(int loA, int hiA, int loB, int hiB, double h) {
  const double d = (double)max(hiA - loB, hiB - loA) * h;
  return d * d;
}

__global__ void unit_filter(const int4* __restrict__ boxes, long long cap, Frame f, int prune,
                            Stats* __restrict__ st, unsigned int* __restrict__ work) {
  const long long n = n_verts(st, cap);
  if (n == 0) return;
  const long long T = (n + kTileV - 1) / kTileV;
  const long long chunks = (n + kChunkV - 1) / kChunkV;
  const long long units = T * (T + 1) / 2 * (kTileV / kChunkV);
  double lb;
  {
    const unsigned long long b = st->lb;
    lb = __longlong_as_double((long long)b);
  }
  const double thr = lb * (1.0 - 1e-9);  // UB and LB are exact up to fp64 rounding
  const double hx = 0.5 * f.sx, hy = 0.5 * f.sy, hz = 0.5 * f.sz;
  const int lane = threadIdx.x & 31;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < units;
       base += (long long)gridDim.x * blockDim.x) {
    const long long u = base + threadIdx.x;
    bool keep = false;
    if (u < units) {
      const long long item = u / (kTileV / kChunkV);
      const int q = (int)(u - item * (kTileV / kChunkV));
      int I, J;
      tile_pair_p(item, T, I, J);
      const long long cj = (long long)J * (kTileV / kChunkV) + q;
      if (cj < chunks) {
        int4 ilo = make_int4(INT_MAX, INT_MAX, INT_MAX, 0), ihi = make_int4(INT_MIN, INT_MIN, INT_MIN, 0);
        for (int r = 0; r < kTileV / kChunkV; r++) {
          const long long ci = (long long)I * (kTileV / kChunkV) + r;
          if (ci >= chunks) break;
          const int4 a = boxes[2 * ci], b = boxes[2 * ci + 1];
          ilo.x = min(ilo.x, a.x); ilo.y = min(ilo.y, a.y); ilo.z = min(ilo.z, a.z);
          ihi.x = max(ihi.x, b.x); ihi.y = max(ihi.y, b.y); ihi.z = max(ihi.z, b.z);
        }
        const int4 jlo = boxes[2 * cj], jhi = boxes[2 * cj + 1];
        const double ub = axis_reach(ilo.x, ihi.x, jlo.x, jhi.x, hx) +
                          axis_reach(ilo.y, ihi.y, jlo.y, jhi.y, hy) +
                          axis_reach(ilo.z, ihi.z, jlo.z, jhi.z, hz);
        keep = !prune || ub >= thr;
      }
    }
    const unsigned int mask = __ballot_sync(0xffffffffu, keep);
    if (!mask) continue;
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(&st->n_work, (unsigned long long)__popc(mask));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (keep) work[pos + __popc(mask & ((1u << lane) - 1))] = (unsigned int)u;
  }
}

}  // namespace sc
