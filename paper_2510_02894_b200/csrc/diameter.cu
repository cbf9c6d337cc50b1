// Diameter stage of the shape-coefficient path (sm_100a).
//
// Replaces reference _diameters_sq_seq / _diameters_sq_par
// (pkg/src/shapecore/features.py:121-192): the maximum over all vertex pairs
// of the squared distance, and the maxima over pairs sharing z (XY), y (XZ)
// and x (YZ) bit for bit (features.py:145-147).
//
//  * diam3d_pass1<R>  -- the O(V^2) hot loop.  Triangular grid of square tile
//    pairs (I <= J); the J tile is staged in shared memory as (x, y, z, |p|^2)
//    and each thread register-blocks R i vertices, so a pair costs three FFMA
//    (dot form) plus half an FMNMX3 on fp32 CUDA cores.  Coordinates are fp32
//    in a bbox-centred frame.  One maximum per (tile pair, warp) is kept and
//    the global maximum is an integer atomicMax on the fp32 bit pattern.
//  * diam3d_select / diam3d_refine -- exactness: every (tile pair, warp)
//    whose pass-1 maximum lies within kRefineRel of the global pass-1 maximum
//    is re-evaluated in fp64 with the reference's own arithmetic on the
//    reference's own coordinates, so the final 3-D diameter is the
//    reference's value bit for bit.  Units below the threshold provably cannot
//    hold the maximum (pass-1 error < ~1e-6 of D^2).
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

constexpr int kWarps = kDiamThreads / 32;

// Pass 1: max over the tile pair of the squared distance in "dot" form,
// |pj|^2 - 2 pi.pj (+ |pi|^2 once per i), i.e. three FFMA per pair plus half a
// 3-input FMNMX3 -- issue-bound at ~3.5 instructions per pair.  The form
// cancels for near pairs but not at the maximum: in the bbox-centred frame
// |p| <= D/2*sqrt(3) so the absolute error is < ~12 * 2^-24 * D^2,
// far inside the kRefineRel margin that decides which warps are re-checked
// exactly.  One maximum per (tile pair, warp) is kept for that selection.
template <int R>
__global__ void __launch_bounds__(kDiamThreads) diam3d_pass1(const int4* __restrict__ keys,
                                                             long long n, int T, long long item0,
                                                             long long n_items, Frame f,
                                                             float* __restrict__ warp_max,
                                                             Stats* __restrict__ st) {
  constexpr int TS = kDiamThreads * R;
  extern __shared__ float4 sj[];  // (x, y, z, |p|^2) of the J tile
  const long long item = item0 + blockIdx.x;
  if (item >= item0 + n_items) return;
  int I, J;
  tile_pair(item, T, I, J);
  for (int t = threadIdx.x; t < TS; t += kDiamThreads) {
    long long j = (long long)J * TS + t;
    if (j >= n) j = n - 1;  // repeats of a real vertex are harmless for a max
    float3 c = frame_coord(keys[j], f);
    sj[t] = make_float4(c.x, c.y, c.z, fmaf(c.x, c.x, fmaf(c.y, c.y, c.z * c.z)));
  }
  float a[R], b[R], c[R], m[R], ni[R];
#pragma unroll
  for (int r = 0; r < R; r++) {
    long long i = (long long)I * TS + r * kDiamThreads + threadIdx.x;
    float3 p = frame_coord(keys[i < n ? i : n - 1], f);
    a[r] = -2.f * p.x;
    b[r] = -2.f * p.y;
    c[r] = -2.f * p.z;
    ni[r] = fmaf(p.x, p.x, fmaf(p.y, p.y, p.z * p.z));
    m[r] = -3.0e38f;
  }
  __syncthreads();
#pragma unroll 2
  for (int j = 0; j < TS; j += 2) {
    const float4 q0 = sj[j], q1 = sj[j + 1];
#pragma unroll
    for (int r = 0; r < R; r++) {
      float t0 = fmaf(q0.x, a[r], q0.w);
      float t1 = fmaf(q1.x, a[r], q1.w);
      t0 = fmaf(q0.y, b[r], t0);
      t1 = fmaf(q1.y, b[r], t1);
      t0 = fmaf(q0.z, c[r], t0);
      t1 = fmaf(q1.z, c[r], t1);
      m[r] = fmax3f(m[r], t0, t1);
    }
  }
  float best = 0.f;
#pragma unroll
  for (int r = 0; r < R; r++) best = fmaxf(best, m[r] + ni[r]);
#pragma unroll
  for (int o = 16; o; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) {
    warp_max[blockIdx.x * (long long)kWarps + (threadIdx.x >> 5)] = best;
    atomic_max_pos_f32(&st->d3_f32, best);
  }
}

// Relative margin of the re-check threshold.  Pass-1 error is below ~1e-6 of
// D^2; a (tile pair, warp) whose pass-1 maximum is below
// M*(1 - kRefineRel) provably cannot hold the exact maximum pair.
constexpr float kRefineRel = 8e-6f;

// Compact the (tile pair, warp) units that may hold the maximum.
__global__ void diam3d_select(const float* __restrict__ warp_max, long long n_units,
                              Stats* __restrict__ st, unsigned int* __restrict__ cand) {
  const float tau = __uint_as_float(st->d3_f32) * (1.f - kRefineRel);
  for (long long base = (long long)blockIdx.x * blockDim.x; base < n_units;
       base += (long long)gridDim.x * blockDim.x) {
    const long long u = base + threadIdx.x;
    const bool hit = u < n_units && warp_max[u] >= tau;
    const unsigned int mask = __ballot_sync(0xffffffffu, hit);
    if (!mask) continue;
    unsigned long long pos = 0;
    const int lane = threadIdx.x & 31;
    if (lane == 0) pos = atomicAdd(&st->n_cand, (unsigned long long)__popc(mask));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (hit) cand[pos + __popc(mask & ((1u << lane) - 1))] = (unsigned int)u;
  }
}

// Exact re-check: every selected warp's 32*R i-rows against its J tile, in
// fp64 with the reference arithmetic on the reference coordinates.  Work unit
// = (candidate, 256-wide j chunk); a persistent grid walks the units.
template <int R>
__global__ void __launch_bounds__(kDiamThreads) diam3d_refine(const int4* __restrict__ keys,
                                                              long long n, int T,
                                                              long long item0, Frame f,
                                                              const unsigned int* __restrict__ cand,
                                                              Stats* __restrict__ st) {
  constexpr int TS = kDiamThreads * R;
  constexpr int CHUNKS = TS / kDiamThreads;
  __shared__ double sx[kDiamThreads], sy[kDiamThreads], sz[kDiamThreads];
  const long long units = (long long)st->n_cand * CHUNKS;
  double best = 0.0;
  for (long long u = blockIdx.x; u < units; u += gridDim.x) {
    const unsigned int cu = cand[u / CHUNKS];
    const int q = (int)(u % CHUNKS);
    const long long item = item0 + cu / kWarps;
    const int warp = cu % kWarps;
    int I, J;
    tile_pair(item, T, I, J);
    __syncthreads();
    {
      long long j = (long long)J * TS + q * kDiamThreads + threadIdx.x;
      int4 kj = keys[j < n ? j : n - 1];
      sx[threadIdx.x] = ref_coord(kj.x, f.sx);
      sy[threadIdx.x] = ref_coord(kj.y, f.sy);
      sz[threadIdx.x] = ref_coord(kj.z, f.sz);
    }
    __syncthreads();
    const int r = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long i = (long long)I * TS + r * kDiamThreads + warp * 32 + lane;
    if (r < R && i < n) {
      int4 ki = keys[i];
      const double xi = ref_coord(ki.x, f.sx), yi = ref_coord(ki.y, f.sy), zi = ref_coord(ki.z, f.sz);
#pragma unroll 4
      for (int t = 0; t < kDiamThreads; t++)
        best = fmax(best, ref_sq_dist(xi, yi, zi, sx[t], sy[t], sz[t]));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best > 0.0) atomic_max_pos_f64(&st->sq[0], best);
}

// ---- planar pass -----------------------------------------------------------
// Plane index space: [0, nZ) XY planes keyed by Z2, [nZ, nZ+nY) XZ by Y2,
// [nZ+nY, P) YZ by X2, where key ranges come from the occupied bbox.
__device__ __forceinline__ void plane_ids(int4 k, const PlaneSpace& ps, int out[3]) {
  out[0] = k.z - ps.lo[0];
  out[1] = ps.cnt[0] + (k.y - ps.lo[1]);
  out[2] = ps.cnt[0] + ps.cnt[1] + (k.x - ps.lo[2]);
}

// Warp-aggregated increment: lanes with equal `id` (vertices of one plane are
// emitted together by the MC warps) share one global atomic.  Returns the
// slot of this lane within its group's reservation.
__device__ __forceinline__ unsigned int group_add(unsigned int* base, int id, bool ok) {
  const int lane = threadIdx.x & 31;
  const unsigned int peers = __match_any_sync(0xffffffffu, ok ? id : -1 - lane);
  const int leader = __ffs(peers) - 1;
  unsigned int pos = 0;
  if (ok && lane == leader) pos = atomicAdd(base + id, (unsigned int)__popc(peers));
  pos = __shfl_sync(0xffffffffu, pos, leader);
  return pos + __popc(peers & ((1u << lane) - 1));
}

__global__ void plane_hist(const int4* __restrict__ keys, long long n, PlaneSpace ps,
                           unsigned int* __restrict__ counts) {
  for (long long base = (long long)blockIdx.x * blockDim.x; base < n;
       base += (long long)gridDim.x * blockDim.x) {
    const long long v = base + threadIdx.x;
    const bool ok = v < n;
    int id[3] = {0, 0, 0};
    if (ok) plane_ids(keys[v], ps, id);
#pragma unroll
    for (int a = 0; a < 3; a++) group_add(counts, id[a], ok);
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
  for (long long base = (long long)blockIdx.x * blockDim.x; base < n;
       base += (long long)gridDim.x * blockDim.x) {
    const long long v = base + threadIdx.x;
    const bool ok = v < n;
    int4 k = make_int4(0, 0, 0, 0);
    int id[3] = {0, 0, 0};
    if (ok) {
      k = keys[v];
      plane_ids(k, ps, id);
    }
    const unsigned int p0 = group_add(cursor, id[0], ok);  // XY: (X, Y)
    const unsigned int p1 = group_add(cursor, id[1], ok);  // XZ: (X, Z)
    const unsigned int p2 = group_add(cursor, id[2], ok);  // YZ: (Y, Z)
    if (ok) {
      sorted[p0] = make_int2(k.x, k.y);
      sorted[p1] = make_int2(k.x, k.z);
      sorted[p2] = make_int2(k.y, k.z);
    }
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
#define SC_INST(RR)                                                                            \
  template __global__ void diam3d_pass1<RR>(const int4*, long long, int, long long, long long,   \
                                            Frame, float*, Stats*);                              \
  template __global__ void diam3d_refine<RR>(const int4*, long long, int, long long, Frame,      \
                                             const unsigned int*, Stats*);
SC_INST(2)
SC_INST(4)
SC_INST(8)
#undef SC_INST

}  // namespace sc
