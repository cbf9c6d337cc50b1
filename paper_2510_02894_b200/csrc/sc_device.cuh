// Shared device-side definitions of the shape-coefficient kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sc {

constexpr int kNumCases = 256;

// Device-resident accumulators of one ROI.  Every field is an exact integer
// (or an fp bit pattern updated with integer atomicMax), so results do not
// depend on block scheduling.
// mc_cells blocks flush their case histograms into kHistCopies copies (block
// index mod kHistCopies) so the end-of-kernel atomics of hundreds of blocks do
// not all queue on the same 256 addresses; the host sums the copies.
constexpr int kHistCopies = 8;

struct Stats {
  unsigned long long hist[kHistCopies][kNumCases];  // active cells per MC case (0/255 never counted)
  unsigned long long n_vert;           // crossed lattice edges == mesh vertices
  long long vol_k;                     // 48*volume/(sx*sy*sz), exact (Appendix A)
  int bbox[6];                         // xmin, ymin, zmin, xmax, ymax, zmax of occupied voxels
  unsigned int d3_f32;                 // fp32 bits of the pass-1 max squared 3-D distance
  unsigned int hist_merged;            // host copy only: hist[0] already holds the sum
  unsigned long long sq[4];            // fp64 bits: exact squared maxima (3d, xy, xz, yz)
  unsigned long long n_cand;           // 3-D (tile pair, warp) units re-checked in fp64
  unsigned long long n_pcand;          // planar tile pairs re-checked in fp64
  unsigned int pl_f32[4];              // fp32 bits of pass-1 planar maxima (xy, xz, yz, -)
  unsigned long long plane_units;      // in-plane tile pairs of the planar pass
  unsigned long long ext[26];          // packed (projection, index) of 13-direction extremes
  unsigned long long lb;               // fp64 bits: exact squared distance lower bound
  unsigned long long n_work;           // surviving 3-D work units after pruning
  unsigned int done1, done2;           // scan_all plane-block / diam_refine tickets
  unsigned int ovf;                    // V exceeded the diameter-side buffers: skip the rest
  unsigned int done3;                  // boxes_extremes block ticket (last block: the 3-D LB)
  unsigned long long plb[3];           // fp64 bits: exact planar lower bounds per family
  unsigned long long n_pwork;          // surviving planar units after pruning
  unsigned long long plane_chunks;     // 256-entry chunks over all planes
  unsigned long long n_sub;            // 3-D 64 x 64 sub-pairs kept (pass 1 evaluates these)
  unsigned long long n_psub;           // planar 64 x 64 sub-pairs kept
  unsigned long long n_super;          // surviving super-chunk pairs (large ROIs)
  // %globaltimer stamps (ns): ROI start (init_stats), end of the marching-cubes
  // stage (scan_all start), end of the diameters (last diam_refine block):
  // mesh_ms / diameters_ms without event nodes in the graph.
  unsigned long long t_start, t_mesh, t_end;
  unsigned int plane_ovf;              // a plane holds more than kPlaneMaxEntries entries
  unsigned int trace_on;               // kernels record their spans (RoiParams::pflags bit 2)
  unsigned int bad_input;              // shard_import: summed vertex count != gathered keys
  unsigned long long n_eval;           // 3-D pair slots pass 1 evaluated (after the vertex filter)
  unsigned long long n_peval;          // planar pair slots pass 1 evaluated
  // %globaltimer of each pipeline kernel's first block start / last block
  // end (index: TraceId), for the batch timeline (SC_TRACE=1 on the host).
  unsigned long long tr[16][2];
  unsigned long long busy[16];         // summed block residency (ns) per kernel
};

enum TraceId {
  kTrPack = 1, kTrMc, kTrScan, kTrScatter, kTrPlaneBoxes, kTrPlaneLb, kTrPlaneFilter, kTrBoxes,
  kTrUnitFilter, kTrUnitExpand, kTrPass1, kTrRefine, kTrCount
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Block-granular kernel span on the ROI record: earliest block start (min),
// latest block end (max; thread 0 leaving the kernel) and summed block
// residency -- three reductions per block, only while tracing (SC_TRACE=1 ->
// RoiParams::pflags bit 2 -> Stats::trace_on).  init_stats seeds the starts.
struct KTrace {
  unsigned long long* e;
  unsigned long long* b;
  unsigned long long t0;
  __device__ __forceinline__ KTrace(const Stats* st, int id)
      : e(const_cast<Stats*>(st)->tr[id]), b(const_cast<Stats*>(st)->busy + id), t0(0) {
    if (threadIdx.x == 0 && st->trace_on) {
      t0 = global_ns();
      atomicMin(e, t0);
    }
  }
  __device__ __forceinline__ ~KTrace() {
    if (threadIdx.x == 0 && t0) {
      const unsigned long long t1 = global_ns();
      atomicMax(e + 1, t1);
      atomicAdd(b, t1 - t0);
    }
  }
};

// 3-D chunk pairs (128 x 128 vertices) tested directly by unit_filter up to
// this many; above it the 1024-vertex super pairs are listed first (slist)
// and expanded by unit_expand.  The host sizes slist from the same constant.
constexpr long long kSingleLevelMax = 1LL << 16;

// Work entries carry, in the top 4 bits of the J field, which 64 x 64 sub-pairs
// of the 128 x 128 chunk pair can reach the lower bound (bit 2a + b: I half a,
// J half b); pass 1 evaluates only those.  0xF = the whole unit.
constexpr unsigned int kSubShift = 28;
constexpr unsigned int kIdxMask = (1u << kSubShift) - 1u;

// Per-case integer tables for the exact volume path: for case k,
// t = sum over its triangles of a.(b x c) and n = sum of (b-a) x (c-a), with
// a, b, c the DOUBLED cell-local vertex coordinates (in {0,1,2}^3).
// Raw corner word of a cell (bits: A_i, A_i+1, B_i, B_i+1, C_i, C_i+1, D_i,
// D_i+1 with A/B = rows (v, w)/(v+1, w), C/D = rows (v, w+1)/(v+1, w+1)) ->
// reference case: occupancy in corner order 0..7 = (A_i, A_i+1, B_i+1, B_i,
// C_i, C_i+1, D_i+1, D_i), complemented (bit set = background corner).
__host__ __device__ __forceinline__ int case_of_idx(int idx) {
  const int occ = (idx & 0x33) | ((idx >> 1) & 0x44) | ((idx << 1) & 0x88);
  return (~occ) & 0xff;
}

struct CaseTables {
  int4 tn[kNumCases];      // (t, n.x, n.y, n.z) by reference case
  int4 tn_raw[kNumCases];  // the same, indexed by mc_cells' raw corner word
};

// Geometry of one launch: doubled-coordinate centre and half spacings used to
// build the pass-1 fp32 frame, and the fp64 spacing for the exact re-check.
struct Frame {
  int cx2, cy2, cz2;   // bbox centre in doubled lattice units (xmin + xmax, ...)
  float hx, hy, hz;    // fp32(0.5 * spacing)
  int ox2, oy2, oz2;   // doubled origin of the (host-cropped) volume in the full grid:
                       // reference coordinates use key + o*2 (0 when uncropped)
  double sx, sy, sz;   // spacing (fp64, reference arithmetic)
};

// Bit-volume segment map: bit s set <=> words [16 s, 16 s + 16) hold a nonzero
// word (one warp-wide 512-byte mask load of the pack = one segment).
__device__ __forceinline__ bool seg_on(const uint32_t* __restrict__ segmap, long long wi) {
  return (__ldg(segmap + (wi >> 9)) >> ((wi >> 4) & 31)) & 1u;
}

// Per-ROI launch parameters, read by the kernels from device memory (one
// record per pipeline slot, written by a 96-byte H2D copy before each launch),
// so a slot's captured CUDA graph is independent of the mask pointer, the
// dims and the spacing and is replayed for every ROI.
struct RoiParams {
  const uint8_t* mask;
  long long nx, ny, nz;
  long long n_chunks;  // nx*ny*nz/16 (fast pack path)
  long long n_words;   // W*ny*nz
  int W;               // 32-bit words per bit-volume row
  int sparse;          // bit 0: the pack writes only nonzero 16-word segments of the bit
                       // volume and marks them in the segment map; readers treat
                       // unmarked segments as zero (0: every word is written); bit 1:
                       // the pack skips the conversion of all-zero segments
  int pflags;          // bit 2: kernels record their timeline spans (SC_TRACE)
  int mc_slab;         // 0, or (nshards << 16) | shard: mc_cells walks only that shard's
                       // contiguous share of the cell layers (two-phase shard entry)
  Frame f;             // cx2..cz2 are filled on the device from the bbox
  long long wcap;      // capacity of the 3-D work list (overflow -> exact re-run)
};

// Planar key space: [0, cnt[0]) XY planes keyed by Z2, then cnt[1] XZ planes
// keyed by Y2, then cnt[2] YZ planes keyed by X2; lo = smallest key per axis.
struct PlaneSpace {
  int lo[3];
  int cnt[3];
};

// ---- vertex binning shared by the MC emission, the sort and the planar pass ----

// Morton brick order: 6 bits per axis (2^18 bins) over the occupied bbox.
// The fine histogram lives in global memory (one atomic per vertex); the top
// 8 bits of the Morton code form 256 super-bins counted in shared memory, so
// every 1024-bin slice of the exclusive scan can start from the super-bin
// prefix without any inter-block communication.
constexpr int kSortBits = 18;
constexpr int kSortBins = 1 << kSortBits;
constexpr int kSortSliceBits = 10;                            // fine bins per scan block
constexpr int kSortSupers = kSortBins >> kSortSliceBits;      // 256 super-bins
constexpr int kScanThreads = 256;                           // scan_all block size
constexpr int kScanSlices = 4;                              // 1024-bin slices per scan block
constexpr int kScanBlocks = kSortSupers / kScanSlices;      // 64 brick-scan blocks
constexpr int kChunk3 = 128;  // vertices per 3-D diameter chunk (pair unit = chunk x chunk)

__device__ __forceinline__ unsigned int spread_bits(unsigned int v) {  // <= 10 bits -> every 3rd bit
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x30000ffu;
  v = (v | (v << 8)) & 0x300f00fu;
  v = (v | (v << 4)) & 0x30c30c3u;
  v = (v | (v << 2)) & 0x9249249u;
  return v;
}

// Brick shift (doubled units) so the bbox spans <= 64 bricks per axis.
__device__ __forceinline__ int brick_shift(const int* bb) {
  const int ext = max(bb[3] - bb[0], max(bb[4] - bb[1], bb[5] - bb[2])) * 2 + 3;
  return max(0, (32 - __clz(ext)) - 6);  // smallest s with (ext >> s) < 64
}

__device__ __forceinline__ unsigned int brick_bin(int X, int Y, int Z, const int* bb, int s) {
  const unsigned int bx = (unsigned int)(X - (2 * bb[0] - 1)) >> s;
  const unsigned int by = (unsigned int)(Y - (2 * bb[1] - 1)) >> s;
  const unsigned int bz = (unsigned int)(Z - (2 * bb[2] - 1)) >> s;
  return spread_bits(bx) | (spread_bits(by) << 1) | (spread_bits(bz) << 2);
}

__device__ __forceinline__ PlaneSpace plane_space(const int* bb) {
  PlaneSpace ps;
  ps.lo[0] = 2 * bb[2] - 1; ps.cnt[0] = 2 * (bb[5] - bb[2]) + 3;
  ps.lo[1] = 2 * bb[1] - 1; ps.cnt[1] = 2 * (bb[4] - bb[1]) + 3;
  ps.lo[2] = 2 * bb[0] - 1; ps.cnt[2] = 2 * (bb[3] - bb[0]) + 3;
  return ps;
}

// XY plane keyed by Z2, XZ by Y2, YZ by X2 (bit-equal fp64 coordinate <=>
// equal doubled lattice key, since (key/2)*s is strictly monotone in key).
__device__ __forceinline__ void plane_ids(int X, int Y, int Z, const PlaneSpace& ps, int out[3]) {
  out[0] = Z - ps.lo[0];
  out[1] = ps.cnt[0] + (Y - ps.lo[1]);
  out[2] = ps.cnt[0] + ps.cnt[1] + (X - ps.lo[2]);
}

// In-plane bricks: each plane family is bucketed by a 16 x 16 Morton brick of
// its two in-plane doubled coordinates (256 bins per plane), so every plane's
// vertex list comes out spatially compact (enables exact planar pruning).
constexpr int kPlaneBins = 256;
constexpr int kPlaneTile = 256;   // in-plane tile edge (first level of plane_filter)
constexpr int kPlaneChunk = 128;  // in-plane chunk edge (planar pair unit)
// Planar work entries hold a plane's chunk indices in 16 bits each, so one
// plane can hold at most this many entries (mesh vertices in that plane; a
// plane's vertices lie on its cross-section contours, far below the bound for
// any real mask).  scan_all checks it per plane at run time.
constexpr long long kPlaneMaxEntries = 65536LL * kPlaneChunk;

__device__ __forceinline__ int axis_shift(int lo, int hi) {  // voxel bbox [lo, hi]
  const int ext = 2 * (hi - lo) + 3;
  return max(0, (32 - __clz(ext)) - 4);  // smallest s with (ext >> s) < 16
}

__device__ __forceinline__ unsigned int spread2x4(unsigned int v) {  // 4 bits -> even bits
  v &= 15u;
  v = (v | (v << 2)) & 0x33u;
  v = (v | (v << 1)) & 0x55u;
  return v;
}

struct PlaneBricks {
  int lo[3];     // smallest doubled key per axis (x, y, z)
  int shift[3];  // brick shift per axis (<= 16 bricks)
};

__device__ __forceinline__ PlaneBricks plane_bricks(const int* bb) {
  PlaneBricks pb;
  for (int a = 0; a < 3; a++) {
    pb.lo[a] = 2 * bb[a] - 1;
    pb.shift[a] = axis_shift(bb[a], bb[a + 3]);
  }
  return pb;
}

// Bin of a vertex inside each of its three planes (XY: (X,Y), XZ: (X,Z), YZ: (Y,Z)).
__device__ __forceinline__ void plane_bins(int X, int Y, int Z, const PlaneBricks& pb,
                                           unsigned int out[3]) {
  const unsigned int bx = (unsigned int)(X - pb.lo[0]) >> pb.shift[0];
  const unsigned int by = (unsigned int)(Y - pb.lo[1]) >> pb.shift[1];
  const unsigned int bz = (unsigned int)(Z - pb.lo[2]) >> pb.shift[2];
  out[0] = spread2x4(bx) | (spread2x4(by) << 1);
  out[1] = spread2x4(bx) | (spread2x4(bz) << 1);
  out[2] = spread2x4(by) | (spread2x4(bz) << 1);
}

// Warp-aggregated increment: lanes with equal `id` share one global atomic.
// Returns this lane's slot within its group's reservation.  All lanes call.
__device__ __forceinline__ unsigned int group_add(unsigned int* base, unsigned int id, bool ok) {
  const int lane = threadIdx.x & 31;
  const unsigned int peers = __match_any_sync(0xffffffffu, ok ? id : 0x80000000u + lane);
  const int leader = __ffs(peers) - 1;
  unsigned int pos = 0;
  if (ok && lane == leader) pos = atomicAdd(base + id, (unsigned int)__popc(peers));
  pos = __shfl_sync(0xffffffffu, pos, leader);
  return pos + __popc(peers & ((1u << lane) - 1));
}

// Same contract as group_add, aggregating runs of equal ids in consecutive
// lanes (one shuffle + two ballots instead of __match_any_sync).  Vertices
// arrive in emission order, so equal bins are mostly adjacent; an id that
// recurs after a break simply takes a second atomic.
__device__ __forceinline__ unsigned int seg_add(unsigned int* base, unsigned int id, bool ok) {
  const int lane = threadIdx.x & 31;
  const unsigned int prev = __shfl_up_sync(0xffffffffu, id, 1);
  const unsigned int okm = __ballot_sync(0xffffffffu, ok);
  const bool start = ok && (lane == 0 || !((okm >> (lane - 1)) & 1u) || prev != id);
  const unsigned int starts = __ballot_sync(0xffffffffu, start);
  const unsigned int upto = (2u << lane) - 1u;  // bits 0..lane (all bits for lane 31)
  const int leader = 31 - __clz(starts & upto);
  const unsigned int after = (starts | ~okm) & ~upto;  // segment breaks past this lane
  unsigned int pos = 0;
  if (start) pos = atomicAdd(base + id, (unsigned int)((after ? __ffs(after) - 1 : 32) - lane));
  pos = __shfl_sync(0xffffffffu, pos, leader & 31);
  return pos + (unsigned int)(lane - leader);
}

// Last-block ticket: returns true in exactly one block, after every block of
// the grid has passed this point (its prior global writes made visible).
__device__ __forceinline__ bool last_block(unsigned int* ticket) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    if (threadIdx.x == 0) *ticket = 0u;  // ready for the next ROI
  }
  return s_last;
}

// ---- helpers shared by the diameter, pruning and planar kernels ----
// Re-check threshold.  Pass 1 evaluates the dot form
// |pj|^2 - 2 pi.pj + |pi|^2 in fp32 on frame coordinates |p| <= R, where R^2
// is the squared half-diagonal of the ROI bbox in the pass's own axes (3-D:
// x, y, z; a plane family: its two in-plane axes).  Its absolute error is
// e <= 35 u R^2 (u = 2^-24: 2u per frame coordinate, 7u R^2 per |p|^2, 3 FMA
// roundings on terms <= 3 R^2, 8u R^2 from the coordinates in the product,
// the |pi|^2 fold).  With M the family's pass-1 maximum (M <= D^2 + e), the
// unit holding the exact maximum pair has pass-1 value >= D^2 - e >= M - 2e,
// so every unit at or above tau = M - 2 e_max is re-checked, e_max = 48 u R^2
// (kRefineAbs = 96 u).  The margin is ABSOLUTE in R^2: a plane family whose
// maximum is far below R^2 (small lesions spread over the field) is covered.
// tau is never above the previous relative rule M (1 - kRefineRel).
constexpr float kRefineRel = 8e-6f;
constexpr double kRefineAbs = 96.0 / 16777216.0;

__device__ __forceinline__ float refine_tau(float M, double R2) {
  const double rel = (double)M * (1.0 - (double)kRefineRel);
  const double abs_ = (double)M - kRefineAbs * R2;
  return __double2float_rd(fmin(rel, abs_));
}

// Squared half-extent of the ROI bbox along one axis in mm^2: vertex keys lie
// in [2 lo - 1, 2 hi + 1] (doubled units), the frame centre at lo + hi, so
// |frame coordinate| <= (hi - lo + 1) * s / 2.
__device__ __forceinline__ double half_extent_sq(int lo, int hi, double s) {
  const double h = 0.5 * (double)(hi - lo + 1) * s;
  return h * h;
}

__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// Upper-triangle pair index -> (I, J), I <= J, row-major over I.
__device__ __forceinline__ void tile_pair(long long t, long long T, int& I, int& J) {
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

__device__ __forceinline__ long long n_vertices(const Stats* st, long long cap) {
  long long n = (long long)st->n_vert;
  return n < cap ? n : cap;
}

// Bbox-centred fp32 frame: centre (doubled units) from the MC bbox.
__device__ __forceinline__ void frame_centre(const Stats* st, Frame& f) {
  f.cx2 = st->bbox[0] + st->bbox[3];
  f.cy2 = st->bbox[1] + st->bbox[4];
  f.cz2 = st->bbox[2] + st->bbox[5];
}

__device__ __forceinline__ float3 frame_coord(int4 k, const Frame& f) {
  return make_float3((float)(k.x - f.cx2) * f.hx, (float)(k.y - f.cy2) * f.hy,
                     (float)(k.z - f.cz2) * f.hz);
}

__device__ __forceinline__ void shard_span(long long n, int shard, int nshards, long long& a,
                                           long long& b) {
  a = n * shard / nshards;
  b = n * (shard + 1) / nshards;
}

__device__ __forceinline__ long long tri(long long T) { return T * (T + 1) / 2; }


__device__ __forceinline__ PlaneSpace plane_space(const Stats* st) {
  int bb[6];
#pragma unroll
  for (int i = 0; i < 6; i++) bb[i] = st->bbox[i];
  return plane_space(bb);
}

struct PlaneAxes {  // in-plane (a, b) coordinate frame of one plane family
  int ca, cb;       // centre, doubled units
  float ha, hb;     // fp32 half spacings
  int oa, ob;       // doubled origin offsets (Frame::ox2 ...)
  double sa, sb;    // fp64 spacings
};

__device__ __forceinline__ PlaneAxes plane_axes(int axis, const Stats* st, const Frame& f) {
  const int* bb = st->bbox;
  PlaneAxes x;
  if (axis == 0) {         // XY plane: (X, Y)
    x.ca = bb[0] + bb[3]; x.cb = bb[1] + bb[4]; x.ha = f.hx; x.hb = f.hy; x.sa = f.sx; x.sb = f.sy;
    x.oa = f.ox2; x.ob = f.oy2;
  } else if (axis == 1) {  // XZ plane: (X, Z)
    x.ca = bb[0] + bb[3]; x.cb = bb[2] + bb[5]; x.ha = f.hx; x.hb = f.hz; x.sa = f.sx; x.sb = f.sz;
    x.oa = f.ox2; x.ob = f.oz2;
  } else {                 // YZ plane: (Y, Z)
    x.ca = bb[1] + bb[4]; x.cb = bb[2] + bb[5]; x.ha = f.hy; x.hb = f.hz; x.sa = f.sy; x.sb = f.sz;
    x.oa = f.oy2; x.ob = f.oz2;
  }
  return x;
}

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

__device__ __forceinline__ int plane_axis(int p, const PlaneSpace& ps) {
  return p < ps.cnt[0] ? 0 : (p < ps.cnt[0] + ps.cnt[1] ? 1 : 2);
}


// Exclusive scan of one value per thread across a 1024-thread block (warp
// shuffles, two levels, 2 barriers).  Returns the exclusive prefix; *total
// receives the block sum.  Must be called by all 1024 threads.
__device__ __forceinline__ unsigned int block_exscan_1024(unsigned int v, unsigned int* total) {
  __shared__ unsigned int wsum[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    unsigned int y = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned int t = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += t;
    }
    wsum[lane] = y;
  }
  __syncthreads();
  const unsigned int excl = x - v + (wid ? wsum[wid - 1] : 0u);
  *total = wsum[31];
  __syncthreads();  // wsum reusable after return
  return excl;
}

// Exclusive scan of one value per thread across a block of any multiple of 32
// threads (<= 1024).  Returns the exclusive prefix; *total receives the block
// sum.  Must be called by all threads of the block.
__device__ __forceinline__ unsigned int block_exscan(unsigned int v, unsigned int* total) {
  __shared__ unsigned int wsum2[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) wsum2[wid] = x;
  __syncthreads();
  if (wid == 0) {
    unsigned int y = lane < nw ? wsum2[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned int t = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += t;
    }
    wsum2[lane] = y;
  }
  __syncthreads();
  const unsigned int excl = x - v + (wid ? wsum2[wid - 1] : 0u);
  *total = wsum2[nw - 1];
  __syncthreads();  // wsum2 reusable after return
  return excl;
}

// fp32 (non-negative) max through the unsigned bit pattern.
__device__ __forceinline__ void atomic_max_pos_f32(unsigned int* addr, float v) {
  atomicMax(addr, __float_as_uint(v));
}
__device__ __forceinline__ void atomic_max_pos_f64(unsigned long long* addr, double v) {
  atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}

// Reference pair distance, features.py:140-143: dx*dx + dy*dy + dz*dz in fp64,
// left to right, every operation rounded (no FMA contraction).
__device__ __forceinline__ double ref_sq_dist(double xi, double yi, double zi, double xj,
                                              double yj, double zj) {
  double dx = __dsub_rn(xj, xi), dy = __dsub_rn(yj, yi), dz = __dsub_rn(zj, zi);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// Programmatic dependent launch: a pipeline kernel launched with the PDL
// attribute may start while its predecessor drains; it waits here until the
// predecessor has completed and its writes are visible (a no-op for a normal
// launch), then lets its own successor launch early.  Called first thing by
// every per-ROI kernel after the pack.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Reference vertex coordinate, mesh.py:184-195: (l - 1 + 0.5*[axis]) * s, which
// in doubled units is (key / 2) * s; key/2 is exact in fp64.
__device__ __forceinline__ double ref_coord(int key2, double s) {
  return __dmul_rn((double)key2 * 0.5, s);
}

}  // namespace sc
