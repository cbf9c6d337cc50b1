// Marching-cubes stage of the shape-coefficient path (sm_100a).
//
// Replaces reference pad_mask + _count_triangles + _count_crossed_edges +
// _emit_mesh (pkg/src/shapecore/mesh.py:55-199) and the triangle gathers of
// surface_area / mesh_volume (features.py:83-110).  Two kernels:
//
//  1. pack_bits_*  -- the one HBM-bound pass: streams the uint8 mask once with
//     128-bit loads (evict-first), writes a 1-bit-per-voxel volume (row-padded
//     to 32-bit words, 1/8 of the mask, stays in L2) and the occupied bounding
//     box.  The reference's 1-voxel zero padding is never materialised: voxels
//     outside the grid read as 0.
//  2. mc_cells     -- walks only the bounding box (+1 shell) of the bit volume,
//     32 cells per thread per step with bitwise ops: active-cell mask, per-case
//     histogram (smem atomics), exact integer volume sum, and crossed-edge
//     masks.  Each crossed lattice edge is one mesh vertex (mesh.py:94-100 ==
//     mesh.py:176 dedup key); vertices are stream-compacted with a warp scan and
//     one global atomic per warp-step, as doubled lattice coordinates.
//
// Triangles are never materialised: T = sum_k hist[k]*TRI_COUNT[k], area =
// sum_k hist[k]*A_k(spacing) and volume = |K| sx sy sz / 48 with K the exact
// integer sum accumulated here.
#include <climits>

#include "sc_device.cuh"

namespace sc {

constexpr unsigned kFull = 0xffffffffu;

// Per-ROI reset: block 0 zeroes the accumulator record; every block clears
// its share of the bit-volume segment map (n_seg words, may be 0).
//
// src_rp (optional): the slot's RoiParams in mapped pinned host memory, read
// over PCIe and stored to dst_rp here, so no separate host->device copy has to
// precede the ROI's graph.
__global__ void init_stats(Stats* st, uint32_t* __restrict__ segmap, long long n_seg,
                           const RoiParams* src_rp, RoiParams* dst_rp) {
  int t = threadIdx.x;
  if (blockIdx.x == 0 && src_rp) {
    static_assert(sizeof(RoiParams) % 4 == 0, "RoiParams is copied as 32-bit words");
    const volatile unsigned int* s = reinterpret_cast<const volatile unsigned int*>(src_rp);
    unsigned int* d = reinterpret_cast<unsigned int*>(dst_rp);
    for (int i = t; i < (int)(sizeof(RoiParams) / 4); i += blockDim.x) d[i] = s[i];
  }
  if (blockIdx.x == 0) {
    for (int i = t; i < (int)(sizeof(Stats) / 8); i += blockDim.x)
      reinterpret_cast<unsigned long long*>(st)[i] = 0ull;
    __syncthreads();
    if (t < 3) st->bbox[t] = INT_MAX;
    if (t >= 3 && t < 6) st->bbox[t] = -1;
    if (t < kTrCount) st->tr[t][0] = ~0ull;
    if (t == 0) {
      st->t_start = global_ns();
      const int pf = src_rp ? reinterpret_cast<const volatile RoiParams*>(src_rp)->pflags
                            : dst_rp->pflags;
      st->trace_on = (unsigned int)(pf >> 2) & 1u;
    }
  }
  for (long long i = (long long)blockIdx.x * blockDim.x + t; i < n_seg;
       i += (long long)gridDim.x * blockDim.x)
    segmap[i] = 0u;
}

// 4 mask bytes -> 4 occupancy bits (byte i nonzero -> bit i).  Bit 7 of each
// byte of t is "byte nonzero" (the classic SWAR zero-byte test); the multiply
// then moves the flag of byte i (bit 7+8i) to bit 28+i with no carries (all 16
// partial products land on distinct bit positions).  3 ALU ops + 1 IMAD.
__device__ __forceinline__ uint32_t nib4(uint32_t v) {
  const uint32_t t = (((v & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | v) & 0x80808080u;
  return (t * 0x00204081u) >> 28;
}

struct BoxAcc {
  int x0 = INT_MAX, y0 = INT_MAX, z0 = INT_MAX, x1 = -1, y1 = -1, z1 = -1;
  __device__ __forceinline__ void add(uint32_t word, long long wi, int W, int ny) {
    long long row = wi / W;
    int w = (int)(wi - row * W);
    int z = (int)(row / ny), y = (int)(row - (long long)z * ny);
    int xa = 32 * w + __ffs(word) - 1, xb = 32 * w + 31 - __clz(word);
    x0 = min(x0, xa); x1 = max(x1, xb);
    y0 = min(y0, y);  y1 = max(y1, y);
    z0 = min(z0, z);  z1 = max(z1, z);
  }
  // Word at column w of row (y, z), already located.
  __device__ __forceinline__ void add_at(uint32_t word, int w, int y, int z) {
    x0 = min(x0, 32 * w + __ffs(word) - 1); x1 = max(x1, 32 * w + 31 - __clz(word));
    y0 = min(y0, y);  y1 = max(y1, y);
    z0 = min(z0, z);  z1 = max(z1, z);
  }
  __device__ __forceinline__ void flush(Stats* st) {
    // Integer warp reductions (REDUX), then one atomic per field per warp.
    int hx1 = __reduce_max_sync(kFull, x1);
    if (hx1 < 0) return;  // warp saw no occupied voxel (uniform)
    int v[6] = {(int)__reduce_min_sync(kFull, (unsigned)x0), (int)__reduce_min_sync(kFull, (unsigned)y0),
                (int)__reduce_min_sync(kFull, (unsigned)z0), hx1,
                __reduce_max_sync(kFull, y1), __reduce_max_sync(kFull, z1)};
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&st->bbox[0], v[0]); atomicMin(&st->bbox[1], v[1]); atomicMin(&st->bbox[2], v[2]);
      atomicMax(&st->bbox[3], v[3]); atomicMax(&st->bbox[4], v[4]); atomicMax(&st->bbox[5], v[5]);
    }
  }
};

// Fast path: nx % 32 == 0 and a 16-byte aligned mask.  A pure stream: one
// 16-byte chunk per thread per step (a warp reads 512 contiguous bytes per
// load instruction), U chunks in flight per thread, lane pairs merge their
// 16-bit halves into one 32-bit word.  The bbox is found afterwards from the
// L2-resident bit volume (bits_bbox), so this loop carries no bookkeeping.
// Grid = resident blocks.  tools/microbench/pack_bench.cu: 5.1 TB/s on a 157 MB
// mask = 88% of the 1 GiB streaming-read rate of the same GPU.
//
// BOX: also accumulate the occupied bbox in registers (32-bit index math, only
// for nonzero words) and flush it once per warp -- replaces bits_bbox.
//
// SPARSE (rp->sparse): a warp-wide load is exactly one 16-word segment of the
// bit volume; all-background segments are not written at all (only the
// nonzero ones, and their bit in the segment map), so the HBM write of the
// bit volume shrinks to the occupied rows and no later pass has to re-read a
// full bit volume (bits_bbox walks the map).
template <int U, bool BOX>
__global__ void __launch_bounds__(256) pack_bits_v16(const RoiParams* __restrict__ rp,
                                                     uint32_t* __restrict__ bits,
                                                     Stats* __restrict__ st,
                                                     uint32_t* __restrict__ segmap) {
  KTrace kt_(st, kTrPack);
  const uint4* __restrict__ mask = reinterpret_cast<const uint4*>(rp->mask);
  const long long n_chunks = rp->n_chunks;
  const unsigned int W = (unsigned int)rp->W, ny = (unsigned int)rp->ny;
  const bool sparse = rp->sparse != 0;
  const bool skip = (rp->sparse & 2) != 0;  // option "pack_skip"
  BoxAcc box;
  const long long step = (long long)gridDim.x * blockDim.x * U;
  for (long long base = (long long)blockIdx.x * blockDim.x * U; base < n_chunks; base += step) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; k++) {
      const long long g = base + (long long)k * blockDim.x + threadIdx.x;
      v[k] = g < n_chunks ? __ldcs(mask + g) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < U; k++) {
      const long long g = base + (long long)k * blockDim.x + threadIdx.x;
      // Sparse: an all-background 512-byte segment (most of a KiTS-like grid)
      // costs 2 LOP3 + 1 vote here and no conversion at all, so the pack
      // leaves the SMs' issue slots to the other ROIs' latency-bound kernels.
      // (out-of-range chunks were loaded as zero)
      if (skip && !__any_sync(kFull, (v[k].x | v[k].y | v[k].z | v[k].w) != 0u)) continue;
      const uint32_t b16 = nib4(v[k].x) | (nib4(v[k].y) << 4) | (nib4(v[k].z) << 8) |
                           (nib4(v[k].w) << 12);
      const uint32_t word = b16 | (__shfl_down_sync(kFull, b16, 1) << 16);
      if (sparse) {
        if ((threadIdx.x & 31) == 0) {
          const long long seg = g >> 5;  // lane 0 holds the segment's first chunk
          atomicOr(segmap + (seg >> 5), 1u << (seg & 31));
        }
      }
      if (!(threadIdx.x & 1) && g < n_chunks) {
        bits[g >> 1] = word;
        if (BOX && word) {
          const unsigned int wi = (unsigned int)(g >> 1), row = wi / W, col = wi - row * W;
          const unsigned int z = row / ny, y = row - z * ny;
          box.x0 = min(box.x0, (int)(32 * col) + __ffs(word) - 1);
          box.x1 = max(box.x1, (int)(32 * col) + 31 - __clz(word));
          box.y0 = min(box.y0, (int)y); box.y1 = max(box.y1, (int)y);
          box.z0 = min(box.z0, (int)z); box.z1 = max(box.z1, (int)z);
        }
      }
    }
  }
  if (BOX) box.flush(st);
}

// ---- TMA bulk-copy variant of the fast pack (option "pack_tma") ----
// One persistent CTA per SM streams a contiguous share of the mask through a
// 4-stage ring of 16 KB shared-memory tiles filled by cp.async.bulk (the copy
// engine tracks the bytes on an mbarrier; no registers hold loads in flight),
// and 8 warps convert each landed tile exactly as pack_bits_v16 does.  The
// CTA holds ~64 KB of shared memory and 256 threads, so most of the SM stays
// free for other ROIs' kernels while the HBM stream runs.
constexpr int kTmaMaxStages = 8;
constexpr int kTmaTile = 16384;  // bytes per stage

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar)), "l"(policy)
      : "memory");
}
// Bounded wait: a lost transaction traps instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  for (long long spin = 0;; spin++) {
    unsigned ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    if (spin > (1LL << 26)) __trap();
  }
}

template <bool BOX, int NT, int TILE>
__global__ void __launch_bounds__(NT, 1) pack_bits_tma(const RoiParams* __restrict__ rp,
                                                      uint32_t* __restrict__ bits,
                                                      Stats* __restrict__ st,
                                                      uint32_t* __restrict__ segmap,
                                                      int stages) {
  KTrace kt_(st, kTrPack);
  extern __shared__ __align__(128) unsigned char s_tiles[];  // stages x TILE
  __shared__ __align__(8) uint64_t s_full[kTmaMaxStages];
  __shared__ int s_tile[kTmaMaxStages];  // tile held by each stage (>= tiles: none)
  const unsigned char* mask = rp->mask;
  const long long n_bytes = 16LL * rp->n_chunks;
  const bool sparse = rp->sparse != 0;
  const bool skip = (rp->sparse & 2) != 0;
  const unsigned int W = (unsigned int)rp->W, ny = (unsigned int)rp->ny;
  BoxAcc box;  // BOX: occupied bbox of the nonzero words (replaces bits_bbox)
  // A contiguous share of tiles per CTA (dynamic per-tile claims measured
  // slower in the batch: C4 +3 us/ROI).
  const int tiles = (int)((n_bytes + TILE - 1) / TILE);
  const int per = (tiles + (int)gridDim.x - 1) / (int)gridDim.x;
  int t_next = min(tiles, (int)blockIdx.x * per);  // static share [t_next, t_end)
  const int t_end = min(tiles, t_next + per);
  uint64_t policy;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  auto issue = [&](int s) {  // thread 0 only: claim the next tile into stage s
    const int t = t_next < t_end ? t_next++ : tiles;
    s_tile[s] = t;
    if (t < tiles) {
      const long long off = (long long)t * TILE;
      const unsigned bytes = (unsigned)min((long long)TILE, n_bytes - off);
      mbar_expect_tx(&s_full[s], bytes);
      bulk_load(s_tiles + s * TILE, mask + off, bytes, &s_full[s], policy);
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; s++) mbar_init(&s_full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < stages; s++) issue(s);
  }
  __syncthreads();
  constexpr int kK = TILE / 16 / NT;  // 16-byte chunks per thread per tile (4 or 8)
  const long long gend = n_bytes / 16;
  // Stage s is consumed at steps s, s + stages, ...; its next claim is
  // written after the step's barrier and read stages - 1 barriers later
  // (stages >= 2: with one stage that read would race the write).
  // Claims only grow, so the first stage without a tile ends the loop.
  for (int k = 0;; k++) {
    const int s = k % stages;
    const int t = s_tile[s];
    if (t >= tiles) break;  // block-uniform
    mbar_wait(&s_full[s], (unsigned)(k / stages) & 1u);
    const long long g0 = (long long)t * (TILE / 16);  // first chunk of the tile
    const uint4* tile = reinterpret_cast<const uint4*>(s_tiles + s * TILE);
    // Only the last tile can be partial: bytes past the mask in its stage are stale.
    const bool full = t + 1 < tiles || n_bytes % TILE == 0;
    // Groups of (up to) 4 chunks per thread: registers stay bounded for any
    // tile / CTA size.
    constexpr int kG = kK < 4 ? kK : 4;
#pragma unroll 1
    for (int q0 = 0; q0 < kK; q0 += kG) {
      uint4 v[kG];
      uint32_t any = 0u;
#pragma unroll
      for (int q = 0; q < kG; q++) {
        const int ci = (q0 + q) * NT + threadIdx.x;
        v[q] = tile[ci];
        if (!full && g0 + ci >= gend) v[q] = make_uint4(0u, 0u, 0u, 0u);
        any |= v[q].x | v[q].y | v[q].z | v[q].w;
      }
      // Sparse: one vote clears the warp's kG segments at once when they are
      // all background -- most of a KiTS-like grid -- so the pack costs a few
      // issue slots per 2 KB there and leaves the SMs to other ROIs' kernels.
      if (skip && !__any_sync(kFull, any != 0u)) continue;
#pragma unroll
      for (int q = 0; q < kG; q++) {
        const int ci = (q0 + q) * NT + threadIdx.x;
        const long long g = g0 + ci;
        if (skip && !__any_sync(kFull, (v[q].x | v[q].y | v[q].z | v[q].w) != 0u)) continue;
        const uint32_t b16 = nib4(v[q].x) | (nib4(v[q].y) << 4) | (nib4(v[q].z) << 8) |
                             (nib4(v[q].w) << 12);
        const uint32_t word = b16 | (__shfl_down_sync(kFull, b16, 1) << 16);
        if (sparse) {
          if (!__any_sync(kFull, word != 0u && !(threadIdx.x & 1) && g < gend)) continue;
          if ((threadIdx.x & 31) == 0) {
            const long long seg = g >> 5;
            atomicOr(segmap + (seg >> 5), 1u << (seg & 31));
          }
        }
        if (!(threadIdx.x & 1) && g < gend) {
          bits[g >> 1] = word;
          if (BOX && word) {
            const unsigned int wi = (unsigned int)(g >> 1), row = wi / W, col = wi - row * W;
            const unsigned int z = row / ny, y = row - z * ny;
            box.x0 = min(box.x0, (int)(32 * col) + __ffs(word) - 1);
            box.x1 = max(box.x1, (int)(32 * col) + 31 - __clz(word));
            box.y0 = min(box.y0, (int)y); box.y1 = max(box.y1, (int)y);
            box.z0 = min(box.z0, (int)z); box.z1 = max(box.z1, (int)z);
          }
        }
      }
    }
    __syncthreads();  // every thread is done with stage s
    if (threadIdx.x == 0) issue(s);
  }
  if (BOX) box.flush(st);
}
#define SC_TMA_INST(BOX, NT, TILE) \
  template __global__ void pack_bits_tma<BOX, NT, TILE>(const RoiParams*, uint32_t*, Stats*, uint32_t*, int);
SC_TMA_INST(false, 256, 16384) SC_TMA_INST(true, 256, 16384)
SC_TMA_INST(false, 128, 16384) SC_TMA_INST(true, 128, 16384)
SC_TMA_INST(false, 256, 32768) SC_TMA_INST(true, 256, 32768)
SC_TMA_INST(false, 256, 8192) SC_TMA_INST(true, 256, 8192)
SC_TMA_INST(false, 128, 32768) SC_TMA_INST(true, 128, 32768)
SC_TMA_INST(false, 64, 32768) SC_TMA_INST(true, 64, 32768)
#undef SC_TMA_INST

// Occupied bbox from the bit volume (L2-resident right after the pack): only
// nonzero words locate themselves.  Four 16-byte loads in flight per thread.
__global__ void __launch_bounds__(256) bits_bbox(const RoiParams* __restrict__ rp,
                                                 const uint4* __restrict__ bits4,
                                                 Stats* __restrict__ st,
                                                 const uint32_t* __restrict__ segmap) {
  pdl_enter();
  constexpr int kU = 4;
  const long long n_words = rp->n_words;
  const int W = rp->W, ny = (int)rp->ny;
  BoxAcc box;
  if (rp->sparse) {
    // Only the marked segments (the occupied rows) are read: one thread per
    // segment, its 16 words as 4 x 16 bytes.
    const long long n_seg = (n_words + 15) / 16;
    const uint32_t* bits = reinterpret_cast<const uint32_t*>(bits4);
    for (long long sgi = (long long)blockIdx.x * blockDim.x + threadIdx.x; sgi < n_seg;
         sgi += (long long)gridDim.x * blockDim.x) {
      if (!seg_on(segmap, 16 * sgi)) continue;
      if (16 * sgi + 16 <= n_words) {
        uint4 v[4];
#pragma unroll
        for (int t = 0; t < 4; t++) v[t] = __ldcg(bits4 + 4 * sgi + t);
        // locate the first word once (one 64-bit division), then step the
        // (w, y, z) position word by word
        const long long row = 16 * sgi / W;
        int w = (int)(16 * sgi - row * W), z = (int)(row / ny), y = (int)(row - (long long)z * ny);
#pragma unroll
        for (int t = 0; t < 4; t++) {
          const uint32_t w4[4] = {v[t].x, v[t].y, v[t].z, v[t].w};
#pragma unroll
          for (int u = 0; u < 4; u++) {
            if (w4[u]) box.add_at(w4[u], w, y, z);
            if (++w == W) {
              w = 0;
              if (++y == ny) { y = 0; z++; }
            }
          }
        }
      } else {
        for (long long wi = 16 * sgi; wi < n_words; wi++) {
          const uint32_t w = __ldcg(bits + wi);
          if (w) box.add(w, wi, W, ny);
        }
      }
    }
    box.flush(st);
    return;
  }
  const long long n4 = n_words / 4;
  const long long step = (long long)gridDim.x * blockDim.x * kU;
  for (long long base = (long long)blockIdx.x * blockDim.x * kU; base < n4; base += step) {
    uint4 v[kU];
#pragma unroll
    for (int k = 0; k < kU; k++) {
      const long long i = base + (long long)k * blockDim.x + threadIdx.x;
      v[k] = i < n4 ? __ldcg(bits4 + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < kU; k++) {
      if (v[k].x | v[k].y | v[k].z | v[k].w) {
        const long long i = base + (long long)k * blockDim.x + threadIdx.x;
        const uint32_t w4[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
        const long long row = 4 * i / W;
        int w = (int)(4 * i - row * W), z = (int)(row / ny), y = (int)(row - (long long)z * ny);
#pragma unroll
        for (int t = 0; t < 4; t++) {
          if (w4[t]) box.add_at(w4[t], w, y, z);
          if (++w == W) {
            w = 0;
            if (++y == ny) { y = 0; z++; }
          }
        }
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (int)(n_words & 3)) {  // 1-3 word tail
    const long long wi = 4 * n4 + threadIdx.x;
    const uint32_t w = __ldcg(reinterpret_cast<const uint32_t*>(bits4) + wi);
    if (w) box.add(w, wi, W, ny);
  }
  box.flush(st);
}

// Generic path: any nx / alignment.  One output word per thread, byte loads
// (still coalesced across the warp within a row).
__global__ void __launch_bounds__(256) pack_bits_generic(const RoiParams* __restrict__ rp,
                                                         uint32_t* __restrict__ bits,
                                                         Stats* __restrict__ st,
                                                         uint32_t* __restrict__ segmap) {
  KTrace kt_(st, kTrPack);
  const uint8_t* __restrict__ mask = rp->mask;
  const long long n_words = rp->n_words;
  const int nx = (int)rp->nx, W = rp->W, ny = (int)rp->ny;
  BoxAcc box;
  const long long step = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < n_words; base += step) {
    long long wi = base + threadIdx.x;
    if (wi < n_words) {
      long long row = wi / W;
      int w = (int)(wi - row * W);
      const uint8_t* src = mask + row * (long long)nx + 32 * w;
      int n = min(32, nx - 32 * w);
      uint32_t word = 0;
      for (int b = 0; b < n; b++) word |= (uint32_t)(__ldcs(src + b) != 0) << b;
      bits[wi] = word;  // every word is written; the map marks the nonzero ones
      if (word) {
        box.add(word, wi, W, ny);
        if (rp->sparse) atomicOr(segmap + (wi >> 9), 1u << ((wi >> 4) & 31));
      }
    }
  }
  box.flush(st);
}

// Lattice row (v, w) seen by word column q: bit i <-> voxel x = 32q - 1 + i,
// i in [0, 32] (word q shifted up by one, bit 31 of word q - 1 below it).
// Out-of-grid voxels are background (this IS the reference's zero padding,
// mesh.py:55-65).
// Word wi of the bit volume; with a sparse bit volume, words of unmarked
// segments read as 0.
__device__ __forceinline__ uint32_t seg_word(const uint32_t* __restrict__ bits,
                                             const uint32_t* __restrict__ segmap, bool sparse,
                                             long long wi) {
  // The map bit first: the data word is only loaded for a marked segment
  // (most rows of a sparse bbox are background: one L1-resident map load).
  if (sparse) {
    const unsigned int lo = (unsigned int)wi;  // bit (wi >> 4) & 31 needs only the low word
    if (!((__ldg(segmap + (wi >> 9)) >> ((lo >> 4) & 31u)) & 1u)) return 0u;
  }
  return bits[wi];
}

// Words q and q - 1 of row (v, w).  All lanes call (converged).  Lanes hold
// consecutive word columns of one row (item order: q fastest), so word q - 1
// is the previous lane's word q; at q == qlo (q_first) it is zero (left of the
// occupied bbox), and only lane 0 with q > qlo loads it itself.
__device__ __forceinline__ void row_words(const uint32_t* __restrict__ bits,
                                          const uint32_t* __restrict__ segmap, bool sparse, int q,
                                          bool q_first, int v, int w, int W, int ny, int nz,
                                          bool on, uint32_t& cur, uint32_t& prev) {
  cur = 0u;
  const bool in = on && v >= 0 && v < ny && w >= 0 && w < nz;
  const long long rb = ((long long)w * ny + v) * W;
  if (in && q < W) cur = seg_word(bits, segmap, sparse, rb + q);
  prev = __shfl_up_sync(kFull, cur, 1);
  if (q_first) prev = 0u;
  else if ((threadIdx.x & 31) == 0) prev = in ? seg_word(bits, segmap, sparse, rb + q - 1) : 0u;
}

constexpr int kStage = 256;  // staged vertices per warp and z step (denser steps emit directly)

// One thread = one (word column q, row v) and kz consecutive z steps (kz is
// chosen per ROI on the device and is grid-uniform, so the rolled step loop
// keeps the warp intrinsics converged).  The step body is not unrolled: the
// 4x-unrolled form (4.1 K SASS instructions) spent a quarter of its warp
// samples in instruction-fetch stalls on C3.
// Cell (u, v, w) has lower corner at unpadded voxel (u, v, w), u,v,w >= -1
// (reference padded cell index minus 1).  The thread owns cells and lattice
// points u = 32q - 1 + i, i in [0, 31].  Row words of the layer two steps
// ahead are loaded at the top of each step (L2-resident bit volume; latency,
// not bandwidth, bound).
//
// Every emitted vertex is also counted into the histograms the diameter stage
// sorts by: its 3-D Morton brick (block-private, flushed once per block) and
// its (plane, in-plane brick) bin in each of its three planes (global).
//
// Cells and vertices are owned by the z layer w of their lower corner (x / y
// edges in layer w, z edges from w to w + 1), so the layers [wlo, whi] of a
// slab split (RoiParams::mc_slab) partition cells and vertices exactly.
__device__ __forceinline__ long long mc_body(int kz, int wlo, int whi,
                                        const RoiParams* __restrict__ rp,
                                        const uint32_t* __restrict__ bits,
                                        const uint32_t* __restrict__ segmap,
                                        Stats* __restrict__ st,
                                        int4* __restrict__ vkeys, long long cap,
                                        unsigned int* __restrict__ sort_counts,
                                        unsigned int* __restrict__ pbin_counts, const int* bb,
                                        unsigned int* s_hist, const int4* __restrict__ tn_raw,
                                        unsigned int* s_sup, int4 (*s_stage)[kStage]) {
  const int ny = (int)rp->ny, nz = (int)rp->nz, W = rp->W;
  const bool sparse = rp->sparse != 0;
  const PlaneSpace ps = plane_space(bb);
  const PlaneBricks pbk = plane_bricks(bb);
  const int bshift = brick_shift(bb);

  const int xmin = bb[0], ymin = bb[1];
  const int xmax = bb[3], ymax = bb[4];
  long long volk = 0;
  const int lane = threadIdx.x & 31;
  // Warp-private vertex stage (warp-uniform fill level), see the emission.
  uint32_t staged = 0;
  // Write the warp's staged vertices at [wbase, wbase + staged) and bin them.
  auto flush_at = [&](unsigned long long wbase) {
    const int4* stg = s_stage[threadIdx.x >> 5];
    for (uint32_t k0 = 0; k0 < staged; k0 += 32) {
      const uint32_t k = k0 + lane;
      const bool ok = k < staged;
      const int4 key = stg[ok ? k : 0];
      const long long g = (long long)wbase + k;
      if (ok && g < cap) vkeys[g] = key;
      const unsigned int bin = brick_bin(key.x, key.y, key.z, bb, bshift);
      seg_add(sort_counts, bin, ok);
      if (ok) atomicAdd(&s_sup[bin >> kSortSliceBits], 1u);
      int id[3];
      unsigned int pbin[3];
      plane_ids(key.x, key.y, key.z, ps, id);
      plane_bins(key.x, key.y, key.z, pbk, pbin);
#pragma unroll
      for (int a2 = 0; a2 < 3; a2++)
        seg_add(pbin_counts, (unsigned int)id[a2] * kPlaneBins + pbin[a2], ok);
    }
    __syncwarp();  // the stage is refilled next
  };
  // Mid-kernel flush of a full stage: the warp reserves its own range.
  auto flush = [&]() {
    __syncwarp();
    unsigned long long wbase = 0;
    if (lane == 0) wbase = atomicAdd(&st->n_vert, (unsigned long long)staged);
    flush_at(__shfl_sync(kFull, wbase, 0));
  };
  if (xmax >= 0) {
    // Points/cells that can be crossed or active: [min-1, max] on every axis.
    const int qlo = xmin >> 5, qhi = (xmax + 1) >> 5;
    const int vlo = ymin - 1;
    const int nq = qhi - qlo + 1, nv = ymax - vlo + 1;
    const int nzc = (whi - wlo + 1 + kz - 1) / kz;
    const long long n_items = (long long)nq * nv * nzc;
    const long long step = (long long)gridDim.x * blockDim.x;
    for (long long base = (long long)blockIdx.x * blockDim.x; base < n_items; base += step) {
      const long long item = base + threadIdx.x;
      const bool valid = item < n_items;
      int q = 0, v = 0, w0 = 0;
      if (valid) {
        if (n_items < (1LL << 32)) {  // (grid-uniform) 32-bit decomposition
          const unsigned int it = (unsigned int)item, r = it / (unsigned int)nq;
          q = qlo + (int)(it - r * (unsigned int)nq);
          const unsigned int r2 = r / (unsigned int)nv;
          v = vlo + (int)(r - r2 * (unsigned int)nv);
          w0 = wlo + (int)r2 * kz;
        } else {
          q = qlo + (int)(item % nq);
          long long r = item / nq;
          v = vlo + (int)(r % nv);
          w0 = wlo + (int)(r / nv) * kz;
        }
      }
      const bool qf = !valid || q == qlo;  // word q - 1 is background (see row_words)
      // Rows (v, w) and (v + 1, w) of the step's two z layers; the layer two
      // steps ahead is loaded at the top of each step (one rolled body keeps
      // the kernel inside the instruction cache).
      uint32_t ca0, pa0, cb0, pb0, ca1, pa1, cb1, pb1;
      {
        const bool on0 = valid && w0 <= whi + 1, on1 = valid && 1 <= kz && w0 + 1 <= whi + 1;
        row_words(bits, segmap, sparse, q, qf, v, w0, W, ny, nz, on0, ca0, pa0);
        row_words(bits, segmap, sparse, q, qf, v + 1, w0, W, ny, nz, on0, cb0, pb0);
        row_words(bits, segmap, sparse, q, qf, v, w0 + 1, W, ny, nz, on1, ca1, pa1);
        row_words(bits, segmap, sparse, q, qf, v + 1, w0 + 1, W, ny, nz, on1, cb1, pb1);
      }
      const int xbase = 32 * q - 1;
#pragma unroll 1
      for (int s = 0; s < kz; s++) {  // kz is grid-uniform: the warp stays converged
        const int w = w0 + s;
        uint32_t ca2, pa2, cb2, pb2;
        const bool on2 = valid && s + 2 <= kz && w + 2 <= whi + 1;
        row_words(bits, segmap, sparse, q, qf, v, w + 2, W, ny, nz, on2, ca2, pa2);
        row_words(bits, segmap, sparse, q, qf, v + 1, w + 2, W, ny, nz, on2, cb2, pb2);
        const bool on = valid && w <= whi;
        const unsigned long long A = ((unsigned long long)ca0 << 1) | (pa0 >> 31);
        const unsigned long long B = ((unsigned long long)cb0 << 1) | (pb0 >> 31);
        const unsigned long long C = ((unsigned long long)ca1 << 1) | (pa1 >> 31);
        const unsigned long long D = ((unsigned long long)cb1 << 1) | (pb1 >> 31);
        ca0 = ca1; pa0 = pa1; cb0 = cb1; pb0 = pb1;
        ca1 = ca2; pa1 = pa2; cb1 = cb2; pb1 = pb2;
        // Background around the whole warp (most steps of a sparse bbox): no
        // active cell, no crossed edge -- nothing else to do this step.
        if (!__any_sync(kFull, on && (A | B | C | D) != 0ull)) continue;
        uint32_t ex = 0, ey = 0, ez = 0, act = 0;
        if (on) {
          ex = (uint32_t)(A ^ (A >> 1));
          ey = (uint32_t)(A ^ B);
          ez = (uint32_t)(A ^ C);
          const unsigned long long all = A & B & C & D, any = A | B | C | D;
          act = (uint32_t)(~(all & (all >> 1)) & (any | (any >> 1)));
        }
        // Active cells.  The shared histogram and the case table (tn_raw,
        // read through L1) are indexed by the raw corner word idx =
        // A[i..i+1] | B[i..i+1]<<2 | C[..]<<4 | D[..]<<6 (4 shift-and pairs);
        // case_of_idx() maps it to the reference case (bit c set when corner
        // c is background, mc_tables.py:10-12, mesh.py:103-128) when the
        // table is built and at the histogram flush.
        // The volume terms are summed in 32 bits per step, widened once.
        int s0 = 0, sx = 0, sy = 0, sz = 0;
        while (act) {
          const int i = __ffs(act) - 1;
          act &= act - 1;
          const uint32_t idx = (uint32_t)((A >> i) & 3) | ((uint32_t)((B >> i) & 3) << 2) |
                               ((uint32_t)((C >> i) & 3) << 4) | ((uint32_t)((D >> i) & 3) << 6);
          atomicAdd(&s_hist[idx], 1u);
          const int4 tn = __ldg(tn_raw + idx);  // L1-resident 4 KB table
          s0 += tn.x;
          sx += (xbase + i) * tn.y;
          sy += tn.z;
          sz += tn.w;
        }
        volk += s0 + 2ll * ((long long)sx + (long long)v * sy + (long long)w * sz);
        // Vertex emission: warp-aggregated stream compaction of crossed edges.
        const uint32_t c = __popc(ex) + __popc(ey) + __popc(ez);
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          uint32_t t = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += t;
        }
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        if (total) {
          const int Y2 = 2 * v, Z2 = 2 * w;
          if (pbin_counts && total <= kStage) {
            // Stage the step's vertices in shared memory (cheap per-lane
            // loop); the stage accumulates over steps and is flushed -- one
            // global reservation, coalesced key stores, converged binning --
            // only when the next step would not fit (or at the end).
            if (staged + total > kStage) {
              flush();
              staged = 0;
            }
            int4* stg = s_stage[threadIdx.x >> 5];
            uint32_t o = staged + incl - c;
            while (ex) {
              const int i = __ffs(ex) - 1; ex &= ex - 1;
              stg[o++] = make_int4(2 * (xbase + i) + 1, Y2, Z2, 0);
            }
            while (ey) {
              const int i = __ffs(ey) - 1; ey &= ey - 1;
              stg[o++] = make_int4(2 * (xbase + i), Y2 + 1, Z2, 0);
            }
            while (ez) {
              const int i = __ffs(ez) - 1; ez &= ez - 1;
              stg[o++] = make_int4(2 * (xbase + i), Y2, Z2 + 1, 0);
            }
            staged += total;
          } else {
            unsigned long long wbase = 0;
            if (lane == 31) wbase = atomicAdd(&st->n_vert, (unsigned long long)total);
            wbase = __shfl_sync(kFull, wbase, 31);
            long long o = (long long)(wbase + incl - c);
            auto emit = [&](int X, int Y, int Z) {
              if (o < cap) vkeys[o] = make_int4(X, Y, Z, 0);
              o++;
              if (pbin_counts) {  // NULL on the mesh-export path (no diameter stage)
                const unsigned int bin = brick_bin(X, Y, Z, bb, bshift);
                atomicAdd(&sort_counts[bin], 1u);
                atomicAdd(&s_sup[bin >> kSortSliceBits], 1u);
                int id[3];
                unsigned int pbin[3];
                plane_ids(X, Y, Z, ps, id);
                plane_bins(X, Y, Z, pbk, pbin);
#pragma unroll
                for (int a2 = 0; a2 < 3; a2++)
                  atomicAdd(&pbin_counts[(long long)id[a2] * kPlaneBins + pbin[a2]], 1u);
              }
            };
            while (ex) {
              const int i = __ffs(ex) - 1; ex &= ex - 1;
              emit(2 * (xbase + i) + 1, Y2, Z2);
            }
            while (ey) {
              const int i = __ffs(ey) - 1; ey &= ey - 1;
              emit(2 * (xbase + i), Y2 + 1, Z2);
            }
            while (ez) {
              const int i = __ffs(ez) - 1; ez &= ez - 1;
              emit(2 * (xbase + i), Y2, Z2 + 1);
            }
          }
        }
      }
    }
  }
  // Final flush: one reservation per block for the last stage of all its
  // warps (every warp ends here; per-warp reservations were thousands of
  // returning atomics on the one n_vert counter per ROI).
  __shared__ unsigned int s_wcnt[256 / 32];
  __shared__ unsigned long long s_wbase;
  if (lane == 0) s_wcnt[threadIdx.x >> 5] = staged;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
      const unsigned int c = s_wcnt[w];
      s_wcnt[w] = tot;
      tot += c;
    }
    s_wbase = tot ? atomicAdd(&st->n_vert, (unsigned long long)tot) : 0ull;
  }
  __syncthreads();
  if (staged) flush_at(s_wbase + s_wcnt[threadIdx.x >> 5]);
  return volk;
}

__global__ void __launch_bounds__(256, 4) mc_cells(const RoiParams* __restrict__ rp,
                                                const uint32_t* __restrict__ bits,
                                                const CaseTables* __restrict__ tabs,
                                                Stats* __restrict__ st, int4* __restrict__ vkeys,
                                                long long cap, unsigned int* __restrict__ sort_counts,
                                                unsigned int* __restrict__ pbin_counts,
                                                const uint32_t* __restrict__ segmap) {
  pdl_enter();
  KTrace kt_(st, kTrMc);
  __shared__ unsigned int s_hist[kNumCases];
  __shared__ unsigned int s_sup[kSortSupers];
  __shared__ int4 s_stage[256 / 32][kStage];  // per-warp vertex stage (blockDim = 256)
  int bb[6];
#pragma unroll
  for (int i = 0; i < 6; i++) bb[i] = st->bbox[i];
  if (bb[3] < 0) return;  // empty ROI (block-uniform)
  // z steps per thread, chosen per ROI from the bbox: the deepest of 8 / 4
  // that still gives every resident thread an item (fewer row loads and chunk
  // prologues per step; C3 single call 162 -> 150 us at 8), 1 or 2 for small
  // bboxes, where parallelism -- not loads -- is the limit (C2: ~22 K items at
  // depth 4 for ~150 K resident threads).
  const long long cols = (long long)(((bb[3] + 1) >> 5) - (bb[0] >> 5) + 1) * (bb[4] - bb[1] + 2);
  // Cell layers [zmin - 1, zmax]; a slab split (the two-phase shard entry)
  // takes the shard's contiguous share of them.
  int wlo = bb[2] - 1, whi = bb[5];
  if (rp->mc_slab) {
    // (32-bit: a 64-bit division would inline a long routine into a kernel
    // that sits at the edge of the instruction cache; L < 2^16, shards < 2^15)
    const unsigned int ns = (unsigned int)rp->mc_slab >> 16, sh = (unsigned int)rp->mc_slab & 0xffffu;
    const unsigned int L = (unsigned int)(whi - wlo + 1);
    const int a = wlo + (int)(L * sh / ns), b = wlo + (int)(L * (sh + 1) / ns);
    wlo = a;
    whi = b - 1;
    if (whi < wlo) return;  // more shards than layers: nothing here (grid-uniform)
  }
  const int zs = whi - wlo + 1;
  const long long threads = (long long)gridDim.x * blockDim.x;
  const int kz = cols * ((zs + 7) / 8) >= threads   ? 8
                 : cols * ((zs + 3) / 4) >= threads ? 4
                 : cols * ((zs + 1) / 2) >= threads ? 2
                                                    : 1;
  // blocks past the bbox's work items have nothing to do: skip the prologue too
  if ((long long)blockIdx.x * blockDim.x >= cols * ((zs + kz - 1) / kz)) return;
  for (int i = threadIdx.x; i < kNumCases; i += blockDim.x) {
    s_hist[i] = 0;
  }
  for (int i = threadIdx.x; i < kSortSupers; i += blockDim.x) s_sup[i] = 0;
  __syncthreads();
  long long volk = mc_body(kz, wlo, whi, rp, bits, segmap, st, vkeys, cap, sort_counts, pbin_counts, bb,
                              s_hist, tabs->tn_raw, s_sup, s_stage);
  const int lane = threadIdx.x & 31;
  // Block flush: exact integer partials.
#pragma unroll
  for (int o = 16; o; o >>= 1) volk += __shfl_xor_sync(kFull, volk, o);
  if (lane == 0 && volk) atomicAdd(reinterpret_cast<unsigned long long*>(&st->vol_k),
                                   (unsigned long long)volk);
  __syncthreads();
  for (int i = threadIdx.x; i < kNumCases; i += blockDim.x)
    if (s_hist[i])
      atomicAdd(&st->hist[blockIdx.x % kHistCopies][case_of_idx(i)], (unsigned long long)s_hist[i]);
  if (sort_counts)
    for (int i = threadIdx.x; i < kSortSupers; i += blockDim.x)
      if (s_sup[i]) atomicAdd(&sort_counts[kSortBins + i], s_sup[i]);
}


template __global__ void pack_bits_v16<4, false>(const RoiParams*, uint32_t*, Stats*, uint32_t*);
template __global__ void pack_bits_v16<4, true>(const RoiParams*, uint32_t*, Stats*, uint32_t*);

}  // namespace sc
