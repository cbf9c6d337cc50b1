// Canonical triangle mesh on the GPU: the
// reference's TriangleMesh bit for bit -- same vertex coordinates, same vertex
// numbering, same triangle list order (pkg/src/shapecore/mesh.py:142-199).
//
// The reference scans cells in (z, y, x) order, emits each active cell's
// triangles in table order and numbers a vertex at its first reference.
// On the GPU:
//   mesh_count   one thread per (w, v, q) item -- 32 cells of one row, items
//                enumerated in exactly that scan order -- counts its triangles;
//   scan         exclusive scan of the counts = each item's first triangle;
//   edge_map     lattice edge -> vertex index (bbox-local dense map);
//   mesh_emit    writes every triangle at its canonical position and
//                atomicMin's the first reference 3t+k of each vertex;
//   flags+scan   vertex id = rank of its first reference;
//   mesh_out     coordinates (key/2)*s in fp64, triangles as ids.
#include "sc_device.cuh"
#include "mc_tables.h"

namespace sc {

__constant__ int8_t c_tri[256][16];
__constant__ int8_t c_edge[12][4];  // axis, dx, dy, dz

struct MeshBox {  // item / lattice ranges derived from the occupied bbox
  int qlo, nq, vlo, nv, wlo, nw;
  int ox, oy, oz;  // lattice origin of the edge map (= min - 1 per axis)
  int mx, my, mz;  // edge-map extents (points)
};

__device__ __forceinline__ MeshBox mesh_box(const Stats* st) {
  const int* bb = st->bbox;
  MeshBox m;
  m.qlo = bb[0] >> 5;
  m.nq = ((bb[3] + 1) >> 5) - m.qlo + 1;
  m.vlo = bb[1] - 1;
  m.nv = bb[4] - m.vlo + 1;
  m.wlo = bb[2] - 1;
  m.nw = bb[5] - m.wlo + 1;
  m.ox = bb[0] - 1; m.oy = bb[1] - 1; m.oz = bb[2] - 1;
  m.mx = bb[3] - bb[0] + 2; m.my = bb[4] - bb[1] + 2; m.mz = bb[5] - bb[2] + 2;
  return m;
}

__device__ __forceinline__ unsigned long long win33(const uint32_t* __restrict__ bits, int q, int v,
                                                    int w, int W, int ny, int nz) {
  if (v < 0 || v >= ny || w < 0 || w >= nz) return 0ull;
  const uint32_t* row = bits + ((long long)w * ny + v) * W;
  const unsigned long long cur = q < W ? row[q] : 0u;
  const unsigned long long prev = q > 0 ? row[q - 1] : 0u;
  return (cur << 1) | (prev >> 31);
}

// Cells of item (q, v, w): active mask and per-cell case via the same bit
// algebra as mc_cells.  Bit i <-> cell u = 32q - 1 + i.
struct ItemCells {
  unsigned long long A, B, C, D;
  uint32_t act;
};

__device__ __forceinline__ ItemCells item_cells(const uint32_t* bits, int q, int v, int w, int W,
                                                int ny, int nz) {
  ItemCells it;
  it.A = win33(bits, q, v, w, W, ny, nz);
  it.B = win33(bits, q, v + 1, w, W, ny, nz);
  it.C = win33(bits, q, v, w + 1, W, ny, nz);
  it.D = win33(bits, q, v + 1, w + 1, W, ny, nz);
  const unsigned long long all = it.A & it.B & it.C & it.D, any = it.A | it.B | it.C | it.D;
  it.act = (uint32_t)(~(all & (all >> 1)) & (any | (any >> 1)));
  return it;
}

__device__ __forceinline__ int cell_case(const ItemCells& it, int i) {
  const uint32_t occ = (uint32_t)((it.A >> i) & 1) | (uint32_t)(((it.A >> (i + 1)) & 1) << 1) |
                       (uint32_t)(((it.B >> (i + 1)) & 1) << 2) | (uint32_t)(((it.B >> i) & 1) << 3) |
                       (uint32_t)(((it.C >> i) & 1) << 4) | (uint32_t)(((it.C >> (i + 1)) & 1) << 5) |
                       (uint32_t)(((it.D >> (i + 1)) & 1) << 6) | (uint32_t)(((it.D >> i) & 1) << 7);
  return (~occ) & 0xff;
}

__device__ __forceinline__ int tri_count(int k) {
  int n = 0;
  while (n < 16 && c_tri[k][n] >= 0) n++;
  return n / 3;
}

// Items in reference scan order: item = ((w - wlo) * nv + (v - vlo)) * nq + (q - qlo).
__global__ void mesh_count(const RoiParams* __restrict__ rp, const uint32_t* __restrict__ bits,
                           const Stats* __restrict__ st, unsigned int* __restrict__ counts) {
  if (st->bbox[3] < 0) return;
  const MeshBox m = mesh_box(st);
  const int W = rp->W, ny = (int)rp->ny, nz = (int)rp->nz;
  const long long items = (long long)m.nq * m.nv * m.nw;
  for (long long it = (long long)blockIdx.x * blockDim.x + threadIdx.x; it < items;
       it += (long long)gridDim.x * blockDim.x) {
    const int q = m.qlo + (int)(it % m.nq);
    const long long r = it / m.nq;
    const int v = m.vlo + (int)(r % m.nv), w = m.wlo + (int)(r / m.nv);
    const ItemCells c = item_cells(bits, q, v, w, W, ny, nz);
    unsigned int n = 0;
    for (uint32_t a = c.act; a; a &= a - 1) n += tri_count(cell_case(c, __ffs(a) - 1));
    counts[it] = n;
  }
}

// ---- device-wide exclusive scan of uint32 (three kernels) -----------------
constexpr int kScanBlock = 1024;

__global__ void __launch_bounds__(kScanBlock) scan_blocks(unsigned int* __restrict__ data,
                                                          long long n,
                                                          unsigned int* __restrict__ block_sums) {
  const long long i = (long long)blockIdx.x * kScanBlock + threadIdx.x;
  const unsigned int v = i < n ? data[i] : 0u;
  unsigned int total;
  const unsigned int ex = block_exscan_1024(v, &total);
  if (i < n) data[i] = ex;
  if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanBlock) scan_sums(unsigned int* __restrict__ sums, int nb,
                                                        unsigned long long* __restrict__ total) {
  __shared__ unsigned int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b = 0; b < nb; b += kScanBlock) {
    const int i = b + threadIdx.x;
    const unsigned int v = i < nb ? sums[i] : 0u;
    unsigned int t;
    const unsigned int ex = block_exscan_1024(v, &t);
    if (i < nb) sums[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += t;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void scan_add(unsigned int* __restrict__ data, long long n,
                         const unsigned int* __restrict__ sums) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) data[i] += sums[i / kScanBlock];
}

// lattice edge (axis, point) -> vertex index; point relative to the map origin.
__device__ __forceinline__ long long emap_index(int axis, int x, int y, int z, const MeshBox& m) {
  return (((long long)axis * m.mz + (z - m.oz)) * m.my + (y - m.oy)) * m.mx + (x - m.ox);
}

__global__ void edge_map_fill(const int4* __restrict__ keys, const Stats* __restrict__ st,
                              int* __restrict__ emap) {
  const MeshBox m = mesh_box(st);
  const long long n = (long long)st->n_vert;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    const int4 k = keys[v];
    const int axis = (k.x & 1) ? 0 : ((k.y & 1) ? 1 : 2);  // the half-integer coordinate
    emap[emap_index(axis, k.x >> 1, k.y >> 1, k.z >> 1, m)] = (int)v;
  }
}

// Every active cell's triangles at their canonical positions; corner k of
// triangle t is reference 3t+k, and a vertex's id is the rank of its first
// reference (mesh.py:176-196).
__global__ void mesh_emit(const RoiParams* __restrict__ rp, const uint32_t* __restrict__ bits,
                          const Stats* __restrict__ st, const unsigned int* __restrict__ offsets,
                          const int* __restrict__ emap, int3* __restrict__ tris,
                          unsigned int* __restrict__ first_ref) {
  if (st->bbox[3] < 0) return;
  const MeshBox m = mesh_box(st);
  const int W = rp->W, ny = (int)rp->ny, nz = (int)rp->nz;
  const long long items = (long long)m.nq * m.nv * m.nw;
  for (long long it = (long long)blockIdx.x * blockDim.x + threadIdx.x; it < items;
       it += (long long)gridDim.x * blockDim.x) {
    const int q = m.qlo + (int)(it % m.nq);
    const long long r = it / m.nq;
    const int v = m.vlo + (int)(r % m.nv), w = m.wlo + (int)(r / m.nv);
    const ItemCells c = item_cells(bits, q, v, w, W, ny, nz);
    unsigned int t = offsets[it];
    for (uint32_t a = c.act; a; a &= a - 1) {  // ascending x = scan order within the row
      const int i = __ffs(a) - 1;
      const int k = cell_case(c, i);
      const int u = 32 * q - 1 + i;
      for (int e3 = 0; e3 < 16 && c_tri[k][e3] >= 0; e3 += 3, t++) {
        int vid[3];
#pragma unroll
        for (int corner = 0; corner < 3; corner++) {
          const int e = c_tri[k][e3 + corner];
          vid[corner] = emap[emap_index(c_edge[e][0], u + c_edge[e][1], v + c_edge[e][2],
                                        w + c_edge[e][3], m)];
          atomicMin(&first_ref[vid[corner]], 3u * t + corner);
        }
        tris[t] = make_int3(vid[0], vid[1], vid[2]);
      }
    }
  }
}

__global__ void id_flags(const unsigned int* __restrict__ first_ref, long long n,
                         unsigned int* __restrict__ flags) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x)
    flags[first_ref[v]] = 1u;
}

// ids[first_ref] is the exclusive scan of the flags: the vertex's id.
__global__ void mesh_out(const int4* __restrict__ keys, const unsigned int* __restrict__ first_ref,
                         const unsigned int* __restrict__ rank, long long n, double sx, double sy,
                         double sz, double* __restrict__ xs, double* __restrict__ ys,
                         double* __restrict__ zs, int* __restrict__ ids) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    const int id = (int)rank[first_ref[v]];
    const int4 k = keys[v];
    ids[v] = id;
    xs[id] = ref_coord(k.x, sx);  // (l - 1 + 0.5*[axis]) * s, mesh.py:184-195
    ys[id] = ref_coord(k.y, sy);
    zs[id] = ref_coord(k.z, sz);
  }
}

__global__ void tris_out(const int3* __restrict__ tris, long long nt, const int* __restrict__ ids,
                         int* __restrict__ out) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
       t += (long long)gridDim.x * blockDim.x) {
    const int3 c = tris[t];
    out[3 * t] = ids[c.x];
    out[3 * t + 1] = ids[c.y];
    out[3 * t + 2] = ids[c.z];
  }
}

cudaError_t upload_mesh_tables() {
  int8_t edge[12][4];
  for (int e = 0; e < 12; e++) {
    edge[e][0] = SC_EDGE_AXIS[e];
    edge[e][1] = SC_EDGE_DX[e];
    edge[e][2] = SC_EDGE_DY[e];
    edge[e][3] = SC_EDGE_DZ[e];
  }
  cudaError_t e = cudaMemcpyToSymbol(c_tri, SC_TRI_TABLE, sizeof(SC_TRI_TABLE));
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(c_edge, edge, sizeof(edge));
}

}  // namespace sc

namespace sc {

// ---- mesh measures with the reference's exact arithmetic ------------------
// features.py:89-118: per-triangle 0.5*sqrt(|(b-a)x(c-a)|^2) and a.(b x c)/6
// with numpy's cross (each component a product minus a product, rounded) and
// a left-to-right 3-term dot, then pairwise_sum (features.py:63-80): zero-pad
// to 2^k and fold halves -- reproduced exactly by fold_pass launches.
__device__ __forceinline__ void cross_rn(double u0, double u1, double u2, double w0, double w1,
                                         double w2, double& c0, double& c1, double& c2) {
  c0 = __dsub_rn(__dmul_rn(u1, w2), __dmul_rn(u2, w1));
  c1 = __dsub_rn(__dmul_rn(u2, w0), __dmul_rn(u0, w2));
  c2 = __dsub_rn(__dmul_rn(u0, w1), __dmul_rn(u1, w0));
}

__device__ __forceinline__ double dot3_rn(double a0, double a1, double a2, double b0, double b1,
                                          double b2) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a0, b0), __dmul_rn(a1, b1)), __dmul_rn(a2, b2));
}

__global__ void tri_terms(const double* __restrict__ xs, const double* __restrict__ ys,
                          const double* __restrict__ zs, const int* __restrict__ tris,
                          long long nt, long long padded, double* __restrict__ area,
                          double* __restrict__ vol) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < padded;
       t += (long long)gridDim.x * blockDim.x) {
    if (t >= nt) { area[t] = 0.0; vol[t] = 0.0; continue; }
    const int ia = tris[3 * t], ib = tris[3 * t + 1], ic = tris[3 * t + 2];
    const double ax = xs[ia], ay = ys[ia], az = zs[ia];
    const double bx = xs[ib], by = ys[ib], bz = zs[ib];
    const double cx = xs[ic], cy = ys[ic], cz = zs[ic];
    double c0, c1, c2;
    cross_rn(__dsub_rn(bx, ax), __dsub_rn(by, ay), __dsub_rn(bz, az), __dsub_rn(cx, ax),
             __dsub_rn(cy, ay), __dsub_rn(cz, az), c0, c1, c2);
    area[t] = __dmul_rn(0.5, __dsqrt_rn(dot3_rn(c0, c1, c2, c0, c1, c2)));
    cross_rn(bx, by, bz, cx, cy, cz, c0, c1, c2);
    vol[t] = __ddiv_rn(dot3_rn(ax, ay, az, c0, c1, c2), 6.0);
  }
}

__global__ void fold_pass(double* __restrict__ a, double* __restrict__ b, long long half) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < half;
       i += (long long)gridDim.x * blockDim.x) {
    a[i] = __dadd_rn(a[i], a[i + half]);
    b[i] = __dadd_rn(b[i], b[i + half]);
  }
}

}  // namespace sc
