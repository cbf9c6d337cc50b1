/* CPU ORACLE -- TEST INFRASTRUCTURE ONLY (see shape_oracle.h).
 *
 * Restates the reference algorithm step by step; each function cites the
 * reference file:line it follows.  Compiled with -ffp-contract=off so every
 * floating-point expression rounds exactly as numba / numpy do (no FMA).
 */
#include "shape_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../paper_2510_02894_b200/csrc/mc_tables.h"

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec / 1e6;
}

void or_free(void* p) { free(p); }

int or_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

static int tri_count(int k) {
  int n = 0;
  while (n < 16 && SC_TRI_TABLE[k][n] >= 0) n++;
  return n / 3;
}

/* mesh.py:55-65 pad_mask.  Nonzero input voxels become 1 (the reference only
 * ever sees binarized masks, volume.py:173-177). */
static uint8_t* pad(const uint8_t* data, int64_t nx, int64_t ny, int64_t nz) {
  int64_t pnx = nx + 2, pny = ny + 2, pnz = nz + 2;
  uint8_t* occ = (uint8_t*)calloc((size_t)(pnx * pny * pnz), 1);
  if (!occ) return NULL;
  for (int64_t z = 0; z < nz; z++)
    for (int64_t y = 0; y < ny; y++) {
      const uint8_t* src = data + (z * ny + y) * nx;
      uint8_t* dst = occ + ((z + 1) * pny + (y + 1)) * pnx + 1;
      for (int64_t x = 0; x < nx; x++) dst[x] = src[x] != 0;
    }
  return occ;
}

/* mesh.py:103-128 _cell_case: bit i set when corner i is background. */
static inline int cell_case(const uint8_t* occ, int64_t p, int64_t pnx, int64_t pny) {
  int c = 0;
  if (occ[p] == 0) c |= 1;
  if (occ[p + 1] == 0) c |= 2;
  if (occ[p + 1 + pnx] == 0) c |= 4;
  if (occ[p + pnx] == 0) c |= 8;
  int64_t q = p + pnx * pny;
  if (occ[q] == 0) c |= 16;
  if (occ[q + 1] == 0) c |= 32;
  if (occ[q + 1 + pnx] == 0) c |= 64;
  if (occ[q + pnx] == 0) c |= 128;
  return c;
}

int64_t or_active_cubes(const uint8_t* data, int64_t nx, int64_t ny, int64_t nz) {
  uint8_t* occ = pad(data, nx, ny, nz);
  if (!occ) return -1;
  int64_t pnx = nx + 2, pny = ny + 2, pnz = nz + 2, n = 0;
  for (int64_t cz = 0; cz < pnz - 1; cz++)
    for (int64_t cy = 0; cy < pny - 1; cy++) {
      int64_t base = (cz * pny + cy) * pnx;
      for (int64_t cx = 0; cx < pnx - 1; cx++) {
        int c = cell_case(occ, base + cx, pnx, pny);
        n += (c != 0 && c != 255);
      }
    }
  free(occ);
  return n;
}

int or_marching_cubes(const uint8_t* data, int64_t nx, int64_t ny, int64_t nz,
                      double sx, double sy, double sz, double** xs_out,
                      double** ys_out, double** zs_out, int32_t** tris_out,
                      int64_t* n_vert_out, int64_t* n_tri_out) {
  /* mesh.py:78-79 EmptyRoi */
  int64_t occupied = 0;
  for (int64_t i = 0; i < nx * ny * nz; i++) occupied += data[i] != 0;
  if (occupied == 0) return 3;

  uint8_t* occ = pad(data, nx, ny, nz);
  if (!occ) return -1;
  int64_t pnx = nx + 2, pny = ny + 2, pnz = nz + 2;
  int64_t n_points = pnx * pny * pnz;

  /* mesh.py:131-139 _count_triangles */
  int tc[256];
  for (int k = 0; k < 256; k++) tc[k] = tri_count(k);
  int64_t n_tri = 0;
  for (int64_t cz = 0; cz < pnz - 1; cz++)
    for (int64_t cy = 0; cy < pny - 1; cy++) {
      int64_t base = (cz * pny + cy) * pnx;
      for (int64_t cx = 0; cx < pnx - 1; cx++) n_tri += tc[cell_case(occ, base + cx, pnx, pny)];
    }

  /* mesh.py:94-100 _count_crossed_edges */
  int64_t n_vert = 0;
  for (int64_t z = 0; z < pnz; z++)
    for (int64_t y = 0; y < pny; y++)
      for (int64_t x = 0; x < pnx; x++) {
        int64_t p = (z * pny + y) * pnx + x;
        if (x + 1 < pnx) n_vert += occ[p] != occ[p + 1];
        if (y + 1 < pny) n_vert += occ[p] != occ[p + pnx];
        if (z + 1 < pnz) n_vert += occ[p] != occ[p + pnx * pny];
      }

  /* mesh.py:142-199 _emit_mesh */
  int32_t* ids = (int32_t*)calloc((size_t)(3 * n_points), sizeof(int32_t));
  double* xs = (double*)malloc(sizeof(double) * (size_t)(n_vert > 0 ? n_vert : 1));
  double* ys = (double*)malloc(sizeof(double) * (size_t)(n_vert > 0 ? n_vert : 1));
  double* zs = (double*)malloc(sizeof(double) * (size_t)(n_vert > 0 ? n_vert : 1));
  int32_t* tris = (int32_t*)malloc(sizeof(int32_t) * 3 * (size_t)(n_tri > 0 ? n_tri : 1));
  if (!ids || !xs || !ys || !zs || !tris) {
    free(ids); free(xs); free(ys); free(zs); free(tris); free(occ);
    return -1;
  }
  int64_t next_id = 0, nt = 0;
  for (int64_t cz = 0; cz < pnz - 1; cz++)
    for (int64_t cy = 0; cy < pny - 1; cy++)
      for (int64_t cx = 0; cx < pnx - 1; cx++) {
        int64_t p = (cz * pny + cy) * pnx + cx;
        int c = cell_case(occ, p, pnx, pny);
        if (c == 0 || c == 255) continue;
        const int8_t* row = SC_TRI_TABLE[c];
        for (int t = 0; t < 16 && row[t] >= 0; t += 3) {
          for (int corner = 0; corner < 3; corner++) {
            int e = row[t + corner];
            int axis = SC_EDGE_AXIS[e];
            int64_t lx = cx + SC_EDGE_DX[e], ly = cy + SC_EDGE_DY[e], lz = cz + SC_EDGE_DZ[e];
            int64_t key = axis * n_points + (lz * pny + ly) * pnx + lx;
            int32_t vid = ids[key];
            if (vid == 0) {
              vid = (int32_t)(++next_id);
              ids[key] = vid;
              double fx = (double)(lx - 1), fy = (double)(ly - 1), fz = (double)(lz - 1);
              if (axis == 0) fx += 0.5;
              else if (axis == 1) fy += 0.5;
              else fz += 0.5;
              xs[vid - 1] = fx * sx;
              ys[vid - 1] = fy * sy;
              zs[vid - 1] = fz * sz;
            }
            tris[3 * nt + corner] = vid - 1;
          }
          nt++;
        }
      }
  free(ids);
  free(occ);
  *xs_out = xs; *ys_out = ys; *zs_out = zs; *tris_out = tris;
  *n_vert_out = n_vert; *n_tri_out = n_tri;
  return 0;
}

/* features.py:63-80 pairwise_sum: zero-pad to 2^k, fold halves. */
double or_pairwise_sum(const double* v, int64_t n) {
  if (n == 0) return 0.0;
  int64_t size = 1;
  while (size < n) size <<= 1;
  double* buf = (double*)calloc((size_t)size, sizeof(double));
  memcpy(buf, v, sizeof(double) * (size_t)n);
  while (size > 1) {
    size /= 2;
    for (int64_t i = 0; i < size; i++) buf[i] = buf[i] + buf[i + size];
  }
  double r = buf[0];
  free(buf);
  return r;
}

/* np.cross(u, w) for 3-vectors: numpy forms each component as a product
 * minus a product, each rounded (numpy/core/numeric.py cross). */
static inline void cross3(const double u[3], const double w[3], double out[3]) {
  out[0] = u[1] * w[2] - u[2] * w[1];
  out[1] = u[2] * w[0] - u[0] * w[2];
  out[2] = u[0] * w[1] - u[1] * w[0];
}

static inline void corner(const double* xs, const double* ys, const double* zs, int32_t i,
                          double out[3]) {
  out[0] = xs[i]; out[1] = ys[i]; out[2] = zs[i];
}

/* features.py:89-96 surface_area */
double or_surface_area(const double* xs, const double* ys, const double* zs,
                       const int32_t* tris, int64_t n_tri) {
  if (n_tri == 0) return 0.0;
  double* areas = (double*)malloc(sizeof(double) * (size_t)n_tri);
  for (int64_t t = 0; t < n_tri; t++) {
    double a[3], b[3], c[3], u[3], w[3], cr[3];
    corner(xs, ys, zs, tris[3 * t], a);
    corner(xs, ys, zs, tris[3 * t + 1], b);
    corner(xs, ys, zs, tris[3 * t + 2], c);
    for (int k = 0; k < 3; k++) { u[k] = b[k] - a[k]; w[k] = c[k] - a[k]; }
    cross3(u, w, cr);
    double dot = cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2];
    areas[t] = 0.5 * sqrt(dot);
  }
  double s = or_pairwise_sum(areas, n_tri);
  free(areas);
  return s;
}

/* features.py:113-118 signed_mesh_volume */
double or_signed_mesh_volume(const double* xs, const double* ys, const double* zs,
                             const int32_t* tris, int64_t n_tri) {
  if (n_tri == 0) return 0.0;
  double* vals = (double*)malloc(sizeof(double) * (size_t)n_tri);
  for (int64_t t = 0; t < n_tri; t++) {
    double a[3], b[3], c[3], cr[3];
    corner(xs, ys, zs, tris[3 * t], a);
    corner(xs, ys, zs, tris[3 * t + 1], b);
    corner(xs, ys, zs, tris[3 * t + 2], c);
    cross3(b, c, cr);
    vals[t] = (a[0] * cr[0] + a[1] * cr[1] + a[2] * cr[2]) / 6.0;
  }
  double s = or_pairwise_sum(vals, n_tri);
  free(vals);
  return s;
}

/* features.py:99-110 mesh_volume: abs applied once at the end. */
double or_mesh_volume(const double* xs, const double* ys, const double* zs,
                      const int32_t* tris, int64_t n_tri) {
  return fabs(or_signed_mesh_volume(xs, ys, zs, tris, n_tri));
}

/* One vertex row of the pair loop, features.py:139-147 (shared by both
 * backends, so they agree bit for bit as the reference's do). */
static inline void row_max(const double* xs, const double* ys, const double* zs, int64_t n,
                           int64_t i, double* m3, double* mxy, double* mxz, double* myz) {
  double xi = xs[i], yi = ys[i], zi = zs[i];
  double a = *m3, b = *mxy, c = *mxz, d = *myz;
  for (int64_t j = i + 1; j < n; j++) {
    double dx = xs[j] - xi, dy = ys[j] - yi, dz = zs[j] - zi;
    double dd = dx * dx + dy * dy + dz * dz;
    if (dd > a) a = dd;
    double pxy = zs[j] == zi ? dd : 0.0;
    double pxz = ys[j] == yi ? dd : 0.0;
    double pyz = xs[j] == xi ? dd : 0.0;
    if (pxy > b) b = pxy;
    if (pxz > c) c = pxz;
    if (pyz > d) d = pyz;
  }
  *m3 = a; *mxy = b; *mxz = c; *myz = d;
}

/* features.py:121-148 _diameters_sq_seq */
void or_diameters_sq_seq(const double* xs, const double* ys, const double* zs, int64_t n,
                         double out[4]) {
  double m3 = 0.0, mxy = 0.0, mxz = 0.0, myz = 0.0;
  for (int64_t i = 0; i + 1 < n; i++) row_max(xs, ys, zs, n, i, &m3, &mxy, &mxz, &myz);
  out[0] = m3; out[1] = mxy; out[2] = mxz; out[3] = myz;
}

/* features.py:151-192 _diameters_sq_par: strip k = rows k and n-1-k. */
void or_diameters_sq_par(const double* xs, const double* ys, const double* zs, int64_t n,
                         int threads, double out[4]) {
  double m3 = 0.0, mxy = 0.0, mxz = 0.0, myz = 0.0;
  int64_t half = (n + 1) / 2;
#ifdef _OPENMP
  int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for num_threads(nt) schedule(static) reduction(max : m3, mxy, mxz, myz)
#endif
  for (int64_t k = 0; k < half; k++) {
    double a = m3, b = mxy, c = mxz, d = myz;
    row_max(xs, ys, zs, n, k, &a, &b, &c, &d);
    int64_t i2 = n - 1 - k;
    if (i2 != k) row_max(xs, ys, zs, n, i2, &a, &b, &c, &d);
    if (a > m3) m3 = a;
    if (b > mxy) mxy = b;
    if (c > mxz) mxz = c;
    if (d > myz) myz = d;
  }
  (void)threads;
  out[0] = m3; out[1] = mxy; out[2] = mxz; out[3] = myz;
}

/* features.py:224-265 extract_features (plus the exact counts the reference
 * does not expose: triangles = mesh.triangle_count, active cubes). */
int or_extract_features(const uint8_t* data, int64_t nx, int64_t ny, int64_t nz,
                        const double spacing[3], int threads, or_features* out) {
  double t0 = now_ms();
  double *xs, *ys, *zs;
  int32_t* tris;
  int64_t nv, nt;
  int rc = or_marching_cubes(data, nx, ny, nz, spacing[0], spacing[1], spacing[2], &xs, &ys,
                             &zs, &tris, &nv, &nt);
  if (rc != 0) return rc;
  double t_mesh = now_ms();
  out->mesh_volume = or_mesh_volume(xs, ys, zs, tris, nt);
  out->surface_area = or_surface_area(xs, ys, zs, tris, nt);
  double t_d0 = now_ms();
  double sq[4];
  if (threads == 1) or_diameters_sq_seq(xs, ys, zs, nv, sq);
  else or_diameters_sq_par(xs, ys, zs, nv, threads, sq);
  double t_end = now_ms();
  out->max_3d_diameter = sqrt(sq[0]);
  out->max_2d_diameter_xy = sqrt(sq[1]);
  out->max_2d_diameter_xz = sqrt(sq[2]);
  out->max_2d_diameter_yz = sqrt(sq[3]);
  out->vertex_count = nv;
  out->triangle_count = nt;
  out->active_cubes = -1; /* filled by or_active_cubes when asked; not on the timed path */
  out->mesh_ms = t_mesh - t0;
  out->diameters_ms = t_end - t_d0;
  out->total_ms = t_end - t0;
  free(xs); free(ys); free(zs); free(tris);
  return 0;
}
