/* shapecore_b200 -- C ABI of the B200-native shape-coefficient path.
 *
 * One call computes the full shape coefficients of a binary ROI mask:
 * marching-cubes surface area and signed-tetrahedron volume, the maximum 3-D
 * diameter and the maximum 2-D diameters in the slice (XY, same z), column
 * (XZ, same y) and row (YZ, same x) planes, plus vertex / triangle /
 * active-cube counts.  All GPU work runs in hand-written sm_100a kernels; there
 * is no CPU fallback: without a usable CUDA device every compute entry returns
 * SC_ERR_CUDA.
 *
 * Reference interfaces replaced (reference = /root/reference/pkg):
 *   sc_calculate_coefficients*  <- shapecore.features.extract_features
 *                                  (src/shapecore/features.py:224-265), i.e.
 *                                  marching_cubes (mesh.py:68-91) -> mesh_volume
 *                                  (features.py:99-110) -> surface_area
 *                                  (features.py:89-96) -> diameters[_parallel]
 *                                  (features.py:205-221); and the engine call
 *                                  behind shapebind.execute (binding
 *                                  src/shapebind/__init__.py:75-117), which today
 *                                  crosses a process boundary (subprocess + NPY).
 *   sc_diameters                <- shapecore.features.diameters / diameters_parallel
 *                                  (features.py:205-221) on raw coordinate arrays.
 *   return codes                <- CLI exit codes (cli.py:23-26): 2 input error,
 *                                  3 empty ROI; exceptions EmptyRoi / NoVertices /
 *                                  NonPositiveSpacing (errors.py:24-40).
 *
 * Data layout (same bytes as the reference MaskVolume, volume.py:59-66): mask
 * is nx*ny*nz bytes in C order with x fastest, index (iz*ny + iy)*nx + ix;
 * any nonzero byte is occupied.  spacing = (sx, sy, sz) in mm, finite, > 0.
 *
 * Threading: every entry is safe to call concurrently from several host
 * threads; calls on the same device are serialised internally.
 */
#ifndef SHAPECORE_B200_H
#define SHAPECORE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SC_ABI_VERSION 4

enum {
  SC_OK = 0,
  SC_ERR_INPUT = 2,       /* bad dims / spacing / pointer (volume.py:74-101)   */
  SC_ERR_EMPTY_ROI = 3,   /* mask has no occupied voxel (mesh.py:78-79)        */
  SC_ERR_NO_VERTICES = 4, /* diameters on an empty set (features.py:198-199)   */
  SC_ERR_CUDA = -1,       /* CUDA runtime / launch failure; see sc_last_error() */
  SC_ERR_NOMEM = -2       /* device or pinned allocation failed                 */
};

/* Output record: the reference ShapeFeatures (features.py:38-60) plus the
 * exact counts and per-stage device times (StageTimings, timing.py:9-20). */
typedef struct {
  double mesh_volume;
  double surface_area;
  double max_3d_diameter;
  double max_2d_diameter_xy; /* slice plane: vertex pairs sharing z  */
  double max_2d_diameter_xz; /* column plane: vertex pairs sharing y */
  double max_2d_diameter_yz; /* row plane: vertex pairs sharing x    */
  int64_t vertex_count;
  int64_t triangle_count;
  int64_t active_cubes;
  double h2d_ms;       /* host->device mask copy (host entry only), CUDA events   */
  double mesh_ms;      /* bit-pack + marching-cubes kernels, CUDA events           */
  double diameters_ms; /* 3-D + planar diameter kernels, CUDA events               */
  double total_ms;     /* host wall time of the whole call                         */
  /* ABI 2: host-mask entries copy only the occupied z/y slab (option
   * "host_crop"); h2d_bytes is what crossed PCIe, host_scan_ms the host scan
   * that found the slab.  Both 0 for device-resident masks. */
  int64_t h2d_bytes;
  double host_scan_ms;
} sc_coeffs;

/* Host mask (pageable or pinned).  device: CUDA ordinal.  The host finds the
 * occupied z/y slab (all host threads) and copies only that slab to the device
 * (option "host_crop", default 1; 0 = copy all nx*ny*nz bytes).  Results are
 * identical either way: everything outside the slab is background. */
int sc_calculate_coefficients(const uint8_t* mask, int64_t nx, int64_t ny, int64_t nz,
                              const double spacing[3], int device, sc_coeffs* out);

/* Typed mask payload straight from an NPY file: `data` is the
 * host payload of an array of NPY shape (s0, s1, s2) = (nz, ny, nx), C order
 * or Fortran order; dtype code 0 |b1, 1 |u1, 2 <i2, 3 <i4, 4 <i8, 5 <f4, 6 <f8
 * (reference volume.py:34-42).  With has_label, voxels equal to the label
 * (label_int for integer/bool codes, label_float for float codes, already
 * converted to the payload dtype) are foreground, otherwise any nonzero voxel
 * (volume.py:173-177).
 * Path: all host threads scan the payload once for its occupied extent over
 * the two slowest axes (C order: z and y; Fortran order: x and y; option
 * "host_crop"); only that slab crosses PCIe, in chunks of whole planes staged
 * through two pinned buffers (the host copies chunk k+1 while chunk k is in
 * flight; a pinned payload is copied directly), and each chunk is binarized on
 * the device as it lands -- Fortran chunks through a shared-memory tile
 * transpose.  h2d_ms covers the copies and the binarization, h2d_bytes the
 * payload bytes that crossed PCIe, host_scan_ms the scan. */
int sc_calculate_coefficients_raw(const void* data, int dtype, const int64_t shape[3],
                                  int fortran_order, int has_label, int64_t label_int,
                                  double label_float, const double spacing[3], int device,
                                  sc_coeffs* out);

/* One typed payload of a raw batch (the arguments of sc_calculate_coefficients_raw). */
typedef struct {
  const void* data;
  int dtype;
  int fortran_order;
  int has_label;
  int64_t label_int;
  double label_float;
  int64_t shape[3]; /* NPY shape (nz, ny, nx) */
} sc_raw_mask;

/* Batch of typed payloads on one device, pipelined over the batch slots like
 * sc_calculate_coefficients_batch (the host scan and staging of ROI i+1 overlap
 * the device work of the ROIs in flight).  spacings[3*i..] per ROI. */
int sc_calculate_coefficients_raw_batch(const sc_raw_mask* masks, const double* spacings,
                                        int64_t count, int device, sc_coeffs* out);

/* Device-resident mask on the CURRENT device; `stream` is a cudaStream_t.  The
 * ROI runs after all prior work on `stream`; NULL means the legacy default
 * stream (ordered the same way; the ROI itself then runs on a library slot
 * stream).  The call is synchronous.  The mask must stay valid for the call. */
int sc_calculate_coefficients_device(const uint8_t* d_mask, int64_t nx, int64_t ny,
                                     int64_t nz, const double spacing[3], void* stream,
                                     sc_coeffs* out);

/* Sharded variant for one very large mesh split across G devices:
 * runs the whole marching-cubes stage, then only shard `shard` of `nshards` of
 * the 3-D pair-tile grid and of the planar groups.  The 4 partial squared
 * maxima (3d, xy, xz, yz; fp64) are written to d_sq4 (device memory, 4
 * doubles) so the caller can ncclAllReduce(MAX) them in place, and also to
 * out (sqrt applied) for convenience.  Counts, area and volume in `out` are
 * complete on every shard. */
int sc_calculate_coefficients_shard(const uint8_t* d_mask, int64_t nx, int64_t ny, int64_t nz,
                                    const double spacing[3], void* stream, int shard,
                                    int nshards, double* d_sq4, sc_coeffs* out);

/* Two-phase (slab-split) shard entry for one very large mesh split across G
 * devices, so that marching cubes -- not only the pair grid -- is divided
 * (replaces the per-rank full mesh of the entry above).  Same pair
 * ownership and results as sc_calculate_coefficients_shard.
 *
 * Phase 1, sc_shard_mesh: bit-pack the whole device mask (every shard gets the
 * global occupied bbox, written to bbox[6] = xmin, ymin, zmin, xmax, ymax,
 * zmax) and run marching cubes over shard `shard`'s contiguous share of the
 * cell layers.  Writes the shard's exact integer partials to d_sums (device,
 * n_sums int64 from sc_shard_exchange_sizes) and its vertex keys (int32 x 4
 * per vertex, device) to d_keys (room for key_cap vertices); *n_keys = the
 * shard's vertex count.  The caller then all-reduces d_sums (SUM, int64) and
 * all-gathers the keys of every shard (any order).
 *
 * Phase 2, sc_shard_diameters: the summed d_sums, the gathered keys
 * (n_keys = their total, must equal the summed vertex count) and phase 1's
 * bbox; evaluates shard `shard` of the pair grid and writes the 4 partial
 * squared maxima (fp64) to d_sq4 for an all-reduce(MAX), as above.  `out`
 * holds the complete counts, area and volume.  Both calls are synchronous and
 * ordered after prior work on `stream` (NULL = the legacy default stream). */
int sc_shard_exchange_sizes(int64_t nx, int64_t ny, int64_t nz, int64_t* n_sums,
                            int64_t* key_cap);
int sc_shard_mesh(const uint8_t* d_mask, int64_t nx, int64_t ny, int64_t nz,
                  const double spacing[3], void* stream, int shard, int nshards,
                  int64_t* d_sums, int32_t* d_keys, int64_t key_cap, int64_t* n_keys,
                  int32_t bbox[6]);
int sc_shard_diameters(const int64_t* d_sums, const int32_t* d_keys, int64_t n_keys, int64_t nx,
                       int64_t ny, int64_t nz, const int32_t bbox[6], const double spacing[3],
                       void* stream, int shard, int nshards, double* d_sq4, sc_coeffs* out);

/* Batch of ROIs on one device (C4): masks[i] are host pointers with dims
 * dims[3*i..3*i+2] and spacing spacings[3*i..]; out[i] per ROI.  Up to 64
 * pipeline slots (option "slots", default 32) round-robin, so the H2D copy and kernels of
 * the next ROIs overlap the current one's.
 * The first failing ROI's code is returned; later ROIs are still processed. */
int sc_calculate_coefficients_batch(const uint8_t* const* masks, const int64_t* dims,
                                    const double* spacings, int64_t count, int device,
                                    sc_coeffs* out);

/* Batch of host ROIs fanned out over several devices (SURVEY 8b "batch entry
 * fans out over devices internally"; replaces the reference's per-case loop,
 * bench.py:122-182, and its worker pinning, dispatch.py:130-146): ROIs are
 * placed on devices[0..ndev) by longest-processing-time on their byte size,
 * one host thread per device entry runs the pipelined single-device batch
 * on its share, and out[i] is ROI i's record whatever device ran it.  A
 * device may be listed more than once (its shares then run one after the
 * other).  The first failing share's code is returned; every ROI is still
 * processed. */
int sc_calculate_coefficients_batch_multi(const uint8_t* const* masks, const int64_t* dims,
                                          const double* spacings, int64_t count,
                                          const int* devices, int ndev, sc_coeffs* out);

/* Same for device-resident masks on the CURRENT device (pipelined likewise).
 * The batch is ordered after prior work on `stream` (cudaStream_t; NULL = the
 * legacy default stream), and work enqueued on it later is ordered after the
 * batch. */
int sc_calculate_coefficients_device_batch(const uint8_t* const* d_masks, const int64_t* dims,
                                           const double* spacings, int64_t count, void* stream,
                                           sc_coeffs* out);

/* Diameters of an arbitrary fp64 point cloud (features.py:205-221), bit-exact
 * with the reference: out = (max3d, xy, xz, yz).  Host arrays. */
int sc_diameters(const double* xs, const double* ys, const double* zs, int64_t n, int device,
                 double out[4]);

/* Marching-cubes vertex set of a host mask as doubled lattice coordinates
 * (2x + [axis==0], 2y + [axis==1], 2z + [axis==2]); vertex i is
 * (keys[3i], keys[3i+1], keys[3i+2]) and the reference coordinate is key/2 *
 * spacing.  Order is unspecified.  *n_out receives the count; at most `cap`
 * entries are written.  For parity tests and mesh export. */
int sc_mesh_vertices(const uint8_t* mask, int64_t nx, int64_t ny, int64_t nz, int device,
                     int32_t* keys, int64_t cap, int64_t* n_out);

/* Measurement hooks (bench.py).  sc_last_kernel_times fills up to n of
 * {pack_ms, mc_ms, prune_ms, pass1_ms, refine_ms, planar_prep_ms, h2d_ms} of the
 * last single-call ROI run on `device` with option "stage_times" = 2 (CUDA
 * events on the launching stream; zeros otherwise) and returns how many were
 * written.  sc_launch_count is the number of kernels this
 * library has launched in the process.  sc_probe_fp32_peak measures the FP32
 * CUDA-core throughput of `device` in TFLOP/s with a dependent-chain-free
 * FFMA2 (mode 0) or scalar FFMA (mode 1) kernel. */
int sc_last_kernel_times(int device, double* ms, int n);
/* Work counters of the last ROI on `device`: {3-D work units kept, 3-D work
 * units total, 3-D fp64 re-check candidates, planar tile pairs total, planar
 * re-check candidates, planar units kept, 3-D 64 x 64 sub-pairs evaluated,
 * planar 64 x 64 sub-pairs listed, 3-D pair slots pass 1 evaluated after its
 * vertex filter, planar pair slots pass 1 evaluated}; a unit is a 128 x 128
 * chunk pair, of which pass 1 evaluates the vertices of the listed 64 x 64
 * sub-pairs that can reach the lower bound.  Returns how many were written
 * (<= 10). */
int sc_last_diagnostics(int device, int64_t* out, int n);
/* Options.  Every call takes a snapshot of the options at entry, so changing
 * them never affects a call already in flight.  sc_set_option sets the
 * process-wide value; sc_set_thread_option overrides it for calls made from
 * the calling thread only (until sc_clear_thread_options).
 * "prune" (default 1) = exact bbox pruning of 3-D and planar work units;
 * "pass1_packed" (1) = FFMA2 variant of the 3-D pass;
 * "graphs" (1) = replay each ROI pipeline as a cached CUDA graph; "slots" (32)
 * = pipeline slots (stream + scratch) the batch entries keep in flight (1-32);
 * "host_crop" (1) = host-mask entries copy only the occupied z/y slab;
 * "host_pack" (-1) = bit-pack the occupied slab on the host and copy only
 * its bits into the device bit volume (1 always, 0 never, -1 when the raw
 * slab would keep PCIe busier than the host scan took);
 * "host_split" (-1) = % of leading slices sent to the device whole while the
 * host scans the rest (-1: balanced from the measured host-scan and PCIe
 * rates and the previous ROI's slab fraction; 0: off);
 * "host_threads" (hardware threads, <= 32) = threads of the host slab scan;
 * "grid_div" (10) / "grid_div_single" (1) = divisor of the per-ROI kernels'
 * grids (SMs x blocks/SM) in batch entries / single calls: fewer resident
 * blocks per ROI let more ROIs share the GPU, a single ROI wants all of it;
 * "zero_copy" (1) = the per-ROI parameter and result records travel through
 * mapped pinned host memory (read by the first kernel, written by the last)
 * instead of copy operations around each ROI's graph;
 * "stage_times" (0) = CUDA events in single-call graphs: 0 none (mesh_ms /
 * diameters_ms then come from device %globaltimer stamps), 1 mesh / diameters
 * boundaries, 2 every stage boundary (sc_last_kernel_times needs 2; each
 * event node adds latency);
 * "batch_stage_times" (0) = per-stage CUDA events in batch graphs (without
 * them mesh_ms / diameters_ms come from the %globaltimer stamps);
 * "pack_tma" (1) / "pack_tma_single" (0) = CTAs per SM of the cp.async.bulk
 * (TMA) pack in batch entries / single calls (0 = the 128-bit-load pack);
 * "pack_chain" (4) = batch entries: a ROI starts only once the pack of the ROI
 * 4 places earlier has finished, so at most 4 HBM passes run at a time and the
 * latency-bound kernels of earlier ROIs overlap them (0 = unchained);
 * "fused_bbox" (1) / "fused_bbox_single" (0) = the pack accumulates the
 * occupied bbox itself (else a separate pass over the bit volume), in batch
 * entries / single calls;
 * "sparse_bits" (1) = the pack writes only nonzero 16-word segments of the
 * bit volume (segment map); "pack_skip" (1) = ... and does no conversion work
 * at all for all-background segments; "pdl" (0) = programmatic dependent
 * launch of the per-ROI kernels in batch graphs; "fork" (1) = the planar
 * filter chain runs on a second stream beside the 3-D one; "dcap" / "wcap" =
 * initial vertex / 3-D work-list capacities (an overflow re-runs the ROI with
 * exact sizes).
 * Measurement / experiment switches: "pack_mode" (0), "pack_bps" (0),
 * "debug_stages" (off; enqueue only the first N kernels, results invalid),
 * "debug_empty" (0; N empty kernels per ROI, a launch-rate probe).
 * Results are identical either way; 0 on success, SC_ERR_INPUT otherwise. */
int sc_set_option(const char* name, int value);
int sc_set_thread_option(const char* name, int value);
void sc_clear_thread_options(void);
uint64_t sc_launch_count(void);
int sc_probe_fp32_peak(int device, int mode, double* tflops);

/* Canonical triangle mesh of a host mask: the reference's
 * marching_cubes output (mesh.py:142-199) bit for bit -- vertices numbered at
 * first reference in (z, y, x) cell-scan order, coordinates (l-1+0.5)*s in
 * fp64, triangles in scan order with the table's winding.  xs/ys/zs hold
 * vcap doubles, tris 3*tcap int32; *n_vert / *n_tri always receive the counts,
 * and the arrays are written only when they are large enough (call once with
 * vcap = tcap = 0 to size them). */
int sc_marching_cubes(const uint8_t* mask, int64_t nx, int64_t ny, int64_t nz,
                      const double spacing[3], int device, double* xs, double* ys, double* zs,
                      int32_t* tris, int64_t vcap, int64_t tcap, int64_t* n_vert,
                      int64_t* n_tri);

/* Surface area, signed volume and volume of an arbitrary triangle mesh with
 * the reference's exact arithmetic (surface_area / signed_mesh_volume /
 * mesh_volume, features.py:89-118, pairwise_sum :63-80): out = (area, signed
 * volume, |volume|), bit-exact with the reference for the same arrays. */
int sc_mesh_measure(const double* xs, const double* ys, const double* zs, int64_t nv,
                    const int32_t* tris, int64_t nt, int device, double out[3]);

/* Host-only helper behind option "host_crop" (no device needed): occupied
 * extent of a host mask as out = (z0, z1, y0, y1), inclusive; returns
 * SC_ERR_EMPTY_ROI (out untouched) when every byte is zero.  threads <= 0 =
 * the "host_threads" option. */
int sc_occupied_slab(const uint8_t* mask, int64_t nx, int64_t ny, int64_t nz, int threads,
                     int64_t out[4]);

const char* sc_last_error(void); /* thread-local message of the last failure */
int sc_abi_version(void);
int sc_device_count(void);

#ifdef __cplusplus
}
#endif
#endif
