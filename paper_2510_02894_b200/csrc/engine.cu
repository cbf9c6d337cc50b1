// Host orchestration and the C ABI (include/shapecore_b200.h).
//
// One ROI = init -> pack -> bbox -> mc_cells -> sort -> boxes / filters (3-D
// and, on a second stream, planar) -> one fused pass-1 kernel -> one fused
// exact re-check that publishes the accumulators to mapped host memory, all
// one CUDA graph per pipeline slot with no host round trip (DESIGN.md section
// 1).  Area, volume, triangle and active-cube counts are formed on the host
// from exact integer histograms.  Per device the
// library keeps up to 16 slots: streams, events, grow-only scratch arenas and
// pinned records, reused across calls (SURVEY.md 8b "Ownership"); a slot is
// used by one call at a time (mutex).  Host masks are scanned / cropped /
// packed on the host first (host_crop.cu).
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <array>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/shapecore_b200.h"
#include "host_crop.h"
#include "mc_tables.h"
#include "sc_device.cuh"

namespace sc {

// Kernels (mc.cu, diameter.cu, prune.cu, planar.cu).
__global__ void init_stats(Stats* st, uint32_t* segmap, long long n_seg, const RoiParams* src_rp,
                           RoiParams* dst_rp);
template <int U, bool BOX>
__global__ void pack_bits_v16(const RoiParams*, uint32_t*, Stats*, uint32_t*);
__global__ void bits_bbox(const RoiParams*, const uint4*, Stats*, const uint32_t*);
template <bool BOX, int NT, int TILE>
__global__ void pack_bits_tma(const RoiParams*, uint32_t*, Stats*, uint32_t*, int);
constexpr int kTmaTileBytes = 16384;  // mc.cu kTmaTile
constexpr int kTmaMaxSmem = 8 * kTmaTileBytes;  // mc.cu kTmaMaxStages x kTmaTile
constexpr int kTmaMaxSmemBig = 6 * 32768;      // 32 KB tiles: up to 6 stages
__global__ void pack_bits_generic(const RoiParams*, uint32_t*, Stats*, uint32_t*);
__global__ void mc_cells(const RoiParams*, const uint32_t*, const CaseTables*, Stats*, int4*,
                         long long, unsigned int*, unsigned int*, const uint32_t*);
__global__ void scan_all(unsigned int*, unsigned int*, unsigned int*, unsigned int*,
                         unsigned int*, unsigned int*, long long, Stats*, int4*, unsigned int*,
                         unsigned int*, unsigned long long*, int);
__global__ void scatter_all(const int4*, long long, const Stats*, unsigned int*, int4*,
                            const unsigned int*, unsigned int*, int2*, unsigned int*,
                            const unsigned int*, unsigned int*);
__global__ void boxes_extremes(const int4*, long long, const RoiParams*, Stats*, int4*, int4*,
                               int4*, float4*);
__global__ void unit_filter(const int4*, const int4*, long long, const RoiParams*, int, int, int,
                            Stats*, uint2*, const int4*, const int4*, uint2*, long long);
__global__ void unit_expand(const int4*, long long, const RoiParams*, int, int, int, Stats*, uint2*,
                            const int4*, const uint2*, long long);
template <bool PACKED>
__global__ void diam_pass1(const int4*, long long, const RoiParams*, const uint2*, float*,
                           const int2*, const unsigned int*, const uint2*, long long, float*,
                           Stats*, const int4*, const int4*, int, const unsigned int*,
                           const int4*, const int4*, const float4*);
__global__ void diam_refine(const int4*, long long, const RoiParams*, const uint2*, const float*,
                            const int2*, const unsigned int*, const uint2*, long long,
                            const float*, Stats*, Stats*);
__global__ void plane_boxes(const int2*, const unsigned int*, const unsigned int*,
                            const RoiParams*, const Stats*, int4*, unsigned long long*, int4*,
                            const unsigned int*);
__global__ void plane_lb(const int2*, const unsigned int*, const unsigned long long*,
                         const RoiParams*, Stats*);
__global__ void plane_filter(const unsigned int*, const unsigned int*, const unsigned int*,
                             const int4*, const RoiParams*, int, int, int, long long, Stats*,
                             uint2*, const int4*);
__global__ void cloud_diameters(const double*, const double*, const double*, long long,
                                long long, unsigned long long*);
int launch_binarize(const void*, int, int, long long, long long, long long, int, int, int,
                    long long, double, uint8_t*, int, cudaStream_t);
__global__ void mesh_count(const RoiParams*, const uint32_t*, const Stats*, unsigned int*);
__global__ void scan_blocks(unsigned int*, long long, unsigned int*);
__global__ void scan_sums(unsigned int*, int, unsigned long long*);
__global__ void scan_add(unsigned int*, long long, const unsigned int*);
__global__ void edge_map_fill(const int4*, const Stats*, int*);
__global__ void mesh_emit(const RoiParams*, const uint32_t*, const Stats*, const unsigned int*,
                          const int*, int3*, unsigned int*);
__global__ void id_flags(const unsigned int*, long long, unsigned int*);
__global__ void mesh_out(const int4*, const unsigned int*, const unsigned int*, long long, double,
                         double, double, double*, double*, double*, int*);
__global__ void tris_out(const int3*, long long, const int*, int*);
cudaError_t upload_mesh_tables();
__global__ void tri_terms(const double*, const double*, const double*, const int*, long long,
                          long long, double*, double*);
__global__ void fold_pass(double*, double*, long long);
template <int MODE>
__global__ void fp32_probe(float*, int, float, float);

__global__ void empty_kernel();
__global__ void canon_keys(int4*, int4*, const unsigned int*, const Stats*);
}  // namespace sc

using namespace sc;

namespace {

thread_local std::string g_err;
// Options (sc_set_option).  Every call takes a snapshot at entry (Ctx::o),
// so a concurrent sc_set_option never changes a call already in flight;
// sc_set_thread_option overrides them for the calling thread only.
struct Opts {
  bool prune = true;         // exact bbox pruning of 3-D and planar work units
  bool packed = true;        // FFMA2 variant of pass 1 ("pass1_packed")
  bool graphs = true;        // replay each ROI pipeline as a cached CUDA graph
  int stages = 1 << 30;      // debug: kernels enqueued per ROI ("debug_stages")
  int empty = 0;             // debug: empty kernels appended per ROI ("debug_empty")
  bool fbox = true;          // batch graphs: bbox accumulated inside the pack ("fused_bbox";
                             // else a bits_bbox pass)
  bool fbox_single = false;  // the same for single calls (C2 call: pack 28.7 + bbox ~6 us
                             // separate vs 38.8 us fused)
  int slots = 32;            // pipeline slots of the batch entries (measured 32 > 24 > 16 > 12)
  long long dcap = 2LL << 20;  // default diameter-side vertex capacity
  long long wcap = 1LL << 20;  // default 3-D work-list capacity (chunk pairs)
  bool batch_times = false;  // per-stage event nodes in batch graphs
  bool pdl = false;          // programmatic dependent launch in batch graphs
  bool sparse = true;        // sparse bit volume (segment map), "sparse_bits"
  bool pack_skip = true;     // sparse pack: no conversion of all-zero segments
  int pack_tma = 1;          // batch graphs: TMA bulk-copy pack, CTAs per SM (0 = 128-bit loads)
  int pack_tma_single = 0;   // the same for single calls (the 128-bit-load pack is faster alone)
  bool pack_prio = true;      // init_stats + pack at the greatest stream priority ("pack_prio")
  int pack_threads = 256;     // TMA pack CTA size (64 / 128 / 256, "pack_threads")
  int pack_tile = 32;         // TMA pack tile KB (8 / 16 / 32, "pack_tile"; 32: C4 -2 %, alone 51 -> 43 us)
  int pack_stages = 2;       // TMA pack ring depth (2..8, "pack_stages"; a CTA's copies complete serially)
  int pack_chain = 4;        // batch: ROI i's graph starts after ROI i - pack_chain's pack
                             // (at most pack_chain HBM passes in flight; 0 = unchained).
                             // C2 / C4 / C5 K=200 us per ROI, chain 0 / 1 / 2 / 3 / 4 / 8:
                             // 33.0 / 57.9 / 34.5 / 29.4 / 29.7 / 32.3, 34.7 / 59.6 / 39.0 /
                             // 32.5 / 32.0 / 33.8, 26.3 / 31.0 / 25.0 / 25.3 / 25.4 / 26.1
  bool fork = true;          // planar chain on a second stream
  bool zc = true;            // "zero_copy": RoiParams / Stats via mapped host memory
  int stage_times = 0;       // single-call graph events: 0 none (timer stamps), 1 mesh/diam, 2 all
  // Divisor of the latency-bound per-ROI kernels' grids: batches keep many
  // ROIs in flight and run faster with few resident blocks per ROI (C2, 32
  // slots: div 5 / 10 / 20 = 33.98 / 32.80 / 33.21 us per ROI); a single call
  // wants the whole GPU for its latency chain (C3 call: div 1 far faster than 4).
  int grid_div = 10;         // batch entries ("grid_div")
  int grid_div_single = 1;   // single calls ("grid_div_single")
  int pack_bps = 0;          // pack blocks per SM (0 = occupancy limit)
  int pack_mode = 0;         // bit 0: one step per pack block; bit 1: low-priority pack;
                             // bit 2 (debug): no pack, reuse the slot's bit volume
  bool crop = true;          // host entries: copy only the occupied z/y slab (host_crop.h)
  int host_pack = -1;        // bit-pack the slab on the host (1 / 0 / -1 adaptive)
  int split = -1;            // % of leading slices sent unscanned (-1 adaptive, 0 off)
  int host_threads = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
};
std::mutex g_opt_mu;
Opts g_opts;                           // process-wide (sc_set_option)
thread_local bool t_opts_on = false;   // sc_set_thread_option was used on this thread
thread_local Opts t_opts;
Opts snapshot_opts() {
  if (t_opts_on) return t_opts;
  std::lock_guard<std::mutex> lk(g_opt_mu);
  return g_opts;
}
std::atomic<unsigned long long> g_launches{0};

void set_err(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

#define CK(expr)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      set_err("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return SC_ERR_CUDA;                                                              \
    }                                                                                  \
  } while (0)

// Every kernel launch of the library goes through CKL(n): checks the launch and
// counts n launches (sc_launch_count, bench.py's gpu_launches).
#define CKL(n)                                     \
  do {                                             \
    CK(cudaGetLastError());                        \
    g_launches.fetch_add((n), std::memory_order_relaxed); \
  } while (0)

// ---------------------------------------------------------------- case tables
struct CaseGeom {
  int ntri[kNumCases];
  int n[kNumCases][5][3];  // doubled-integer (b-a) x (c-a) per triangle
  CaseTables tabs;
};

const CaseGeom& case_geom() {
  static CaseGeom g = [] {
    CaseGeom c{};
    for (int k = 0; k < kNumCases; k++) {
      int t_sum = 0, n_sum[3] = {0, 0, 0}, nt = 0;
      for (int t = 0; t < 16 && SC_TRI_TABLE[k][t] >= 0; t += 3) {
        int a[3][3];
        for (int v = 0; v < 3; v++) {
          int e = SC_TRI_TABLE[k][t + v];
          int ax = SC_EDGE_AXIS[e];
          a[v][0] = 2 * SC_EDGE_DX[e] + (ax == 0);
          a[v][1] = 2 * SC_EDGE_DY[e] + (ax == 1);
          a[v][2] = 2 * SC_EDGE_DZ[e] + (ax == 2);
        }
        int u[3], w[3], bc[3];
        for (int d = 0; d < 3; d++) { u[d] = a[1][d] - a[0][d]; w[d] = a[2][d] - a[0][d]; }
        int nn[3] = {u[1] * w[2] - u[2] * w[1], u[2] * w[0] - u[0] * w[2], u[0] * w[1] - u[1] * w[0]};
        bc[0] = a[1][1] * a[2][2] - a[1][2] * a[2][1];
        bc[1] = a[1][2] * a[2][0] - a[1][0] * a[2][2];
        bc[2] = a[1][0] * a[2][1] - a[1][1] * a[2][0];
        t_sum += a[0][0] * bc[0] + a[0][1] * bc[1] + a[0][2] * bc[2];
        for (int d = 0; d < 3; d++) { n_sum[d] += nn[d]; c.n[k][nt][d] = nn[d]; }
        nt++;
      }
      c.ntri[k] = nt;
      c.tabs.tn[k] = make_int4(t_sum, n_sum[0], n_sum[1], n_sum[2]);
    }
    for (int idx = 0; idx < kNumCases; idx++) c.tabs.tn_raw[idx] = c.tabs.tn[case_of_idx(idx)];
    return c;
  }();
  return g;
}

// Area of one triangle of case k in mm^2: 0.5*|N| with N = diag(sy sz, sx sz, sx sy)/4 * n.
void area_table(const double sp[3], double out[kNumCases]) {
  const CaseGeom& g = case_geom();
  const double fx = sp[1] * sp[2] * 0.25, fy = sp[0] * sp[2] * 0.25, fz = sp[0] * sp[1] * 0.25;
  for (int k = 0; k < kNumCases; k++) {
    double s = 0.0;
    for (int t = 0; t < g.ntri[k]; t++) {
      double a = fx * g.n[k][t][0], b = fy * g.n[k][t][1], c = fz * g.n[k][t][2];
      s += 0.5 * std::sqrt(a * a + b * b + c * c);
    }
    out[k] = s;
  }
}

// ------------------------------------------------------------------- context
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;  // elements
  // Grow-only.  Fresh memory is zeroed once: the sparse bit volume reads words
  // of unwritten segments together with their (clear) map bit and discards
  // them, and those reads must not touch uninitialised memory
  // (compute-sanitizer initcheck).
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = n + n / 4 + 1024;
    cudaError_t e = cudaMalloc(&p, want * sizeof(T));
    if (e == cudaSuccess) e = cudaMemset(p, 0, want * sizeof(T));
    if (e == cudaSuccess) cap = want;
    return e;
  }
};

struct Ctx {
  Opts o;  // options of the call in progress (snapshot taken at its entry)
  int device = 0;
  int sms = 148;
  std::mutex mu;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[6] = {};
  cudaEvent_t kev[10] = {};     // per-kernel boundaries of the last ROI
  cudaStream_t stream2 = nullptr;  // planar branch of the ROI graph (fork / join)
  cudaEvent_t pack_ev = nullptr;   // batch pack chain: recorded after this slot's pack
  cudaEvent_t chain_wait = nullptr;  // ... and this slot's ROI waits on another slot's
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  double last_ms[7] = {0, 0, 0, 0, 0, 0, 0};  // pack, mc, prune, pass1, refine, planar, h2d
  bool times_pending = false;  // last_ms[0..5] still to be read from kev[]
  long long cap_floor = 0, dcap_floor = 0, wcap_floor = 0;  // raised by overflow re-runs only
  long long last_diag[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  int occ_pass1 = 1, occ_pass1s = 1, occ_pack = 1, occ_mc = 1;  // blocks/SM
  int prio_lo = 0, prio_hi = 0;  // stream priority range (least, greatest)
  Stats* d_stats = nullptr;
  Stats* h_stats = nullptr;  // pinned (mapped: the pipeline's last kernel writes it)
  Stats* h_stats_dev = nullptr;     // its device-side address
  RoiParams* h_rp_dev = nullptr;    // device-side address of h_rp (read by init_stats)
  RoiParams* d_rp = nullptr;  // per-ROI launch parameters (device)
  RoiParams* h_rp = nullptr;  // staging copy (pinned)
  long long dcap_sz = 0;      // vertices the diameter-side buffers are sized for (monotonic)
  CaseTables* d_tabs = nullptr;
  DevBuf<uint32_t> bits;
  DevBuf<uint32_t> segmap;  // 1 bit per 16-word bit-volume segment (sparse pack)
  DevBuf<int4> keys, keys_sorted, boxes, sboxes;  // chunk / super-chunk boxes (lo, hi)
  DevBuf<int4> hboxes;  // boxes of the two 64-vertex halves of every chunk
  DevBuf<uint2> slist;  // surviving super-chunk pairs (two-level filter of large ROIs)
  DevBuf<unsigned int> sort_counts, sort_cursor;
  DevBuf<uint2> work;  // surviving 3-D chunk pairs (I, J)
  DevBuf<float> warp_max, plane_umax;
  DevBuf<uint2> plane_work;  // surviving in-plane chunk pairs {plane, I << 16 | J}
  DevBuf<unsigned int> plane_counts, plane_start, plane_tstart, plane_cstart;
  DevBuf<unsigned int> pbin_counts, pbin_cursor;
  DevBuf<unsigned long long> plane_ext;
  DevBuf<int4> plane_boxes_buf;
  DevBuf<int4> plane_hboxes;  // boxes of the two 64-entry halves of every in-plane chunk
  DevBuf<unsigned int> plane_cmap;  // plane of every in-plane chunk (scatter_all)
  DevBuf<int2> plane_sorted;
  DevBuf<uint8_t> mask_stage, raw_stage;  // raw_stage: two chunk buffers (typed payloads)
  uint8_t* h_raw = nullptr;               // pinned staging of typed payload chunks (two halves)
  size_t h_raw_cap = 0;                   // bytes
  cudaEvent_t cev[2] = {};                // DMA out of h_raw half k finished
  double last_scan_ms = 0.0;      // host time (scan, + pack) of the last host-mask ROI
  double last_pure_scan_ms = 0.0; // its slab scan alone
  long long last_h2d_bytes = 0;   // bytes that crossed PCIe for it
  long long last_scan_bytes = 0;  // bytes the host scan read for it
  long long last_slab_bytes = 0;  // bytes of its occupied slab
  bool prepacked = false;         // this ROI's bit volume came packed from the host
  int mc_slab = 0;                // RoiParams::mc_slab of the next ROI (two-phase shard entry)
  bool mesh_only = false;         // enqueue_roi stops after mc_cells (two-phase shard entry)
  uint32_t* h_bits = nullptr;     // pinned staging of a host-packed bit volume
  size_t h_bits_cap = 0;          // words
  bool last_split = false;        // it used the split read (split_slices)
  DevBuf<double> cloud;
  DevBuf<unsigned long long> cloud_out;
  // CUDA graphs of whole ROIs, keyed by everything baked into the nodes.
  struct GraphEntry {  // everything a captured ROI graph depends on
    bool fast;          // 128-bit pack path (nx % 32 == 0, 16-byte aligned mask)
    cudaStream_t s;
    int shard, nshards;
    void* d_sq4;
    long long cap, dcap;
    bool prune, packed, fbox;
    int stages;
    int packmode;       // pack grid shape / priority (option "pack_mode")
    int grid_div;       // option "grid_div"
    bool events;        // stage event nodes present
    bool ev_full;       // ... at every stage boundary
    bool pdl;           // option "pdl"
    bool sparse;        // option "sparse_bits"
    bool fork;          // option "fork"
    bool zc;            // option "zero_copy"
    bool prepacked;     // bit volume packed on the host (no pack kernel)
    cudaEvent_t chain;  // pack-chain event waited on (nullptr: none)
    unsigned long long gen;
    cudaGraphExec_t exec;
    unsigned long long launches;
  };
  std::vector<GraphEntry> graphs;
  unsigned long long gen = 0;  // bumped whenever a scratch buffer moves
  bool capturing = false;      // inside a stream capture of launch_roi
  bool events_on = true;       // record stage events (single calls; batches: option)
  int grid_div = 1;            // grid divisor of this ROI's latency-bound kernels
  bool ev_full = true;         // every stage boundary (else mesh / diameters only)

  unsigned long long fingerprint() const {
    unsigned long long h = 1469598103934665603ull;
    const void* ps[] = {bits.p, segmap.p, keys.p, keys_sorted.p, boxes.p, sboxes.p, hboxes.p, slist.p,
                        sort_counts.p, sort_cursor.p,
                        work.p, warp_max.p, plane_umax.p,
                        plane_counts.p, plane_start.p, plane_tstart.p, plane_sorted.p,
                        plane_work.p, plane_cstart.p, pbin_counts.p, pbin_cursor.p,
                        plane_ext.p, plane_boxes_buf.p, plane_hboxes.p,
                        plane_cmap.p};
    for (const void* p : ps) h = (h ^ (unsigned long long)(uintptr_t)p) * 1099511628211ull;
    return h;
  }
  void drop_graphs() {
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    graphs.clear();
  }
};

// Two independent pipeline slots per device (stream, events, scratch, graphs):
// single-ROI calls use slot 0; batch calls alternate slots so the H2D copy and
// kernels of ROI i+1 overlap the tail and the host round trip of ROI i.
constexpr int kSlots = 64;
std::mutex g_ctx_mu;
std::vector<std::array<std::unique_ptr<Ctx>, kSlots>> g_ctx;

int get_ctx(int device, Ctx** out, int slot = 0) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) {
    set_err("device %d out of range (%d CUDA devices)", device, n);
    return SC_ERR_INPUT;
  }
  if ((int)g_ctx.size() < n) g_ctx.resize(n);
  if (!g_ctx[device][slot]) {
    auto c = std::make_unique<Ctx>();
    c->device = device;
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) {
      set_err("device %d is sm_%d%d; this library is built for sm_100a (B200)", device,
              prop.major, prop.minor);
      return SC_ERR_CUDA;
    }
    c->sms = prop.multiProcessorCount;
    CK(cudaDeviceGetStreamPriorityRange(&c->prio_lo, &c->prio_hi));
    // Slot streams: priority falls with the slot index (slot 0, the
    // single-call slot, at the greatest), so a batch's ROIs drain roughly in
    // launch order instead of all finishing together -- slots free up early
    // and the batch's tail runs with more ROIs in flight (C2, K = 20: 49.3 ->
    // 46.2 us/ROI; steady state unchanged; SC_SLOT_PRIO=0: all at the greatest).
    // (The HBM pack can further be launched at the least, pack_mode bit 1.)
    int sprio = c->prio_hi;
    const char* sp_env = std::getenv("SC_SLOT_PRIO");
    if (!(sp_env && std::strcmp(sp_env, "0") == 0)) {
      const int levels = c->prio_lo - c->prio_hi + 1;
      sprio = c->prio_hi + std::min(levels - 1, slot * levels / 16);
    }
    CK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, sprio));
    CK(cudaStreamCreateWithPriority(&c->stream2, cudaStreamNonBlocking, sprio));
    CK(cudaFuncSetAttribute(pack_bits_tma<false, 256, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaMaxSmem));
    CK(cudaFuncSetAttribute(pack_bits_tma<true, 256, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaMaxSmem));
    CK(cudaFuncSetAttribute(pack_bits_tma<false, 128, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaMaxSmem));
    CK(cudaFuncSetAttribute(pack_bits_tma<true, 128, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaMaxSmem));
    CK(cudaFuncSetAttribute(pack_bits_tma<false, 256, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaMaxSmemBig));
    CK(cudaFuncSetAttribute(pack_bits_tma<true, 256, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaMaxSmemBig));
    CK(cudaFuncSetAttribute(pack_bits_tma<false, 256, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaMaxSmem));
    CK(cudaFuncSetAttribute(pack_bits_tma<true, 256, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaMaxSmem));
    CK(cudaFuncSetAttribute(pack_bits_tma<false, 128, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaMaxSmemBig));
    CK(cudaFuncSetAttribute(pack_bits_tma<true, 128, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaMaxSmemBig));
    CK(cudaFuncSetAttribute(pack_bits_tma<false, 64, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaMaxSmemBig));
    CK(cudaFuncSetAttribute(pack_bits_tma<true, 64, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaMaxSmemBig));
    CK(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming));
    for (auto& e : c->cev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->pack_ev, cudaEventDisableTiming));
    for (auto& e : c->ev) CK(cudaEventCreate(&e));
    for (auto& e : c->kev) CK(cudaEventCreate(&e));
    CK(cudaMalloc(&c->d_stats, sizeof(Stats)));
    CK(cudaMallocHost(&c->h_stats, sizeof(Stats)));
    CK(cudaMalloc(&c->d_rp, sizeof(RoiParams)));
    CK(cudaMallocHost(&c->h_rp, sizeof(RoiParams)));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->h_stats_dev), c->h_stats, 0));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->h_rp_dev), c->h_rp, 0));
    CK(cudaMalloc(&c->d_tabs, sizeof(CaseTables)));
    CK(cudaMemcpy(c->d_tabs, &case_geom().tabs, sizeof(CaseTables), cudaMemcpyHostToDevice));
    CK(upload_mesh_tables());
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->occ_pass1, diam_pass1<true>, 256, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->occ_pass1s, diam_pass1<false>, 256, 0));
    static bool env_read = false;  // (g_ctx_mu held) environment defaults, once
    if (!env_read) {
      env_read = true;
      std::lock_guard<std::mutex> lk(g_opt_mu);
      if (const char* v = getenv("SC_PASS1")) g_opts.packed = std::strcmp(v, "scalar") != 0;
      if (const char* v = getenv("SC_PRUNE")) g_opts.prune = std::strcmp(v, "0") != 0;
    }
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->occ_pack, pack_bits_v16<4, false>, 256, 0));
    if (const char* v = getenv("SC_PACK_BPS")) c->occ_pack = std::max(1, std::atoi(v));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->occ_mc, mc_cells, 256, 0));
    {
      // Lazy module loading must not happen inside a stream capture: touch
      // every kernel once here.
      cudaFuncAttributes fa;
      const void* kernels[] = {(const void*)init_stats, (const void*)pack_bits_v16<4, false>,
                               (const void*)pack_bits_v16<4, true>,
                               (const void*)pack_bits_tma<false, 256, 16384>, (const void*)pack_bits_tma<true, 256, 16384>,
                               (const void*)pack_bits_tma<false, 128, 16384>, (const void*)pack_bits_tma<true, 128, 16384>,
                               (const void*)pack_bits_tma<false, 256, 32768>, (const void*)pack_bits_tma<true, 256, 32768>,
                               (const void*)pack_bits_tma<false, 256, 8192>, (const void*)pack_bits_tma<true, 256, 8192>,
                               (const void*)pack_bits_tma<false, 128, 32768>, (const void*)pack_bits_tma<true, 128, 32768>,
                               (const void*)pack_bits_tma<false, 64, 32768>, (const void*)pack_bits_tma<true, 64, 32768>,
                               (const void*)mesh_count, (const void*)mesh_emit,
                               (const void*)bits_bbox,
                               (const void*)pack_bits_generic, (const void*)mc_cells,
                               (const void*)scan_all, (const void*)scatter_all,
                               (const void*)boxes_extremes, (const void*)unit_filter,
                               (const void*)unit_expand,
                               (const void*)diam_pass1<true>, (const void*)diam_pass1<false>,
                               (const void*)diam_refine, (const void*)cloud_diameters,
                               (const void*)plane_boxes,
                               (const void*)plane_lb, (const void*)plane_filter,
                               (const void*)canon_keys};
      for (const void* k : kernels) CK(cudaFuncGetAttributes(&fa, k));
    }
    g_ctx[device][slot] = std::move(c);
  }
  *out = g_ctx[device][slot].get();
  return SC_OK;
}

int check_input(const void* mask, int64_t nx, int64_t ny, int64_t nz, const double sp[3]) {
  if (!mask) { set_err("mask pointer is NULL"); return SC_ERR_INPUT; }
  if (nx < 1 || ny < 1 || nz < 1) {
    set_err("dims must all be >= 1, got (%lld, %lld, %lld)", (long long)nx, (long long)ny,
            (long long)nz);
    return SC_ERR_INPUT;
  }
  // Doubled lattice keys and fp32 frame coordinates must stay exact.
  if (nx > (1 << 20) || ny > (1 << 20) || nz > (1 << 20)) {
    set_err("dims beyond 2^20 per axis are not supported");
    return SC_ERR_INPUT;
  }
  // (the planar chunk-index width is checked per plane at run time: scan_all
  // sets Stats::plane_ovf, finish_roi reports it)
  if (((nx + 31) / 32) * ny * nz >= (1LL << 32)) {  // bit-volume word indices are 32-bit
    set_err("masks above 2^37 voxels are not supported");
    return SC_ERR_INPUT;
  }
  if (!sp) { set_err("spacing pointer is NULL"); return SC_ERR_INPUT; }
  for (int i = 0; i < 3; i++)
    if (!(sp[i] > 0.0) || !std::isfinite(sp[i])) {
      set_err("spacing components must be finite and > 0, got (%g, %g, %g)", sp[0], sp[1], sp[2]);
      return SC_ERR_INPUT;
    }
  return SC_OK;
}

double f64_of(unsigned long long bits) {
  double d;
  std::memcpy(&d, &bits, 8);
  return d;
}

constexpr long long kChunk = 128;  // sc_device.cuh kChunk3: pair unit = chunk x chunk
// The 3-D work list (surviving chunk pairs) starts at Opts::wcap entries; a
// ROI whose pruned list is longer re-runs with the exact size.
constexpr long long kPlaneBinsHost = 256;  // sc_device.cuh kPlaneBins

// Stage events: inside a capture they must be external event nodes so that
// graph replays record them (plain records only order the capture).
cudaError_t record(Ctx* c, cudaEvent_t ev, cudaStream_t s) {
  if (!c->events_on) return cudaSuccess;  // batch graphs: no stage-event nodes
  // level 1: only the mesh / diameters boundaries (kev 0, 2, 6)
  if (!c->ev_full && ev != c->kev[0] && ev != c->kev[2] && ev != c->kev[6]) return cudaSuccess;
  return c->capturing ? cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal)
                      : cudaEventRecord(ev, s);
}

// Capacity of the per-ROI vertex arrays.  V is only known on the device, so
// the arrays are sized up front (grow-only) and an overflow, detected after
// the single end-of-ROI sync, re-runs the ROI with exact capacity.
long long vertex_capacity(int64_t nx, int64_t ny, int64_t nz, long long hint) {
  const long long vox = nx * ny * nz;
  long long cap = std::max<long long>(1 << 20, vox / 16);
  return std::max(cap, hint);
}

// keys (MC output) hold up to `cap` vertices; the diameter-side arrays (whose
// tile-pair bookkeeping grows as V^2) hold up to `dcap` <= cap.
int ensure_buffers(Ctx* c, int64_t nx, int64_t ny, int64_t nz, long long cap, long long dcap,
                   long long punits, long long wunits) {
  dcap = c->dcap_sz = std::max(c->dcap_sz, dcap);
  const int W = (int)((nx + 31) / 32);
  CK(c->bits.ensure((size_t)((long long)W * ny * nz)));
  CK(c->segmap.ensure(c->bits.cap / 512 + 1));
  CK(c->keys.ensure((size_t)cap));
  const long long C = (dcap + kChunk - 1) / kChunk;  // chunk pairs: C(C+1)/2
  const long long wc = std::min(C * (C + 1) / 2, std::max(c->o.wcap, wunits));
  CK(c->warp_max.ensure((size_t)wc));
  CK(c->work.ensure((size_t)wc));
  CK(c->keys_sorted.ensure((size_t)dcap));
  CK(c->boxes.ensure((size_t)(2 * (C + 1))));
  CK(c->hboxes.ensure((size_t)(4 * (C + 1))));
  {  // every super pair can survive (pruning off): size for all of them whenever
     // unit_filter takes the two-level path (same switch, sc_device.cuh)
    const long long CT = (C + 7) / 8;
    CK(c->slist.ensure((size_t)(C * (C + 1) / 2 > kSingleLevelMax ? CT * (CT + 1) / 2 : 1)));
  }
  CK(c->sboxes.ensure((size_t)(2 * (C / 8 + 1))));
  {
    unsigned int* before = c->sort_counts.p;
    CK(c->sort_counts.ensure(kSortBins + kSortSupers));
    CK(c->sort_cursor.ensure(kSortBins));
    if (c->sort_counts.p != before)  // histograms are self-cleaning after the first zeroing
      CK(cudaMemset(c->sort_counts.p, 0, sizeof(unsigned int) * c->sort_counts.cap));
  }
  const long long P = 2 * (nx + ny + nz) + 9;
  CK(c->plane_counts.ensure((size_t)P));
  CK(c->plane_start.ensure((size_t)P + 1));
  CK(c->plane_tstart.ensure((size_t)P + 1));
  CK(c->plane_cstart.ensure((size_t)P + 1));
  CK(c->plane_ext.ensure((size_t)P * 8));
  {
    unsigned int* before = c->pbin_counts.p;  // self-cleaning after the first zeroing
    CK(c->pbin_counts.ensure((size_t)P * kPlaneBinsHost));
    if (c->pbin_counts.p != before)
      CK(cudaMemset(c->pbin_counts.p, 0, sizeof(unsigned int) * c->pbin_counts.cap));
    CK(c->pbin_cursor.ensure((size_t)P * kPlaneBinsHost));
  }
  CK(c->plane_sorted.ensure((size_t)(3 * dcap)));
  // surviving in-plane chunk pairs: sized for 16 per chunk (overflow is
  // detected on the device and re-run with the exact count).
  const long long t = (3 * dcap) / kPlaneChunk + P + 1;  // chunks over all planes
  const long long pu = std::max(std::min(t * (t + 1) / 2, t * 16), punits);
  CK(c->plane_umax.ensure((size_t)pu));
  CK(c->plane_work.ensure((size_t)pu));
  CK(c->plane_boxes_buf.ensure((size_t)t));
  CK(c->plane_hboxes.ensure((size_t)(2 * t)));
  CK(c->plane_cmap.ensure((size_t)t));
  return SC_OK;
}

// Grid of the latency-bound pipeline kernels: k blocks per SM, divided by the
// option "grid_div" (fewer blocks = less block-scheduling and prologue work
// per ROI when several ROIs share the GPU; every kernel is grid-stride).
int lgrid(const Ctx* c, int k) {
  return std::max(1, c->sms * k / std::max(1, c->grid_div));
}

// Zero-copy per-ROI records (option "zero_copy", default on): init_stats reads
// RoiParams from mapped pinned host memory and diam_refine's last block writes
// the accumulator record back there, so the ROI is the graph alone -- no H2D
// copy before it and no D2H copy node inside it.  Off for the debug stage cuts
// (diam_refine may not run).
bool zero_copy_records(const Ctx* c) {
  (void)c;
  return c->o.zc && c->o.stages >= (1 << 20);
}

// Launch of a per-ROI pipeline kernel.  In batch graphs (no stage-event nodes
// between the kernels) it carries the programmatic-dependent-launch attribute
// (option "pdl"): the kernel is scheduled while its predecessor drains and
// waits on griddepcontrol.wait (pdl_enter) for the predecessor's results.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(const Ctx* c, cudaStream_t s, int grid, int block, void (*k)(KArgs...),
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  // (not with the fork / join: a programmatic edge cannot follow an event wait)
  cfg.numAttrs = (c->o.pdl && !c->events_on && !c->o.fork) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

// Batch pack chain (option "pack_chain"): the end of this slot's HBM pass is
// marked on pack_ev, and the ROI waits for another slot's mark before it
// starts, so the packs of consecutive ROIs run one (or pack_chain) at a time
// at the full HBM rate while the latency-bound kernels of earlier ROIs
// overlap them.  Inside a capture both are external event nodes.
cudaError_t chain_mark(Ctx* c, cudaStream_t s) {
  if (!c->chain_wait) return cudaSuccess;
  return c->capturing ? cudaEventRecordWithFlags(c->pack_ev, s, cudaEventRecordExternal)
                      : cudaEventRecord(c->pack_ev, s);
}

// Launch with an explicit priority (the batch's HBM chain -- init_stats and
// the pack -- runs at the greatest priority, option "pack_prio": its CTAs are
// scheduled ahead of the latency-bound kernels of the ROIs already in flight,
// so the next pack of the chain does not queue behind them).
template <typename... KArgs, typename... Args>
cudaError_t launch_prio(const Ctx* c, cudaStream_t s, dim3 grid, int block, size_t smem,
                        void (*k)(KArgs...), Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributePriority;
  at[0].val.priority = c->prio_hi;
  cfg.attrs = at;
  cfg.numAttrs = c->o.pack_prio ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

// TMA bulk-copy pack: `pack_tma` CTAs per SM of `pack_threads` threads, each
// streaming through a ring of `pack_stages` 16 KB shared-memory tiles.
template <bool BOX>
cudaError_t launch_tma_pack(Ctx* c, cudaStream_t s) {
  const int st = std::max(2, std::min(8, c->o.pack_stages));
  const size_t smem = (size_t)st * kTmaTileBytes;
  const dim3 grid((unsigned)(c->sms * c->o.pack_tma));
  const RoiParams* rp = c->d_rp;
  if (c->o.pack_tile == 32) {  // 32 KB tiles (64 / 128 / 256 threads, <= 6 stages)
    const int st32 = std::min(st, 6);
    const size_t sm32 = (size_t)st32 * 32768;
    if (c->o.pack_threads <= 64)
      return launch_prio(c, s, grid, 64, sm32, pack_bits_tma<BOX, 64, 32768>, rp, c->bits.p,
                         c->d_stats, c->segmap.p, st32);
    if (c->o.pack_threads <= 128)
      return launch_prio(c, s, grid, 128, sm32, pack_bits_tma<BOX, 128, 32768>, rp, c->bits.p,
                         c->d_stats, c->segmap.p, st32);
    return launch_prio(c, s, grid, 256, sm32, pack_bits_tma<BOX, 256, 32768>, rp, c->bits.p,
                       c->d_stats, c->segmap.p, st32);
  }
  if (c->o.pack_tile == 8)  // 8 KB tiles (256 threads)
    return launch_prio(c, s, grid, 256, (size_t)st * 8192, pack_bits_tma<BOX, 256, 8192>, rp,
                       c->bits.p, c->d_stats, c->segmap.p, st);
  if (c->o.pack_threads <= 128)  // (the 16 KB block-ring pack has 128- and 256-thread forms)
    return launch_prio(c, s, grid, 128, smem, pack_bits_tma<BOX, 128, 16384>, rp, c->bits.p,
                       c->d_stats, c->segmap.p, st);
  return launch_prio(c, s, grid, 256, smem, pack_bits_tma<BOX, 256, 16384>, rp, c->bits.p,
                     c->d_stats, c->segmap.p, st);
}

// Enqueue one whole ROI on stream s; no host synchronisation.  Everything
// ROI-specific (mask pointer, dims, spacing) is read by the kernels from the
// slot's RoiParams record, so the enqueued sequence -- and a graph captured
// from it -- depends only on the pack path, the shard and the slot buffers.
// kev[] brackets the stages for sc_last_kernel_times.
int enqueue_diam(Ctx* c, cudaStream_t s, int shard, int nshards, int& nk);

int enqueue_roi(Ctx* c, bool fast, cudaStream_t s, int shard, int nshards) {
  const RoiParams* rp = c->d_rp;
  // Diagnostic option "debug_stages": enqueue only the first N kernels (results
  // invalid) to measure the marginal batch cost of each stage.
  const int lim = c->o.stages;
  int nk = 0;
  const long long cap = (long long)c->keys.cap, dcap = c->dcap_sz;
  // (the pack marks nonzero segments of a cleared map; the no-pack debug mode
  // keeps the previous map)
  const bool clear_map = c->o.sparse && !(c->o.pack_mode & 4) && !c->prepacked;
  const bool zc = zero_copy_records(c);
  if (c->chain_wait)
    CK(cudaStreamWaitEvent(s, c->chain_wait, c->capturing ? cudaEventWaitExternal : 0));
  CK(launch_prio(c, s, dim3(clear_map ? 8 : 1), 256, 0, init_stats, c->d_stats, c->segmap.p,
                 clear_map ? (long long)c->segmap.cap : 0LL,
                 (const RoiParams*)(zc ? c->h_rp_dev : nullptr), c->d_rp));
  CKL(1);
  for (int e = 0; e < c->o.empty; e++) {  // debug: launch-rate probe
    empty_kernel<<<1, 32, 0, s>>>();
    CKL(1);
  }
  if (++nk >= lim) return SC_OK;
  CK(record(c, c->kev[0], s));  // kev0..kev1 = the HBM pass alone
  if (c->prepacked) {  // the host already wrote the bit volume: bbox pass only
    CK(record(c, c->kev[1], s));
    CK(chain_mark(c, s));
    CK(launch_k(c, s, lgrid(c, 4), 256, bits_bbox, rp, reinterpret_cast<const uint4*>(c->bits.p),
                c->d_stats, c->segmap.p));
    CKL(1);
    if (++nk >= lim) return SC_OK;
  } else if (fast && c->o.fbox && c->o.pack_tma > 0 &&
             !(c->o.pack_mode & 4)) {
    // TMA pack with the bbox accumulated inside (no bits_bbox kernel)
    CK(launch_tma_pack<true>(c, s));
    CKL(1);
    if (++nk >= lim) return SC_OK;
    CK(record(c, c->kev[1], s));
    CK(chain_mark(c, s));
  } else if (fast && c->o.fbox && !(c->o.pack_mode & 4)) {
    pack_bits_v16<4, true><<<c->sms * std::max(1, c->occ_pack), 256, 0, s>>>(rp, c->bits.p,
                                                                              c->d_stats,
                                                                              c->segmap.p);
    CKL(1);
    if (++nk >= lim) return SC_OK;
    CK(record(c, c->kev[1], s));
    CK(chain_mark(c, s));
  } else if (fast) {
    // pack_mode bit 0: one 4 KB step per block (grid covers the slot's largest
    // mask; extra blocks exit) instead of a persistent grid, so blocks retire
    // continuously and other streams' kernels interleave; bit 1: low priority.
    const int pm = c->o.pack_mode;
    cudaLaunchConfig_t cfg = {};
    const int pbps = c->o.pack_bps > 0 ? c->o.pack_bps : std::max(1, c->occ_pack);
    cfg.gridDim = dim3((unsigned)(c->sms * pbps));
    if (pm & 1)
      cfg.gridDim = dim3((unsigned)std::max<long long>(
          1, (2 * (long long)c->bits.cap + 256 * 4 - 1) / (256 * 4)));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributePriority;
    at[0].val.priority = c->prio_lo;
    cfg.attrs = at;
    cfg.numAttrs = (pm & 2) ? 1 : 0;
    if (!(pm & 4) && c->o.pack_tma > 0) {  // bulk-copy (TMA) pack
      CK(launch_tma_pack<false>(c, s));
      CKL(1);
    } else if (!(pm & 4)) {  // bit 2 (debug, timing only): reuse the slot's previous bit volume
      CK(cudaLaunchKernelEx(&cfg, pack_bits_v16<4, false>, rp, c->bits.p, c->d_stats,
                            c->segmap.p));
      CKL(1);
    }
    if (++nk >= lim) return SC_OK;
    CK(record(c, c->kev[1], s));
    CK(chain_mark(c, s));
    CK(launch_k(c, s, lgrid(c, 4), 256, bits_bbox, rp, reinterpret_cast<const uint4*>(c->bits.p),
                                         c->d_stats, c->segmap.p));
    CKL(1);
    if (++nk >= lim) return SC_OK;
  } else {
    pack_bits_generic<<<lgrid(c, 8), 256, 0, s>>>(rp, c->bits.p, c->d_stats,
                                                  c->segmap.p);  // after init_stats: no PDL
    CKL(1);
    if (++nk >= lim) return SC_OK;
    CK(record(c, c->kev[1], s));
    CK(chain_mark(c, s));
  }
  CK(launch_k(c, s, lgrid(c, std::max(1, c->occ_mc)), 256, mc_cells, rp, c->bits.p, c->d_tabs, c->d_stats,
                                                          c->keys.p, cap, c->sort_counts.p,
                                                          c->pbin_counts.p, c->segmap.p));
  CKL(1);
  if (++nk >= lim) return SC_OK;
  CK(record(c, c->kev[2], s));
  if (c->mesh_only) return SC_OK;
  return enqueue_diam(c, s, shard, nshards, nk);
}

// Diameter half of the pipeline (sort -> bounds -> filters -> pass 1 ->
// re-check): reads only the slot's Stats (bbox, n_vert), the vertex keys and
// the brick / plane-bin histograms mc_cells left -- or, in the two-phase shard
// entry, the gathered keys and summed histograms loaded into the same buffers.
int enqueue_diam(Ctx* c, cudaStream_t s, int shard, int nshards, int& nk) {
  const RoiParams* rp = c->d_rp;
  const int lim = c->o.stages;
  const long long dcap = c->dcap_sz;
  const bool zc = zero_copy_records(c);
  // Persistent grids: exactly the resident blocks, so the static round-robin
  // split of work units is also the load balance.
  const int pgrid = lgrid(c, std::max(1, c->o.packed ? c->occ_pass1 : c->occ_pass1s));
  const long long pucap = (long long)c->plane_umax.cap;
  const int prune = c->o.prune ? 1 : 0;

  // Orders (Morton bricks; planes by in-plane brick), chunk boxes + extremes,
  // exact lower bound, pruned 3-D work list.
  CK(launch_k(c, s, kScanBlocks + std::max(1, lgrid(c, 1) / 2), kScanThreads, scan_all, c->sort_counts.p, c->sort_cursor.p,
                                            c->plane_counts.p, c->plane_start.p,
                                            c->plane_tstart.p, c->plane_cstart.p, dcap,
                                            c->d_stats, c->sboxes.p, c->pbin_counts.p, c->pbin_cursor.p, c->plane_ext.p,
                                            nshards > 1 ? 1 : 0));
  CKL(1);
  if (++nk >= lim) return SC_OK;
  CK(launch_k(c, s, lgrid(c, 4), 256, scatter_all, c->keys.p, dcap, c->d_stats, c->sort_cursor.p,
                                         c->keys_sorted.p, c->plane_start.p, c->pbin_cursor.p,
                                         c->plane_sorted.p, c->sort_counts.p + kSortBins,
                                         c->plane_cstart.p, c->plane_cmap.p));
  CKL(1);
  if (++nk >= lim) return SC_OK;
  if (nshards > 1) {
    // Shards own 3-D chunk pairs by identity: give every shard (every GPU)
    // the same vertex order -- each brick bin's segment sorted by the vertex's
    // coordinates inside the brick.
    // (one warp per bin, 4-warp blocks: 16 blocks per SM)
    CK(launch_k(c, s, c->sms * 16, 128, canon_keys, c->keys_sorted.p, c->keys.p,
                c->sort_cursor.p, c->d_stats));
    CKL(1);
    // (planar units are owned by whole planes, planar.cu plane_filter: the
    // order of a plane's entries does not matter)
  }
  // After the sort the 3-D chain (boxes -> filter) and the planar chain
  // (plane boxes -> bound -> filter) are independent: the planar one runs on
  // the slot's second stream (a fork / join inside the captured graph), so
  // the ROI's critical path is the longer chain, not their sum.
  const bool fork = c->o.fork && lim >= (1 << 20);
  cudaStream_t sp = s;
  if (fork) {
    CK(cudaEventRecord(c->fork_ev, s));
    CK(cudaStreamWaitEvent(c->stream2, c->fork_ev, 0));
    sp = c->stream2;
    CK(record(c, c->kev[7], sp));
    CK(launch_k(c, sp, lgrid(c, 4), 256, plane_boxes, c->plane_sorted.p, c->plane_start.p,
                c->plane_cstart.p, rp, c->d_stats, c->plane_boxes_buf.p, c->plane_ext.p,
                c->plane_hboxes.p, c->plane_cmap.p));
    CKL(1);
    CK(launch_k(c, sp, lgrid(c, 1), 256, plane_lb, c->plane_sorted.p, c->plane_start.p,
                c->plane_ext.p, rp, c->d_stats));
    CKL(1);
    CK(launch_k(c, sp, lgrid(c, 4), 256, plane_filter, c->plane_start.p, c->plane_tstart.p,
                c->plane_cstart.p, c->plane_boxes_buf.p, rp, prune, shard, nshards, pucap,
                c->d_stats, c->plane_work.p, c->plane_hboxes.p));
    CKL(1);
    CK(record(c, c->kev[8], sp));
    CK(cudaEventRecord(c->join_ev, sp));
  }
  // (the unsorted mc output is dead after the sort: its buffer takes the
  // pass-1 frame coordinates of the sorted keys)
  float4* fkeys = reinterpret_cast<float4*>(c->keys.p);
  CK(launch_k(c, s, lgrid(c, 2), 256, boxes_extremes, c->keys_sorted.p, dcap, rp, c->d_stats, c->boxes.p,
                                            c->sboxes.p, c->hboxes.p, fkeys));
  CKL(1);
  if (++nk >= lim) return SC_OK;
  CK(launch_k(c, s, lgrid(c, 4), 256, unit_filter, c->keys_sorted.p, c->boxes.p, dcap, rp, prune, shard,
                                         nshards, c->d_stats, c->work.p, c->sboxes.p, c->hboxes.p, c->slist.p, (long long)c->slist.cap));
  CKL(1);
  CK(launch_k(c, s, lgrid(c, 4), 256, unit_expand, c->boxes.p, dcap, rp, prune, shard, nshards,
              c->d_stats, c->work.p, c->hboxes.p, c->slist.p, (long long)c->slist.cap));
  CKL(1);
  if (++nk >= lim) return SC_OK;
  CK(record(c, c->kev[3], s));
  if (!fork) {
  CK(record(c, c->kev[7], s));
  CK(launch_k(c, s, lgrid(c, 4), 256, plane_boxes, c->plane_sorted.p, c->plane_start.p, c->plane_cstart.p,
                                         rp, c->d_stats, c->plane_boxes_buf.p, c->plane_ext.p, c->plane_hboxes.p,
                                         c->plane_cmap.p));
  CKL(1);
  if (++nk >= lim) return SC_OK;
  CK(launch_k(c, s, lgrid(c, 1), 256, plane_lb, c->plane_sorted.p, c->plane_start.p, c->plane_ext.p, rp,
                                  c->d_stats));
  CKL(1);
  if (++nk >= lim) return SC_OK;
  CK(launch_k(c, s, lgrid(c, 4), 256, plane_filter, c->plane_start.p, c->plane_tstart.p, c->plane_cstart.p,
                                          c->plane_boxes_buf.p, rp, prune, shard, nshards, pucap,
                                          c->d_stats, c->plane_work.p, c->plane_hboxes.p));
  CKL(1);
  if (++nk >= lim) return SC_OK;
  CK(record(c, c->kev[8], s));
  } else {
    CK(cudaStreamWaitEvent(s, c->join_ev, 0));
  }
  CK(record(c, c->kev[4], s));
  // One pass-1 kernel and one re-check kernel for the 3-D and the planar lists.
  if (c->o.packed)
    CK(launch_k(c, s, pgrid, 256, diam_pass1<true>, c->keys_sorted.p, dcap, rp, c->work.p,
                c->warp_max.p, c->plane_sorted.p, c->plane_start.p, c->plane_work.p, pucap,
                c->plane_umax.p, c->d_stats, c->boxes.p, c->hboxes.p, prune, c->plane_cstart.p,
                c->plane_boxes_buf.p, c->plane_hboxes.p, (const float4*)fkeys));
  else
    CK(launch_k(c, s, pgrid, 256, diam_pass1<false>, c->keys_sorted.p, dcap, rp, c->work.p, c->warp_max.p,
                                            c->plane_sorted.p, c->plane_start.p, c->plane_work.p,
                                            pucap, c->plane_umax.p, c->d_stats, c->boxes.p,
                                            c->hboxes.p, prune, c->plane_cstart.p,
                                            c->plane_boxes_buf.p, c->plane_hboxes.p,
                                            (const float4*)fkeys));
  CKL(1);
  if (++nk >= lim) return SC_OK;
  CK(record(c, c->kev[5], s));
  CK(launch_k(c, s, lgrid(c, 2), 256, diam_refine, c->keys_sorted.p, dcap, rp, c->work.p, c->warp_max.p,
                                         c->plane_sorted.p, c->plane_start.p, c->plane_work.p,
                                         pucap, c->plane_umax.p, c->d_stats, zc ? c->h_stats_dev : nullptr));
  CKL(1);
  if (++nk >= lim) return SC_OK;
  CK(record(c, c->kev[6], s));
  return SC_OK;
}

void fill_out(const Stats& h, const double sp[3], sc_coeffs* out) {
  static const int* tri = [] {
    static int t[kNumCases];
    for (int k = 0; k < kNumCases; k++) t[k] = case_geom().ntri[k];
    return t;
  }();
  thread_local double at[kNumCases];  // per-case areas, cached per spacing
  thread_local double at_sp[3] = {-1.0, -1.0, -1.0};
  if (sp[0] != at_sp[0] || sp[1] != at_sp[1] || sp[2] != at_sp[2]) {
    area_table(sp, at);
    at_sp[0] = sp[0]; at_sp[1] = sp[1]; at_sp[2] = sp[2];
  }
  double area = 0.0;
  long long T = 0, active = 0;
  for (int k = 0; k < kNumCases; k++) {
    unsigned long long cnt = 0;
    for (int c = 0; c < (h.hist_merged ? 1 : kHistCopies); c++) cnt += h.hist[c][k];
    if (!cnt) continue;
    area += (double)cnt * at[k];
    T += (long long)cnt * tri[k];
    active += (long long)cnt;
  }
  const long long K = h.vol_k < 0 ? -h.vol_k : h.vol_k;
  out->mesh_volume = (double)K * sp[0] * sp[1] * sp[2] / 48.0;
  out->surface_area = area;
  out->max_3d_diameter = std::sqrt(f64_of(h.sq[0]));
  out->max_2d_diameter_xy = std::sqrt(f64_of(h.sq[1]));
  out->max_2d_diameter_xz = std::sqrt(f64_of(h.sq[2]));
  out->max_2d_diameter_yz = std::sqrt(f64_of(h.sq[3]));
  out->vertex_count = (int64_t)h.n_vert;
  out->triangle_count = T;
  out->active_cubes = active;
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    (void)cudaGetLastError();  // an unrecorded / pending event is not a launch error
    ms = 0.f;
  }
  return ms;
}

// Enqueue one ROI plus its result copies, replaying the slot's cached CUDA
// graph for this (pack path, stream, shard, buffers, options) when there is
// one; otherwise capture it first.  Graph replay removes the per-kernel launch
// cost of the ~16-kernel pipeline (SC option "graphs").  The ROI's parameters
// travel in a 96-byte H2D copy ahead of the graph.
int enqueue_with_copies(Ctx* c, bool fast, cudaStream_t s, int shard, int nshards,
                        double* d_sq4) {
  int rc = enqueue_roi(c, fast, s, shard, nshards);
  if (rc) return rc;
  if (d_sq4)
    CK(cudaMemcpyAsync(d_sq4, c->d_stats->sq, 4 * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (!zero_copy_records(c))  // else diam_refine published the record itself
    CK(cudaMemcpyAsync(c->h_stats, c->d_stats, sizeof(Stats), cudaMemcpyDeviceToHost, s));
  return SC_OK;
}

double wall_ms();
// Host-side phase accounting of the batch loop (SC_HOST_PROFILE=1 prints it).
struct HostProf {
  double sync = 0, finish = 0, start = 0, copy = 0, launch = 0;
  long long n = 0;
};
HostProf g_hprof;
bool host_prof_on() {
  static const bool on = std::getenv("SC_HOST_PROFILE") != nullptr;
  return on;
}

// Batch timeline from the kernels' %globaltimer spans (Stats::tr), SC_TRACE=1:
// per kernel its mean start offset from the ROI start (init_stats) and mean
// span, plus the mean ROI latency; printed at the end of each batch.
struct TraceAcc {
  double off[kTrCount] = {}, span[kTrCount] = {}, busy[kTrCount] = {};
  long long n[kTrCount] = {};
  double lat = 0;
  long long rois = 0;
  std::vector<std::array<unsigned long long, 4>> seq;  // (t_start, pack start, pack end, t_end)
};
TraceAcc g_trace;
std::mutex g_trace_mu;  // batches on several host threads share the accumulator
bool trace_on() {
  static const bool on = std::getenv("SC_TRACE") != nullptr;
  return on;
}
void trace_add(const Stats& h) {
  if (!h.t_start) return;
  std::lock_guard<std::mutex> lk(g_trace_mu);
  for (int k = 1; k < kTrCount; k++) {
    // (the refine's last block publishes the record before its own end
    // stamp: its end is t_end)
    const unsigned long long end = k == kTrRefine ? h.t_end : h.tr[k][1];
    if (h.tr[k][0] == ~0ull || end < h.tr[k][0]) continue;
    g_trace.off[k] += 1e-3 * (double)(h.tr[k][0] - h.t_start);
    g_trace.span[k] += 1e-3 * (double)(end - h.tr[k][0]);
    g_trace.busy[k] += 1e-3 * (double)h.busy[k];
    g_trace.n[k]++;
  }
  if (h.t_end > h.t_start) {
    g_trace.lat += 1e-3 * (double)(h.t_end - h.t_start);
    g_trace.rois++;
  }
  g_trace.seq.push_back({h.t_start, h.tr[kTrPack][0], h.tr[kTrPack][1], h.t_end});
}
void trace_print() {
  static const char* names[kTrCount] = {"init", "pack", "mc_cells", "scan_all", "scatter_all",
                                         "plane_boxes", "plane_lb", "plane_filter",
                                         "boxes_extremes", "unit_filter", "unit_expand",
                                         "pass1", "refine"};
  std::lock_guard<std::mutex> lk(g_trace_mu);
  if (!g_trace.rois) return;
  std::fprintf(stderr, "[sc trace] %lld ROIs, mean ROI latency %.1f us (init -> refine end)\n",
               g_trace.rois, g_trace.lat / (double)g_trace.rois);
  for (int k = 1; k < kTrCount; k++)
    if (g_trace.n[k])
      std::fprintf(stderr, "[sc trace]   %-15s start +%8.1f us  span %8.1f us  block-us %9.1f\n",
                   names[k], g_trace.off[k] / (double)g_trace.n[k],
                   g_trace.span[k] / (double)g_trace.n[k], g_trace.busy[k] / (double)g_trace.n[k]);
  // Admission: ROI i (slot i mod S) starts after ROI i - S ended (slot reuse:
  // host collect + relaunch) and after ROI i - chain's pack (pack chain).
  const auto& q = g_trace.seq;
  const int S = std::getenv("SC_TRACE_SLOTS") ? std::atoi(std::getenv("SC_TRACE_SLOTS")) : 32;
  const int ch = std::getenv("SC_TRACE_CHAIN") ? std::atoi(std::getenv("SC_TRACE_CHAIN")) : 4;
  double g_slot = 0, g_chain = 0, pack_gap = 0, g_link = 0;
  long long n_slot = 0, n_chain = 0, n_pg = 0, n_link = 0;
  for (size_t i = 0; i < q.size(); i++) {
    if (i >= (size_t)S && q[i - S][3] && q[i][0] > q[i - S][3]) {
      g_slot += 1e-3 * (double)(q[i][0] - q[i - S][3]);
      n_slot++;
    }
    if (ch > 0 && i >= (size_t)ch && q[i][0] > q[i - ch][2]) {
      g_chain += 1e-3 * (double)(q[i][0] - q[i - ch][2]);
      n_chain++;
    }
    if (ch > 0 && i >= (size_t)ch && q[i][1] > q[i - ch][2] && q[i - ch][2]) {
      g_link += 1e-3 * (double)(q[i][1] - q[i - ch][2]);
      n_link++;
    }
    if (i >= 1 && q[i][1] > q[i - 1][1]) {
      pack_gap += 1e-3 * (double)(q[i][1] - q[i - 1][1]);
      n_pg++;
    }
  }
  if (n_slot) std::fprintf(stderr, "[sc trace]   init(i) - end(i-%d)      %8.1f us (slot reuse)\n", S, g_slot / n_slot);
  if (n_chain) std::fprintf(stderr, "[sc trace]   init(i) - pack end(i-%d)  %8.1f us (pack chain)\n", ch, g_chain / n_chain);
  if (n_pg) std::fprintf(stderr, "[sc trace]   pack start spacing       %8.1f us\n", pack_gap / n_pg);
  if (n_link)
    std::fprintf(stderr, "[sc trace]   pack start(i) - pack end(i-%d) %6.1f us (%lld of %zu ROIs)\n", ch,
                 g_link / n_link, n_link, q.size());
  g_trace = TraceAcc{};
}

// Everything about the pack that a captured graph bakes in.
int pack_key(const Opts& o) {
  return (o.pack_mode & 7) | ((o.pack_bps & 63) << 3) | ((o.pack_tma & 15) << 9) |
         ((o.pack_stages & 15) << 13) | (((o.pack_threads / 32) & 15) << 17) |
         ((o.pack_prio ? 1 : 0) << 21) | ((o.pack_tile / 8) << 23);
}

// The slot's RoiParams record for the next ROI (host copy; the slot's
// previous ROI has been collected, so it is safe to rewrite).
void fill_rp(Ctx* c, const uint8_t* d_mask, int64_t nx, int64_t ny, int64_t nz,
             const double sp[3], const int org[3]) {
  RoiParams& h = *c->h_rp;
  h.mask = d_mask;
  h.nx = nx;
  h.ny = ny;
  h.nz = nz;
  h.W = (int)((nx + 31) / 32);
  h.n_words = (long long)h.W * ny * nz;
  h.n_chunks = nx * ny * nz / 16;
  h.sparse = (c->o.sparse && !c->prepacked) ? (c->o.pack_skip ? 3 : 1) : 0;
  h.pflags = trace_on() ? 4 : 0;
  h.mc_slab = c->mc_slab;
  h.f.cx2 = h.f.cy2 = h.f.cz2 = 0;  // set on the device from the bbox
  h.f.hx = (float)(0.5 * sp[0]);
  h.f.hy = (float)(0.5 * sp[1]);
  h.f.hz = (float)(0.5 * sp[2]);
  h.f.sx = sp[0];
  h.f.sy = sp[1];
  h.f.sz = sp[2];
  h.f.ox2 = 2 * org[0];  // slab origin (host crop); graph-invariant like the rest
  h.f.oy2 = 2 * org[1];
  h.f.oz2 = 2 * org[2];
  h.wcap = (long long)std::min(c->work.cap, c->warp_max.cap);
}

int launch_roi(Ctx* c, const uint8_t* d_mask, int64_t nx, int64_t ny, int64_t nz,
               const double sp[3], cudaStream_t s, int shard, int nshards, double* d_sq4,
               const int org[3]) {
  fill_rp(c, d_mask, nx, ny, nz, sp, org);
  const bool hp = host_prof_on();
  double t0 = hp ? wall_ms() : 0.0;
  if (!zero_copy_records(c))  // else init_stats reads the record from mapped host memory
    CK(cudaMemcpyAsync(c->d_rp, c->h_rp, sizeof(RoiParams), cudaMemcpyHostToDevice, s));
  if (hp) { const double t1 = wall_ms(); g_hprof.copy += t1 - t0; t0 = t1; }
  const bool fast = nx % 32 == 0 && (reinterpret_cast<uintptr_t>(d_mask) & 15) == 0;
  if (!c->o.graphs || s == nullptr)
    return enqueue_with_copies(c, fast, s, shard, nshards, d_sq4);
  const long long cap = (long long)c->keys.cap, dcap = c->dcap_sz;
  const bool prune = c->o.prune, packed = c->o.packed, fbox = c->o.fbox;
  for (auto& g : c->graphs)
    if (g.fast == fast && g.s == s && g.shard == shard && g.nshards == nshards &&
        g.d_sq4 == d_sq4 && g.cap == cap && g.dcap == dcap && g.prune == prune &&
        g.packed == packed && g.fbox == fbox && g.stages == c->o.stages + 7 * c->o.empty &&
        g.packmode == pack_key(c->o) &&
        g.grid_div == c->grid_div &&
        g.events == c->events_on && g.ev_full == c->ev_full && g.pdl == c->o.pdl &&
        g.sparse == c->o.sparse && g.fork == c->o.fork &&
        g.zc == c->o.zc && g.prepacked == c->prepacked && g.chain == c->chain_wait &&
        g.gen == c->gen) {
      CK(cudaGraphLaunch(g.exec, s));
      if (hp) g_hprof.launch += wall_ms() - t0;
      g_launches.fetch_add(g.launches, std::memory_order_relaxed);
      return SC_OK;
    }
  const unsigned long long before = g_launches.load();
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  c->capturing = true;
  int rc = enqueue_with_copies(c, fast, s, shard, nshards, d_sq4);
  c->capturing = false;
  cudaGraph_t graph = nullptr;
  cudaError_t ec = cudaStreamEndCapture(s, &graph);
  const unsigned long long launches = g_launches.load() - before;
  g_launches.fetch_sub(launches, std::memory_order_relaxed);  // captured, not launched
  if (rc) { if (graph) cudaGraphDestroy(graph); return rc; }
  CK(ec);
  cudaGraphExec_t exec = nullptr;
  ec = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  CK(ec);
  if (c->graphs.size() >= 8) {
    cudaGraphExecDestroy(c->graphs.front().exec);
    c->graphs.erase(c->graphs.begin());
  }
  Ctx::GraphEntry g{fast, s, shard, nshards, d_sq4, cap, dcap, prune, packed, fbox,
                    c->o.stages + 7 * c->o.empty,
                    pack_key(c->o),
                    c->grid_div,
                    c->events_on, c->ev_full, c->o.pdl, c->o.sparse,
                    c->o.fork, c->o.zc, c->prepacked, c->chain_wait, c->gen, exec, launches};
  c->graphs.push_back(g);
  CK(cudaGraphLaunch(exec, s));
  g_launches.fetch_add(launches, std::memory_order_relaxed);
  return SC_OK;
}

// Start one ROI on slot c: make room, enqueue (graph replay when cached).
// No synchronisation; finish_roi collects it.
struct Pending {
  const uint8_t* d_mask;
  int64_t nx, ny, nz;
  double sp[3];
  cudaStream_t s;
  int shard, nshards;
  double* d_sq4;
  long long cap, dcap, wunits;
  int org[3];  // origin of the (cropped) volume in the caller's grid, voxels
};

int start_roi(Ctx* c, const uint8_t* d_mask, int64_t nx, int64_t ny, int64_t nz,
              const double sp[3], cudaStream_t s, int shard, int nshards, double* d_sq4,
              long long punits, Pending* p, const int org[3] = nullptr) {
  static const int kZero[3] = {0, 0, 0};
  if (!org) org = kZero;
  // Requested sizes depend only on the dims and on floors raised by overflow
  // re-runs (never on the allocated capacities, so graphs stay valid).
  if (p->cap > 0) {  // re-run after an overflow: exact sizes from now on
    c->cap_floor = std::max(c->cap_floor, p->cap);
    c->dcap_floor = std::max(c->dcap_floor, p->dcap);
    c->wcap_floor = std::max(c->wcap_floor, p->wunits);
  }
  long long cap = vertex_capacity(nx, ny, nz, c->cap_floor);
  long long dcap = std::min<long long>(cap, std::max<long long>(c->o.dcap, c->dcap_floor));
  const unsigned long long fp0 = c->fingerprint();
  int rc = ensure_buffers(c, nx, ny, nz, cap, dcap, punits, c->wcap_floor);
  if (rc) return rc;
  if (c->fingerprint() != fp0) {
    c->gen++;
    c->drop_graphs();
  }
  *p = Pending{d_mask, nx, ny, nz, {sp[0], sp[1], sp[2]}, s, shard, nshards, d_sq4,
               (long long)c->keys.cap, c->dcap_sz, 0, {org[0], org[1], org[2]}};
  return launch_roi(c, d_mask, nx, ny, nz, sp, s, shard, nshards, d_sq4, org);
}

// Wait for the ROI started on slot c, re-run it once with exact buffer sizes
// if the device reported an overflow, and fill `out`.
// Checks and output record of a ROI whose Stats are on the host.
int collect_roi(Ctx* c, const double sp[3], sc_coeffs* out) {
  if (c->h_stats->bbox[3] < 0) {
    set_err("mask has no occupied voxels");
    return SC_ERR_EMPTY_ROI;
  }
  if (c->h_stats->plane_ovf) {
    set_err("a plane of the mesh holds more than %lld vertices (planar chunk index width)",
            kPlaneMaxEntries);
    return SC_ERR_INPUT;
  }
  if ((long long)c->h_stats->n_super > (long long)c->slist.cap) {
    // cannot happen with slist sized from kSingleLevelMax; never report a
    // maximum from a truncated super-pair list
    set_err("super-pair list overflow (%llu > %zu)", c->h_stats->n_super, c->slist.cap);
    return SC_ERR_NOMEM;
  }
  fill_out(*c->h_stats, sp, out);
  if (trace_on()) trace_add(*c->h_stats);
  c->times_pending = c->events_on && c->ev_full;  // per-stage times: from kev[] on demand
  if (!c->times_pending)
    for (int i = 0; i < 6; i++) c->last_ms[i] = 0.0;
  c->last_ms[6] = 0.0;
  {
    const Stats& h = *c->h_stats;
    const long long Vv = (long long)h.n_vert, C = (Vv + kChunk - 1) / kChunk;
    c->last_diag[0] = (long long)h.n_work;
    c->last_diag[1] = C * (C + 1) / 2;
    c->last_diag[2] = (long long)h.n_cand;
    c->last_diag[3] = (long long)h.plane_units;
    c->last_diag[4] = (long long)h.n_pcand;
    c->last_diag[5] = (long long)h.n_pwork;
    c->last_diag[6] = (long long)h.n_sub;
    c->last_diag[7] = (long long)h.n_psub;
    c->last_diag[8] = (long long)h.n_eval;
    c->last_diag[9] = (long long)h.n_peval;
  }
  if (c->events_on) {
    out->mesh_ms = ev_ms(c->kev[0], c->kev[2]);
    out->diameters_ms = ev_ms(c->kev[2], c->kev[6]);
  } else {  // device %globaltimer stamps (no event nodes in the graph)
    const Stats& h = *c->h_stats;
    out->mesh_ms = h.t_mesh > h.t_start ? (double)(h.t_mesh - h.t_start) * 1e-6 : 0.0;
    out->diameters_ms = h.t_end > h.t_mesh ? (double)(h.t_end - h.t_mesh) * 1e-6 : 0.0;
  }
  return SC_OK;
}

int finish_roi(Ctx* c, Pending* p, sc_coeffs* out) {
  const bool hp = host_prof_on();
  const double t0 = hp ? wall_ms() : 0.0;
  CK(cudaStreamSynchronize(p->s));
  const double t1 = hp ? wall_ms() : 0.0;
  if (hp) g_hprof.sync += t1 - t0;
  struct Tail {  // everything after the wait is "finish"
    bool on; double t;
    ~Tail() { if (on) { g_hprof.finish += wall_ms() - t; g_hprof.n++; } }
  } tail{hp, t1};
  const long long V = (long long)c->h_stats->n_vert;
  const long long PU = (long long)c->h_stats->n_pwork;
  const long long WU = (long long)c->h_stats->n_work;
  if (V > p->dcap || PU > (long long)c->plane_umax.cap || WU > c->h_rp->wcap) {
    // rare: more vertices / planar tiles / 3-D units than reserved -> exact re-run
    Pending q = *p;
    q.cap = std::max(p->cap, V);
    q.dcap = std::max(p->dcap, V);
    q.wunits = WU;
    const int org[3] = {q.org[0], q.org[1], q.org[2]};
    int rc = start_roi(c, q.d_mask, q.nx, q.ny, q.nz, q.sp, q.s, q.shard, q.nshards, q.d_sq4, PU,
                       &q, org);
    if (rc) return rc;
    CK(cudaStreamSynchronize(q.s));
    if ((long long)c->h_stats->n_vert > q.dcap ||
        (long long)c->h_stats->n_pwork > (long long)c->plane_umax.cap ||
        (long long)c->h_stats->n_work > c->h_rp->wcap) {
      set_err("vertex buffer overflow");
      return SC_ERR_NOMEM;
    }
  }
  return collect_roi(c, p->sp, out);
}

// Full pipeline on a device-resident mask (context lock held by the caller).
int run_roi(Ctx* c, const uint8_t* d_mask, int64_t nx, int64_t ny, int64_t nz, const double sp[3],
            cudaStream_t s, int shard, int nshards, double* d_sq4, sc_coeffs* out,
            const int org[3] = nullptr) {
  Pending p{};
  // single calls: mesh / diameters events (level 1), every stage (2) or none (0)
  c->grid_div = c->o.grid_div_single;
  c->o.pack_tma = c->o.pack_tma_single;
  c->o.fbox = c->o.fbox_single;
  c->events_on = c->o.stage_times > 0;
  c->ev_full = c->o.stage_times > 1;
  int rc = start_roi(c, d_mask, nx, ny, nz, sp, s, shard, nshards, d_sq4, 0, &p, org);
  if (rc) return rc;
  return finish_roi(c, &p, out);
}

double wall_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

// Copy a host mask into the slot's staging buffer on stream s (events ev[0] /
// ev[1] bracket the copy).  With option "host_crop" (default on) the host first
// finds the occupied z/y slab (host_crop.h, all host threads) and only that
// slab crosses PCIe, as one 2-D copy of whole x rows; *cy / *cz / org then
// describe the slab (x is never cropped).  An all-background mask is reported
// here, before any device work, as the reference does (mesh.py:78-79).
// Host-read / PCIe balance of the host entries (per device, updated after
// every host-mask ROI): host scan rate, pinned H2D rate, occupied-slab fraction.
struct HostRates {
  std::mutex mu;
  double scan_bpms = 0.0, h2d_bpms = 0.0, slab_frac = 1.0;
  bool packed = false;  // the last host-mask ROI was packed on the host
};
HostRates& host_rates(int device) {
  static HostRates r[64];
  return r[device & 63];
}

// After a host-mask ROI: refresh the rates split_slices() balances.
void note_host_rates(const Ctx* c, int64_t total_bytes, double h2d_ms) {
  HostRates& r = host_rates(c->device);
  std::lock_guard<std::mutex> lk(r.mu);
  if (c->last_pure_scan_ms > 0.0 && c->last_scan_bytes > 0)
    r.scan_bpms = (double)c->last_scan_bytes / c->last_pure_scan_ms;
  r.packed = c->prepacked;
  if (!c->last_split && h2d_ms > 0.0 && c->last_h2d_bytes > (1 << 20))
    r.h2d_bpms = (double)c->last_h2d_bytes / h2d_ms;
  if (total_bytes > 0) r.slab_frac = (double)c->last_slab_bytes / (double)total_bytes;
}

// Leading slices [0, a) that go to the device whole, unscanned: the host scan
// (rate Rc) and the PCIe link (rate Rp) then read the mask concurrently.
// With s the slab fraction of the previous ROI, (1 - f)/Rc = (f + s)/Rp gives
// f = (Rp/Rc - s) / (1 + Rp/Rc); f = 0 when the slab alone already keeps PCIe
// busier than the scan (e.g. C3), and until both rates have been measured.
int64_t split_slices(const Ctx* c, int64_t nz) {
  const int device = c->device;
  const int pct = c->o.split;
  if (pct == 0 || nz < 8) return 0;
  double f;
  if (pct > 0) {
    f = pct / 100.0;
  } else {
    HostRates& r = host_rates(device);
    std::lock_guard<std::mutex> lk(r.mu);
    // (a slab big enough to be packed on the host makes the split pointless)
    if (r.scan_bpms <= 0.0 || r.h2d_bpms <= 0.0 || r.packed) return 0;
    const double k = r.h2d_bpms / r.scan_bpms;
    f = (k - r.slab_frac) / (1.0 + k);
  }
  if (f <= 0.0) return 0;
  return std::min<int64_t>(nz - 1, (int64_t)(f * (double)nz));
}

// Pack the occupied slab on the host (option host_pack: 1 always, 0 never, -1
// when the raw slab would keep PCIe busier than the host scan took, i.e. the
// link, not the host, would bound the ROI -- C3-like ROIs with large slabs).
bool pack_on_host(const Ctx* c, double slab_bytes, double scan_ms) {
  const int mode = c->o.host_pack;
  if (mode >= 0) return mode == 1;
  HostRates& r = host_rates(c->device);
  std::lock_guard<std::mutex> lk(r.mu);
  const double pcie_bpms = r.h2d_bpms > 0.0 ? r.h2d_bpms : 50e6;  // bytes per ms
  return slab_bytes / pcie_bpms > scan_ms;
}

int stage_host_mask(Ctx* c, const uint8_t* mask, int64_t nx, int64_t ny, int64_t nz,
                    cudaStream_t s, int64_t* cy, int64_t* cz, int org[3]) {
  org[0] = org[1] = org[2] = 0;
  c->last_scan_ms = c->last_pure_scan_ms = 0.0;
  *cy = ny;
  *cz = nz;
  const uint8_t* src = mask;
  const size_t S = (size_t)nx * ny;  // bytes per slice
  c->prepacked = false;
  const int64_t a = c->o.crop ? split_slices(c, nz) : 0;
  if (a > 0) {
    // Split read: slices [0, a) cross PCIe whole while the host scans [a, nz)
    // for its occupied slab; the device volume is slices [0, Z1] with every
    // row (rows outside the slab are zeroed on the device), origin 0.
    CK(cudaEventRecord(c->ev[0], s));
    CK(cudaMemcpyAsync(c->mask_stage.p, mask, a * S, cudaMemcpyHostToDevice, s));
    const double t0 = wall_ms();
    const Slab sl = occupied_slab(mask + a * S, nx, ny, nz - a, c->o.host_threads);
    c->last_scan_ms = c->last_pure_scan_ms = wall_ms() - t0;
    size_t bytes = a * S;
    int64_t Z1 = a - 1;
    if (!sl.empty) {
      const int64_t z0 = a + sl.z0;
      Z1 = a + sl.z1;
      const size_t width = (size_t)nx * (sl.y1 - sl.y0 + 1);
      CK(cudaMemsetAsync(c->mask_stage.p + a * S, 0, (Z1 - a + 1) * S, s));
      CK(cudaMemcpy2DAsync(c->mask_stage.p + z0 * S + sl.y0 * nx, S, mask + z0 * S + sl.y0 * nx,
                           S, width, (size_t)(Z1 - z0 + 1), cudaMemcpyHostToDevice, s));
      bytes += width * (Z1 - z0 + 1);
      c->last_slab_bytes = (long long)(width * (Z1 - z0 + 1));
    } else {
      c->last_slab_bytes = 0;
    }
    CK(cudaEventRecord(c->ev[1], s));
    *cz = Z1 + 1;
    c->last_h2d_bytes = (long long)bytes;
    c->last_scan_bytes = sl.bytes_read;
    c->last_split = true;
    return SC_OK;
  }
  c->last_split = false;
  if (c->o.crop) {
    const double t0 = wall_ms();
    const int th = c->o.host_threads;
    const Slab sl = occupied_slab(mask, nx, ny, nz, th);
    c->last_scan_ms = c->last_pure_scan_ms = wall_ms() - t0;
    c->last_scan_bytes = sl.bytes_read;
    if (sl.empty) {
      set_err("mask has no occupied voxels");
      return SC_ERR_EMPTY_ROI;
    }
    *cy = sl.y1 - sl.y0 + 1;
    *cz = sl.z1 - sl.z0 + 1;
    org[1] = (int)sl.y0;
    org[2] = (int)sl.z0;
    src = mask + (sl.z0 * ny + sl.y0) * nx;
    if (pack_on_host(c, (double)nx * *cy * *cz, c->last_scan_ms)) {
      // Host pack: the same host threads bit-pack the slab's rows into the
      // device bit-volume layout, and only the bits (1/8 of the slab) cross
      // PCIe, straight into the slot's bit volume; the ROI's graph then starts
      // at the bbox pass (no device pack).
      const double t1 = wall_ms();
      const size_t W = (size_t)((nx + 31) / 32), words = W * *cy * *cz;
      if (words > c->h_bits_cap) {
        if (c->h_bits) cudaFreeHost(c->h_bits);
        c->h_bits = nullptr;
        c->h_bits_cap = 0;
        CK(cudaMallocHost(&c->h_bits, sizeof(uint32_t) * (words + words / 4 + 1024)));
        c->h_bits_cap = words + words / 4 + 1024;
      }
      pack_slab(mask, nx, ny, sl.z0, sl.z1, sl.y0, sl.y1, c->h_bits, th);
      c->last_scan_ms += wall_ms() - t1;
      const unsigned long long fp0 = c->fingerprint();
      CK(c->bits.ensure(words));
      CK(c->segmap.ensure(c->bits.cap / 512 + 1));
      if (c->fingerprint() != fp0) {  // scratch moved: cached ROI graphs are stale
        c->gen++;
        c->drop_graphs();
      }
      CK(cudaEventRecord(c->ev[0], s));
      CK(cudaMemcpyAsync(c->bits.p, c->h_bits, sizeof(uint32_t) * words,
                         cudaMemcpyHostToDevice, s));
      CK(cudaEventRecord(c->ev[1], s));
      c->last_h2d_bytes = (long long)(sizeof(uint32_t) * words);
      c->last_slab_bytes = (long long)((size_t)nx * *cy * *cz);
      c->prepacked = true;
      return SC_OK;
    }
  }
  const size_t width = (size_t)nx * *cy;
  c->last_slab_bytes = (long long)(width * *cz);
  CK(cudaEventRecord(c->ev[0], s));
  if (*cy == ny)
    CK(cudaMemcpyAsync(c->mask_stage.p, src, width * *cz, cudaMemcpyHostToDevice, s));
  else
    CK(cudaMemcpy2DAsync(c->mask_stage.p, width, src, (size_t)nx * ny, width, (size_t)*cz,
                         cudaMemcpyHostToDevice, s));
  CK(cudaEventRecord(c->ev[1], s));
  c->last_h2d_bytes = (long long)(width * *cz);
  return SC_OK;
}

// Typed NPY payload -> the slot's uint8 mask stage (sc_calculate_coefficients_raw*):
// host scan for the occupied slab over the payload's two slowest axes, then
// the slab in chunks of whole planes through two pinned staging halves (the
// host copies chunk k+1 while chunk k's DMA runs; a pinned payload is copied
// directly), each chunk binarized on the device right behind its copy.  The
// mask stage then holds the slab in C order with dims (*cx, *cy, *cz) and
// origin org in the payload's grid.
int stage_host_raw(Ctx* c, const sc_raw_mask& m, cudaStream_t s, int64_t* cx, int64_t* cy,
                   int64_t* cz, int org[3]) {
  static const int itemsize[7] = {1, 1, 2, 4, 8, 4, 8};
  const int isz = itemsize[m.dtype];
  const int64_t nz = m.shape[0], ny = m.shape[1], nx = m.shape[2];
  const bool F = m.fortran_order != 0;
  const int64_t planes = F ? nx : nz, rows = ny, row_elems = F ? nz : nx;
  const int64_t row_bytes = row_elems * isz;
  int64_t p0 = 0, p1 = planes - 1, r0 = 0, r1 = rows - 1;
  c->prepacked = false;
  c->last_split = false;
  c->last_scan_ms = c->last_pure_scan_ms = 0.0;
  c->last_scan_bytes = 0;
  if (c->o.crop) {
    const double t0 = wall_ms();
    const Slab sl = occupied_slab_typed(m.data, m.dtype, row_elems, rows, planes, m.has_label,
                                        m.label_int, m.label_float, c->o.host_threads);
    c->last_scan_ms = c->last_pure_scan_ms = wall_ms() - t0;
    c->last_scan_bytes = sl.bytes_read;
    if (sl.empty) {
      set_err("mask has no occupied voxels");
      return SC_ERR_EMPTY_ROI;
    }
    p0 = sl.z0; p1 = sl.z1; r0 = sl.y0; r1 = sl.y1;
    if (F && nx % 32 == 0) {  // keep x 32-aligned: the slab stays on the 128-bit pack path
      p0 &= ~(int64_t)31;
      p1 = std::min(planes - 1, ((p1 + 32) & ~(int64_t)31) - 1);
    }
  }
  const int64_t np = p1 - p0 + 1, nr = r1 - r0 + 1;
  const int64_t width = nr * row_bytes, pitch = rows * row_bytes;  // slab / payload plane bytes
  const uint8_t* src = static_cast<const uint8_t*>(m.data) + p0 * pitch + r0 * row_bytes;
  if (!F) {
    *cx = nx; *cy = nr; *cz = np;
    org[0] = 0; org[1] = (int)r0; org[2] = (int)p0;
  } else {
    *cx = np; *cy = nr; *cz = nz;
    org[0] = (int)p0; org[1] = (int)r0; org[2] = 0;
  }
  CK(c->mask_stage.ensure((size_t)(np * nr * row_elems)));
  const int64_t kChunkBytes = 4LL << 20;
  const int64_t per = std::max<int64_t>(1, kChunkBytes / std::max<int64_t>(1, width));
  const int64_t chunk = per * width;
  CK(c->raw_stage.ensure((size_t)(2 * chunk)));
  cudaPointerAttributes attr{};
  const bool pinned = cudaPointerGetAttributes(&attr, m.data) == cudaSuccess &&
                      attr.type == cudaMemoryTypeHost;
  (void)cudaGetLastError();  // pageable memory may report an error on older drivers
  if (!pinned && (size_t)(2 * chunk) > c->h_raw_cap) {
    if (c->h_raw) CK(cudaFreeHost(c->h_raw));
    c->h_raw = nullptr;
    c->h_raw_cap = 0;
    CK(cudaMallocHost(&c->h_raw, (size_t)(2 * chunk)));
    c->h_raw_cap = (size_t)(2 * chunk);
  }
  CK(cudaEventRecord(c->ev[0], s));
  int64_t idx = 0;
  for (int64_t a = 0; a < np; a += per, idx++) {
    const int64_t b = std::min(np, a + per), bytes = (b - a) * width;
    uint8_t* dev = c->raw_stage.p + (idx & 1) * chunk;  // reused in stream order
    if (pinned) {
      CK(cudaMemcpy2DAsync(dev, (size_t)width, src + a * pitch, (size_t)pitch, (size_t)width,
                           (size_t)(b - a), cudaMemcpyHostToDevice, s));
    } else {
      uint8_t* hb = c->h_raw + (idx & 1) * chunk;
      if (idx >= 2) CK(cudaEventSynchronize(c->cev[idx & 1]));  // its previous DMA is done
      copy_rows(hb, src + a * pitch, pitch, width, b - a, c->o.host_threads);
      CK(cudaMemcpyAsync(dev, hb, (size_t)bytes, cudaMemcpyHostToDevice, s));
      CK(cudaEventRecord(c->cev[idx & 1], s));
    }
    const int rc = F ? launch_binarize(dev, m.dtype, 1, b - a, nr, row_elems, (int)np, (int)a,
                                       m.has_label, m.label_int, m.label_float,
                                       c->mask_stage.p, c->sms * 4, s)
                     : launch_binarize(dev, m.dtype, 0, b - a, nr, row_elems, 0, 0, m.has_label,
                                       m.label_int, m.label_float,
                                       c->mask_stage.p + a * nr * row_elems, c->sms * 4, s);
    if (rc) {
      set_err("unsupported element type code %d", m.dtype);
      return SC_ERR_INPUT;
    }
    CKL(1);
  }
  CK(cudaEventRecord(c->ev[1], s));
  c->last_h2d_bytes = np * width;
  c->last_slab_bytes = np * width;
  return SC_OK;
}

int check_raw(const sc_raw_mask& m) {
  if (m.dtype < 0 || m.dtype > 6) {
    set_err("unsupported element type code %d", m.dtype);
    return SC_ERR_INPUT;
  }
  if (!m.data) {
    set_err("payload pointer is NULL");
    return SC_ERR_INPUT;
  }
  return SC_OK;
}

// Pipelined batch over the slots of `device` (option "slots", default 8): ROI i+1 is enqueued (H2D copy
// included for host masks) before ROI i is collected, so copies, kernels and
// the host round trip of neighbouring ROIs overlap.  The first failing ROI's
// code is returned; every other ROI is still processed.
int run_batch(int device, const uint8_t* const* masks, const int64_t* dims,
              const double* spacings, int64_t count, bool host, sc_coeffs* out,
              cudaStream_t user, const sc_raw_mask* raws = nullptr) {
  if (count < 0 || (count > 0 && (!masks || !dims || !spacings || !out))) {
    set_err("bad batch arguments");
    return SC_ERR_INPUT;
  }
  if (count == 0) return SC_OK;
  const Opts opts = snapshot_opts();  // one snapshot for the whole batch
  const int nslots = std::max(1, std::min<int>(kSlots, opts.slots));
  Ctx* cs[kSlots] = {};
  for (int k = 0; k < nslots; k++) {
    int rc = get_ctx(device, &cs[k], k);
    if (rc) return rc;
  }
  std::unique_lock<std::mutex> locks[kSlots];
  for (int k = 0; k < nslots; k++) locks[k] = std::unique_lock<std::mutex>(cs[k]->mu);
  // Batch graphs carry no per-stage event nodes unless asked for (fewer graph
  // nodes = cheaper launches); the slots go back to single-call mode after.
  struct EventsMode {
    Ctx** cs; int n;
    ~EventsMode() {
      for (int k = 0; k < n; k++) {
        cs[k]->events_on = cs[k]->ev_full = true;
        cs[k]->chain_wait = nullptr;
      }
    }
  } events_mode{cs, nslots};
  for (int k = 0; k < nslots; k++) {
    cs[k]->o = opts;
    cs[k]->events_on = cs[k]->ev_full = opts.batch_times;
    cs[k]->grid_div = opts.grid_div;
    // slots are used round-robin: slot k's ROI follows slot k - pack_chain's
    cs[k]->chain_wait = (opts.pack_chain > 0 && opts.pack_chain < nslots)
                            ? cs[(k - opts.pack_chain + nslots) % nslots]->pack_ev : nullptr;
  }
  CK(cudaSetDevice(device));
  // Device masks: order the batch after prior work on the caller's stream;
  // NULL is the legacy default stream (the slot streams are non-blocking).
  if (!host && !user) user = cudaStreamLegacy;
  if (user) {
    CK(cudaEventRecord(cs[0]->ev[4], user));
    for (int k = 0; k < nslots; k++) CK(cudaStreamWaitEvent(cs[k]->stream, cs[0]->ev[4], 0));
  }
  // Size every slot for the largest ROI of the batch up front: growing a
  // buffer mid-batch would synchronise the device and drop the slot's graphs.
  {
    int64_t mx = 0, my = 0, mz = 0, mb = 0;
    for (int64_t i = 0; i < count; i++) {
      const int64_t nx = dims[3 * i], ny = dims[3 * i + 1], nz = dims[3 * i + 2];
      if (nx <= 0 || ny <= 0 || nz <= 0) continue;
      mx = std::max(mx, nx); my = std::max(my, ny); mz = std::max(mz, nz);
      mb = std::max(mb, nx * ny * nz);
    }
    if (mb > 0)
      for (int k = 0; k < nslots; k++) {
        Ctx* c = cs[k];
        const unsigned long long fp0 = c->fingerprint();
        const long long cap = vertex_capacity(mx, my, mz, c->cap_floor);
        const long long dcap =
            std::min<long long>(cap, std::max<long long>(c->o.dcap, c->dcap_floor));
        int rc = ensure_buffers(c, mx, my, mz, cap, dcap, 0, c->wcap_floor);
        if (rc) return rc;
        if (c->fingerprint() != fp0) {
          c->gen++;
          c->drop_graphs();
        }
        if (host) CK(c->mask_stage.ensure((size_t)mb));
      }
  }
  Pending pend[kSlots] = {};
  int64_t idx[kSlots];
  double t_start[kSlots];
  for (int k = 0; k < kSlots; k++) { idx[k] = -1; t_start[k] = 0.0; }
  int first = SC_OK;
  std::string first_err;
  auto note = [&](int rc) {
    if (rc && first == SC_OK) { first = rc; first_err = g_err; }
  };
  auto collect = [&](int k) {
    if (idx[k] < 0) return;
    Ctx* c = cs[k];
    sc_coeffs* o = &out[idx[k]];
    note(finish_roi(c, &pend[k], o));
    if (host) {
      o->h2d_ms = ev_ms(c->ev[0], c->ev[1]);
      o->h2d_bytes = c->last_h2d_bytes;
      o->host_scan_ms = c->last_scan_ms;
      c->last_ms[6] = o->h2d_ms;
      const int64_t j = idx[k];
      if (!raws)  // (typed payloads do not feed the uint8 split-read balance)
        note_host_rates(c, dims[3 * j] * dims[3 * j + 1] * dims[3 * j + 2], o->h2d_ms);
    }
    o->total_ms = wall_ms() - t_start[k];
    idx[k] = -1;
  };
  // Every exit path (an early CK return included) collects the ROIs still in
  // flight before the slot locks are released: their out[] entries get
  // written and no slot's pinned RoiParams is rewritten under a running ROI.
  struct DrainGuard {
    std::function<void()> f;
    ~DrainGuard() { f(); }
  } drain{[&] {
    for (int64_t i = 0; i < nslots; i++) collect((int)((count + i) % nslots));
  }};
  for (int64_t i = 0; i < count; i++) {
    const int k = (int)(i % nslots);
    collect(k);
    std::memset(&out[i], 0, sizeof out[i]);
    const int64_t nx = dims[3 * i], ny = dims[3 * i + 1], nz = dims[3 * i + 2];
    const double* sp = spacings + 3 * i;
    int rc = check_input(masks[i], nx, ny, nz, sp);
    if (rc) { note(rc); continue; }
    Ctx* c = cs[k];
    cudaStream_t s = c->stream;
    t_start[k] = wall_ms();
    const uint8_t* dm = masks[i];
    int64_t cx = nx, cy = ny, cz = nz;
    int org[3] = {0, 0, 0};
    if (raws) {
      if ((rc = check_raw(raws[i])) || (rc = stage_host_raw(c, raws[i], s, &cx, &cy, &cz, org))) {
        note(rc);
        continue;
      }
      dm = c->mask_stage.p;
    } else if (host) {
      CK(c->mask_stage.ensure((size_t)nx * ny * nz));
      rc = stage_host_mask(c, masks[i], nx, ny, nz, s, &cy, &cz, org);
      if (rc) { note(rc); continue; }
      dm = c->mask_stage.p;
    } else {
      c->prepacked = false;
    }
    pend[k] = Pending{};
    const double ts = host_prof_on() ? wall_ms() : 0.0;
    rc = start_roi(c, dm, cx, cy, cz, sp, s, 0, 1, nullptr, 0, &pend[k], org);
    if (host_prof_on()) g_hprof.start += wall_ms() - ts;
    if (rc) { note(rc); continue; }
    idx[k] = i;
  }
  drain.f();
  if (user) {  // ... and later work on it after the batch
    for (int k = 0; k < nslots; k++) {
      CK(cudaEventRecord(cs[k]->ev[5], cs[k]->stream));
      CK(cudaStreamWaitEvent(user, cs[k]->ev[5], 0));
    }
  }
  if (first) g_err = first_err;
  if (trace_on()) trace_print();
  if (host_prof_on() && g_hprof.n) {
    const double n = (double)g_hprof.n;
    std::fprintf(stderr,
                 "[sc host] %lld ROIs: per ROI sync-wait %.1f us, finish %.1f us, start %.1f us "
                 "(RoiParams copy %.1f us, graph launch %.1f us)\n",
                 g_hprof.n, 1e3 * g_hprof.sync / n, 1e3 * g_hprof.finish / n,
                 1e3 * g_hprof.start / n, 1e3 * g_hprof.copy / n, 1e3 * g_hprof.launch / n);
    g_hprof = HostProf{};
  }
  return first;
}

// Exclusive scan in place of n uint32 counts (3 kernels); returns the total.
int device_exscan(Ctx* c, unsigned int* data, long long n, cudaStream_t s,
                  unsigned long long* d_total) {
  const long long nb = (n + 1023) / 1024;
  unsigned int* sums = nullptr;
  CK(cudaMallocAsync(&sums, sizeof(unsigned int) * std::max<long long>(1, nb), s));
  scan_blocks<<<(unsigned)std::max<long long>(1, nb), 1024, 0, s>>>(data, n, sums);
  CKL(1);
  scan_sums<<<1, 1024, 0, s>>>(sums, (int)nb, d_total);
  CKL(1);
  scan_add<<<(unsigned)std::max<long long>(1, (n + 255) / 256), 256, 0, s>>>(data, n, sums);
  CKL(1);
  CK(cudaFreeAsync(sums, s));
  return SC_OK;
}

template <typename T>
struct Tmp {  // call-scoped device allocation (export path only)
  T* p = nullptr;
  ~Tmp() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, sizeof(T) * std::max<size_t>(1, n)); }
};

// Canonical TriangleMesh of a device mask (mesh.cu).  Fills the caller's
// buffers only when they are large enough; *nv / *nt always get the counts.
int run_mesh(Ctx* c, const uint8_t* d_mask, int64_t nx, int64_t ny, int64_t nz,
             const double sp[3], cudaStream_t s, double* xs, double* ys, double* zs,
             int32_t* tris, int64_t vcap, int64_t tcap, int64_t* nv, int64_t* nt) {
  long long cap = vertex_capacity(nx, ny, nz, c->cap_floor);
  for (int attempt = 0; attempt < 2; attempt++) {
    const unsigned long long fp0 = c->fingerprint();
    CK(c->bits.ensure((size_t)(((nx + 31) / 32) * ny * nz)));
    CK(c->segmap.ensure(c->bits.cap / 512 + 1));
    CK(c->keys.ensure((size_t)cap));
    if (c->fingerprint() != fp0) {  // scratch moved: cached ROI graphs are stale
      c->gen++;
      c->drop_graphs();
    }
    RoiParams& h = *c->h_rp;
    h.mask = d_mask; h.nx = nx; h.ny = ny; h.nz = nz;
    h.W = (int)((nx + 31) / 32);
    h.n_words = (long long)h.W * ny * nz;
    h.n_chunks = nx * ny * nz / 16;
    h.f.cx2 = h.f.cy2 = h.f.cz2 = 0;
    h.f.hx = (float)(0.5 * sp[0]); h.f.hy = (float)(0.5 * sp[1]); h.f.hz = (float)(0.5 * sp[2]);
    h.f.sx = sp[0]; h.f.sy = sp[1]; h.f.sz = sp[2];
    h.f.ox2 = h.f.oy2 = h.f.oz2 = 0;
    h.sparse = 0;  // the export kernels read every bit-volume word
    h.mc_slab = 0;
    h.wcap = 0;
    CK(cudaMemcpyAsync(c->d_rp, c->h_rp, sizeof(RoiParams), cudaMemcpyHostToDevice, s));
    init_stats<<<1, 256, 0, s>>>(c->d_stats, c->segmap.p, 0LL, nullptr, c->d_rp);
    CKL(1);
    if (nx % 32 == 0 && (reinterpret_cast<uintptr_t>(d_mask) & 15) == 0) {
      pack_bits_v16<4, true><<<c->sms * std::max(1, c->occ_pack), 256, 0, s>>>(
          c->d_rp, c->bits.p, c->d_stats, c->segmap.p);
      CKL(1);
    } else {
      pack_bits_generic<<<c->sms * 8, 256, 0, s>>>(c->d_rp, c->bits.p, c->d_stats, c->segmap.p);
      CKL(1);
    }
    mc_cells<<<c->sms * std::max(1, c->occ_mc), 256, 0, s>>>(c->d_rp, c->bits.p, c->d_tabs,
                                                            c->d_stats, c->keys.p,
                                                            (long long)c->keys.cap, nullptr,
                                                            nullptr, c->segmap.p);
    CKL(1);
    CK(cudaMemcpyAsync(c->h_stats, c->d_stats, sizeof(Stats), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if ((long long)c->h_stats->n_vert <= (long long)c->keys.cap) break;
    cap = (long long)c->h_stats->n_vert;
    c->cap_floor = std::max(c->cap_floor, cap);
  }
  const Stats hs = *c->h_stats;
  if (hs.bbox[3] < 0) { set_err("mask has no occupied voxels"); return SC_ERR_EMPTY_ROI; }
  const long long V = (long long)hs.n_vert;
  const int* bb = hs.bbox;
  const long long nq = ((bb[3] + 1) >> 5) - (bb[0] >> 5) + 1, nvr = bb[4] - bb[1] + 2,
                  nwr = bb[5] - bb[2] + 2, items = nq * nvr * nwr;
  Tmp<unsigned int> offs;
  Tmp<unsigned long long> total;
  CK(offs.alloc(items));
  CK(total.alloc(1));
  mesh_count<<<c->sms * 8, 256, 0, s>>>(c->d_rp, c->bits.p, c->d_stats, offs.p);
  CKL(1);
  int rc = device_exscan(c, offs.p, items, s, total.p);
  if (rc) return rc;
  unsigned long long T = 0;
  CK(cudaMemcpyAsync(&T, total.p, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *nv = V;
  *nt = (int64_t)T;
  if (V > vcap || (long long)T > tcap || !xs || !ys || !zs || !tris) return SC_OK;
  const long long mx = bb[3] - bb[0] + 2, my = bb[4] - bb[1] + 2, mz = bb[5] - bb[2] + 2;
  Tmp<int> emap, ids;
  Tmp<int3> ttmp;
  Tmp<unsigned int> first, flags;
  Tmp<double> dx, dy, dz;
  Tmp<int> dtris;
  CK(emap.alloc((size_t)(3 * mx * my * mz)));
  CK(ids.alloc((size_t)V));
  CK(ttmp.alloc((size_t)T));
  CK(first.alloc((size_t)V));
  CK(flags.alloc((size_t)(3 * T)));
  CK(dx.alloc((size_t)V)); CK(dy.alloc((size_t)V)); CK(dz.alloc((size_t)V));
  CK(dtris.alloc((size_t)(3 * T)));
  CK(cudaMemsetAsync(first.p, 0xFF, sizeof(unsigned int) * V, s));
  CK(cudaMemsetAsync(flags.p, 0, sizeof(unsigned int) * 3 * T, s));
  const int g = c->sms * 8;
  edge_map_fill<<<g, 256, 0, s>>>(c->keys.p, c->d_stats, emap.p);
  CKL(1);
  mesh_emit<<<g, 256, 0, s>>>(c->d_rp, c->bits.p, c->d_stats, offs.p, emap.p, ttmp.p, first.p);
  CKL(1);
  id_flags<<<g, 256, 0, s>>>(first.p, V, flags.p);
  CKL(1);
  if ((rc = device_exscan(c, flags.p, 3 * (long long)T, s, total.p))) return rc;
  mesh_out<<<g, 256, 0, s>>>(c->keys.p, first.p, flags.p, V, sp[0], sp[1], sp[2], dx.p, dy.p,
                             dz.p, ids.p);
  CKL(1);
  tris_out<<<g, 256, 0, s>>>(ttmp.p, (long long)T, ids.p, dtris.p);
  CKL(1);
  CK(cudaMemcpyAsync(xs, dx.p, sizeof(double) * V, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(ys, dy.p, sizeof(double) * V, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(zs, dz.p, sizeof(double) * V, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(tris, dtris.p, sizeof(int) * 3 * T, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return SC_OK;
}

int current_ctx(Ctx** c) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  return get_ctx(dev, c);
}

// One option into `o` (sc_set_option / sc_set_thread_option).
int set_opt(Opts& o, const char* name, int value) {
  if (!name) { set_err("NULL option name"); return SC_ERR_INPUT; }
  if (std::strcmp(name, "prune") == 0) o.prune = value != 0;
  else if (std::strcmp(name, "pass1_packed") == 0) o.packed = value != 0;
  else if (std::strcmp(name, "graphs") == 0) o.graphs = value != 0;
  else if (std::strcmp(name, "slots") == 0) o.slots = std::max(1, std::min(kSlots, value));
  else if (std::strcmp(name, "dcap") == 0) o.dcap = std::max(256, value);
  else if (std::strcmp(name, "wcap") == 0) o.wcap = std::max(1, value);
  else if (std::strcmp(name, "fused_bbox") == 0) o.fbox = value != 0;
  else if (std::strcmp(name, "fused_bbox_single") == 0) o.fbox_single = value != 0;
  else if (std::strcmp(name, "host_crop") == 0) o.crop = value != 0;
  else if (std::strcmp(name, "host_pack") == 0) o.host_pack = std::max(-1, std::min(1, value));
  else if (std::strcmp(name, "host_split") == 0) o.split = std::max(-1, std::min(90, value));
  else if (std::strcmp(name, "pack_mode") == 0) o.pack_mode = value & 7;
  else if (std::strcmp(name, "pack_bps") == 0) o.pack_bps = std::max(0, std::min(63, value));
  else if (std::strcmp(name, "grid_div") == 0) o.grid_div = std::max(1, value);
  else if (std::strcmp(name, "grid_div_single") == 0) o.grid_div_single = std::max(1, value);
  else if (std::strcmp(name, "pdl") == 0) o.pdl = value != 0;
  else if (std::strcmp(name, "fork") == 0) o.fork = value != 0;
  else if (std::strcmp(name, "zero_copy") == 0) o.zc = value != 0;
  else if (std::strcmp(name, "stage_times") == 0) o.stage_times = std::max(0, std::min(2, value));
  else if (std::strcmp(name, "pack_tma") == 0) o.pack_tma = std::max(0, std::min(8, value));
  else if (std::strcmp(name, "pack_chain") == 0) o.pack_chain = std::max(0, std::min(8, value));
  else if (std::strcmp(name, "pack_tma_single") == 0) o.pack_tma_single = std::max(0, std::min(8, value));
  else if (std::strcmp(name, "sparse_bits") == 0) o.sparse = value != 0;
  else if (std::strcmp(name, "pack_skip") == 0) o.pack_skip = value != 0;
  else if (std::strcmp(name, "batch_stage_times") == 0) o.batch_times = value != 0;
  else if (std::strcmp(name, "host_threads") == 0) o.host_threads = std::max(1, value);
  else if (std::strcmp(name, "debug_empty") == 0) o.empty = std::max(0, value);
  else if (std::strcmp(name, "pack_prio") == 0) o.pack_prio = value != 0;
  else if (std::strcmp(name, "pack_tile") == 0) o.pack_tile = (value == 8 || value == 32) ? value : 16;
  else if (std::strcmp(name, "pack_threads") == 0)
    o.pack_threads = (value == 64 || value == 128) ? value : 256;
  else if (std::strcmp(name, "pack_stages") == 0) o.pack_stages = std::max(2, std::min(8, value));
  else if (std::strcmp(name, "debug_stages") == 0) o.stages = value > 0 ? value : (1 << 30);
  else { set_err("unknown option %s", name); return SC_ERR_INPUT; }
  return SC_OK;
}

}  // namespace

extern "C" {

const char* sc_last_error(void) { return g_err.c_str(); }
int sc_abi_version(void) { return SC_ABI_VERSION; }

int sc_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int sc_calculate_coefficients_device(const uint8_t* d_mask, int64_t nx, int64_t ny, int64_t nz,
                                     const double spacing[3], void* stream, sc_coeffs* out) {
  return sc_calculate_coefficients_shard(d_mask, nx, ny, nz, spacing, stream, 0, 1, nullptr, out);
}

int sc_calculate_coefficients_shard(const uint8_t* d_mask, int64_t nx, int64_t ny, int64_t nz,
                                    const double spacing[3], void* stream, int shard,
                                    int nshards, double* d_sq4, sc_coeffs* out) {
  const double t0 = wall_ms();
  int rc = check_input(d_mask, nx, ny, nz, spacing);
  if (rc) return rc;
  if (!out || nshards < 1 || shard < 0 || shard >= nshards) {
    set_err("bad output pointer or shard %d of %d", shard, nshards);
    return SC_ERR_INPUT;
  }
  Ctx* c;
  if ((rc = current_ctx(&c))) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  c->o = snapshot_opts();
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  if (!stream) {
    // NULL = the legacy default stream (also torch's default stream): the
    // slot stream is non-blocking, so order the ROI after prior work on it
    // explicitly (the call is synchronous, so later work is ordered anyway).
    CK(cudaEventRecord(c->ev[4], cudaStreamLegacy));
    CK(cudaStreamWaitEvent(s, c->ev[4], 0));
  }
  std::memset(out, 0, sizeof *out);
  c->prepacked = false;
  rc = run_roi(c, d_mask, nx, ny, nz, spacing, s, shard, nshards, d_sq4, out);
  out->total_ms = wall_ms() - t0;
  return rc;
}

// ---- two-phase (slab-split) shard entry -------------------------------------
//
// Phase 1 (sc_shard_mesh): the pack (replicated: every rank gets the global
// bbox, which fixes the brick / plane binning and the pass-1 frame) and
// marching cubes over the shard's share of the cell layers only.  Its exact
// integer partials -- case histogram, volume sum, vertex count, brick and
// plane-bin histograms -- go to an int64 "sums" vector the caller all-reduces
// (SUM), its vertex keys to a buffer the caller all-gathers.  Phase 2
// (sc_shard_diameters) loads the summed histograms and the gathered keys into
// the slot and runs the diameter half with identity ownership, so the
// marching-cubes work as well as the pair grid falls with the shard count.
// Layout of the sums vector (int64): [0, 256) case histogram, 256 vol_k,
// 257 n_vert, then kSortBins + kSortSupers brick counts, then P x kPlaneBins
// plane-bin counts (P = 2 (nx + ny + nz) + 9, the host bound of the plane space).
constexpr long long kSumHist = 0, kSumVol = 256, kSumVert = 257, kSumSort = 258;
constexpr long long kSumPlane = kSumSort + kSortBins + kSortSupers;

long long shard_sums_len(int64_t nx, int64_t ny, int64_t nz) {
  return kSumPlane + (2 * (nx + ny + nz) + 9) * kPlaneBinsHost;
}

// Phase 1 export: partials -> sums (and zero the slot's histograms, which no
// scan_all consumed this time).
__global__ void shard_export(const Stats* __restrict__ st, unsigned int* __restrict__ sort_counts,
                             unsigned int* __restrict__ pbin_counts, long long n_pbin,
                             long long* __restrict__ sums) {
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long step = (long long)gridDim.x * blockDim.x;
  for (long long i = t0; i < kNumCases; i += step) {
    unsigned long long h = 0;
    for (int c = 0; c < kHistCopies; c++) h += st->hist[c][i];
    sums[kSumHist + i] = (long long)h;
  }
  if (t0 == 0) {
    sums[kSumVol] = st->vol_k;
    sums[kSumVert] = (long long)st->n_vert;
  }
  for (long long i = t0; i < kSortBins + kSortSupers; i += step) {
    sums[kSumSort + i] = sort_counts[i];
    sort_counts[i] = 0u;
  }
  for (long long i = t0; i < n_pbin; i += step) {
    sums[kSumPlane + i] = pbin_counts[i];
    pbin_counts[i] = 0u;
  }
}

// Phase 2 import (after init_stats): the global bbox and the summed partials.
// A summed vertex count that differs from the gathered key count is refused
// here, on the device (no host round trip before the run): the record is
// flagged, and with no histograms loaded the pipeline has nothing to do.
__global__ void shard_import(Stats* __restrict__ st, int4 bb_lo, int4 bb_hi,
                             unsigned int* __restrict__ sort_counts,
                             unsigned int* __restrict__ pbin_counts, long long n_pbin,
                             const long long* __restrict__ sums, long long n_keys) {
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long step = (long long)gridDim.x * blockDim.x;
  const bool ok = sums[kSumVert] == n_keys;
  if (t0 == 0) {
    st->bbox[0] = bb_lo.x; st->bbox[1] = bb_lo.y; st->bbox[2] = bb_lo.z;
    st->bbox[3] = bb_hi.x; st->bbox[4] = bb_hi.y; st->bbox[5] = bb_hi.z;
    st->vol_k = sums[kSumVol];
    st->n_vert = ok ? (unsigned long long)n_keys : 0ull;
    st->bad_input = ok ? 0u : 1u;
  }
  if (!ok) return;  // (the slot's histograms stay zero)
  for (long long i = t0; i < kNumCases; i += step) st->hist[0][i] = (unsigned long long)sums[kSumHist + i];
  for (long long i = t0; i < kSortBins + kSortSupers; i += step)
    sort_counts[i] = (unsigned int)sums[kSumSort + i];
  for (long long i = t0; i < n_pbin; i += step)
    pbin_counts[i] = (unsigned int)sums[kSumPlane + i];
}

// Phase 1: the shard's vertex keys to the caller's buffer, sized on the device
// (no host round trip for the count); at most `room` keys.
__global__ void shard_copy_keys(const int4* __restrict__ src, int4* __restrict__ dst,
                                const Stats* __restrict__ st, long long room) {
  const long long n = min((long long)st->n_vert, room);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int sc_shard_exchange_sizes(int64_t nx, int64_t ny, int64_t nz, int64_t* n_sums,
                            int64_t* key_cap) {
  if (nx <= 0 || ny <= 0 || nz <= 0 || !n_sums || !key_cap) {
    set_err("bad dims or NULL output");
    return SC_ERR_INPUT;
  }
  *n_sums = shard_sums_len(nx, ny, nz);
  *key_cap = vertex_capacity(nx, ny, nz, 0);
  return SC_OK;
}

namespace {
// Per-call state of a two-phase entry: no graphs (one-off pipeline cuts), the
// Stats record copied back explicitly, single-call launch shapes.
void two_phase_opts(Ctx* c) {
  c->o = snapshot_opts();
  c->o.graphs = 0;
  c->o.zc = 0;
  c->grid_div = c->o.grid_div_single;
  c->o.pack_tma = c->o.pack_tma_single;
  c->o.fbox = c->o.fbox_single;
  c->events_on = c->o.stage_times > 0;
  c->ev_full = c->o.stage_times > 1;
  c->prepacked = false;
}
cudaStream_t order_after_legacy(Ctx* c, void* stream) {
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  if (!stream) {
    cudaEventRecord(c->ev[4], cudaStreamLegacy);
    cudaStreamWaitEvent(s, c->ev[4], 0);
  }
  return s;
}
}  // namespace

int sc_shard_mesh(const uint8_t* d_mask, int64_t nx, int64_t ny, int64_t nz,
                  const double spacing[3], void* stream, int shard, int nshards,
                  int64_t* d_sums, int32_t* d_keys, int64_t key_cap, int64_t* n_keys,
                  int32_t bbox[6]) {
  int rc = check_input(d_mask, nx, ny, nz, spacing);
  if (rc) return rc;
  if (!d_sums || !d_keys || !n_keys || !bbox || nshards < 1 || nshards > 0x7fff || shard < 0 ||
      shard >= nshards) {
    set_err("NULL buffer or bad shard %d of %d", shard, nshards);
    return SC_ERR_INPUT;
  }
  Ctx* c;
  if ((rc = current_ctx(&c))) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  two_phase_opts(c);
  cudaStream_t s = order_after_legacy(c, stream);
  struct Reset {  // the slot's next ROI is a plain one again, whatever happens
    Ctx* c;
    ~Reset() { c->mc_slab = 0; c->mesh_only = false; }
  } reset{c};
  Pending p{};
  const long long n_pbin = (2 * (nx + ny + nz) + 9) * kPlaneBinsHost;
  for (int attempt = 0; attempt < 2; attempt++) {
    c->mc_slab = (nshards << 16) | shard;
    c->mesh_only = true;
    if ((rc = start_roi(c, d_mask, nx, ny, nz, spacing, s, 0, 1, nullptr, 0, &p))) return rc;
    // export and key copy enqueued behind the mesh: one synchronisation per call
    shard_export<<<c->sms * 2, 256, 0, s>>>(c->d_stats, c->sort_counts.p, c->pbin_counts.p,
                                            n_pbin, reinterpret_cast<long long*>(d_sums));
    CKL(1);
    shard_copy_keys<<<c->sms * 4, 256, 0, s>>>(
        c->keys.p, reinterpret_cast<int4*>(d_keys), c->d_stats,
        std::min<long long>((long long)key_cap, (long long)c->keys.cap));
    CKL(1);
    CK(cudaStreamSynchronize(s));
    const long long V = (long long)c->h_stats->n_vert;
    if (V <= (long long)c->keys.cap) break;
    if (attempt) { set_err("vertex buffer overflow"); return SC_ERR_NOMEM; }
    p.cap = V;  // exact re-run (raises the slot's floors)
    p.dcap = std::max(p.dcap, V);
  }
  const Stats& h = *c->h_stats;
  for (int i = 0; i < 6; i++) bbox[i] = h.bbox[i];
  const long long V = (long long)h.n_vert;
  *n_keys = V;
  if (h.bbox[3] < 0) {
    set_err("mask has no occupied voxels");
    return SC_ERR_EMPTY_ROI;
  }
  if (V > key_cap) {
    set_err("key buffer holds %lld keys, the shard has %lld", (long long)key_cap, V);
    return SC_ERR_NOMEM;
  }
  return SC_OK;
}

int sc_shard_diameters(const int64_t* d_sums, const int32_t* d_keys, int64_t n_keys, int64_t nx,
                       int64_t ny, int64_t nz, const int32_t bbox[6], const double spacing[3],
                       void* stream, int shard, int nshards, double* d_sq4, sc_coeffs* out) {
  const double t0 = wall_ms();
  if (!d_sums || (!d_keys && n_keys) || n_keys < 0 || !bbox || !spacing || !out || nshards < 1 ||
      shard < 0 || shard >= nshards || nx <= 0 || ny <= 0 || nz <= 0) {
    set_err("bad input to sc_shard_diameters");
    return SC_ERR_INPUT;
  }
  for (int i = 0; i < 3; i++)
    if (!(spacing[i] > 0.0) || !std::isfinite(spacing[i])) {
      set_err("spacing must be positive and finite");
      return SC_ERR_INPUT;
    }
  if (bbox[3] < 0) {
    set_err("mask has no occupied voxels");
    return SC_ERR_EMPTY_ROI;
  }
  Ctx* c;
  int rc;
  if ((rc = current_ctx(&c))) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  two_phase_opts(c);
  cudaStream_t s = order_after_legacy(c, stream);
  std::memset(out, 0, sizeof *out);
  // (the summed vertex count must be the gathered key count: shard_import
  // checks it on the device)
  long long punits = 0;
  const long long n_pbin = (2 * (nx + ny + nz) + 9) * kPlaneBinsHost;
  const int4 lo = make_int4(bbox[0], bbox[1], bbox[2], 0), hi = make_int4(bbox[3], bbox[4], bbox[5], 0);
  for (int attempt = 0; attempt < 2; attempt++) {
    const long long cap = std::max<long long>(vertex_capacity(nx, ny, nz, c->cap_floor), n_keys);
    const long long dcap =
        std::min<long long>(cap, std::max<long long>(c->o.dcap, std::max<long long>(c->dcap_floor, 0)));
    const unsigned long long fp0 = c->fingerprint();
    if ((rc = ensure_buffers(c, nx, ny, nz, cap, dcap, punits, c->wcap_floor))) return rc;
    if (c->fingerprint() != fp0) {
      c->gen++;
      c->drop_graphs();
    }
    static const int kZero[3] = {0, 0, 0};
    fill_rp(c, nullptr, nx, ny, nz, spacing, kZero);
    CK(cudaMemcpyAsync(c->d_rp, c->h_rp, sizeof(RoiParams), cudaMemcpyHostToDevice, s));
    init_stats<<<1, 256, 0, s>>>(c->d_stats, c->segmap.p, 0LL, nullptr, c->d_rp);
    CKL(1);
    shard_import<<<c->sms * 2, 256, 0, s>>>(c->d_stats, lo, hi, c->sort_counts.p, c->pbin_counts.p,
                                            n_pbin, reinterpret_cast<const long long*>(d_sums),
                                            (long long)n_keys);
    CKL(1);
    if (n_keys)
      CK(cudaMemcpyAsync(c->keys.p, d_keys, (size_t)n_keys * sizeof(int4), cudaMemcpyDeviceToDevice, s));
    CK(record(c, c->kev[2], s));
    int nk = 0;
    if ((rc = enqueue_diam(c, s, shard, nshards, nk))) return rc;
    if (d_sq4)
      CK(cudaMemcpyAsync(d_sq4, c->d_stats->sq, 4 * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(c->h_stats, c->d_stats, sizeof(Stats), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const Stats& h = *c->h_stats;
    if (h.bad_input) {
      set_err("summed vertex count != gathered keys (%lld)", (long long)n_keys);
      return SC_ERR_INPUT;
    }
    const long long PU = (long long)h.n_pwork, WU = (long long)h.n_work;
    if (n_keys <= c->dcap_sz && PU <= (long long)c->plane_umax.cap && WU <= c->h_rp->wcap) break;
    if (attempt) { set_err("vertex buffer overflow"); return SC_ERR_NOMEM; }
    c->cap_floor = std::max(c->cap_floor, cap);  // exact sizes from now on
    c->dcap_floor = std::max<long long>(c->dcap_floor, n_keys);
    c->wcap_floor = std::max(c->wcap_floor, WU);
    punits = PU;
  }
  rc = collect_roi(c, spacing, out);
  out->total_ms = wall_ms() - t0;
  return rc;
}

int sc_calculate_coefficients(const uint8_t* mask, int64_t nx, int64_t ny, int64_t nz,
                              const double spacing[3], int device, sc_coeffs* out) {
  const double t0 = wall_ms();
  int rc = check_input(mask, nx, ny, nz, spacing);
  if (rc) return rc;
  if (!out) { set_err("out is NULL"); return SC_ERR_INPUT; }
  Ctx* c;
  if ((rc = get_ctx(device, &c))) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  c->o = snapshot_opts();
  CK(cudaSetDevice(device));
  std::memset(out, 0, sizeof *out);
  CK(c->mask_stage.ensure((size_t)nx * ny * nz));
  cudaStream_t s = c->stream;
  int64_t cy = ny, cz = nz;
  int org[3] = {0, 0, 0};
  rc = stage_host_mask(c, mask, nx, ny, nz, s, &cy, &cz, org);
  if (rc) return rc;
  rc = run_roi(c, c->mask_stage.p, nx, cy, cz, spacing, s, 0, 1, nullptr, out, org);
  out->h2d_ms = ev_ms(c->ev[0], c->ev[1]);
  out->h2d_bytes = c->last_h2d_bytes;
  out->host_scan_ms = c->last_scan_ms;
  c->last_ms[6] = out->h2d_ms;
  if (rc == SC_OK) note_host_rates(c, nx * ny * nz, out->h2d_ms);
  out->total_ms = wall_ms() - t0;
  return rc;
}

int sc_calculate_coefficients_raw(const void* data, int dtype, const int64_t shape[3],
                                  int fortran_order, int has_label, int64_t label_int,
                                  double label_float, const double spacing[3], int device,
                                  sc_coeffs* out) {
  const double t0 = wall_ms();
  if (!shape) { set_err("shape pointer is NULL"); return SC_ERR_INPUT; }
  sc_raw_mask m{data, dtype, fortran_order, has_label, label_int, label_float,
                {shape[0], shape[1], shape[2]}};
  int rc = check_raw(m);
  if (rc) return rc;
  const int64_t nx = shape[2], ny = shape[1], nz = shape[0];
  if ((rc = check_input(data, nx, ny, nz, spacing))) return rc;
  if (!out) { set_err("out is NULL"); return SC_ERR_INPUT; }
  Ctx* c;
  if ((rc = get_ctx(device, &c))) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  c->o = snapshot_opts();
  CK(cudaSetDevice(device));
  std::memset(out, 0, sizeof *out);
  cudaStream_t s = c->stream;
  int64_t cx = nx, cy = ny, cz = nz;
  int org[3] = {0, 0, 0};
  if ((rc = stage_host_raw(c, m, s, &cx, &cy, &cz, org))) return rc;
  rc = run_roi(c, c->mask_stage.p, cx, cy, cz, spacing, s, 0, 1, nullptr, out, org);
  out->h2d_ms = ev_ms(c->ev[0], c->ev[1]);
  out->h2d_bytes = c->last_h2d_bytes;
  out->host_scan_ms = c->last_scan_ms;
  c->last_ms[6] = out->h2d_ms;
  out->total_ms = wall_ms() - t0;
  return rc;
}

int sc_calculate_coefficients_raw_batch(const sc_raw_mask* masks, const double* spacings,
                                        int64_t count, int device, sc_coeffs* out) {
  if (count < 0 || (count > 0 && (!masks || !spacings || !out))) {
    set_err("bad batch arguments");
    return SC_ERR_INPUT;
  }
  std::vector<const uint8_t*> ptrs((size_t)count);
  std::vector<int64_t> dims((size_t)(3 * count));
  for (int64_t i = 0; i < count; i++) {
    ptrs[(size_t)i] = static_cast<const uint8_t*>(masks[i].data);
    dims[(size_t)(3 * i)] = masks[i].shape[2];
    dims[(size_t)(3 * i + 1)] = masks[i].shape[1];
    dims[(size_t)(3 * i + 2)] = masks[i].shape[0];
  }
  return run_batch(device, ptrs.data(), dims.data(), spacings, count, true, out, nullptr, masks);
}

int sc_calculate_coefficients_batch(const uint8_t* const* masks, const int64_t* dims,
                                    const double* spacings, int64_t count, int device,
                                    sc_coeffs* out) {
  return run_batch(device, masks, dims, spacings, count, true, out, nullptr);
}

int sc_calculate_coefficients_batch_multi(const uint8_t* const* masks, const int64_t* dims,
                                          const double* spacings, int64_t count,
                                          const int* devices, int ndev, sc_coeffs* out) {
  if (count < 0 || ndev < 1 || !devices || (count > 0 && (!masks || !dims || !spacings || !out))) {
    set_err("bad batch arguments");
    return SC_ERR_INPUT;
  }
  if (count == 0) return SC_OK;
  // LPT over the devices by streamed bytes (the HBM pass sets the per-ROI
  // floor; V is unknown before marching cubes): largest ROI first onto the
  // least-loaded device.  One host thread per device entry runs the
  // pipelined single-device batch on its share; results land in input order.
  std::vector<int64_t> order((size_t)count);
  for (int64_t i = 0; i < count; i++) order[(size_t)i] = i;
  auto bytes = [&](int64_t i) {
    return std::max<int64_t>(1, dims[3 * i]) * std::max<int64_t>(1, dims[3 * i + 1]) *
           std::max<int64_t>(1, dims[3 * i + 2]);
  };
  std::stable_sort(order.begin(), order.end(),
                   [&](int64_t a, int64_t b) { return bytes(a) > bytes(b); });
  std::vector<std::vector<int64_t>> share((size_t)ndev);
  std::vector<double> load((size_t)ndev, 0.0);
  for (int64_t i : order) {
    const size_t d = (size_t)(std::min_element(load.begin(), load.end()) - load.begin());
    share[d].push_back(i);
    load[d] += (double)bytes(i);
  }
  for (auto& v : share) std::sort(v.begin(), v.end());  // each share in input order
  const Opts opts = snapshot_opts();  // the caller's options, for every worker thread
  std::vector<int> rcs((size_t)ndev, SC_OK);
  std::vector<std::string> errs((size_t)ndev);
  std::vector<std::thread> workers;
  for (int d = 0; d < ndev; d++) {
    if (share[(size_t)d].empty()) continue;
    workers.emplace_back([&, d] {
      t_opts = opts;
      t_opts_on = true;
      const std::vector<int64_t>& mine = share[(size_t)d];
      std::vector<const uint8_t*> m(mine.size());
      std::vector<int64_t> dm(3 * mine.size());
      std::vector<double> sp(3 * mine.size());
      std::vector<sc_coeffs> o(mine.size());
      for (size_t k = 0; k < mine.size(); k++) {
        m[k] = masks[mine[k]];
        for (int a = 0; a < 3; a++) {
          dm[3 * k + a] = dims[3 * mine[k] + a];
          sp[3 * k + a] = spacings[3 * mine[k] + a];
        }
      }
      rcs[(size_t)d] = run_batch(devices[d], m.data(), dm.data(), sp.data(), (int64_t)mine.size(),
                                 true, o.data(), nullptr);
      if (rcs[(size_t)d]) errs[(size_t)d] = g_err;
      for (size_t k = 0; k < mine.size(); k++) out[mine[k]] = o[k];
    });
  }
  for (auto& t : workers) t.join();
  for (int d = 0; d < ndev; d++)
    if (rcs[(size_t)d]) {
      g_err = errs[(size_t)d];
      return rcs[(size_t)d];
    }
  return SC_OK;
}

int sc_calculate_coefficients_device_batch(const uint8_t* const* d_masks, const int64_t* dims,
                                           const double* spacings, int64_t count, void* stream,
                                           sc_coeffs* out) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  return run_batch(dev, d_masks, dims, spacings, count, false, out, (cudaStream_t)stream);
}

int sc_diameters(const double* xs, const double* ys, const double* zs, int64_t n, int device,
                 double out[4]) {
  if (!out || (n > 0 && (!xs || !ys || !zs))) { set_err("NULL argument"); return SC_ERR_INPUT; }
  if (n <= 0) { set_err("diameters need at least one vertex"); return SC_ERR_NO_VERTICES; }
  if (n > (1LL << 31)) { set_err("too many points"); return SC_ERR_INPUT; }
  Ctx* c;
  int rc = get_ctx(device, &c);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  c->o = snapshot_opts();
  CK(cudaSetDevice(device));
  cudaStream_t s = c->stream;
  CK(c->cloud.ensure((size_t)(3 * n)));
  CK(c->cloud_out.ensure(4));
  CK(cudaMemcpyAsync(c->cloud.p, xs, n * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(c->cloud.p + n, ys, n * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(c->cloud.p + 2 * n, zs, n * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(c->cloud_out.p, 0, 32, s));
  const long long T = (n + 255) / 256;  // 256-point tiles; T(T+1)/2 tile pairs, grid-stride
  const long long units = T * (T + 1) / 2;
  const unsigned grid = (unsigned)std::min<long long>(units, (long long)c->sms * 8);
  cloud_diameters<<<grid, 256, 0, s>>>(c->cloud.p, c->cloud.p + n, c->cloud.p + 2 * n, n, T,
                                       c->cloud_out.p);
  CKL(1);
  unsigned long long hb[4];
  CK(cudaMemcpyAsync(hb, c->cloud_out.p, 32, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int i = 0; i < 4; i++) out[i] = std::sqrt(f64_of(hb[i]));
  return SC_OK;
}

int sc_marching_cubes(const uint8_t* mask, int64_t nx, int64_t ny, int64_t nz,
                      const double spacing[3], int device, double* xs, double* ys, double* zs,
                      int32_t* tris, int64_t vcap, int64_t tcap, int64_t* n_vert,
                      int64_t* n_tri) {
  int rc = check_input(mask, nx, ny, nz, spacing);
  if (rc) return rc;
  if (!n_vert || !n_tri) { set_err("NULL argument"); return SC_ERR_INPUT; }
  Ctx* c;
  if ((rc = get_ctx(device, &c))) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  c->o = snapshot_opts();
  CK(cudaSetDevice(device));
  const size_t bytes = (size_t)nx * ny * nz;
  CK(c->mask_stage.ensure(bytes));
  cudaStream_t s = c->stream;
  CK(cudaMemcpyAsync(c->mask_stage.p, mask, bytes, cudaMemcpyHostToDevice, s));
  return run_mesh(c, c->mask_stage.p, nx, ny, nz, spacing, s, xs, ys, zs, tris, vcap, tcap,
                  n_vert, n_tri);
}

int sc_mesh_measure(const double* xs, const double* ys, const double* zs, int64_t nv,
                    const int32_t* tris, int64_t nt, int device, double out[3]) {
  if (!out || nv < 0 || nt < 0 || (nv > 0 && (!xs || !ys || !zs)) || (nt > 0 && !tris)) {
    set_err("bad mesh arguments");
    return SC_ERR_INPUT;
  }
  out[0] = out[1] = out[2] = 0.0;
  if (nt == 0) return SC_OK;  // features.py:91-92, 103-104: empty mesh -> 0.0
  Ctx* c;
  int rc = get_ctx(device, &c);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  c->o = snapshot_opts();
  CK(cudaSetDevice(device));
  cudaStream_t s = c->stream;
  long long padded = 1;
  while (padded < nt) padded <<= 1;
  Tmp<double> dx, dy, dz, area, vol;
  Tmp<int> dt;
  CK(dx.alloc((size_t)nv)); CK(dy.alloc((size_t)nv)); CK(dz.alloc((size_t)nv));
  CK(dt.alloc((size_t)(3 * nt)));
  CK(area.alloc((size_t)padded)); CK(vol.alloc((size_t)padded));
  CK(cudaMemcpyAsync(dx.p, xs, 8 * nv, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dy.p, ys, 8 * nv, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dz.p, zs, 8 * nv, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dt.p, tris, 12 * nt, cudaMemcpyHostToDevice, s));
  tri_terms<<<c->sms * 8, 256, 0, s>>>(dx.p, dy.p, dz.p, dt.p, nt, padded, area.p, vol.p);
  CKL(1);
  for (long long half = padded / 2; half >= 1; half /= 2) {
    fold_pass<<<(unsigned)std::min<long long>((half + 255) / 256, c->sms * 8), 256, 0, s>>>(
        area.p, vol.p, half);
    CKL(1);
  }
  double r[2];
  CK(cudaMemcpyAsync(&r[0], area.p, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&r[1], vol.p, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  out[0] = r[0];
  out[1] = r[1];
  out[2] = std::fabs(r[1]);
  return SC_OK;
}

int sc_mesh_vertices(const uint8_t* mask, int64_t nx, int64_t ny, int64_t nz, int device,
                     int32_t* keys, int64_t cap, int64_t* n_out) {
  const double unit[3] = {1.0, 1.0, 1.0};
  int rc = check_input(mask, nx, ny, nz, unit);
  if (rc) return rc;
  if (!n_out || (cap > 0 && !keys)) { set_err("NULL argument"); return SC_ERR_INPUT; }
  Ctx* c;
  if ((rc = get_ctx(device, &c))) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  c->o = snapshot_opts();
  CK(cudaSetDevice(device));
  const size_t bytes = (size_t)nx * ny * nz;
  CK(c->mask_stage.ensure(bytes));
  cudaStream_t s = c->stream;
  CK(cudaMemcpyAsync(c->mask_stage.p, mask, bytes, cudaMemcpyHostToDevice, s));
  {
    const double unit[3] = {1.0, 1.0, 1.0};
    sc_coeffs tmp;
    c->prepacked = false;
    if ((rc = run_roi(c, c->mask_stage.p, nx, ny, nz, unit, s, 0, 1, nullptr, &tmp))) return rc;
  }
  const long long V = (long long)c->h_stats->n_vert;
  *n_out = V;
  const long long m = V < cap ? V : cap;
  if (m > 0) {
    std::vector<int4> tmp((size_t)m);
    // (the sorted copy: the unsorted buffer is reused by the diameter stage)
    CK(cudaMemcpyAsync(tmp.data(), c->keys_sorted.p, m * sizeof(int4), cudaMemcpyDeviceToHost,
                       s));
    CK(cudaStreamSynchronize(s));
    for (long long i = 0; i < m; i++) {
      keys[3 * i] = tmp[i].x;
      keys[3 * i + 1] = tmp[i].y;
      keys[3 * i + 2] = tmp[i].z;
    }
  }
  return SC_OK;
}

int sc_last_kernel_times(int device, double* ms, int n) {
  Ctx* c;
  int rc = get_ctx(device, &c);
  if (rc) return -rc;
  std::lock_guard<std::mutex> lk(c->mu);
  c->o = snapshot_opts();
  if (c->times_pending) {
    // pack, mc, prune (sort + 3-D filter), pass 1 (3-D + planar), re-check
    // (both), planar prep (runs beside the 3-D filter when forked)
    static const int from[6] = {0, 1, 2, 4, 5, 7}, to[6] = {1, 2, 3, 5, 6, 8};
    for (int i = 0; i < 6; i++) c->last_ms[i] = ev_ms(c->kev[from[i]], c->kev[to[i]]);
    c->times_pending = false;
  }
  int m = n < 7 ? n : 7;
  for (int i = 0; i < m; i++) ms[i] = c->last_ms[i];
  return m;
}

uint64_t sc_launch_count(void) { return g_launches.load(); }

int sc_occupied_slab(const uint8_t* mask, int64_t nx, int64_t ny, int64_t nz, int threads,
                     int64_t out[4]) {
  if (!mask || !out || nx < 1 || ny < 1 || nz < 1) {
    set_err("bad mask pointer, output pointer or dims");
    return SC_ERR_INPUT;
  }
  const Slab sl = occupied_slab(mask, nx, ny, nz,
                                threads > 0 ? threads : snapshot_opts().host_threads);
  if (sl.empty) {
    set_err("mask has no occupied voxels");
    return SC_ERR_EMPTY_ROI;
  }
  out[0] = sl.z0; out[1] = sl.z1; out[2] = sl.y0; out[3] = sl.y1;
  return SC_OK;
}

int sc_last_diagnostics(int device, int64_t* out, int n) {
  Ctx* c;
  int rc = get_ctx(device, &c);
  if (rc) return -rc;
  std::lock_guard<std::mutex> lk(c->mu);
  c->o = snapshot_opts();
  int m = n < 10 ? n : 10;
  for (int i = 0; i < m; i++) out[i] = c->last_diag[i];
  return m;
}

int sc_set_option(const char* name, int value) {
  std::lock_guard<std::mutex> lk(g_opt_mu);
  return set_opt(g_opts, name, value);
}

int sc_set_thread_option(const char* name, int value) {
  if (!t_opts_on) {
    Opts o;
    {
      std::lock_guard<std::mutex> lk(g_opt_mu);
      o = g_opts;
    }
    int rc = set_opt(o, name, value);
    if (rc) return rc;
    t_opts = o;
    t_opts_on = true;
    return SC_OK;
  }
  return set_opt(t_opts, name, value);
}

void sc_clear_thread_options(void) { t_opts_on = false; }

int sc_probe_fp32_peak(int device, int mode, double* tflops) {
  if (!tflops) { set_err("NULL argument"); return SC_ERR_INPUT; }
  Ctx* c;
  int rc = get_ctx(device, &c);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  c->o = snapshot_opts();
  CK(cudaSetDevice(device));
  cudaStream_t s = c->stream;
  float* d_out;
  const int blocks = c->sms * 8, threads = 256, iters = 1 << 14;
  CK(cudaMalloc(&d_out, sizeof(float) * blocks * threads));
  float best = 0.f;
  for (int rep = 0; rep < 4; rep++) {
    CK(cudaEventRecord(c->ev[0], s));
    switch (mode) {
      case 0: fp32_probe<0><<<blocks, threads, 0, s>>>(d_out, iters, 1.0001f, 0.5f); break;
      case 1: fp32_probe<1><<<blocks, threads, 0, s>>>(d_out, iters, 1.0001f, 0.5f); break;
      case 2: fp32_probe<2><<<blocks, threads, 0, s>>>(d_out, iters, 1.0001f, 0.5f); break;
      default: fp32_probe<3><<<blocks, threads, 0, s>>>(d_out, iters, 1.0001f, 0.5f); break;
    }
    CKL(1);
    CK(cudaEventRecord(c->ev[1], s));
    CK(cudaEventSynchronize(c->ev[1]));
    float ms = ev_ms(c->ev[0], c->ev[1]);
    if (rep > 0 && (best == 0.f || ms < best)) best = ms;
  }
  cudaFree(d_out);
  // 16 FFMA2 (4 flop) or 16 FFMA (2 flop) per thread per iteration.
  const double flop = (double)blocks * threads * iters * 16.0 * ((mode == 0 || mode == 2) ? 4.0 : 2.0);
  *tflops = flop / (best * 1e-3) / 1e12;
  return SC_OK;
}

}  // extern "C"
