// Host-side occupied-slab detection (see host_crop.h).  Plain host C++; lives
// in a .cu file only so the library builds from one nvcc command.
#include "host_crop.h"

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace sc {
namespace {

// Minimal persistent worker pool: run(n, fn) calls fn(t) for t in [0, n) on the
// workers and the calling thread, and returns when every call has finished.
class Pool {
 public:
  explicit Pool(int workers) {
    for (int i = 0; i < workers; i++) th_.emplace_back([this, i] { loop(i); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return (int)th_.size() + 1; }

  void run(int64_t n, int max_threads, const std::function<void(int64_t)>& fn) {
    std::lock_guard<std::mutex> serial(run_mu_);  // one job at a time
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      next_.store(0);
      active_ = std::max(0, std::min<int>(max_threads - 1, (int)th_.size()));
      pending_ = active_;
      gen_++;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void work() {
    for (int64_t t; (t = next_.fetch_add(1)) < n_;) (*fn_)(t);
  }
  void loop(int idx) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        if (idx >= active_) continue;  // not needed for this job
      }
      work();
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }

  std::vector<std::thread> th_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int64_t)>* fn_ = nullptr;
  std::atomic<int64_t> next_{0};
  int64_t n_ = 0;
  int active_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

Pool& pool() {
  static Pool p(std::max(0, (int)std::thread::hardware_concurrency() - 1));
  return p;
}

// Any nonzero byte in p[0, n)?  OR over the whole row (no data-dependent exit
// inside a row: rows are short and mostly background).  The AVX2 form (4 x 32
// B loads in flight per step) reads ~23 GB/s per core on the B200 hosts vs ~12
// for the portable 64-bit form (tools/microbench/scan_bench.cpp).
__attribute__((target("avx2"))) bool row_any_avx2(const uint8_t* p, int64_t n) {
  __m256i acc = _mm256_setzero_si256();
  int64_t i = 0;
  for (; i + 128 <= n; i += 128) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(p + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(p + i + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(p + i + 64));
    const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(p + i + 96));
    acc = _mm256_or_si256(acc, _mm256_or_si256(_mm256_or_si256(a, b), _mm256_or_si256(c, d)));
  }
  bool any = !_mm256_testz_si256(acc, acc);
  for (; i < n && !any; i++) any = p[i] != 0;
  return any;
}

inline bool row_any_u64(const uint8_t* p, int64_t n) {
  uint64_t acc = 0;
  int64_t i = 0;
  for (; i + 32 <= n; i += 32) {
    uint64_t w[4];
    std::memcpy(w, p + i, 32);
    acc |= w[0] | w[1] | w[2] | w[3];
  }
  for (; i < n; i++) acc |= p[i];
  return acc != 0;
}

// One row of nx bytes -> W words.
__attribute__((target("avx2"))) void pack_row_avx2(const uint8_t* p, int64_t nx, uint32_t* out) {
  const __m256i zero = _mm256_setzero_si256();
  int64_t i = 0, w = 0;
  for (; i + 32 <= nx; i += 32, w++) {
    const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(p + i));
    out[w] = ~(uint32_t)_mm256_movemask_epi8(_mm256_cmpeq_epi8(v, zero));
  }
  if (i < nx) {
    uint32_t word = 0;
    for (int64_t b = 0; i + b < nx; b++) word |= (uint32_t)(p[i + b] != 0) << b;
    out[w] = word;
  }
}

void pack_row_scalar(const uint8_t* p, int64_t nx, uint32_t* out) {
  for (int64_t w = 0; 32 * w < nx; w++) {
    uint32_t word = 0;
    for (int64_t b = 0; b < 32 && 32 * w + b < nx; b++) word |= (uint32_t)(p[32 * w + b] != 0) << b;
    out[w] = word;
  }
}

}  // namespace

void pack_slab(const uint8_t* mask, int64_t nx, int64_t ny, int64_t z0, int64_t z1, int64_t y0,
               int64_t y1, uint32_t* out, int threads) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  const int64_t W = (nx + 31) / 32, rows = y1 - y0 + 1, nzs = z1 - z0 + 1;
  if (nzs <= 0 || rows <= 0) return;
  // tasks of ~256 KB of mask rows (enough of them for every thread)
  const int64_t per = std::max<int64_t>(1, (int64_t(1) << 18) / std::max<int64_t>(1, nx * rows));
  const int64_t ntask = (nzs + per - 1) / per;
  auto job = [&](int64_t t) {
    for (int64_t zz = t * per; zz < std::min(nzs, (t + 1) * per); zz++)
      for (int64_t r = 0; r < rows; r++) {
        const uint8_t* src = mask + ((z0 + zz) * ny + y0 + r) * nx;
        uint32_t* dst = out + (zz * rows + r) * W;
        if (avx2) pack_row_avx2(src, nx, dst);
        else pack_row_scalar(src, nx, dst);
      }
  };
  const int nt = std::max(1, threads);
  if (nt == 1 || ntask == 1) {
    for (int64_t t = 0; t < ntask; t++) job(t);
  } else {
    pool().run(ntask, nt, job);
  }
}

Slab occupied_slab(const uint8_t* mask, int64_t nx, int64_t ny, int64_t nz, int threads) {
  struct Part {
    int64_t z0 = INT64_MAX, z1 = -1, y0 = INT64_MAX, y1 = -1, read = 0;
  };
  static const bool avx2 = __builtin_cpu_supports("avx2");
  auto row_any = [](const uint8_t* p, int64_t n) {
    return avx2 ? row_any_avx2(p, n) : row_any_u64(p, n);
  };
  const int64_t slice = nx * ny;
  // ~1 MB tasks: enough of them to balance, few enough to keep the counter cold.
  const int64_t per = std::max<int64_t>(1, (int64_t(1) << 20) / std::max<int64_t>(1, slice));
  const int64_t ntask = (nz + per - 1) / per;
  std::vector<Part> parts((size_t)ntask);
  auto scan = [&](int64_t t) {
    Part& r = parts[(size_t)t];
    const int64_t za = t * per, zb = std::min(nz, za + per);
    for (int64_t z = za; z < zb; z++) {
      const uint8_t* s = mask + z * slice;
      int64_t lo = -1;
      for (int64_t y = 0; y < ny; y++)
        if (row_any(s + y * nx, nx)) { lo = y; break; }
      if (lo < 0) { r.read += slice; continue; }
      int64_t hi = lo;
      for (int64_t y = ny - 1; y > lo; y--)
        if (row_any(s + y * nx, nx)) { hi = y; break; }
      r.read += (lo + 1 + (ny - hi)) * nx;
      r.z0 = std::min(r.z0, z);
      r.z1 = std::max(r.z1, z);
      r.y0 = std::min(r.y0, lo);
      r.y1 = std::max(r.y1, hi);
    }
  };
  const int nt = std::max(1, threads);
  if (nt == 1 || ntask == 1) {
    for (int64_t t = 0; t < ntask; t++) scan(t);
  } else {
    pool().run(ntask, nt, scan);
  }
  Part all;
  for (const Part& r : parts) {
    all.z0 = std::min(all.z0, r.z0); all.z1 = std::max(all.z1, r.z1);
    all.y0 = std::min(all.y0, r.y0); all.y1 = std::max(all.y1, r.y1);
    all.read += r.read;
  }
  Slab out;
  out.empty = all.z1 < 0;
  out.z0 = out.empty ? 0 : all.z0;
  out.z1 = out.empty ? -1 : all.z1;
  out.y0 = out.empty ? 0 : all.y0;
  out.y1 = out.empty ? -1 : all.y1;
  out.bytes_read = all.read;
  return out;
}

namespace {

template <typename T>
bool row_has(const uint8_t* p, int64_t n, T label) {
  T v;
  bool any = false;
  for (int64_t i = 0; i < n; i++) {
    std::memcpy(&v, p + i * (int64_t)sizeof(T), sizeof(T));
    any |= v == label;
  }
  return any;
}

}  // namespace

Slab occupied_slab_typed(const void* data, int dtype, int64_t row_elems, int64_t rows,
                         int64_t planes, int has_label, int64_t label_i, double label_f,
                         int threads) {
  static const int itemsize[7] = {1, 1, 2, 4, 8, 4, 8};
  const int isz = itemsize[dtype];
  const uint8_t* base = static_cast<const uint8_t*>(data);
  if (!has_label)  // any nonzero byte: the uint8 scanner over rows of row_elems * isz bytes
    return occupied_slab(base, row_elems * isz, rows, planes, threads);
  struct Part {
    int64_t z0 = INT64_MAX, z1 = -1, y0 = INT64_MAX, y1 = -1, read = 0;
  };
  const int64_t row_bytes = row_elems * isz, plane = row_bytes * rows;
  auto row_any = [&](const uint8_t* p) -> bool {
    switch (dtype) {
      case 0: case 1: return row_has<uint8_t>(p, row_elems, (uint8_t)label_i);
      case 2: return row_has<int16_t>(p, row_elems, (int16_t)label_i);
      case 3: return row_has<int32_t>(p, row_elems, (int32_t)label_i);
      case 4: return row_has<int64_t>(p, row_elems, (int64_t)label_i);
      case 5: return row_has<float>(p, row_elems, (float)label_f);
      default: return row_has<double>(p, row_elems, label_f);
    }
  };
  const int64_t per = std::max<int64_t>(1, (int64_t(1) << 20) / std::max<int64_t>(1, plane));
  const int64_t ntask = (planes + per - 1) / per;
  std::vector<Part> parts((size_t)ntask);
  auto scan = [&](int64_t t) {
    Part& r = parts[(size_t)t];
    for (int64_t z = t * per; z < std::min(planes, (t + 1) * per); z++) {
      const uint8_t* s = base + z * plane;
      int64_t lo = -1;
      for (int64_t y = 0; y < rows; y++)
        if (row_any(s + y * row_bytes)) { lo = y; break; }
      if (lo < 0) { r.read += plane; continue; }
      int64_t hi = lo;
      for (int64_t y = rows - 1; y > lo; y--)
        if (row_any(s + y * row_bytes)) { hi = y; break; }
      r.read += (lo + 1 + (rows - hi)) * row_bytes;
      r.z0 = std::min(r.z0, z); r.z1 = std::max(r.z1, z);
      r.y0 = std::min(r.y0, lo); r.y1 = std::max(r.y1, hi);
    }
  };
  const int nt = std::max(1, threads);
  if (nt == 1 || ntask == 1) {
    for (int64_t t = 0; t < ntask; t++) scan(t);
  } else {
    pool().run(ntask, nt, scan);
  }
  Part all;
  for (const Part& r : parts) {
    all.z0 = std::min(all.z0, r.z0); all.z1 = std::max(all.z1, r.z1);
    all.y0 = std::min(all.y0, r.y0); all.y1 = std::max(all.y1, r.y1);
    all.read += r.read;
  }
  Slab out;
  out.empty = all.z1 < 0;
  out.z0 = out.empty ? 0 : all.z0;
  out.z1 = out.empty ? -1 : all.z1;
  out.y0 = out.empty ? 0 : all.y0;
  out.y1 = out.empty ? -1 : all.y1;
  out.bytes_read = all.read;
  return out;
}

void copy_rows(void* dst, const void* src, int64_t pitch, int64_t width, int64_t nrows,
               int threads) {
  uint8_t* d = static_cast<uint8_t*>(dst);
  const uint8_t* s = static_cast<const uint8_t*>(src);
  // tasks of ~1 MB
  const int64_t per = std::max<int64_t>(1, (int64_t(1) << 20) / std::max<int64_t>(1, width));
  const int64_t ntask = (nrows + per - 1) / per;
  auto job = [&](int64_t t) {
    const int64_t a = t * per, b = std::min(nrows, a + per);
    if (pitch == width) {
      std::memcpy(d + a * width, s + a * pitch, (size_t)((b - a) * width));
      return;
    }
    for (int64_t r = a; r < b; r++) std::memcpy(d + r * width, s + r * pitch, (size_t)width);
  };
  const int nt = std::max(1, threads);
  if (nt == 1 || ntask == 1) {
    for (int64_t t = 0; t < ntask; t++) job(t);
  } else {
    pool().run(ntask, nt, job);
  }
}

}  // namespace sc
