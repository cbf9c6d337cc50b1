// Host scan microbenchmark: read rate of "is this row all zero" over a
// 157 MB mask (C2 size) with several loop variants and thread counts.
// Build: g++ -O3 -std=c++17 -pthread scan_bench.cpp -o scan_bench
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static const int64_t NX = 512, NY = 512, NZ = 600;

static inline bool row_any_u64(const uint8_t* p, int64_t n) {
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

__attribute__((target("avx2"))) static bool row_any_avx2(const uint8_t* p, int64_t n) {
  __m256i acc = _mm256_setzero_si256();
  int64_t i = 0;
  for (; i + 128 <= n; i += 128) {
    __m256i a = _mm256_loadu_si256((const __m256i*)(p + i));
    __m256i b = _mm256_loadu_si256((const __m256i*)(p + i + 32));
    __m256i c = _mm256_loadu_si256((const __m256i*)(p + i + 64));
    __m256i d = _mm256_loadu_si256((const __m256i*)(p + i + 96));
    acc = _mm256_or_si256(acc, _mm256_or_si256(_mm256_or_si256(a, b), _mm256_or_si256(c, d)));
  }
  bool any = !_mm256_testz_si256(acc, acc);
  for (; i < n; i++) any |= p[i] != 0;
  return any;
}

// Whole-slice variant: OR the slice in big strides (fast path for empty
// slices), fall back to rows only when the slice is nonzero.
__attribute__((target("avx2"))) static bool block_any_avx2_pf(const uint8_t* p, int64_t n) {
  __m256i acc = _mm256_setzero_si256();
  int64_t i = 0;
  for (; i + 256 <= n; i += 256) {
    _mm_prefetch((const char*)(p + i + 4096), _MM_HINT_T0);
    _mm_prefetch((const char*)(p + i + 4096 + 64), _MM_HINT_T0);
    _mm_prefetch((const char*)(p + i + 4096 + 128), _MM_HINT_T0);
    _mm_prefetch((const char*)(p + i + 4096 + 192), _MM_HINT_T0);
    __m256i a = _mm256_loadu_si256((const __m256i*)(p + i));
    __m256i b = _mm256_loadu_si256((const __m256i*)(p + i + 32));
    __m256i c = _mm256_loadu_si256((const __m256i*)(p + i + 64));
    __m256i d = _mm256_loadu_si256((const __m256i*)(p + i + 96));
    __m256i e = _mm256_loadu_si256((const __m256i*)(p + i + 128));
    __m256i f = _mm256_loadu_si256((const __m256i*)(p + i + 160));
    __m256i g = _mm256_loadu_si256((const __m256i*)(p + i + 192));
    __m256i h = _mm256_loadu_si256((const __m256i*)(p + i + 224));
    acc = _mm256_or_si256(acc, _mm256_or_si256(_mm256_or_si256(_mm256_or_si256(a, b), _mm256_or_si256(c, d)),
                                               _mm256_or_si256(_mm256_or_si256(e, f), _mm256_or_si256(g, h))));
  }
  bool any = !_mm256_testz_si256(acc, acc);
  for (; i < n; i++) any |= p[i] != 0;
  return any;
}

__attribute__((target("avx2"))) static bool block_any_avx2(const uint8_t* p, int64_t n) {
  __m256i acc = _mm256_setzero_si256();
  int64_t i = 0;
  for (; i + 256 <= n; i += 256) {
    __m256i x = _mm256_loadu_si256((const __m256i*)(p + i));
#pragma GCC unroll 8
    for (int k = 32; k < 256; k += 32) x = _mm256_or_si256(x, _mm256_loadu_si256((const __m256i*)(p + i + k)));
    acc = _mm256_or_si256(acc, x);
  }
  bool any = !_mm256_testz_si256(acc, acc);
  for (; i < n; i++) any |= p[i] != 0;
  return any;
}

__attribute__((target("avx512f,avx512bw"))) static bool row_any_avx512(const uint8_t* p, int64_t n) {
  __m512i acc = _mm512_setzero_si512();
  int64_t i = 0;
  for (; i + 256 <= n; i += 256) {
    __m512i a = _mm512_loadu_si512((const void*)(p + i));
    __m512i b = _mm512_loadu_si512((const void*)(p + i + 64));
    __m512i c = _mm512_loadu_si512((const void*)(p + i + 128));
    __m512i d = _mm512_loadu_si512((const void*)(p + i + 192));
    acc = _mm512_or_si512(acc, _mm512_or_si512(_mm512_or_si512(a, b), _mm512_or_si512(c, d)));
  }
  bool any = _mm512_test_epi64_mask(acc, acc) != 0;
  for (; i < n; i++) any |= p[i] != 0;
  return any;
}

int main() {
  const int64_t bytes = NX * NY * NZ;
  uint8_t* m = (uint8_t*)aligned_alloc(64, bytes);
  std::memset(m, 0, bytes);
  // KiTS-like occupancy: a blob in slices 228..354, rows 245..319
  for (int64_t z = 228; z <= 354; z++)
    for (int64_t y = 245; y <= 319; y++) std::memset(m + (z * NY + y) * NX + 100, 1, 300);
  const int hw = (int)std::thread::hardware_concurrency();
  printf("hw threads %d, avx2 %d\n", hw, __builtin_cpu_supports("avx2"));
  auto run = [&](const char* name, int threads, int variant) {
    std::vector<double> ts;
    for (int rep = 0; rep < 7; rep++) {
      std::atomic<int64_t> next{0};
      std::atomic<int64_t> found{0};
      auto t0 = std::chrono::steady_clock::now();
      auto work = [&]() {
        int64_t z;
        int64_t f = 0;
        while ((z = next.fetch_add(2)) < NZ) {
          for (int64_t zz = z; zz < std::min(NZ, z + 2); zz++) {
            const uint8_t* s = m + zz * NX * NY;
            if (variant == 0) {
              for (int64_t y = 0; y < NY; y++) if (row_any_u64(s + y * NX, NX)) { f++; break; }
            } else if (variant == 1) {
              for (int64_t y = 0; y < NY; y++) if (row_any_avx2(s + y * NX, NX)) { f++; break; }
            } else if (variant == 4) {
              for (int64_t y = 0; y < NY; y++) if (row_any_avx512(s + y * NX, NX)) { f++; break; }
            } else if (variant == 2) {
              if (block_any_avx2(s, NX * NY)) f++;
            } else {
              if (block_any_avx2_pf(s, NX * NY)) f++;
            }
          }
        }
        found += f;
      };
      std::vector<std::thread> th;
      for (int t = 1; t < threads; t++) th.emplace_back(work);
      work();
      for (auto& t : th) t.join();
      ts.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    std::sort(ts.begin(), ts.end());
    printf("%-22s threads %3d: %.3f ms  %.1f GB/s\n", name, threads, ts[3] * 1e3, bytes / ts[3] / 1e9);
  };
  const char* names[5] = {"rows u64 (current)", "rows avx2", "slice avx2", "slice avx2+prefetch",
                          "rows avx512"};
  for (int v : {0, 1, 4, 2})
    for (int t : {1, 4, 8, hw}) run(names[v], t, v);
  return 0;
}
