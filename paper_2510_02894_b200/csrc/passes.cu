// The two O(pairs) kernels of the diameter stage (sm_100a): one pass-1 kernel
// and one exact re-check kernel, each running the 3-D and the planar work
// lists back to back (pass_bodies.cuh).  Fusing them halves the kernel
// boundaries of the diameter stage; the two lists are independent, so every
// warp simply works through its share of the first list, then of the second.
#include "pass_bodies.cuh"

namespace sc {

template <bool PACKED>
__global__ void __launch_bounds__(kDiamThreads, 4) diam_pass1(
    const int4* __restrict__ keys, long long cap, const RoiParams* __restrict__ rp,
    const uint2* __restrict__ work, float* __restrict__ umax, const int2* __restrict__ sorted,
    const unsigned int* __restrict__ start, const uint2* __restrict__ pwork, long long pwcap,
    float* __restrict__ pumax, Stats* __restrict__ st, const int4* __restrict__ boxes,
    const int4* __restrict__ hboxes, int vfilter, const unsigned int* __restrict__ cstart,
    const int4* __restrict__ pboxes, const int4* __restrict__ hpboxes,
    const float4* __restrict__ fkeys) {
  pdl_enter();
  KTrace kt_(st, kTrPass1);
  if (st->ovf || st->bbox[3] < 0) return;  // re-run pending (scan_all) / empty
  __shared__ float4 sj_all[kWarps][kChunk];  // per-warp J chunk, (x, y, z | -, |p|^2)
  __shared__ float4 si_all[kWarps][kChunk];  // per-warp filtered I list
  float4* sj = sj_all[threadIdx.x >> 5];
  float4* si = si_all[threadIdx.x >> 5];
  // A list longer than its buffer means a re-run with exact sizes is pending.
  if ((long long)st->n_work <= rp->wcap)
    pass1_3d<PACKED>(keys, fkeys, cap, rp, work, umax, st, sj, si, boxes, hboxes, vfilter);
  __syncwarp();
  if ((long long)st->n_pwork <= pwcap)
    pass1_planar(sorted, start, pwork, rp, pumax, st, sj, si, cstart, pboxes, hpboxes, vfilter);
}
template __global__ void diam_pass1<true>(const int4*, long long, const RoiParams*, const uint2*,
                                          float*, const int2*, const unsigned int*, const uint2*,
                                          long long, float*, Stats*, const int4*, const int4*, int,
                                          const unsigned int*, const int4*, const int4*,
                                          const float4*);
template __global__ void diam_pass1<false>(const int4*, long long, const RoiParams*, const uint2*,
                                           float*, const int2*, const unsigned int*,
                                           const uint2*, long long, float*, Stats*, const int4*,
                                           const int4*, int, const unsigned int*, const int4*,
                                           const int4*, const float4*);

__global__ void __launch_bounds__(kDiamThreads) diam_refine(
    const int4* __restrict__ keys, long long cap, const RoiParams* __restrict__ rp,
    const uint2* __restrict__ work, const float* __restrict__ umax,
    const int2* __restrict__ sorted, const unsigned int* __restrict__ start,
    const uint2* __restrict__ pwork, long long pwcap, const float* __restrict__ pumax,
    Stats* __restrict__ st, Stats* out_host) {
  pdl_enter();
  KTrace kt_(st, kTrRefine);
  __shared__ double s_a[kChunk], s_b[kChunk], s_c[kChunk];
  __shared__ double s_red[kDiamThreads / 32];
  __shared__ unsigned int s_list[kDiamThreads];
  __shared__ int s_n;
  if (!st->ovf && st->bbox[3] >= 0) {  // block-uniform
    if ((long long)st->n_work <= rp->wcap)
      refine_3d(keys, cap, rp, work, umax, st, s_a, s_b, s_c, s_list, s_n);
    __syncthreads();
    if ((long long)st->n_pwork <= pwcap)
      refine_planar(sorted, start, pwork, rp, pumax, st, s_a, s_b, s_red, s_list, s_n);
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&st->t_end, global_ns());
  }
  // out_host (optional): the slot's accumulator record in mapped pinned host
  // memory; the last block to finish publishes the complete record there, so
  // no device->host copy follows the ROI's graph.
  // The case histogram goes out merged (hist[0] = sum of the kHistCopies
  // copies, marked by hist_merged), so 2.5 KB cross PCIe instead of 16.8 KB.
  if (out_host && last_block(&st->done2)) {
    const volatile unsigned long long* s = reinterpret_cast<const volatile unsigned long long*>(st);
    unsigned long long* d = reinterpret_cast<unsigned long long*>(out_host);
    for (int k = threadIdx.x; k < kNumCases; k += blockDim.x) {
      unsigned long long sum = 0;
#pragma unroll
      for (int c = 0; c < kHistCopies; c++) sum += s[c * kNumCases + k];
      d[k] = sum;
    }
    constexpr int kTail = kHistCopies * kNumCases;  // first word after the histograms
    for (int i = kTail + threadIdx.x; i < (int)(sizeof(Stats) / 8); i += blockDim.x) d[i] = s[i];
    __syncthreads();
    if (threadIdx.x == 0) out_host->hist_merged = 1u;
    __threadfence_system();
  }
}

}  // namespace sc
