// Device top-K with the reference ranking (K9): score descending, document id ascending
// (maxsim/streamio.py:230-262 TopKHeap, maxsim/cli.py:88-92 _ranked).
//
// (score, id) pairs are totally ordered, so the r-th best element is the best element that is
// strictly worse than the (r-1)-th: every round is one block-wide argmax, no "taken" flags.
// Pass 1: each block selects the top-K of its contiguous slice; pass 2 (same kernel) reduces
// the n_blocks * K candidates in a single block.
#pragma once
#include "ptx.cuh"

namespace mxs {

MXS_DEV bool better(double s1, long long i1, double s2, long long i2) {
  return s1 > s2 || (s1 == s2 && i1 < i2);
}

// in_ids == nullptr means ids are positions + id_offset.
__global__ void __launch_bounds__(512) topk_kernel(const double* __restrict__ in_s, const long long* __restrict__ in_ids,
                                                   long long n, int k, long long chunk, long long id_offset,
                                                   double* __restrict__ out_s, long long* __restrict__ out_ids) {
  __shared__ double ws[16];
  __shared__ long long wi[16];
  __shared__ double last_s;
  __shared__ long long last_i;
  const long long lo = (long long)blockIdx.x * chunk;
  const long long hi = min(n, lo + chunk);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double ls = INFINITY;
  long long li = -1;  // sentinel: everything is "worse" than (+inf, -1)
  for (int r = 0; r < k; ++r) {
    double bs = -INFINITY;
    long long bi = LLONG_MAX;
    bool have = false;
    for (long long e = lo + threadIdx.x; e < hi; e += blockDim.x) {
      const double s = in_s[e];
      const long long id = in_ids ? in_ids[e] : e + id_offset;
      if (s != s || id < 0) continue;       // NaN / empty candidate slots never rank
      if (!better(ls, li, s, id)) continue; // must be strictly worse than the last pick
      if (!have || better(s, id, bs, bi)) {
        bs = s;
        bi = id;
        have = true;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double os = __shfl_xor_sync(0xffffffffu, bs, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(os, oi, bs, bi)) {
        bs = os;
        bi = oi;
      }
    }
    if (lane == 0) {
      ws[w] = bs;
      wi[w] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = ws[0];
      long long id = wi[0];
      for (int j = 1; j < nw; ++j)
        if (better(ws[j], wi[j], s, id)) {
          s = ws[j];
          id = wi[j];
        }
      last_s = s;
      last_i = id;
      out_s[(long long)blockIdx.x * k + r] = s;
      out_ids[(long long)blockIdx.x * k + r] = (id == LLONG_MAX) ? -1 : id;
    }
    __syncthreads();
    ls = last_s;
    li = last_i;
  }
}

}  // namespace mxs
