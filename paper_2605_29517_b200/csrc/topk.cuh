// Device top-K with the reference ranking (K9): score descending, document id ascending
// (maxsim/streamio.py:230-262 TopKHeap, maxsim/cli.py:88-92 _ranked).
//
// (score, id) pairs are totally ordered (ids are unique), so a sorting network under that order
// reproduces the heap's result exactly, ties included.
#pragma once
#include "ptx.cuh"

namespace mxs {

MXS_DEV bool better(double s1, long long i1, double s2, long long i2) {
  return s1 > s2 || (s1 == s2 && i1 < i2);
}

constexpr int kTopkThreads = 1024;
constexpr int kTopkSlice = 4096;  // elements sorted per block (64 KB of shared memory)

// Each block sorts one slice of (score, id) pairs with a bitonic network under the reference
// order (score desc, id asc; invalid slots -- past the end, NaN, id < 0 -- sort last) and keeps
// the first k.  Repeated over the surviving candidates until one slice remains.
// in_ids == nullptr means ids are positions + id_offset.
__global__ void __launch_bounds__(kTopkThreads) topk_kernel(const double* __restrict__ in_s,
                                                            const long long* __restrict__ in_ids, long long n, int k,
                                                            long long chunk, long long id_offset,
                                                            double* __restrict__ out_s, long long* __restrict__ out_ids) {
  extern __shared__ uint8_t tk_smem[];
  double* ss = reinterpret_cast<double*>(tk_smem);
  long long* si = reinterpret_cast<long long*>(tk_smem + kTopkSlice * sizeof(double));
  const long long lo = (long long)blockIdx.x * chunk;
  const long long hi = min(n, lo + chunk);
  for (int e = threadIdx.x; e < kTopkSlice; e += blockDim.x) {
    double s = -INFINITY;
    long long id = LLONG_MAX;
    const long long g = lo + e;
    if (g < hi) {
      const double v = in_s[g];
      const long long i = in_ids ? in_ids[g] : g + id_offset;
      if (v == v && i >= 0) {
        s = v;
        id = i;
      }
    }
    ss[e] = s;
    si[e] = id;
  }
  __syncthreads();
  for (int size = 2; size <= kTopkSlice; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < kTopkSlice / 2; t += blockDim.x) {
        const int a = 2 * t - (t & (stride - 1));  // first element of the pair
        const int b = a + stride;
        const bool desc_block = (a & size) == 0;   // this run is sorted "best first"
        const double sa = ss[a], sb = ss[b];
        const long long ia = si[a], ib = si[b];
        // b strictly better than a under (score desc, id asc, invalid last)?
        const bool b_first = (ib != LLONG_MAX) && (ia == LLONG_MAX || better(sb, ib, sa, ia));
        if (b_first == desc_block) {
          ss[a] = sb;
          ss[b] = sa;
          si[a] = ib;
          si[b] = ia;
        }
      }
      __syncthreads();
    }
  }
  for (int r = threadIdx.x; r < k; r += blockDim.x) {
    const long long id = si[r];
    out_s[(long long)blockIdx.x * k + r] = (id == LLONG_MAX) ? -INFINITY : ss[r];
    out_ids[(long long)blockIdx.x * k + r] = (id == LLONG_MAX) ? -1 : id;
  }
}

}  // namespace mxs
