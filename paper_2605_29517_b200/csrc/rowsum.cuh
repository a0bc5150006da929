// S4 per-pair score kernel (separate pass; the tensor-core forwards fold it into their epilogue).
#pragma once
#include "score_sum.cuh"

namespace mxs {

// Separate S4 pass over materialised row maxima [n_pairs, l_q] (opt-in rowmax outputs, the
// SIMT kernels and shapes whose query spans more than one CTA cluster).  One warp per pair.
__global__ void rowsum_kernel(const float* __restrict__ rowmax, long long n_pairs, int l_q, double* __restrict__ scores) {
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= n_pairs) return;
  const double s = warp_score_sum(rowmax + warp * l_q, l_q);
  if ((threadIdx.x & 31u) == 0) scores[warp] = s;
}

}  // namespace mxs
