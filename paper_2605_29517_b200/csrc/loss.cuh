// In-batch contrastive loss of the C3 training step (maxsim/cli.py:198-206 _softmax_ce), fused:
// float64 scores [n_q, b] with the positives on the diagonal -> loss (f64 scalar) and the score
// gradient (probs - eye) / n_q for the column slice [col0, col0 + ncols) in fp32 -- the
// upstream gradient of the backward gathers.  Replaces ~15 small elementwise / reduction
// launches of the torch restatement (parallel.softmax_ce) with one block.
//
// One CTA; warp w takes rows w, w + W, ... in order; per row: max, sum of exp(s - max) (lane
// partials then a fixed butterfly), lse = log(sum) + max, the row term lse - s[q, q]; the loss
// is the fixed-order sum of the warps' row terms / n_q, so the result is deterministic.
#pragma once
#include <cstdint>

namespace mxs {

constexpr int kLossThreads = 256;

__global__ void __launch_bounds__(kLossThreads) softmax_ce_kernel(const double* __restrict__ s, int n_q, int b,
                                                                 int col0, int ncols, double* __restrict__ loss,
                                                                 float* __restrict__ g) {
  __shared__ double wsum[kLossThreads / 32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0.0;  // this warp's row terms, rows in increasing order
  for (int q = w; q < n_q; q += kLossThreads / 32) {
    const double* row = s + (long long)q * b;
    double mx = -INFINITY;
    for (int j = lane; j < b; j += 32) mx = fmax(mx, row[j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    double se = 0.0;
    for (int j = lane; j < b; j += 32) se += exp(row[j] - mx);
#pragma unroll
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const double lse = log(se) + mx;
    acc += lse - row[q];
    float* grow = g + (long long)q * ncols;
    for (int j = lane; j < ncols; j += 32) {
      const int c = col0 + j;
      grow[j] = (float)((exp(row[c] - lse) - (c == q ? 1.0 : 0.0)) / n_q);
    }
  }
  if (lane == 0) wsum[w] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < kLossThreads / 32; ++i) t += wsum[i];
    *loss = t / n_q;
  }
}

}  // namespace mxs
