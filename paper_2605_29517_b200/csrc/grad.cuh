// Exact MaxSim backward gathers (K7, K8).  The max is resolved by the saved argmax, so the
// score is piecewise linear (maxsim/backward.py:1-21):
//   dD[r]    = sum over the CSR bucket of r (ascending source) of g[q,b] * Q[q_row(s)]   (K7)
//   dQ[q, i] = sum over b ascending of g[q,b] * D_b[argmax[q,b,i]]                       (K8)
// Both are destination-owned: one warp owns one output row, accumulates it in fp32 registers in
// the reference's order (maxsim/backward.py:165-172, :225-231) and stores it exactly once -- no
// atomics anywhere.  Lanes split the embedding axis (VEC contiguous elements per lane).
#pragma once
#include "fwd_exact.cuh"  // to_f32

namespace mxs {

struct GradParams {
  int n_q, n_docs, l_q, dim;
  const float* g;              // [n_q, n_docs]
  // K7
  const int32_t* row_ptr;      // [n_dest + 1]
  const int32_t* col_idx;      // [n_src]
  long long n_dest;
  float* dD;                   // [n_dest, dim]
  // K8
  const int32_t* argmax;       // [n_q, n_docs, l_q]
  const long long* doc_row_off;  // [n_docs] first row of each document in D
  float* dQ;                   // [n_q, l_q, dim]
};

// K7: warp per destination row.  Q rows are gathered through L2 (Q is small and hot).
template <typename T>
__global__ void __launch_bounds__(256) grad_docs_kernel(const T* __restrict__ Q, const GradParams p) {
  const long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= p.n_dest) return;
  const int nchunk = (p.dim + 31) >> 5;  // <= 8 (dim <= 512 on this path)
  float acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) acc[c] = 0.f;
  const int lo = p.row_ptr[r], hi = p.row_ptr[r + 1];
  const long long per_q = (long long)p.n_docs * p.l_q;
  for (int t0 = lo; t0 < hi; t0 += 32) {
    const int n = min(32, hi - t0);
    const int my = (lane < n) ? p.col_idx[t0 + lane] : 0;
    for (int j = 0; j < n; ++j) {
      const long long s = __shfl_sync(0xffffffffu, my, j);
      const int q = (int)(s / per_q);
      const int b = (int)((s / p.l_q) % p.n_docs);
      const long long qrow = (long long)q * p.l_q + s % p.l_q;
      const float w = __ldg(p.g + (long long)q * p.n_docs + b);
      const T* row = Q + qrow * p.dim;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        if (c >= nchunk) break;
        const int k = c * 32 + lane;
        if (k < p.dim) acc[c] = __fmaf_rn(w, to_f32(row[k]), acc[c]);
      }
    }
  }
  float* out = p.dD + r * p.dim;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    if (c >= nchunk) break;
    const int k = c * 32 + lane;
    if (k < p.dim) out[k] = acc[c];
  }
}

// K8: warp per (q, i) query row; b ascending.
template <typename T>
__global__ void __launch_bounds__(256) grad_query_kernel(const T* __restrict__ D, const GradParams p) {
  const long long wq = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wq >= (long long)p.n_q * p.l_q) return;
  const int q = (int)(wq / p.l_q), i = (int)(wq % p.l_q);
  const int nchunk = (p.dim + 31) >> 5;
  float acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) acc[c] = 0.f;
  for (int b0 = 0; b0 < p.n_docs; b0 += 32) {
    const int n = min(32, p.n_docs - b0);
    int my_a = 0;
    float my_w = 0.f;
    long long my_off = 0;
    if (lane < n) {
      my_a = p.argmax[((long long)q * p.n_docs + b0 + lane) * p.l_q + i];
      my_w = p.g[(long long)q * p.n_docs + b0 + lane];
      my_off = p.doc_row_off[b0 + lane];
    }
    for (int j = 0; j < n; ++j) {
      const int a = __shfl_sync(0xffffffffu, my_a, j);
      const float w = __shfl_sync(0xffffffffu, my_w, j);
      const long long off = __shfl_sync(0xffffffffu, my_off, j);
      const T* row = D + (off + a) * p.dim;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        if (c >= nchunk) break;
        const int k = c * 32 + lane;
        if (k < p.dim) acc[c] = __fmaf_rn(w, to_f32(row[k]), acc[c]);
      }
    }
  }
  float* out = p.dQ + wq * p.dim;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    if (c >= nchunk) break;
    const int k = c * 32 + lane;
    if (k < p.dim) out[k] = acc[c];
  }
}

}  // namespace mxs
