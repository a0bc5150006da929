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


// ---------------------------------------------------------------------------------------------
// Vectorised variants: each lane owns VEC = 8 B / sizeof(T) consecutive elements per pass, so one
// warp instruction moves a 256 B row slice; U source rows are in flight per warp.  Accumulation
// order per output element is unchanged (sources in bucket / b order), fp32 FMA.
template <typename T>
struct Vec8;
template <>
struct Vec8<float> {
  static constexpr int N = 2;
  MXS_DEV static void load(const float* p, float (&o)[2]) {
    const float2 t = __ldg(reinterpret_cast<const float2*>(p));
    o[0] = t.x;
    o[1] = t.y;
  }
};
template <>
struct Vec8<__nv_bfloat16> {
  static constexpr int N = 4;
  MXS_DEV static void load(const __nv_bfloat16* p, float (&o)[4]) {
    const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
    o[0] = __uint_as_float(t.x << 16);
    o[1] = __uint_as_float(t.x & 0xffff0000u);
    o[2] = __uint_as_float(t.y << 16);
    o[3] = __uint_as_float(t.y & 0xffff0000u);
  }
};
template <>
struct Vec8<__half> {
  static constexpr int N = 4;
  MXS_DEV static void load(const __half* p, float (&o)[4]) {
    const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
    const __half2 a = *reinterpret_cast<const __half2*>(&t.x);
    const __half2 b = *reinterpret_cast<const __half2*>(&t.y);
    const float2 fa = __half22float2(a), fb = __half22float2(b);
    o[0] = fa.x;
    o[1] = fa.y;
    o[2] = fb.x;
    o[3] = fb.y;
  }
};

constexpr int kGradU = 4;  // source rows in flight per warp

// K7 vectorised: warp per destination row; NP passes of 32 * VEC elements cover dim.
template <typename T, int NP>
__global__ void __launch_bounds__(256) grad_docs_vec_kernel(const T* __restrict__ Q, const GradParams p) {
  constexpr int V = Vec8<T>::N;
  const long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= p.n_dest) return;
  float acc[NP][V];
#pragma unroll
  for (int a = 0; a < NP; ++a)
#pragma unroll
    for (int v = 0; v < V; ++v) acc[a][v] = 0.f;
  const int lo = __ldg(p.row_ptr + r), hi = __ldg(p.row_ptr + r + 1);
  const long long per_q = (long long)p.n_docs * p.l_q;
  for (int t0 = lo; t0 < hi; t0 += 32) {
    const int n = min(32, hi - t0);
    // lane j decodes source t0 + j: Q row and weight
    long long my_row = 0;
    float my_w = 0.f;
    if (lane < n) {
      const long long s = __ldg(p.col_idx + t0 + lane);
      const int q = (int)(s / per_q);
      const int b = (int)((s / p.l_q) % p.n_docs);
      my_row = (long long)q * p.l_q + s % p.l_q;
      my_w = __ldg(p.g + (long long)q * p.n_docs + b);
    }
    for (int j0 = 0; j0 < n; j0 += kGradU) {
      float x[kGradU][NP][V];
      float w[kGradU];
#pragma unroll
      for (int u = 0; u < kGradU; ++u) {
        const int j = j0 + u;
        const long long row = __shfl_sync(0xffffffffu, my_row, j & 31);
        w[u] = (j < n) ? __shfl_sync(0xffffffffu, my_w, j & 31) : 0.f;
#pragma unroll
        for (int a = 0; a < NP; ++a) {
          const int k = (a * 32 + lane) * V;
          if (j < n && k < p.dim)
            Vec8<T>::load(Q + row * p.dim + k, x[u][a]);
          else
#pragma unroll
            for (int v = 0; v < V; ++v) x[u][a][v] = 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < kGradU; ++u)
        if (j0 + u < n)
#pragma unroll
          for (int a = 0; a < NP; ++a)
#pragma unroll
            for (int v = 0; v < V; ++v) acc[a][v] = __fmaf_rn(w[u], x[u][a][v], acc[a][v]);
    }
  }
  float* out = p.dD + r * p.dim;
#pragma unroll
  for (int a = 0; a < NP; ++a) {
    const int k = (a * 32 + lane) * V;
    if (k < p.dim) {
      if constexpr (V == 4)
        *reinterpret_cast<float4*>(out + k) = make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
      else
        *reinterpret_cast<float2*>(out + k) = make_float2(acc[a][0], acc[a][1]);
    }
  }
}

// K8 vectorised: warp per (q, i) query row; documents b ascending.
template <typename T, int NP>
__global__ void __launch_bounds__(256) grad_query_vec_kernel(const T* __restrict__ D, const GradParams p) {
  constexpr int V = Vec8<T>::N;
  const long long wq = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wq >= (long long)p.n_q * p.l_q) return;
  const int q = (int)(wq / p.l_q), i = (int)(wq % p.l_q);
  float acc[NP][V];
#pragma unroll
  for (int a = 0; a < NP; ++a)
#pragma unroll
    for (int v = 0; v < V; ++v) acc[a][v] = 0.f;
  for (int b0 = 0; b0 < p.n_docs; b0 += 32) {
    const int n = min(32, p.n_docs - b0);
    long long my_row = 0;
    float my_w = 0.f;
    if (lane < n) {
      const int a_ = __ldg(p.argmax + ((long long)q * p.n_docs + b0 + lane) * p.l_q + i);
      my_w = __ldg(p.g + (long long)q * p.n_docs + b0 + lane);
      my_row = __ldg(p.doc_row_off + b0 + lane) + a_;
    }
    for (int j0 = 0; j0 < n; j0 += kGradU) {
      float x[kGradU][NP][V];
      float w[kGradU];
#pragma unroll
      for (int u = 0; u < kGradU; ++u) {
        const int j = j0 + u;
        const long long row = __shfl_sync(0xffffffffu, my_row, j & 31);
        w[u] = (j < n) ? __shfl_sync(0xffffffffu, my_w, j & 31) : 0.f;
#pragma unroll
        for (int a = 0; a < NP; ++a) {
          const int k = (a * 32 + lane) * V;
          if (j < n && k < p.dim)
            Vec8<T>::load(D + row * p.dim + k, x[u][a]);
          else
#pragma unroll
            for (int v = 0; v < V; ++v) x[u][a][v] = 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < kGradU; ++u)
        if (j0 + u < n)
#pragma unroll
          for (int a = 0; a < NP; ++a)
#pragma unroll
            for (int v = 0; v < V; ++v) acc[a][v] = __fmaf_rn(w[u], x[u][a][v], acc[a][v]);
    }
  }
  float* out = p.dQ + wq * p.dim;
#pragma unroll
  for (int a = 0; a < NP; ++a) {
    const int k = (a * 32 + lane) * V;
    if (k < p.dim) {
      if constexpr (V == 4)
        *reinterpret_cast<float4*>(out + k) = make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
      else
        *reinterpret_cast<float2*>(out + k) = make_float2(acc[a][0], acc[a][1]);
    }
  }
}

}  // namespace mxs
