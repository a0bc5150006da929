// Exact MaxSim backward gathers (K7, K8).  The max is resolved by the saved argmax, so the
// score is piecewise linear (maxsim/backward.py:1-21):
//   dD[r]    = sum over the CSR bucket of r (ascending source) of g[q,b] * Q[q_row(s)]   (K7)
//   dQ[q, i] = sum over b ascending of g[q,b] * D_b[argmax[q,b,i]]                       (K8)
// Both are destination-owned: one warp owns one output row, accumulates it in fp32 registers in
// the reference's order (maxsim/backward.py:165-172, :225-231) and stores it exactly once -- no
// atomics anywhere.  Lanes split the embedding axis (VEC contiguous elements per lane).
#pragma once
#include "convert.cuh"  // to_f32
#include "fastdiv.cuh"

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
  // debug ownership ledger (MXS_DEBUG_WRITES=1, else null): the owning warp of output row r
  // bumps wcount[r] once when it stores the row -- the launcher then checks every count is 1
  // (reference WriteTracking, tests/test_backward.py:94-108)
  int32_t* wcount;
  FastDiv per_q_div, lq_div;   // K7 source decoding: s / (n_docs * l_q), rem / l_q
};

MXS_DEV void note_row_write(const GradParams& p, long long r, int lane) {
  if (p.wcount != nullptr && lane == 0) atomicAdd(p.wcount + r, 1);
}

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
  note_row_write(p, r, lane);
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
  note_row_write(p, wq, lane);
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
  // source ids are < 2^31 (checked on the host): 32-bit unsigned decode
  const uint32_t per_q = (uint32_t)p.n_docs * (uint32_t)p.l_q, lq = (uint32_t)p.l_q;
  for (int t0 = lo; t0 < hi; t0 += 32) {
    const int n = min(32, hi - t0);
    // lane j decodes source t0 + j: Q row and weight
    long long my_row = 0;
    float my_w = 0.f;
    if (lane < n) {
      const uint32_t s = (uint32_t)__ldg(p.col_idx + t0 + lane);
      const uint32_t q = s / per_q, rem = s - q * per_q;
      const uint32_t b = rem / lq, i = rem - b * lq;
      my_row = (long long)q * lq + i;
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
  note_row_write(p, r, lane);
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
  note_row_write(p, wq, lane);
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

// ---------------------------------------------------------------------------------------------
// Row-group variants: a gathered row is covered by LPR lanes x 16 B, so one warp load instruction
// moves SP = 32 / LPR source rows (d = 128 bf16: two 256-B rows per LDG.128).  Lane group h
// accumulates the sources j = h (mod SP) in order (fp32, FFMA2); the SP partial sums are added
// in a fixed order at the end -- deterministic, no atomics, still destination-owned.
template <typename T>
struct Vec16;
template <>
struct Vec16<__nv_bfloat16> {
  static constexpr int N = 8;
  MXS_DEV static void load(const __nv_bfloat16* p, float (&o)[8]) {
    const uint4 t = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      o[2 * i] = __uint_as_float(w[i] << 16);
      o[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
};
template <>
struct Vec16<__half> {
  static constexpr int N = 8;
  MXS_DEV static void load(const __half* p, float (&o)[8]) {
    const uint4 t = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
      o[2 * i] = f.x;
      o[2 * i + 1] = f.y;
    }
  }
};
template <>
struct Vec16<float> {
  static constexpr int N = 4;
  MXS_DEV static void load(const float* p, float (&o)[4]) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = t.x;
    o[1] = t.y;
    o[2] = t.z;
    o[3] = t.w;
  }
};

#ifndef MXS_GRAD_GU
#define MXS_GRAD_GU 8
#endif
#ifndef GRAD_LOAD
#define GRAD_LOAD(p) __ldg(reinterpret_cast<const uint4*>(p))
#endif
constexpr int kGradGU = MXS_GRAD_GU;  // source rows per lane group and step (dD)
// dQ (K8) keeps twice as many rows in flight: 81 vs 86 us at C3, where dD runs slower with 16
// (88 vs 82 us) -- scripts/ab_grad.sh
#ifndef MXS_GRAD_GU_Q
#define MXS_GRAD_GU_Q 16
#endif
constexpr int kGradWarps = 8;  // warps per block of the row-group kernels

// Per-warp staging of one chunk of up to 32 sources: (gathered row, weight), written once by the
// lane that decoded the source and read back as a half-warp broadcast (no per-source shuffles).
struct GradStage {
  int row[32];
  float w[32];
};

// 16-byte gather load, read-only, not allocated in L1 (the rows are L2-resident and not reused by
// the SM).
MXS_DEV uint4 ldg_stream16(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

template <typename T>
MXS_DEV void unpack16(const uint4& t, float (&o)[Vec16<T>::N]);
template <>
MXS_DEV void unpack16<__nv_bfloat16>(const uint4& t, float (&o)[8]) {
  const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o[2 * i] = __uint_as_float(w[i] << 16);
    o[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
template <>
MXS_DEV void unpack16<__half>(const uint4& t, float (&o)[8]) {
  const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
    o[2 * i] = f.x;
    o[2 * i + 1] = f.y;
  }
}
template <>
MXS_DEV void unpack16<float>(const uint4& t, float (&o)[4]) {
  o[0] = __uint_as_float(t.x);
  o[1] = __uint_as_float(t.y);
  o[2] = __uint_as_float(t.z);
  o[3] = __uint_as_float(t.w);
}

// One step = kGradGU source rows per lane group.  Latency is hidden by occupancy (32-40
// registers, 64 warps per SM), not by deeper per-warp pipelining: a software-pipelined variant
// (two steps in flight, 70 registers) measured 126 us vs 87 us at C3 (scripts/probe_grad.py).
template <typename T, int LPR, int GU = kGradGU>
MXS_DEV void grad_rowgroup_chunk(const T* __restrict__ base, int dim, const GradStage& st, int n,
                                 float (&acc)[Vec16<T>::N], int h, int lp) {
  constexpr int V = Vec16<T>::N, SP = 32 / LPR;
  constexpr int G = (SP * GU > 32) ? 32 / SP : GU;  // one step never reaches past the 32 staged sources
  for (int j0 = 0; j0 < n; j0 += SP * G) {
    uint4 raw[G];
    float ws[G];
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int j = j0 + u * SP + h;  // entries past n hold (row 0, weight 0)
      ws[u] = st.w[j & 31];
      raw[u] = GRAD_LOAD(base + (long long)st.row[j & 31] * dim + lp * V);
    }
#pragma unroll
    for (int u = 0; u < G; ++u) {
      float x[V];
      unpack16<T>(raw[u], x);
#pragma unroll
      for (int v = 0; v < V; v += 2) ffma2_rn(acc[v], acc[v + 1], ws[u], ws[u], x[v], x[v + 1]);
    }
  }
}

template <typename T, int LPR>
MXS_DEV void grad_rowgroup_store(float (&acc)[Vec16<T>::N], float* out, int lane) {
  constexpr int V = Vec16<T>::N;
#pragma unroll
  for (int off = LPR; off < 32; off <<= 1)
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], off);
  if (lane < LPR) {
#pragma unroll
    for (int v = 0; v < V; v += 4)
      *reinterpret_cast<float4*>(out + lane * V + v) = make_float4(acc[v], acc[v + 1], acc[v + 2], acc[v + 3]);
  }
}

// K7 row-group: warp per destination row (CSR bucket), dim = LPR * V.  Chunks of 32 sources:
// coalesced col_idx load, source decode (two invariant divisions), weight load, staged in shared
// memory; then kGradGU rows in flight per lane group.
template <typename T, int LPR>
__global__ void __launch_bounds__(32 * kGradWarps) grad_docs_rg_kernel(const T* __restrict__ Q, const GradParams p) {
  constexpr int V = Vec16<T>::N;
  __shared__ GradStage stage[kGradWarps];
  const long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, h = lane / LPR, lp = lane % LPR;
  GradStage& st = stage[threadIdx.x >> 5];
  if (r >= p.n_dest) return;
  float acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.f;
  const int lo = __ldg(p.row_ptr + r), hi = __ldg(p.row_ptr + r + 1);
  const uint32_t per_q = (uint32_t)p.n_docs * (uint32_t)p.l_q, lq = (uint32_t)p.l_q;
  for (int t0 = lo; t0 < hi; t0 += 32) {
    const int n = min(32, hi - t0);
    int my_row = 0;
    float my_w = 0.f;
    if (lane < n) {
      const uint32_t s = (uint32_t)__ldg(p.col_idx + t0 + lane);
      const uint32_t q = fdiv(s, p.per_q_div), rem = s - q * per_q;
      const uint32_t b = fdiv(rem, p.lq_div), i = rem - b * lq;
      my_row = (int)(q * lq + i);
      my_w = __ldg(p.g + (long long)q * p.n_docs + b);
    }
    __syncwarp();  // the previous chunk's readers are done with the stage
    st.row[lane] = my_row;
    st.w[lane] = my_w;
    __syncwarp();
    grad_rowgroup_chunk<T, LPR>(Q, p.dim, st, n, acc, h, lp);
  }
  note_row_write(p, r, lane);
  grad_rowgroup_store<T, LPR>(acc, p.dD + r * p.dim, lane);
}

// K8 row-group: warp per (q, i) query row, documents b ascending (chunks of 32 documents).
template <typename T, int LPR>
__global__ void __launch_bounds__(32 * kGradWarps) grad_query_rg_kernel(const T* __restrict__ D, const GradParams p) {
  constexpr int V = Vec16<T>::N;
  __shared__ GradStage stage[kGradWarps];
  const long long wq = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, h = lane / LPR, lp = lane % LPR;
  GradStage& st = stage[threadIdx.x >> 5];
  if (wq >= (long long)p.n_q * p.l_q) return;
  const int q = (int)(wq / p.l_q), i = (int)(wq % p.l_q);
  float acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.f;
  for (int b0 = 0; b0 < p.n_docs; b0 += 32) {
    const int n = min(32, p.n_docs - b0);
    int my_row = 0;
    float my_w = 0.f;
    if (lane < n) {
      const int a_ = __ldg(p.argmax + ((long long)q * p.n_docs + b0 + lane) * p.l_q + i);
      my_w = __ldg(p.g + (long long)q * p.n_docs + b0 + lane);
      my_row = (int)(__ldg(p.doc_row_off + b0 + lane) + a_);
    }
    __syncwarp();
    st.row[lane] = my_row;
    st.w[lane] = my_w;
    __syncwarp();
    grad_rowgroup_chunk<T, LPR, MXS_GRAD_GU_Q>(D, p.dim, st, n, acc, h, lp);
  }
  note_row_write(p, wq, lane);
  grad_rowgroup_store<T, LPR>(acc, p.dQ + wq * p.dim, lane);
}

// ---------------------------------------------------------------------------------------------
// FP32 inputs, the reference's exact arithmetic: float64 accumulation in the reference's order
// (maxsim/backward.py:165-172: acc += w[s] * q_row, sources ascending per bucket, a rounded f64
// product then a rounded f64 add -- no FMA; :225-231: d_q[q] += g[q, b] * D_b[idx], b ascending),
// so dD and dQ are bit-identical to the reference's float64 gradients.  Warp per output row,
// lane k owns elements k, k + 32, ... (NC per lane); 32 sources decoded per chunk in parallel.
struct GradParams64 {
  int n_q, n_docs, l_q, dim;
  const double* g;             // [n_q, n_docs]
  const int32_t* row_ptr;      // K7
  const int32_t* col_idx;
  long long n_dest;
  double* dD;                  // [n_dest, dim]
  const int32_t* argmax;       // K8
  const long long* doc_row_off;
  double* dQ;                  // [n_q, l_q, dim]
  int32_t* wcount;             // debug ownership ledger (see GradParams)
};

template <int NC>
__global__ void __launch_bounds__(256) grad_docs_f64_kernel(const float* __restrict__ Q, const GradParams64 p) {
  const long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= p.n_dest) return;
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  const int lo = __ldg(p.row_ptr + r), hi = __ldg(p.row_ptr + r + 1);
  const long long per_q = (long long)p.n_docs * p.l_q;
  for (int t0 = lo; t0 < hi; t0 += 32) {
    const int n = min(32, hi - t0);
    long long my_row = 0;
    double my_w = 0.0;
    if (lane < n) {
      const long long s = __ldg(p.col_idx + t0 + lane);
      const long long q = s / per_q, b = (s / p.l_q) % p.n_docs;
      my_row = q * p.l_q + s % p.l_q;
      my_w = __ldg(p.g + q * p.n_docs + b);
    }
    for (int j = 0; j < n; ++j) {
      const long long row = __shfl_sync(0xffffffffu, my_row, j);
      const double w = __shfl_sync(0xffffffffu, my_w, j);
      const float* src = Q + row * p.dim;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int k = c * 32 + lane;
        if (k < p.dim) acc[c] = __dadd_rn(acc[c], __dmul_rn(w, (double)__ldg(src + k)));
      }
    }
  }
  if (p.wcount != nullptr && lane == 0) atomicAdd(p.wcount + r, 1);
  double* out = p.dD + r * p.dim;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int k = c * 32 + lane;
    if (k < p.dim) out[k] = acc[c];
  }
}

template <int NC>
__global__ void __launch_bounds__(256) grad_query_f64_kernel(const float* __restrict__ D, const GradParams64 p) {
  const long long wq = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wq >= (long long)p.n_q * p.l_q) return;
  const int q = (int)(wq / p.l_q), i = (int)(wq % p.l_q);
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  for (int b0 = 0; b0 < p.n_docs; b0 += 32) {
    const int n = min(32, p.n_docs - b0);
    long long my_row = 0;
    double my_w = 0.0;
    if (lane < n) {
      my_row = __ldg(p.doc_row_off + b0 + lane) + __ldg(p.argmax + ((long long)q * p.n_docs + b0 + lane) * p.l_q + i);
      my_w = __ldg(p.g + (long long)q * p.n_docs + b0 + lane);
    }
    for (int j = 0; j < n; ++j) {
      const long long row = __shfl_sync(0xffffffffu, my_row, j);
      const double w = __shfl_sync(0xffffffffu, my_w, j);
      const float* src = D + row * p.dim;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int k = c * 32 + lane;
        if (k < p.dim) acc[c] = __dadd_rn(acc[c], __dmul_rn(w, (double)__ldg(src + k)));
      }
    }
  }
  if (p.wcount != nullptr && lane == 0) atomicAdd(p.wcount + wq, 1);
  double* out = p.dQ + wq * p.dim;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int k = c * 32 + lane;
    if (k < p.dim) out[k] = acc[c];
  }
}

// out[0] = number of rows whose write count is not exactly 1, out[1] = the first such row (or -1)
__global__ void __launch_bounds__(256) write_once_check_kernel(const int32_t* __restrict__ wcount, long long n,
                                                               unsigned long long* out) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
    if (wcount[r] != 1) {
      atomicAdd(out, 1ull);
      atomicMin(out + 1, (unsigned long long)r);
    }
}

}  // namespace mxs
