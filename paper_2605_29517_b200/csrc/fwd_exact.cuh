// Bit-exact FP32 MaxSim forward on CUDA cores (K10).
//
// Restates the reference element arithmetic exactly (S1): every similarity is the strict
// left-to-right fp32 fold `acc = fl(acc + fl(q_k * d_k))` of `maxsim/kernels.py:29-38`
// (dot_block), with no FMA contraction (__fmul_rn / __fadd_rn), so scores and argmax match
// the numpy oracle bit for bit, including ties.  Masking (S2) and the strict-> lowest-index
// fold (S3) follow `maxsim/forward.py:146-155` and `maxsim/kernels.py:69-93`.
//
// One CTA folds one (query, document) pair at a time: 32 query rows x 64 document tokens per
// sub-tile, 8 accumulators per thread, the embedding axis streamed through shared memory in
// chunks of 64 (the fold order over k is preserved across chunks).  Four k steps per LDS.128
// (query row and the 8 broadcast document rows); one rounding per product and per add, in k order.
#pragma once
#include "convert.cuh"

namespace mxs {

struct FwdExactParams {
  int n_q, l_q, n_docs, l_pad, dim;
  const int32_t* valid_lens;  // nullable
  const long long* cu_seqlens;  // packed layout when non-null (then l_pad unused)
  float* rowmax;
  int32_t* argmax;
};

constexpr int kExRows = 32, kExCols = 64, kExK = 64, kExThreads = 256;
constexpr int kExStride = kExK + 4;  // row pitch in floats: 16-B aligned rows, conflict-free LDS.128

// rows x kw elements of a row-major [*, dim] operand starting at (row0, k0) -> smem [rows][kExStride],
// zero outside (rows_valid, kw).  fp32 with dim % 4 == 0: float4 loads.
template <typename T, int ROWS>
MXS_DEV void ex_stage(float (*dst)[kExStride], const T* src, int rows_valid, int dim, int k0, int kw, bool vec4) {
  if constexpr (sizeof(T) == 4) {
    if (vec4) {
      for (int e = threadIdx.x; e < ROWS * (kExK / 4); e += kExThreads) {
        const int rr = e / (kExK / 4), kk = (e % (kExK / 4)) * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (rr < rows_valid && kk < kw) v = __ldg(reinterpret_cast<const float4*>(src + (long long)rr * dim + k0 + kk));
        *reinterpret_cast<float4*>(&dst[rr][kk]) = v;
      }
      return;
    }
  }
  for (int e = threadIdx.x; e < ROWS * kExK; e += kExThreads) {
    const int rr = e / kExK, kk = e % kExK;
    dst[rr][kk] = (rr < rows_valid && kk < kw) ? to_f32(src[(long long)rr * dim + k0 + kk]) : 0.f;
  }
}

// one k step of the sequential fold for the thread's 8 columns: __fmul_rn then __fadd_rn (scalar on
// purpose -- ptxas contracts a packed mul.rn.f32x2 + add.rn.f32x2 pair into FFMA2, which would
// round once instead of twice)
template <bool kFirst>
MXS_DEV void ex_step(float (&acc)[8], float qv, const float (&d)[8]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float t = __fmul_rn(qv, d[c]);
    acc[c] = kFirst ? t : __fadd_rn(acc[c], t);
  }
}

template <typename T>
__global__ void __launch_bounds__(kExThreads, 3) fwd_exact_kernel(const T* __restrict__ Q, const T* __restrict__ D,
                                                                const FwdExactParams p) {
  __shared__ __align__(16) float sQ[kExRows][kExStride];
  __shared__ __align__(16) float sD[kExCols][kExStride];
  __shared__ float xm[8][kExRows];
  __shared__ int xi[8][kExRows];
  const int tid = threadIdx.x;
  const int i = tid & 31;   // query row within the row tile
  const int jg = tid >> 5;  // column phase: columns jg, jg+8, ...
  const long long n_pairs = (long long)p.n_q * p.n_docs;
  const bool vec4 = sizeof(T) == 4 && (p.dim & 3) == 0;
  for (long long pr = blockIdx.x; pr < n_pairs; pr += gridDim.x) {
    const int q = (int)(pr / p.n_docs), b = (int)(pr % p.n_docs);
    long long drow0;
    int vl;
    if (p.cu_seqlens) {
      drow0 = p.cu_seqlens[b];
      vl = (int)(p.cu_seqlens[b + 1] - drow0);
    } else {
      drow0 = (long long)b * p.l_pad;
      vl = p.valid_lens ? min(max(p.valid_lens[b], 0), p.l_pad) : p.l_pad;  // clamped: memory-safe on unvalidated input
    }
    const T* qbase = Q + (long long)q * p.l_q * p.dim;
    const T* dbase = D + drow0 * p.dim;
    const bool v4 = vec4 && ((reinterpret_cast<uintptr_t>(qbase) | reinterpret_cast<uintptr_t>(dbase)) & 15u) == 0;
    for (int r0 = 0; r0 < p.l_q; r0 += kExRows) {
      float m = -INFINITY;
      int ix = 0;
      for (int c0 = 0; c0 < vl; c0 += kExCols) {
        float acc[8];
        for (int k0 = 0; k0 < p.dim; k0 += kExK) {
          const int kw = min(kExK, p.dim - k0);
          __syncthreads();
          ex_stage<T, kExRows>(sQ, qbase + (long long)r0 * p.dim, p.l_q - r0, p.dim, k0, kw, v4);
          ex_stage<T, kExCols>(sD, dbase + (long long)c0 * p.dim, vl - c0, p.dim, k0, kw, v4);
          __syncthreads();
          const int kw4 = kw & ~3;
          for (int k = 0; k < kw4; k += 4) {
            const float4 qv = *reinterpret_cast<const float4*>(&sQ[i][k]);
            float d0[8], d1[8], d2[8], d3[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const float4 dv = *reinterpret_cast<const float4*>(&sD[jg + 8 * c][k]);
              d0[c] = dv.x;
              d1[c] = dv.y;
              d2[c] = dv.z;
              d3[c] = dv.w;
            }
            if (k0 == 0 && k == 0)
              ex_step<true>(acc, qv.x, d0);
            else
              ex_step<false>(acc, qv.x, d0);
            ex_step<false>(acc, qv.y, d1);
            ex_step<false>(acc, qv.z, d2);
            ex_step<false>(acc, qv.w, d3);
          }
          for (int k = kw4; k < kw; ++k) {  // dim % 4 tail
            float dk[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) dk[c] = sD[jg + 8 * c][k];
            if (k0 == 0 && k == 0)
              ex_step<true>(acc, sQ[i][k], dk);
            else
              ex_step<false>(acc, sQ[i][k], dk);
          }
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int j = c0 + jg + 8 * c;
          if (j < vl && acc[c] > m) {
            m = acc[c];
            ix = j;
          }
        }
      }
      xm[jg][i] = m;
      xi[jg][i] = ix;
      __syncthreads();
      if (jg == 0 && r0 + i < p.l_q) {
        float bm = xm[0][i];
        int bi = xi[0][i];
        for (int w = 1; w < 8; ++w) {
          const float om = xm[w][i];
          const int oi = xi[w][i];
          if (om > bm || (om == bm && oi < bi)) {
            bm = om;
            bi = oi;
          }
        }
        const long long o = ((long long)q * p.n_docs + b) * p.l_q + r0 + i;
        p.rowmax[o] = bm;
        if (p.argmax) p.argmax[o] = bi;
      }
      __syncthreads();
    }
  }
}

// fp32 rows, dim % 4 == 0, 16-B aligned: the same fold with the (column tile, k chunk) stages
// double-buffered through cp.async (16-B LDGSTS, zero-fill outside the valid rows / width), so
// stage s + 1 streams in while stage s is folded.  Dynamic smem: 2 x (32 + 64) rows x 68 floats.
MXS_DEV void cp_async16(void* smem_dst, const void* gsrc, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)), "l"(gsrc),
               "r"(valid ? 16 : 0)
               : "memory");
}
MXS_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
MXS_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr size_t kExV4Smem = (size_t)2 * (kExRows + kExCols) * kExStride * sizeof(float);

__global__ void __launch_bounds__(kExThreads, 3) fwd_exact_f32v_kernel(const float* __restrict__ Q,
                                                                       const float* __restrict__ D,
                                                                       const FwdExactParams p) {
  extern __shared__ __align__(16) float ex_smem[];
  float(*sQ)[kExRows][kExStride] = reinterpret_cast<float(*)[kExRows][kExStride]>(ex_smem);
  float(*sD)[kExCols][kExStride] = reinterpret_cast<float(*)[kExCols][kExStride]>(ex_smem + 2 * kExRows * kExStride);
  __shared__ float xm[8][kExRows];
  __shared__ int xi[8][kExRows];
  const int tid = threadIdx.x;
  const int i = tid & 31;
  const int jg = tid >> 5;
  const long long n_pairs = (long long)p.n_q * p.n_docs;
  const int nk = (p.dim + kExK - 1) / kExK;
  for (long long pr = blockIdx.x; pr < n_pairs; pr += gridDim.x) {
    const int q = (int)(pr / p.n_docs), b = (int)(pr % p.n_docs);
    long long drow0;
    int vl;
    if (p.cu_seqlens) {
      drow0 = p.cu_seqlens[b];
      vl = (int)(p.cu_seqlens[b + 1] - drow0);
    } else {
      drow0 = (long long)b * p.l_pad;
      vl = p.valid_lens ? min(max(p.valid_lens[b], 0), p.l_pad) : p.l_pad;  // clamped: memory-safe on unvalidated input
    }
    const float* qbase = Q + (long long)q * p.l_q * p.dim;
    const float* dbase = D + drow0 * p.dim;
    const int nc = (vl + kExCols - 1) / kExCols;
    for (int r0 = 0; r0 < p.l_q; r0 += kExRows) {
      auto issue = [&](int st, int buf) {
        const int c0 = (st / nk) * kExCols, k0 = (st % nk) * kExK;
        const int kw = min(kExK, p.dim - k0);
        for (int e = tid; e < kExRows * (kExK / 4); e += kExThreads) {
          const int rr = e / (kExK / 4), kk = (e % (kExK / 4)) * 4;
          const bool ok = r0 + rr < p.l_q && kk < kw;
          cp_async16(&sQ[buf][rr][kk], ok ? qbase + (long long)(r0 + rr) * p.dim + k0 + kk : qbase, ok);
        }
        for (int e = tid; e < kExCols * (kExK / 4); e += kExThreads) {
          const int cc = e / (kExK / 4), kk = (e % (kExK / 4)) * 4;
          const bool ok = c0 + cc < vl && kk < kw;
          cp_async16(&sD[buf][cc][kk], ok ? dbase + (long long)(c0 + cc) * p.dim + k0 + kk : dbase, ok);
        }
        cp_async_commit();
      };
      float m = -INFINITY;
      int ix = 0;
      float acc[8];
      const int nst = nc * nk;
      if (nst > 0) issue(0, 0);
      for (int st = 0; st < nst; ++st) {
        const int buf = st & 1;
        if (st + 1 < nst) {
          issue(st + 1, buf ^ 1);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncthreads();
        const int c0 = (st / nk) * kExCols, k0 = (st % nk) * kExK;
        const int kw = min(kExK, p.dim - k0);
        for (int k = 0; k < kw; k += 4) {
          const float4 qv = *reinterpret_cast<const float4*>(&sQ[buf][i][k]);
          float d0[8], d1[8], d2[8], d3[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 dv = *reinterpret_cast<const float4*>(&sD[buf][jg + 8 * c][k]);
            d0[c] = dv.x;
            d1[c] = dv.y;
            d2[c] = dv.z;
            d3[c] = dv.w;
          }
          if (k0 == 0 && k == 0)
            ex_step<true>(acc, qv.x, d0);
          else
            ex_step<false>(acc, qv.x, d0);
          ex_step<false>(acc, qv.y, d1);
          ex_step<false>(acc, qv.z, d2);
          ex_step<false>(acc, qv.w, d3);
        }
        if (st % nk == nk - 1) {  // column tile complete: fold in column order
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int j = c0 + jg + 8 * c;
            if (j < vl && acc[c] > m) {
              m = acc[c];
              ix = j;
            }
          }
        }
        __syncthreads();  // buffer `buf` is refilled by the issue of stage st + 2
      }
      xm[jg][i] = m;
      xi[jg][i] = ix;
      __syncthreads();
      if (jg == 0 && r0 + i < p.l_q) {
        float bm = xm[0][i];
        int bi = xi[0][i];
        for (int w = 1; w < 8; ++w) {
          const float om = xm[w][i];
          const int oi = xi[w][i];
          if (om > bm || (om == bm && oi < bi)) {
            bm = om;
            bi = oi;
          }
        }
        const long long o = ((long long)q * p.n_docs + b) * p.l_q + r0 + i;
        p.rowmax[o] = bm;
        if (p.argmax) p.argmax[o] = bi;
      }
      __syncthreads();
    }
  }
}

// INT8 x INT8 on CUDA cores, for widths beyond the tensor-core tiles (maxsim/quant.py:171-179):
// exact int32 dot (wrapping like numpy's int32 matmul), f32(acc) round-to-nearest, then
// fl(fl(acc * s_q) * s_d) in the reference order, masked strict-> fold.  Same tiling as
// fwd_exact_kernel.
__global__ void __launch_bounds__(kExThreads, 3) fwd_exact_i8_kernel(const int8_t* __restrict__ Q,
                                                                     const float* __restrict__ qs,
                                                                     const int8_t* __restrict__ D,
                                                                     const float* __restrict__ ds,
                                                                     const FwdExactParams p) {
  __shared__ int sQ[kExRows][kExK + 1];
  __shared__ int sD[kExCols][kExK + 1];
  __shared__ float xm[8][kExRows];
  __shared__ int xi[8][kExRows];
  const int tid = threadIdx.x;
  const int i = tid & 31;
  const int jg = tid >> 5;
  const long long n_pairs = (long long)p.n_q * p.n_docs;
  for (long long pr = blockIdx.x; pr < n_pairs; pr += gridDim.x) {
    const int q = (int)(pr / p.n_docs), b = (int)(pr % p.n_docs);
    const int vl = p.valid_lens ? min(max(p.valid_lens[b], 0), p.l_pad) : p.l_pad;  // clamped: memory-safe on unvalidated input
    const int8_t* qbase = Q + (long long)q * p.l_q * p.dim;
    const int8_t* dbase = D + (long long)b * p.l_pad * p.dim;
    for (int r0 = 0; r0 < p.l_q; r0 += kExRows) {
      const float sq = (r0 + i < p.l_q) ? qs[(long long)q * p.l_q + r0 + i] : 1.f;
      float m = -INFINITY;
      int ix = 0;
      for (int c0 = 0; c0 < vl; c0 += kExCols) {
        int acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int k0 = 0; k0 < p.dim; k0 += kExK) {
          const int kw = min(kExK, p.dim - k0);
          __syncthreads();
          for (int e = tid; e < kExRows * kExK; e += kExThreads) {
            const int rr = e / kExK, kk = e % kExK;
            sQ[rr][kk] = (r0 + rr < p.l_q && kk < kw) ? (int)qbase[(long long)(r0 + rr) * p.dim + k0 + kk] : 0;
          }
          for (int e = tid; e < kExCols * kExK; e += kExThreads) {
            const int cc = e / kExK, kk = e % kExK;
            sD[cc][kk] = (c0 + cc < vl && kk < kw) ? (int)dbase[(long long)(c0 + cc) * p.dim + k0 + kk] : 0;
          }
          __syncthreads();
          for (int k = 0; k < kw; ++k) {
            const int qv = sQ[i][k];
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[c] = (int)((unsigned)acc[c] + (unsigned)(qv * sD[jg + 8 * c][k]));
          }
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int j = c0 + jg + 8 * c;
          if (j < vl) {
            const float v = __fmul_rn(__fmul_rn(__int2float_rn(acc[c]), sq), ds[(long long)b * p.l_pad + j]);
            if (v > m) {
              m = v;
              ix = j;
            }
          }
        }
      }
      xm[jg][i] = m;
      xi[jg][i] = ix;
      __syncthreads();
      if (jg == 0 && r0 + i < p.l_q) {
        float bm = xm[0][i];
        int bi = xi[0][i];
        for (int w = 1; w < 8; ++w) {
          const float om = xm[w][i];
          const int oi = xi[w][i];
          if (om > bm || (om == bm && oi < bi)) {
            bm = om;
            bi = oi;
          }
        }
        const long long o = ((long long)q * p.n_docs + b) * p.l_q + r0 + i;
        p.rowmax[o] = bm;
        if (p.argmax) p.argmax[o] = bi;
      }
      __syncthreads();
    }
  }
}

}  // namespace mxs
