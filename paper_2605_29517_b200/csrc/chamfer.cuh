// Chamfer distance (maxsim/chamfer.py:49-199): the hard-selection pattern with an online MIN
// over squared Euclidean distances, bit-exact with the reference's float32 arithmetic.
//
//   sq_norms   : n[i] = fl(x0*x0), then fl(n + fl(xk*xk)) for k = 1..dim-1   (maxsim/kernels.py:41-47)
//   distance   : d = fl(fl(fl(<p,s>) * -2) + |p|^2) + |s|^2 with <p,s> the S1 sequential fold
//                (maxsim/kernels.py:29-38, 50-66)
//   fold       : strict <, columns ascending -> lowest index on ties (maxsim/kernels.py:69-93)
// Point clouds are 3-D (any dim; <= kChDimMax keeps the point in registers): K = 3 gives a tensor core nothing to do, so
// this is an FP32-ALU kernel -- one thread per point of the first set, the second set streamed
// through shared memory in tiles, every product / add an explicit _rn intrinsic (no FMA
// contraction) so the bits match numpy's.
//
// Backward (maxsim/chamfer.py:167-199), float64 like the reference, same operation order:
//   dP[i]  = c_ps * (p_i - s_{a1[i]})                     (gather half)
//   dP[r] += c_sp * (p_r - s_j)  for j in CSR_p bucket r  (scatter half, ascending j)
// and symmetrically for dS; the CSR inversions come from the shared builder (K6).
#pragma once
#include "ptx.cuh"

namespace mxs {

constexpr int kChDimMax = 16;
constexpr int kChTile = 1024;  // second-set points per shared-memory tile
constexpr int kChThreads = 256;

__global__ void __launch_bounds__(256) sq_norms_kernel(const float* __restrict__ X, long long rows, int dim,
                                                       float* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const float* x = X + i * dim;
  float acc = __fmul_rn(x[0], x[0]);
  for (int k = 1; k < dim; ++k) acc = __fadd_rn(acc, __fmul_rn(x[k], x[k]));
  out[i] = acc;
}

template <int DIM>
__global__ void __launch_bounds__(kChThreads) chamfer_nn_kernel(const float* __restrict__ A,
                                                                const float* __restrict__ an, long long n,
                                                                const float* __restrict__ B,
                                                                const float* __restrict__ bn, long long m, int dim,
                                                                float* __restrict__ best, int32_t* __restrict__ idx) {
  constexpr int kTile = DIM > 0 ? kChTile : kChTile / 2;  // <= 32 KB of static shared memory
  __shared__ float sB[kTile * (DIM > 0 ? DIM : kChDimMax)];
  __shared__ float sBn[kTile];
  const int D = DIM > 0 ? DIM : dim;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  float a[kChDimMax];
  float ai = 0.f;
  if (i < n) {
#pragma unroll
    for (int k = 0; k < kChDimMax; ++k)
      if (k < D) a[k] = A[i * D + k];
    ai = an[i];
  }
  float bd = INFINITY;
  int bj = 0;
  for (long long t0 = 0; t0 < m; t0 += kTile) {
    const int cnt = (int)min((long long)kTile, m - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * D; e += blockDim.x) sB[e] = B[t0 * D + e];
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) sBn[e] = bn[t0 + e];
    __syncthreads();
    if (i < n) {
      for (int j = 0; j < cnt; ++j) {
        const float* b = sB + j * D;
        float dot = __fmul_rn(a[0], b[0]);
#pragma unroll
        for (int k = 1; k < kChDimMax; ++k)
          if (k < D) dot = __fadd_rn(dot, __fmul_rn(a[k], b[k]));
        const float d = __fadd_rn(__fadd_rn(__fmul_rn(dot, -2.0f), ai), sBn[j]);
        if (d < bd) {  // strict: the lowest index wins ties
          bd = d;
          bj = (int)(t0 + j);
        }
      }
    }
  }
  if (i < n) {
    best[i] = bd;
    idx[i] = bj;
  }
}

// Any dimension (> kChDimMax): the point of the first set stays in global memory (L1-resident,
// one row per thread), the second set streams through shared memory in tiles of 8192 floats.
// Same S1 fold, same strict-< scan, so the bits match the register kernel's and the reference's.
__global__ void __launch_bounds__(kChThreads) chamfer_nn_any_kernel(const float* __restrict__ A,
                                                                    const float* __restrict__ an, long long n,
                                                                    const float* __restrict__ B,
                                                                    const float* __restrict__ bn, long long m,
                                                                    int dim, float* __restrict__ best,
                                                                    int32_t* __restrict__ idx) {
  constexpr int kFloats = 8192;
  __shared__ float sB[kFloats];
  __shared__ float sBn[kFloats / (kChDimMax + 1) + 1];  // dim > kChDimMax -> tile <= 481
  const int tile = max(1, kFloats / dim);
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const float* a = A + (i < n ? i : 0) * dim;
  const float ai = i < n ? an[i] : 0.f;
  float bd = INFINITY;
  int bj = 0;
  for (long long t0 = 0; t0 < m; t0 += tile) {
    const int cnt = (int)min((long long)tile, m - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * dim; e += blockDim.x) sB[e] = B[t0 * dim + e];
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) sBn[e] = bn[t0 + e];
    __syncthreads();
    if (i < n) {
      for (int j = 0; j < cnt; ++j) {
        const float* b = sB + j * dim;
        float dot = __fmul_rn(a[0], b[0]);
        for (int k = 1; k < dim; ++k) dot = __fadd_rn(dot, __fmul_rn(a[k], b[k]));
        const float d = __fadd_rn(__fadd_rn(__fmul_rn(dot, -2.0f), ai), sBn[j]);
        if (d < bd) {
          bd = d;
          bj = (int)(t0 + j);
        }
      }
    }
  }
  if (i < n) {
    best[i] = bd;
    idx[i] = bj;
  }
}

// One thread per (destination point r, coordinate k): the gather half first, then the CSR
// bucket in ascending source order (maxsim/chamfer.py:178-197).
__global__ void __launch_bounds__(256) chamfer_grad_kernel(const float* __restrict__ X, long long nx,
                                                           const float* __restrict__ Y, int dim,
                                                           const int32_t* __restrict__ nn,       // [nx] into Y
                                                           const int32_t* __restrict__ row_ptr,  // [nx + 1]
                                                           const int32_t* __restrict__ col_idx,  // sources in Y
                                                           double c_gather, double c_scatter,
                                                           double* __restrict__ dX) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nx * dim) return;
  const long long r = t / dim;
  const int k = (int)(t - r * dim);
  const double xr = (double)X[r * dim + k];
  double acc = __dadd_rn(0.0, __dmul_rn(c_gather, __dsub_rn(xr, (double)Y[(long long)nn[r] * dim + k])));
  for (int e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
    const long long j = col_idx[e];
    acc = __dadd_rn(acc, __dmul_rn(c_scatter, __dsub_rn(xr, (double)Y[j * dim + k])));
  }
  dX[t] = acc;
}

}  // namespace mxs
