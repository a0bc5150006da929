// Per-token symmetric INT8 quantisation (K4), bit-exact with maxsim/quant.py:104-120:
//   scale = fl32(maxabs / levels), 1e-12 for an all-zero row (ZERO_ROW_SCALE, quant.py:27)
//   q     = clamp(rint_half_even(fl32(x / scale)), -levels, levels)
// One warp per row; IEEE division (__fdiv_rn) and rintf, no fast-math.
#pragma once
#include "fwd_exact.cuh"  // to_f32

namespace mxs {

template <typename T>
__global__ void __launch_bounds__(256) quantize_kernel(const T* __restrict__ x, long long rows, int dim, int levels,
                                                       int8_t* __restrict__ q, float* __restrict__ scale) {
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const T* xr = x + warp * dim;
  float mx = 0.f;
  for (int k = lane; k < dim; k += 32) mx = fmaxf(mx, fabsf(to_f32(xr[k])));
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float s = __fdiv_rn(mx, (float)levels);
  if (s == 0.f) s = 1e-12f;
  if (lane == 0) scale[warp] = s;
  const float lv = (float)levels;
  int8_t* qr = q + warp * dim;
  for (int k = lane; k < dim; k += 32) {
    float t = rintf(__fdiv_rn(to_f32(xr[k]), s));
    t = fminf(fmaxf(t, -lv), lv);
    qr[k] = (int8_t)(int)t;
  }
}

}  // namespace mxs
