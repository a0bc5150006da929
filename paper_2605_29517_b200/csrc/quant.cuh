// Per-token symmetric INT8 quantisation (K4), bit-exact with maxsim/quant.py:104-120:
//   scale = fl32(maxabs / levels), 1e-12 for an all-zero row (ZERO_ROW_SCALE, quant.py:27)
//   q     = clamp(rint_half_even(fl32(x / scale)), -levels, levels)
// One warp per row; IEEE division (__fdiv_rn) and rintf, no fast-math.
#pragma once
#include "convert.cuh"  // to_f32

namespace mxs {

// rint_half_even(fl32(x / s)) without an IEEE division per element: r = 1/s is within 1 ulp, so
// y = x * r is within a few ulp of the correctly rounded quotient; the nearest integer can only
// differ if y lies within a hair of a half-integer, and exactly those elements (rare) take the
// exact __fdiv_rn path.  |x / s| <= levels + 1 <= 128, so 2^-12 is >> 4 ulp of y.
MXS_DEV float quant_round(float x, float s, float r) {
  const float y = __fmul_rn(x, r);
  const float fy = floorf(y);
  const float frac = y - fy;  // exact (Sterbenz-range subtraction)
  if (fabsf(frac - 0.5f) < 0x1p-12f) return rintf(__fdiv_rn(x, s));
  return rintf(y);
}

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
  const float lv = (float)levels, r = __frcp_rn(s);
  int8_t* qr = q + warp * dim;
  for (int k = lane; k < dim; k += 32) {
    float t = quant_round(to_f32(xr[k]), s, r);
    t = fminf(fmaxf(t, -lv), lv);
    qr[k] = (int8_t)(int)t;
  }
}

// Vectorised variant for bf16 / f16 rows with dim == 128: a warp owns a row, a lane 4 elements
// (one 8-byte load, one 4-byte int8 store); the row stays in registers for both passes.
template <typename T>
__global__ void __launch_bounds__(256) quantize128_kernel(const T* __restrict__ x, long long rows, int levels,
                                                          int8_t* __restrict__ q, float* __restrict__ scale) {
  static_assert(sizeof(T) == 2, "16-bit rows");
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const uint2 raw = __ldg(reinterpret_cast<const uint2*>(x + warp * 128) + lane);
  float v[4];
  {
    const T* h = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = to_f32(h[j]);
  }
  float mx = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3])));
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float s = __fdiv_rn(mx, (float)levels);
  if (s == 0.f) s = 1e-12f;
  if (lane == 0) scale[warp] = s;
  const float r = __frcp_rn(s), lv = (float)levels;
  uint32_t packed = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float t = fminf(fmaxf(quant_round(v[j], s, r), -lv), lv);
    packed |= ((uint32_t)(uint8_t)(int8_t)(int)t) << (8 * j);
  }
  reinterpret_cast<uint32_t*>(q + warp * 128)[lane] = packed;
}


// Streaming variant for bf16 / f16 rows with dim == 128 (the C4 corpus, HBM-bound): 8 lanes own
// a row (32 B = 16 elements each, so the per-row reduction / division / reciprocal is amortised
// over 16 elements per lane), each 8-lane group keeps two rows in flight, and the grid is
// persistent (grid-stride), so one row's arithmetic overlaps the next rows' loads.  Same
// arithmetic as quantize128_kernel (bit-exact); the rounding check is on the distance to the
// nearest integer (|y - rint(y)| near 1/2 <=> y near a half-integer).
MXS_DEV float quant_round_fast(float x, float s, float r) {
  const float y = __fmul_rn(x, r);
  const float t = rintf(y);
  if (fabsf(y - t) > 0.5f - 0x1p-12f) return rintf(__fdiv_rn(x, s));
  return t;
}

// The same rounding for a pair, without FRND / F2I: z = fl(y + 1.5 * 2^23) rounds y to the
// nearest integer, ties to even (exactly rintf for |y| < 2^22), and z's bit pattern is
// 0x4B400000 + rint(y), whose low byte is rint(y) as an int8 (|rint(y)| <= 127 here).  The
// half-integer check uses t = z - 1.5 * 2^23 (exact).  Packed FMUL2 / FADD2 on the FMA pipe
// instead of FRND + F2I per element.
MXS_DEV void quant_round_magic2(uint32_t& o0, uint32_t& o1, float x0, float x1, float s, float r) {
  constexpr float kM = 12582912.0f;  // 1.5 * 2^23
  float y0, y1, z0, z1, t0, t1, d0, d1;
  fmul2_rn(y0, y1, x0, x1, r, r);
  fadd2_rn(z0, z1, y0, y1, kM, kM);
  fadd2_rn(t0, t1, z0, z1, -kM, -kM);
  fadd2_rn(d0, d1, y0, y1, -t0, -t1);
  o0 = __float_as_uint(z0);
  o1 = __float_as_uint(z1);
  // near a half-integer (rare): the exact division decides, as in quant_round_fast.  (Collecting
  // the flags and redoing flagged elements in one loop after the row measured slower: 0.98 vs
  // 0.82 ms at C4.)
  if (fabsf(d0) > 0.5f - 0x1p-12f) o0 = (uint32_t)(int)rintf(__fdiv_rn(x0, s));
  if (fabsf(d1) > 0.5f - 0x1p-12f) o1 = (uint32_t)(int)rintf(__fdiv_rn(x1, s));
}

template <typename T, int U>
__global__ void __launch_bounds__(256) quantize128_stream_kernel(const T* __restrict__ x, long long rows, int levels,
                                                                 int8_t* __restrict__ q, float* __restrict__ scale) {
  static_assert(sizeof(T) == 2, "16-bit rows");
  const int l8 = threadIdx.x & 7;
  const long long grp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 3;  // 8-lane group id
  const long long n_grp = ((long long)gridDim.x * blockDim.x) >> 3;
  const float lv = (float)levels;
  // the next pass's rows are loaded before this pass's arithmetic (software prefetch: twice the
  // bytes in flight per lane group)
  auto load_rows = [&](long long r0, uint4 (&raw)[U][2]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long rr = r0 + u * n_grp;
      raw[u][0] = raw[u][1] = make_uint4(0u, 0u, 0u, 0u);
      if (rr < rows) {
        const uint4* src = reinterpret_cast<const uint4*>(x + rr * 128) + 2 * l8;
        raw[u][0] = __ldg(src);
        raw[u][1] = __ldg(src + 1);
      }
    }
  };
  uint4 nxt[U][2];
  load_rows(grp, nxt);
  for (long long r0 = grp; r0 - grp < rows; r0 += U * n_grp) {  // warp-uniform trip count
    long long row[U];
#pragma unroll
    for (int u = 0; u < U; ++u) row[u] = r0 + u * n_grp;
    uint4 raw[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      raw[u][0] = nxt[u][0];
      raw[u][1] = nxt[u][1];
    }
    load_rows(r0 + U * n_grp, nxt);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float v[16];
      const T* h = reinterpret_cast<const T*>(&raw[u][0]);
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = to_f32(h[j]);
      float mx = fabsf(v[0]);
#pragma unroll
      for (int j = 1; j < 16; ++j) mx = fmaxf(mx, fabsf(v[j]));
#pragma unroll
      for (int o = 4; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));  // within the 8 lanes
      if (row[u] < rows) {
        float s = __fdiv_rn(mx, lv);
        if (s == 0.f) s = 1e-12f;
        if (l8 == 0) scale[row[u]] = s;
        const float r = __frcp_rn(s);
        // no clamp needed here: |x| <= maxabs and s = fl(maxabs / levels) give |x / s| <= levels
        // (1 + 2^-23), and x * fl(1 / s) adds two more ulps -- far below the 0.5 that rint would
        // need to reach levels + 1 (zero rows: x = 0).  The reference's clip is a no-op on them.
        uint32_t w[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t t[4];
#pragma unroll
          for (int j = 0; j < 4; j += 2) quant_round_magic2(t[j], t[j + 1], v[4 * c + j], v[4 * c + j + 1], s, r);
          // the low byte of each rounded value's bit pattern is its int8 two's-complement byte
          w[c] = __byte_perm(__byte_perm(t[0], t[1], 0x0040), __byte_perm(t[2], t[3], 0x0040), 0x5410);
        }
        reinterpret_cast<uint4*>(q + row[u] * 128)[l8] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
}

}  // namespace mxs
