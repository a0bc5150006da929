// S4: the per-pair score is the strict left-to-right float64 sum of the fp32 row maxima
// (`maxsim/kernels.py:22-26` seq_sum_f64, called at `maxsim/forward.py:216`).  One warp computes it
// in parallel when that is provably bit-identical to the sequential chain.
//
// Every fp32 value is a multiple of its ulp 2^(E-150) (E = biased exponent, 1 for subnormals) and
// smaller than 2^(E-126).  If Emax - Emin <= 29 - ceil(log2 n), every partial sum of any subset is
// a multiple of 2^(Emin-150) below 2^(53+Emin-150): exactly representable in f64.  Then the
// sequential sum and any tree sum are both the exact sum -- bit-identical.  Pairs that fail the
// certificate (maxima spanning > 2^19 in magnitude, or non-finite) take the sequential chain.
#pragma once
#include "ptx.cuh"

namespace mxs {

// Per-lane accumulator of the certificate (sum, exponent range, finiteness).
struct CertSum {
  double s = 0.0;
  int emin = 255, emax = 0;
  bool finite = true;
  MXS_DEV void add(float v) {
    const uint32_t bits = __float_as_uint(v) & 0x7fffffffu;
    if (bits >= 0x7f800000u) finite = false;
    if (bits != 0u) {
      const int e = max((int)(bits >> 23), 1);
      emin = min(emin, e);
      emax = max(emax, e);
    }
    s += (double)v;
  }
  // butterfly over the warp: every lane ends with the totals
  MXS_DEV void warp_reduce() {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      emin = min(emin, __shfl_xor_sync(0xffffffffu, emin, o));
      emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    }
    finite = __all_sync(0xffffffffu, finite);
  }
  MXS_DEV bool exact(int n) const {
    const int log2n = 32 - __clz(max(n - 1, 1));
    return finite && (emax == 0 || emax - emin <= 29 - log2n);
  }
};

// Whole warp: S4 score of the n values load(0..n-1).  The result is valid in every lane.
template <typename Load>
MXS_DEV double warp_score_sum_fn(int n, Load load) {
  const int lane = (int)(threadIdx.x & 31u);
  CertSum c;
  for (int i = lane; i < n; i += 32) c.add(load(i));
  c.warp_reduce();
  if (c.exact(n)) return c.s;
  double t = 0.0;  // sequential fallback (rare): the reference order itself
  if (lane == 0) {
    t = (double)load(0);
    for (int i = 1; i < n; ++i) t = __dadd_rn(t, (double)load(i));
  }
  return __shfl_sync(0xffffffffu, t, 0);
}

// Whole warp: S4 score of v[0..n) (global or shared memory).
MXS_DEV double warp_score_sum(const float* v, int n) {
  return warp_score_sum_fn(n, [v](int i) { return v[i]; });
}

}  // namespace mxs
