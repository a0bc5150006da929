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

// Exact sum under the certificate in INTEGER fixed point (no FP64 per value: on this B200 an
// F2F + DADD per value, even in a side warp, cost several percent of a tensor-core kernel's
// throughput).  With emax the largest biased exponent and S = 29 - ceil(log2 n), every value is
// M * 2^(e - 150) with a 24-bit significand M, i.e. the integer M << (e - emax + S) in units of
// 2^(emax - 150 - S).  Under the certificate (emax - emin <= S) every shift is >= 0, every term is
// < 2^(24 + S) and the sum of the n terms is < 2^53: an exact int64 that converts to f64 exactly
// -- the exact sum, i.e. the sequential f64 sum bit for bit.
MXS_DEV int fix_shift(int n) { return 29 - (32 - __clz(max(n - 1, 1))); }
MXS_DEV long long fix_term(uint32_t bits, int emax, int S) {  // 0 for +-0
  const uint32_t mag = bits & 0x7fffffffu;
  const int e = (int)(mag >> 23);
  const int sh = max(e, 1) - emax + S;
  if (mag == 0u || sh < 0) return 0ll;  // sh < 0 only when the certificate fails (the chain is used)
  const long long t = (long long)(e ? ((mag & 0x7fffffu) | 0x800000u) : mag) << sh;
  return (bits >> 31) ? -t : t;
}
MXS_DEV double fix_to_double(long long k, int emax, int S) {  // k * 2^(emax - 150 - S), exact
  return __dmul_rn(__ll2double_rn(k), __longlong_as_double((long long)(emax - 150 - S + 1023) << 52));
}
MXS_DEV void exp_range(uint32_t bits, int& emin, int& emax, bool& fin) {
  const uint32_t mag = bits & 0x7fffffffu;
  if (mag >= 0x7f800000u) fin = false;
  if (mag != 0u) {
    const int e = max((int)(mag >> 23), 1);
    emin = min(emin, e);
    emax = max(emax, e);
  }
}
MXS_DEV bool certified(int emin, int emax, bool fin, int n) {
  return fin && emax != 0 && emax - emin <= fix_shift(n);  // emax == 0 (all +-0): only the chain gets the sign
}

// Whole warp: S4 score of the n values load(0..n-1).  The result is valid in every lane.
template <typename Load>
MXS_DEV double warp_score_sum_fn(int n, Load load) {
  const int lane = (int)(threadIdx.x & 31u);
  int emin = 255, emax = 0;
  bool fin = true;
  for (int i = lane; i < n; i += 32) exp_range(__float_as_uint(load(i)), emin, emax, fin);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    emin = min(emin, __shfl_xor_sync(0xffffffffu, emin, o));
    emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  }
  fin = __all_sync(0xffffffffu, fin);
  if (certified(emin, emax, fin, n)) {
    const int S = fix_shift(n);
    long long k = 0;
    for (int i = lane; i < n; i += 32) k += fix_term(__float_as_uint(load(i)), emax, S);
#pragma unroll
    for (int o = 16; o; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
    return fix_to_double(k, emax, S);
  }
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
