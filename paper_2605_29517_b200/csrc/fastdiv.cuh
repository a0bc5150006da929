// Division by run-time invariant 32-bit divisors (CSR source walk, gather source decoding).
#pragma once
#include "ptx.cuh"

namespace mxs {

// n / d for 32-bit unsigned n and a run-time invariant d >= 1 (Granlund-Montgomery): a mulhi, a
// subtract and two shifts instead of the ~20-instruction division subroutine per source.
struct FastDiv {
  uint32_t d, m, s1, s2;
};
inline FastDiv make_fastdiv(uint32_t d) {
  uint32_t l = 0;
  while (l < 32 && (1ull << l) < d) ++l;
  FastDiv f;
  f.d = d;
  f.m = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
  f.s1 = l < 1 ? l : 1;
  f.s2 = l > 1 ? l - 1 : 0;
  return f;
}
MXS_DEV uint32_t fdiv(uint32_t n, const FastDiv& f) {
  const uint32_t t = __umulhi(n, f.m);
  return (t + ((n - t) >> f.s1)) >> f.s2;
}

}  // namespace mxs
