// Launchers of the bit-exact SIMT forward kernels (K10, K10b) and the separate S4 rowsum pass.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "fwd_exact.cuh"
#include "rowsum.cuh"
#include "host.h"

namespace mxs_host {

int launch_rowsum(const float* rowmax, int64_t n_pairs, int64_t l_q, double* scores, cudaStream_t st) {
  if (n_pairs <= 0) return MXS_OK;
  const int threads = 256;
  const long long blocks = (n_pairs * 32 + threads - 1) / threads;
  mxs::rowsum_kernel<<<(unsigned)blocks, threads, 0, st>>>(rowmax, n_pairs, (int)l_q, scores);
  return check_launch("rowsum_kernel");
}

namespace {

template <typename T>
int launch_fwd_exact_t(const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad,
                     int64_t dim, const int32_t* valid_lens, const long long* cu, float* rowmax, int32_t* argmax,
                     cudaStream_t st) {
  mxs::FwdExactParams p;
  p.n_q = (int)n_q;
  p.l_q = (int)l_q;
  p.n_docs = (int)n_docs;
  p.l_pad = (int)l_pad;
  p.dim = (int)dim;
  p.valid_lens = valid_lens;
  p.cu_seqlens = cu;
  p.rowmax = rowmax;
  p.argmax = argmax;
  const long long pairs = n_q * n_docs;
  const int nsm = sm_count();
  long long grid = pairs < (long long)nsm * 16 ? pairs : (long long)nsm * 16;
  if (grid <= 0) return MXS_OK;
  if constexpr (std::is_same<T, float>::value) {
    // double-buffered cp.async variant: 16-B aligned rows (dim % 4 == 0, aligned bases)
    if (dim % 4 == 0 && ((reinterpret_cast<uintptr_t>(Q) | reinterpret_cast<uintptr_t>(D)) & 15) == 0 &&
        !getenv("MXS_EXACT_V1")) {
      int s;
      if ((s = ensure_smem((const void*)mxs::fwd_exact_f32v_kernel, mxs::kExV4Smem)) != MXS_OK) return s;
      mxs::fwd_exact_f32v_kernel<<<(unsigned)grid, mxs::kExThreads, mxs::kExV4Smem, st>>>(
          static_cast<const float*>(Q), static_cast<const float*>(D), p);
      return check_launch("fwd_exact_f32v_kernel");
    }
  }
  mxs::fwd_exact_kernel<T><<<(unsigned)grid, mxs::kExThreads, 0, st>>>(static_cast<const T*>(Q),
                                                                        static_cast<const T*>(D), p);
  return check_launch("fwd_exact_kernel");
}

}  // namespace

int launch_fwd_exact_i8(const int8_t* Q, const float* qs, int64_t n_q, int64_t l_q, const int8_t* D, const float* ds,
                        int64_t n_docs, int64_t l_pad, int64_t dim, const int32_t* valid_lens, float* rowmax,
                        int32_t* argmax, cudaStream_t st) {
  mxs::FwdExactParams p;
  p.n_q = (int)n_q;
  p.l_q = (int)l_q;
  p.n_docs = (int)n_docs;
  p.l_pad = (int)l_pad;
  p.dim = (int)dim;
  p.valid_lens = valid_lens;
  p.cu_seqlens = nullptr;
  p.rowmax = rowmax;
  p.argmax = argmax;
  const long long pairs = n_q * n_docs;
  const long long grid = pairs < (long long)sm_count() * 16 ? pairs : (long long)sm_count() * 16;
  if (grid <= 0) return MXS_OK;
  mxs::fwd_exact_i8_kernel<<<(unsigned)grid, mxs::kExThreads, 0, st>>>(Q, qs, D, ds, p);
  return check_launch("fwd_exact_i8_kernel");
}

int launch_fwd_exact(int dtype, const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad,
                     int64_t dim, const int32_t* valid_lens, const int64_t* cu, float* rowmax, int32_t* argmax,
                     cudaStream_t st) {
  const long long* c = (const long long*)cu;
  switch (dtype) {
    case MXS_F32: return launch_fwd_exact_t<float>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, c, rowmax, argmax, st);
    case MXS_BF16:
      return launch_fwd_exact_t<__nv_bfloat16>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, c, rowmax, argmax, st);
    case MXS_F16: return launch_fwd_exact_t<__half>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, c, rowmax, argmax, st);
    default: return fail(MXS_UNSUPPORTED, "exact forward: dtype %d not a float type", dtype);
  }
}

}  // namespace mxs_host
