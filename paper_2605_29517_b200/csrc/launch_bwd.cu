// Backward entry points: inverse-grid CSR build (K6) and the destination-owned gathers (K7, K8).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "csr.cuh"
#include "grad.cuh"
#include "host.h"

using namespace mxs_host;

namespace {

// Vectorised gather dispatch: rows must be 8-byte aligned (dim * sizeof(T) % 8 == 0) and the
// dimension must fit NP <= 4 passes of 32 lanes x 8 bytes; otherwise the scalar kernels run.
// Row-group kernels when a row is exactly 8, 16 or 32 lanes x 16 B (bf16/f16 d = 64/128/256,
// f32 d = 32/64/128).
template <typename T>
static int rowgroup_lanes(int dim) {
  const int bytes = dim * (int)sizeof(T);
  if (bytes % 16) return 0;
  const int lpr = bytes / 16;
  return (lpr == 8 || lpr == 16 || lpr == 32) ? lpr : 0;
}
template <typename T>
static bool launch_grad_docs_rg(const T* Q, const mxs::GradParams& p, long long blocks, cudaStream_t st) {
  switch (rowgroup_lanes<T>(p.dim)) {
    case 8: mxs::grad_docs_rg_kernel<T, 8><<<(unsigned)blocks, 256, 0, st>>>(Q, p); return true;
    case 16: mxs::grad_docs_rg_kernel<T, 16><<<(unsigned)blocks, 256, 0, st>>>(Q, p); return true;
    case 32: mxs::grad_docs_rg_kernel<T, 32><<<(unsigned)blocks, 256, 0, st>>>(Q, p); return true;
    default: return false;
  }
}
template <typename T>
static bool launch_grad_query_rg(const T* D, const mxs::GradParams& p, long long blocks, cudaStream_t st) {
  switch (rowgroup_lanes<T>(p.dim)) {
    case 8: mxs::grad_query_rg_kernel<T, 8><<<(unsigned)blocks, 256, 0, st>>>(D, p); return true;
    case 16: mxs::grad_query_rg_kernel<T, 16><<<(unsigned)blocks, 256, 0, st>>>(D, p); return true;
    case 32: mxs::grad_query_rg_kernel<T, 32><<<(unsigned)blocks, 256, 0, st>>>(D, p); return true;
    default: return false;
  }
}
template <typename T>
static bool launch_grad_docs_vec(const T* Q, const mxs::GradParams& p, long long blocks, cudaStream_t st) {
  if (launch_grad_docs_rg<T>(Q, p, blocks, st)) return true;
  constexpr int V = mxs::Vec8<T>::N;
  if ((p.dim * (int)sizeof(T)) % 8 != 0) return false;
  const int np = (p.dim + 32 * V - 1) / (32 * V);
  switch (np) {
    case 1: mxs::grad_docs_vec_kernel<T, 1><<<(unsigned)blocks, 256, 0, st>>>(Q, p); return true;
    case 2: mxs::grad_docs_vec_kernel<T, 2><<<(unsigned)blocks, 256, 0, st>>>(Q, p); return true;
    case 3: mxs::grad_docs_vec_kernel<T, 3><<<(unsigned)blocks, 256, 0, st>>>(Q, p); return true;
    case 4: mxs::grad_docs_vec_kernel<T, 4><<<(unsigned)blocks, 256, 0, st>>>(Q, p); return true;
    default: return false;
  }
}
template <typename T>
static bool launch_grad_query_vec(const T* D, const mxs::GradParams& p, long long blocks, cudaStream_t st) {
  if (launch_grad_query_rg<T>(D, p, blocks, st)) return true;
  constexpr int V = mxs::Vec8<T>::N;
  if ((p.dim * (int)sizeof(T)) % 8 != 0) return false;
  const int np = (p.dim + 32 * V - 1) / (32 * V);
  switch (np) {
    case 1: mxs::grad_query_vec_kernel<T, 1><<<(unsigned)blocks, 256, 0, st>>>(D, p); return true;
    case 2: mxs::grad_query_vec_kernel<T, 2><<<(unsigned)blocks, 256, 0, st>>>(D, p); return true;
    case 3: mxs::grad_query_vec_kernel<T, 3><<<(unsigned)blocks, 256, 0, st>>>(D, p); return true;
    case 4: mxs::grad_query_vec_kernel<T, 4><<<(unsigned)blocks, 256, 0, st>>>(D, p); return true;
    default: return false;
  }
}

}  // namespace

extern "C" {

size_t mxs_csr_workspace_bytes(int64_t n_q, int64_t n_dest) { return (size_t)(n_q * n_dest) * sizeof(int32_t); }

int mxs_build_inverse_csr(const int32_t* argmax, int64_t n_q, int64_t n_docs, int64_t l_q, const int64_t* dest_off,
                          const int64_t* dest_len, int64_t n_dest, int64_t max_dest_len, int32_t* row_ptr,
                          int32_t* col_idx, void* ws, size_t ws_bytes, void* stream) {
  if (!argmax || !dest_off || !dest_len || !row_ptr || !col_idx || !ws)
    return fail(MXS_INVALID_ARGUMENT, "mxs_build_inverse_csr: null pointer");
  if (n_q < 1 || n_docs < 1 || l_q < 1 || n_dest < 1) return fail(MXS_SHAPE_MISMATCH, "mxs_build_inverse_csr: bad shape");
  if (n_q * n_docs * l_q >= (1LL << 31) || n_dest >= (1LL << 31))
    return fail(MXS_UNSUPPORTED, "mxs_build_inverse_csr: more than 2^31 sources or destinations");
  if (ws_bytes < mxs_csr_workspace_bytes(n_q, n_dest))
    return fail(MXS_INVALID_ARGUMENT, "mxs_build_inverse_csr: workspace too small");
  const size_t hist_bytes = (size_t)max_dest_len * sizeof(int32_t);
  if (hist_bytes > 200 * 1024) return fail(MXS_UNSUPPORTED, "document longer than %lld rows", (long long)(200 * 256));
  mxs::CsrParams p;
  p.argmax = argmax;
  p.dest_off = (const long long*)dest_off;
  p.dest_len = (const long long*)dest_len;
  p.n_q = (int)n_q;
  p.n_docs = (int)n_docs;
  p.l_q = (int)l_q;
  p.n_dest = n_dest;
  p.cnt = (int32_t*)ws;
  p.row_ptr = row_ptr;
  p.col_idx = col_idx;
  cudaStream_t st = (cudaStream_t)stream;
  int s;
  if ((s = ensure_smem((const void*)mxs::csr_count_kernel, 200 * 1024)) != MXS_OK ||
      (s = ensure_smem((const void*)mxs::csr_place_kernel, 200 * 1024)) != MXS_OK ||
      (s = ensure_smem((const void*)mxs::csr_place_v2_kernel, 200 * 1024)) != MXS_OK ||
      (s = ensure_smem((const void*)mxs::csr_count_w_kernel, 64 * 1024)) != MXS_OK ||
      (s = ensure_smem((const void*)mxs::csr_place_w_kernel, 64 * 1024)) != MXS_OK)
    return s;
  const unsigned segs = (unsigned)(n_q * n_docs);
  // rows that belong to no document (never the case for padded / packed layouts) stay zero
  if (cudaMemsetAsync(ws, 0, mxs_csr_workspace_bytes(n_q, n_dest), st) != cudaSuccess)
    return fail(MXS_CUDA_ERROR, "memset");
  if (cudaMemsetAsync(row_ptr, 0, sizeof(int32_t) * (size_t)(n_dest + 1), st) != cudaSuccess)
    return fail(MXS_CUDA_ERROR, "memset");
  const bool warp_seg = max_dest_len <= mxs::kCsrWarpLenMax && !getenv("MXS_CSR_BLOCK");
  const int hist_len = (int)((max_dest_len + 3) & ~3LL);
  const size_t wsh = (size_t)mxs::kCsrWW * hist_len * sizeof(int32_t);
  const unsigned wblocks = (unsigned)((segs + mxs::kCsrWW - 1) / mxs::kCsrWW);
  if (warp_seg)
    mxs::csr_count_w_kernel<<<wblocks, 32 * mxs::kCsrWW, wsh, st>>>(p, hist_len);
  else
    mxs::csr_count_kernel<<<segs, 256, hist_bytes, st>>>(p);
  if ((s = check_launch("csr_count_kernel")) != MXS_OK) return s;
  mxs::csr_scan_kernel<<<(unsigned)n_docs, 1024, 0, st>>>(p);
  if ((s = check_launch("csr_scan_kernel")) != MXS_OK) return s;
  if (warp_seg)
    mxs::csr_place_w_kernel<<<wblocks, 32 * mxs::kCsrWW, wsh, st>>>(p, hist_len);
  else if (hist_bytes * mxs::kCsrWarps <= 200 * 1024)
    mxs::csr_place_v2_kernel<<<segs, 32 * mxs::kCsrWarps, hist_bytes * mxs::kCsrWarps, st>>>(p);
  else
    mxs::csr_place_kernel<<<segs, 256, hist_bytes, st>>>(p);
  return check_launch("csr_place_kernel");
}

int mxs_grad_docs_csr(int dtype, const int32_t* row_ptr, const int32_t* col_idx, int64_t n_dest, const float* g,
                      const void* Q, int64_t n_q, int64_t n_docs, int64_t l_q, int64_t dim, float* dD, void* stream) {
  if (!row_ptr || !col_idx || !g || !Q || !dD) return fail(MXS_INVALID_ARGUMENT, "mxs_grad_docs_csr: null pointer");
  if (dim < 1 || dim > 512) return fail(MXS_UNSUPPORTED, "mxs_grad_docs_csr: dim %lld outside [1, 512]", (long long)dim);
  if (n_dest < 1) return MXS_OK;
  mxs::GradParams p = {};
  p.n_q = (int)n_q;
  p.n_docs = (int)n_docs;
  p.l_q = (int)l_q;
  p.dim = (int)dim;
  p.g = g;
  p.row_ptr = row_ptr;
  p.col_idx = col_idx;
  p.n_dest = n_dest;
  p.dD = dD;
  cudaStream_t st = (cudaStream_t)stream;
  const long long blocks = (n_dest * 32 + 255) / 256;
  if (dtype == MXS_F32) {
    if (!launch_grad_docs_vec<float>((const float*)Q, p, blocks, st))
      mxs::grad_docs_kernel<float><<<(unsigned)blocks, 256, 0, st>>>((const float*)Q, p);
  } else if (dtype == MXS_BF16) {
    if (!launch_grad_docs_vec<__nv_bfloat16>((const __nv_bfloat16*)Q, p, blocks, st))
      mxs::grad_docs_kernel<__nv_bfloat16><<<(unsigned)blocks, 256, 0, st>>>((const __nv_bfloat16*)Q, p);
  } else if (dtype == MXS_F16) {
    if (!launch_grad_docs_vec<__half>((const __half*)Q, p, blocks, st))
      mxs::grad_docs_kernel<__half><<<(unsigned)blocks, 256, 0, st>>>((const __half*)Q, p);
  } else
    return fail(MXS_UNSUPPORTED, "mxs_grad_docs_csr: dtype %d", dtype);
  return check_launch("grad_docs_kernel");
}

int mxs_grad_query(int dtype, const int32_t* argmax, const float* g, const void* D, const int64_t* doc_row_off,
                   int64_t n_q, int64_t n_docs, int64_t l_q, int64_t dim, float* dQ, void* stream) {
  if (!argmax || !g || !D || !doc_row_off || !dQ) return fail(MXS_INVALID_ARGUMENT, "mxs_grad_query: null pointer");
  if (dim < 1 || dim > 512) return fail(MXS_UNSUPPORTED, "mxs_grad_query: dim %lld outside [1, 512]", (long long)dim);
  mxs::GradParams p = {};
  p.n_q = (int)n_q;
  p.n_docs = (int)n_docs;
  p.l_q = (int)l_q;
  p.dim = (int)dim;
  p.g = g;
  p.argmax = argmax;
  p.doc_row_off = (const long long*)doc_row_off;
  p.dQ = dQ;
  cudaStream_t st = (cudaStream_t)stream;
  const long long blocks = (n_q * l_q * 32 + 255) / 256;
  if (blocks == 0) return MXS_OK;
  if (dtype == MXS_F32) {
    if (!launch_grad_query_vec<float>((const float*)D, p, blocks, st))
      mxs::grad_query_kernel<float><<<(unsigned)blocks, 256, 0, st>>>((const float*)D, p);
  } else if (dtype == MXS_BF16) {
    if (!launch_grad_query_vec<__nv_bfloat16>((const __nv_bfloat16*)D, p, blocks, st))
      mxs::grad_query_kernel<__nv_bfloat16><<<(unsigned)blocks, 256, 0, st>>>((const __nv_bfloat16*)D, p);
  } else if (dtype == MXS_F16) {
    if (!launch_grad_query_vec<__half>((const __half*)D, p, blocks, st))
      mxs::grad_query_kernel<__half><<<(unsigned)blocks, 256, 0, st>>>((const __half*)D, p);
  } else
    return fail(MXS_UNSUPPORTED, "mxs_grad_query: dtype %d", dtype);
  return check_launch("grad_query_kernel");
}

}  // extern "C"
