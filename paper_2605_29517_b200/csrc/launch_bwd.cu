// Backward entry points: inverse-grid CSR build (K6) and the destination-owned gathers (K7, K8).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include <cub/device/device_radix_sort.cuh>

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

// MXS_DEBUG_WRITES=1: ownership ledger of the destination-owned gathers.  Every output row must
// be stored by exactly one warp (the reference's WriteTracking assertion, tests/test_backward.py:
// 94-108); the check is synchronous and reports the first offending row.
struct WriteLedger {
  int32_t* counts = nullptr;
  unsigned long long* result = nullptr;
  long long n = 0;
  template <typename P>
  int arm(P& p, long long rows, cudaStream_t st) {
    if (!env_is("MXS_DEBUG_WRITES", "1") || rows < 1) return MXS_OK;
    n = rows;
    if (scratch_alloc((void**)&counts, (size_t)((rows + 3) & ~3LL) * sizeof(int32_t) + 16, st) != MXS_OK)
      return fail(MXS_CUDA_ERROR, "write ledger: allocation failed");
    result = reinterpret_cast<unsigned long long*>(counts + ((rows + 3) & ~3LL));
    // counts = 0, result = {0, ~0}: two memsets (0x00 then 0xff over the second word)
    if (cudaMemsetAsync(counts, 0, (size_t)((rows + 3) & ~3LL) * sizeof(int32_t) + 8, st) != cudaSuccess ||
        cudaMemsetAsync(result + 1, 0xff, 8, st) != cudaSuccess)
      return fail(MXS_CUDA_ERROR, "write ledger: memset failed");
    p.wcount = counts;
    return MXS_OK;
  }
  int check(const char* what, cudaStream_t st) {
    if (!counts) return MXS_OK;
    const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 4096);
    mxs::write_once_check_kernel<<<blocks, 256, 0, st>>>(counts, n, result);
    unsigned long long h[2] = {0ull, 0ull};
    cudaMemcpyAsync(h, result, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(counts, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail(MXS_CUDA_ERROR, "write ledger: sync failed");
    if (h[0] != 0)
      return fail(MXS_CUDA_ERROR, "%s: %llu output rows not written exactly once (first: row %llu)", what, h[0], h[1]);
    return MXS_OK;
  }
};

// f64 gathers for fp32 inputs (bit-identical to the reference's float64 gradients)
template <typename KernelFn>
static int launch_f64(KernelFn pick, int64_t dim, long long warps, const char* what, cudaStream_t st) {
  const long long blocks = (warps * 32 + 255) / 256;
  if (blocks == 0) return MXS_OK;
  const int nc = (int)((dim + 31) / 32);
  if (!pick(nc <= 1 ? 1 : nc <= 2 ? 2 : nc <= 4 ? 4 : nc <= 8 ? 8 : 16, (unsigned)blocks, st))
    return fail(MXS_UNSUPPORTED, "%s: dim %lld", what, (long long)dim);
  return check_launch(what);
}

}  // namespace

extern "C" {

// The CSR build needs no caller workspace any more (csr_doc_kernel keeps its histograms in shared
// memory; the radix-sort path allocates stream-ordered scratch itself).  The entry point and the
// ws arguments stay for ABI stability.
size_t mxs_csr_workspace_bytes(int64_t n_q, int64_t n_dest) {
  (void)n_q;
  (void)n_dest;
  return 0;
}

int mxs_build_inverse_csr(const int32_t* argmax, int64_t n_q, int64_t n_docs, int64_t l_q, const int64_t* dest_off,
                          const int64_t* dest_len, int64_t n_dest, int64_t max_dest_len, int32_t* row_ptr,
                          int32_t* col_idx, void* ws, size_t ws_bytes, void* stream) {
  (void)ws;
  (void)ws_bytes;
  if (!argmax || !dest_off || !dest_len || !row_ptr || !col_idx)
    return fail(MXS_INVALID_ARGUMENT, "mxs_build_inverse_csr: null pointer");
  if (n_q < 1 || n_docs < 1 || l_q < 1 || n_dest < 1 || max_dest_len < 1)
    return fail(MXS_SHAPE_MISMATCH, "mxs_build_inverse_csr: bad shape");
  if (n_q * n_docs * l_q >= (1LL << 31) || n_dest >= (1LL << 31) - 1)
    return fail(MXS_UNSUPPORTED, "mxs_build_inverse_csr: more than 2^31 sources or destinations");
  mxs::CsrParams p;
  p.argmax = argmax;
  p.dest_off = (const long long*)dest_off;
  p.dest_len = (const long long*)dest_len;
  p.n_q = (int)n_q;
  p.n_docs = (int)n_docs;
  p.l_q = (int)l_q;
  p.n_dest = n_dest;
  p.row_ptr = row_ptr;
  p.col_idx = col_idx;
  cudaStream_t st = (cudaStream_t)stream;
  int s;
  // shared-memory plan of csr_doc_kernel: (2W + 3) rows of H 32-bit words per CTA
  constexpr size_t kSmemMax = 227 * 1024 - 256;
  const long long H = (max_dest_len + 3) & ~3LL;
  const long long w_cap = ((long long)(kSmemMax / (4 * (size_t)H)) - 3) / 2;
  if (w_cap >= 1 && !env_is("MXS_CSR_IMPL", "sort")) {
    const long long n_src = n_q * l_q;
    const long long per_warp = std::max(32, env_int("MXS_CSR_SRC_PER_WARP", 2048));
    const long long nwt = std::min<long long>(8 * mxs::kCsrMaxWarps, std::max(1LL, (n_src + per_warp - 1) / per_warp));
    const int W = (int)std::min<long long>(std::min<long long>(env_int("MXS_CSR_WARPS", mxs::kCsrMaxWarps), w_cap), nwt);
    const int CL = (int)std::min<long long>(8, (nwt + W - 1) / W);
    p.hist_len = (int)H;
    p.lq_div = mxs::make_fastdiv((uint32_t)l_q);
    const size_t smem = (size_t)(2 * W + 3) * (size_t)H * sizeof(int32_t);
    if ((s = ensure_smem((const void*)mxs::csr_doc_kernel, smem)) != MXS_OK) return s;
    void* args[] = {&p};
    return launch_cluster((const void*)mxs::csr_doc_kernel, n_docs * CL, CL, 32 * W, smem, st, args, "csr_doc_kernel");
  }
  // general path: stable radix sort of (destination row, source) pairs
  const long long n = n_q * n_docs * l_q;
  int end_bit = 1;
  while (end_bit < 31 && (1LL << end_bit) <= n_dest) ++end_bit;
  size_t temp = 0;
  cub::DoubleBuffer<int32_t> dk(nullptr, nullptr), dv(nullptr, nullptr);
  if (cub::DeviceRadixSort::SortPairs(nullptr, temp, dk, dv, (int)n, 0, end_bit, st) != cudaSuccess)
    return fail(MXS_CUDA_ERROR, "csr radix sort: temp query failed");
  const size_t arr = ((size_t)n * sizeof(int32_t) + 255) & ~(size_t)255;
  char* buf = nullptr;
  if (scratch_alloc((void**)&buf, 3 * arr + temp, st) != MXS_OK)
    return fail(MXS_CUDA_ERROR, "csr radix sort: cannot allocate %zu bytes of scratch", 3 * arr + temp);
  int32_t* k0 = (int32_t*)buf;
  int32_t* k1 = (int32_t*)(buf + arr);
  int32_t* v0 = (int32_t*)(buf + 2 * arr);
  const int nsm = sm_count();
  const unsigned blocks = (unsigned)std::max(1LL, std::min<long long>((n + 255) / 256, (long long)nsm * 8));
  mxs::csr_sort_keys_kernel<<<blocks, 256, 0, st>>>(p, k0, v0);
  s = check_launch("csr_sort_keys_kernel");
  if (s == MXS_OK) {
    // values ping-pong between v0 and col_idx; keys between k0 and k1
    cub::DoubleBuffer<int32_t> keys(k0, k1), vals(v0, col_idx);
    if (cub::DeviceRadixSort::SortPairs(buf + 3 * arr, temp, keys, vals, (int)n, 0, end_bit, st) != cudaSuccess)
      s = fail(MXS_CUDA_ERROR, "csr radix sort failed");
    if (s == MXS_OK && vals.Current() != col_idx &&
        cudaMemcpyAsync(col_idx, vals.Current(), (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      s = fail(MXS_CUDA_ERROR, "csr radix sort: copy");
    if (s == MXS_OK) {
      const unsigned rb = (unsigned)std::max(1LL, std::min<long long>((n_dest + 256) / 256, (long long)nsm * 8));
      mxs::csr_sort_rowptr_kernel<<<rb, 256, 0, st>>>(keys.Current(), n, n_dest, row_ptr);
      s = check_launch("csr_sort_rowptr_kernel");
    }
  }
  cudaFreeAsync(buf, st);
  return s;
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
  p.per_q_div = mxs::make_fastdiv((uint32_t)(n_docs * l_q));
  p.lq_div = mxs::make_fastdiv((uint32_t)l_q);
  cudaStream_t st = (cudaStream_t)stream;
  WriteLedger ledger;
  int s = ledger.arm(p, n_dest, st);
  if (s != MXS_OK) return s;
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
  if ((s = check_launch("grad_docs_kernel")) != MXS_OK) return s;
  return ledger.check("mxs_grad_docs_csr", st);
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
  WriteLedger ledger;
  int s = ledger.arm(p, n_q * l_q, st);
  if (s != MXS_OK) return s;
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
  if ((s = check_launch("grad_query_kernel")) != MXS_OK) return s;
  return ledger.check("mxs_grad_query", st);
}

int mxs_grad_docs_csr_f64(const int32_t* row_ptr, const int32_t* col_idx, int64_t n_dest, const double* g,
                          const float* Q, int64_t n_q, int64_t n_docs, int64_t l_q, int64_t dim, double* dD,
                          void* stream) {
  if (!row_ptr || !col_idx || !g || !Q || !dD) return fail(MXS_INVALID_ARGUMENT, "mxs_grad_docs_csr_f64: null pointer");
  if (dim < 1 || dim > 512) return fail(MXS_UNSUPPORTED, "mxs_grad_docs_csr_f64: dim %lld outside [1, 512]", (long long)dim);
  if (n_dest < 1) return MXS_OK;
  mxs::GradParams64 p = {};
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
  WriteLedger ledger;
  int s = ledger.arm(p, n_dest, st);
  if (s != MXS_OK) return s;
  s = launch_f64(
      [&](int nc, unsigned blocks, cudaStream_t stm) {
        switch (nc) {
          case 1: mxs::grad_docs_f64_kernel<1><<<blocks, 256, 0, stm>>>(Q, p); return true;
          case 2: mxs::grad_docs_f64_kernel<2><<<blocks, 256, 0, stm>>>(Q, p); return true;
          case 4: mxs::grad_docs_f64_kernel<4><<<blocks, 256, 0, stm>>>(Q, p); return true;
          case 8: mxs::grad_docs_f64_kernel<8><<<blocks, 256, 0, stm>>>(Q, p); return true;
          case 16: mxs::grad_docs_f64_kernel<16><<<blocks, 256, 0, stm>>>(Q, p); return true;
          default: return false;
        }
      },
      dim, n_dest, "grad_docs_f64_kernel", st);
  if (s != MXS_OK) return s;
  return ledger.check("mxs_grad_docs_csr_f64", st);
}

int mxs_grad_query_f64(const int32_t* argmax, const double* g, const float* D, const int64_t* doc_row_off, int64_t n_q,
                       int64_t n_docs, int64_t l_q, int64_t dim, double* dQ, void* stream) {
  if (!argmax || !g || !D || !doc_row_off || !dQ) return fail(MXS_INVALID_ARGUMENT, "mxs_grad_query_f64: null pointer");
  if (dim < 1 || dim > 512) return fail(MXS_UNSUPPORTED, "mxs_grad_query_f64: dim %lld outside [1, 512]", (long long)dim);
  mxs::GradParams64 p = {};
  p.n_q = (int)n_q;
  p.n_docs = (int)n_docs;
  p.l_q = (int)l_q;
  p.dim = (int)dim;
  p.g = g;
  p.argmax = argmax;
  p.doc_row_off = (const long long*)doc_row_off;
  p.dQ = dQ;
  cudaStream_t st = (cudaStream_t)stream;
  WriteLedger ledger;
  int s = ledger.arm(p, n_q * l_q, st);
  if (s != MXS_OK) return s;
  s = launch_f64(
      [&](int nc, unsigned blocks, cudaStream_t stm) {
        switch (nc) {
          case 1: mxs::grad_query_f64_kernel<1><<<blocks, 256, 0, stm>>>(D, p); return true;
          case 2: mxs::grad_query_f64_kernel<2><<<blocks, 256, 0, stm>>>(D, p); return true;
          case 4: mxs::grad_query_f64_kernel<4><<<blocks, 256, 0, stm>>>(D, p); return true;
          case 8: mxs::grad_query_f64_kernel<8><<<blocks, 256, 0, stm>>>(D, p); return true;
          case 16: mxs::grad_query_f64_kernel<16><<<blocks, 256, 0, stm>>>(D, p); return true;
          default: return false;
        }
      },
      dim, n_q * l_q, "grad_query_f64_kernel", st);
  if (s != MXS_OK) return s;
  return ledger.check("mxs_grad_query_f64", st);
}

}  // extern "C"
