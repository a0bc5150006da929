// Entry points of the small kernels: INT8 quantiser (K4), device top-K (K9), Chamfer (K11).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "quant.cuh"
#include "topk.cuh"
#include "chamfer.cuh"
#include "loss.cuh"

#ifndef MXS_QUANT_U
#define MXS_QUANT_U 1  // rows per pass and 8-lane group of the streaming quantiser (+ the prefetched next pass)
#endif
#include "host.h"

using namespace mxs_host;

static const long long kTopkChunk = mxs::kTopkSlice;
static const size_t kTopkSmem = mxs::kTopkSlice * (sizeof(double) + sizeof(long long));

static bool use_select(long long k) { return k <= mxs::kSelMaxK; }
// elements per CTA slice; ids are implicit (positions) only for the first pass of mxs_topk
static long long topk_slice(long long k, bool explicit_ids) {
  if (!use_select(k)) return kTopkChunk;
  return explicit_ids ? mxs::kSelChunkExplicit : mxs::kSelChunkImplicit;
}
static size_t select_smem(long long chunk, long long k, bool explicit_ids) {
  (void)k;
  return (size_t)chunk * (explicit_ids ? 16 : 8) + (size_t)(mxs::kSelThreads / 32) * mxs::kSelMaxK * 16 +
         (size_t)mxs::kSelSurvivors * 16;
}

// Passes until one CTA remains: each pass keeps k candidates per slice.
static long long topk_ws_elems(long long n, long long k, bool explicit_ids = false) {
  long long total = 0;
  long long slice = topk_slice(k, explicit_ids);
  while (n > slice) {
    const long long blocks = (n + slice - 1) / slice;
    n = blocks * k;
    total += n;
    slice = topk_slice(k, true);
  }
  return total;
}

static int topk_launch(const double* s, const long long* ids, long long n, long long k, long long blocks,
                       long long chunk, long long id_offset, double* os, long long* oi, cudaStream_t st) {
  if (use_select(k)) {
    mxs::topk_select_kernel<<<(unsigned)blocks, mxs::kSelThreads, select_smem(chunk, k, ids != nullptr), st>>>(
        s, ids, n, (int)k, chunk, id_offset, os, oi);
    return check_launch("topk_select_kernel");
  }
  mxs::topk_kernel<<<(unsigned)blocks, mxs::kTopkThreads, kTopkSmem, st>>>(s, ids, n, (int)k, chunk, id_offset, os, oi);
  return check_launch("topk_kernel");
}

static int topk_run(const double* s, const long long* ids, long long n, long long k, long long id_offset, double* top_s,
                    long long* top_id, void* ws, cudaStream_t st) {
  int r0;
  if ((r0 = ensure_smem((const void*)mxs::topk_kernel, kTopkSmem)) != MXS_OK ||
      (r0 = ensure_smem((const void*)mxs::topk_select_kernel,
                        std::max(select_smem(mxs::kSelChunkImplicit, mxs::kSelMaxK, false),
                                 select_smem(mxs::kSelChunkExplicit, mxs::kSelMaxK, true)))) != MXS_OK)
    return r0;
  double* cs = (double*)ws;
  const long long cap = topk_ws_elems(n, k, ids != nullptr);
  long long* ci = (long long*)(cs + cap);
  long long used = 0;
  long long slice = topk_slice(k, ids != nullptr);
  while (n > slice) {
    const long long blocks = (n + slice - 1) / slice;
    const long long chunk = use_select(k) ? (n + blocks - 1) / blocks : slice;  // balanced slices
    double* os = cs + used;
    long long* oi = ci + used;
    int r;
    if ((r = topk_launch(s, ids, n, k, blocks, chunk, id_offset, os, oi, st)) != MXS_OK) return r;
    s = os;
    ids = oi;
    id_offset = 0;
    n = blocks * k;
    used += n;
    slice = topk_slice(k, true);
  }
  return topk_launch(s, ids, n, k, 1, n, id_offset, top_s, top_id, st);
}

extern "C" {

int mxs_quantize_per_token(int dtype, const void* x, int64_t rows, int64_t dim, int levels, int8_t* q, float* scale,
                           void* stream) {
  if (!x || !q || !scale) return fail(MXS_INVALID_ARGUMENT, "mxs_quantize_per_token: null pointer");
  if (rows < 0 || dim < 1) return fail(MXS_SHAPE_MISMATCH, "mxs_quantize_per_token: bad shape");
  if (levels < 1 || levels > 127) return fail(MXS_INVALID_ARGUMENT, "levels must be in [1, 127], got %d", levels);
  if (rows == 0) return MXS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const long long blocks = (rows * 32 + 255) / 256;
  if (dtype == MXS_F32)
    mxs::quantize_kernel<float><<<(unsigned)blocks, 256, 0, st>>>((const float*)x, rows, (int)dim, levels, q, scale);
  else if ((dtype == MXS_BF16 || dtype == MXS_F16) && dim == 128 &&
           (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(q) & 15) == 0) {
    // persistent 8-lanes-per-row kernel: 8 blocks of 256 threads per SM
    const long long want = (rows + 32 * MXS_QUANT_U - 1) / (32 * MXS_QUANT_U);  // 32 groups x U rows per block pass
    const long long sblocks = want < (long long)sm_count() * 8 ? want : (long long)sm_count() * 8;
    if (dtype == MXS_BF16)
      mxs::quantize128_stream_kernel<__nv_bfloat16, MXS_QUANT_U>
          <<<(unsigned)sblocks, 256, 0, st>>>((const __nv_bfloat16*)x, rows, levels, q, scale);
    else
      mxs::quantize128_stream_kernel<__half, MXS_QUANT_U><<<(unsigned)sblocks, 256, 0, st>>>((const __half*)x, rows, levels, q, scale);
  } else if (dtype == MXS_BF16 && dim == 128)
    mxs::quantize128_kernel<__nv_bfloat16>
        <<<(unsigned)blocks, 256, 0, st>>>((const __nv_bfloat16*)x, rows, levels, q, scale);
  else if (dtype == MXS_F16 && dim == 128)
    mxs::quantize128_kernel<__half><<<(unsigned)blocks, 256, 0, st>>>((const __half*)x, rows, levels, q, scale);
  else if (dtype == MXS_BF16)
    mxs::quantize_kernel<__nv_bfloat16>
        <<<(unsigned)blocks, 256, 0, st>>>((const __nv_bfloat16*)x, rows, (int)dim, levels, q, scale);
  else if (dtype == MXS_F16)
    mxs::quantize_kernel<__half><<<(unsigned)blocks, 256, 0, st>>>((const __half*)x, rows, (int)dim, levels, q, scale);
  else
    return fail(MXS_UNSUPPORTED, "mxs_quantize_per_token: dtype %d", dtype);
  return check_launch("quantize_kernel");
}

size_t mxs_topk_workspace_bytes(int64_t n, int64_t k) {
  return (size_t)topk_ws_elems(n, k) * (sizeof(double) + sizeof(long long));
}

int mxs_topk(const double* scores, int64_t n, int64_t k, int64_t id_offset, double* top_s, int64_t* top_id, void* ws,
             size_t ws_bytes, void* stream) {
  if (!scores || !top_s || !top_id) return fail(MXS_INVALID_ARGUMENT, "mxs_topk: null pointer");
  if (k > n) return fail(MXS_K_TOO_LARGE, "top-%lld requested from a corpus of %lld documents", (long long)k, (long long)n);
  if (k <= 0) return MXS_OK;
  if (k > 2048) return fail(MXS_UNSUPPORTED, "mxs_topk: k > 2048");
  if (mxs_topk_workspace_bytes(n, k) > 0 && (!ws || ws_bytes < mxs_topk_workspace_bytes(n, k)))
    return fail(MXS_INVALID_ARGUMENT, "mxs_topk: workspace too small");
  return topk_run(scores, nullptr, n, k, id_offset, top_s, (long long*)top_id, ws, (cudaStream_t)stream);
}

int mxs_topk_candidates(const double* scores, const int64_t* ids, int64_t n, int64_t k, double* top_s, int64_t* top_id,
                        void* stream) {
  if (!scores || !ids || !top_s || !top_id) return fail(MXS_INVALID_ARGUMENT, "mxs_topk_candidates: null pointer");
  if (k <= 0) return MXS_OK;
  if (k > 2048) return fail(MXS_UNSUPPORTED, "mxs_topk_candidates: k > 2048");
  if (n > topk_slice(k, true))
    return fail(MXS_UNSUPPORTED, "mxs_topk_candidates: more than %lld candidates", topk_slice(k, true));
  return topk_run(scores, (const long long*)ids, n, k, 0, top_s, (long long*)top_id, nullptr, (cudaStream_t)stream);
}

// ------------------------------------------------------------------ Chamfer
int mxs_sq_norms(const float* X, int64_t rows, int64_t dim, float* out, void* stream) {
  if (!X || !out) return fail(MXS_INVALID_ARGUMENT, "mxs_sq_norms: null pointer");
  if (rows < 1 || dim < 1) return fail(MXS_SHAPE_MISMATCH, "mxs_sq_norms: empty input");
  const long long blocks = (rows + 255) / 256;
  mxs::sq_norms_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(X, rows, (int)dim, out);
  return check_launch("sq_norms_kernel");
}

int mxs_chamfer_nn(const float* A, const float* a_norms, int64_t n, const float* B, const float* b_norms, int64_t m,
                   int64_t dim, float* best, int32_t* idx, void* stream) {
  if (!A || !a_norms || !B || !b_norms || !best || !idx) return fail(MXS_INVALID_ARGUMENT, "mxs_chamfer_nn: null");
  if (n < 1 || m < 1) return fail(MXS_SHAPE_MISMATCH, "point set must hold at least one point");
  if (dim < 1 || dim > 8192) return fail(MXS_UNSUPPORTED, "mxs_chamfer_nn: dim %lld outside [1, 8192]", (long long)dim);
  if (m >= (1LL << 31)) return fail(MXS_UNSUPPORTED, "mxs_chamfer_nn: more than 2^31 points");
  const long long blocks = (n + mxs::kChThreads - 1) / mxs::kChThreads;
  cudaStream_t st = (cudaStream_t)stream;
  if (dim > mxs::kChDimMax)
    mxs::chamfer_nn_any_kernel<<<(unsigned)blocks, mxs::kChThreads, 0, st>>>(A, a_norms, n, B, b_norms, m, (int)dim,
                                                                             best, idx);
  else if (dim == 3)
    mxs::chamfer_nn_kernel<3><<<(unsigned)blocks, mxs::kChThreads, 0, st>>>(A, a_norms, n, B, b_norms, m, 3, best, idx);
  else
    mxs::chamfer_nn_kernel<0><<<(unsigned)blocks, mxs::kChThreads, 0, st>>>(A, a_norms, n, B, b_norms, m, (int)dim,
                                                                            best, idx);
  return check_launch("chamfer_nn_kernel");
}

int mxs_chamfer_grad(const float* X, int64_t nx, const float* Y, int64_t dim, const int32_t* nn,
                     const int32_t* row_ptr, const int32_t* col_idx, double c_gather, double c_scatter, double* dX,
                     void* stream) {
  if (!X || !Y || !nn || !row_ptr || !col_idx || !dX) return fail(MXS_INVALID_ARGUMENT, "mxs_chamfer_grad: null");
  if (nx < 1 || dim < 1) return fail(MXS_SHAPE_MISMATCH, "mxs_chamfer_grad: empty input");
  const long long total = nx * dim, blocks = (total + 255) / 256;
  mxs::chamfer_grad_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(X, nx, Y, (int)dim, nn, row_ptr,
                                                                               col_idx, c_gather, c_scatter, dX);
  return check_launch("chamfer_grad_kernel");
}

}  // extern "C"

// ------------------------------------------------------------------ input validation
namespace {

// out[0] = lowest bad index (atomicMin), grid-stride over the entries
__global__ void check_lens_kernel(const int32_t* __restrict__ vl, long long n, long long l_pad,
                                  unsigned long long* out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int v = vl[i];
    if (v < 1 || v > l_pad) atomicMin(out, (unsigned long long)i);
  }
}
// out[0] = lowest document whose step cu[i+1] - cu[i] <= 0; out[1] = 1 if cu[0] != 0, 2 if cu[B] != n_tokens
__global__ void check_cu_kernel(const long long* __restrict__ cu, long long n_docs, long long n_tokens,
                                unsigned long long* out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0) {
    if (cu[0] != 0) atomicOr(out + 1, 1ull);
    if (cu[n_docs] != n_tokens) atomicOr(out + 1, 2ull);
  }
  for (long long i = t; i < n_docs; i += (long long)gridDim.x * blockDim.x)
    if (cu[i + 1] <= cu[i]) atomicMin(out, (unsigned long long)i);
}

// Runs `launch(dev_out)` into a zero-initialised 2-word device scratch and reads it back.
template <typename F>
int run_check(cudaStream_t st, unsigned long long (&host)[2], F launch) {
  unsigned long long* d = nullptr;
  if (scratch_alloc((void**)&d, 16, st) != MXS_OK) return fail(MXS_CUDA_ERROR, "validation scratch allocation failed");
  const unsigned long long init[2] = {~0ull, 0ull};
  cudaMemcpyAsync(d, init, 16, cudaMemcpyHostToDevice, st);
  launch(d);
  int s = check_launch("validation kernel");
  cudaMemcpyAsync(host, d, 16, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d, st);
  if (cudaStreamSynchronize(st) != cudaSuccess && s == MXS_OK) s = fail(MXS_CUDA_ERROR, "validation: stream sync failed");
  return s;
}

unsigned checks_grid(long long n) {
  const long long b = (n + 255) / 256;
  return (unsigned)std::max<long long>(1, std::min<long long>(b, 4LL * std::max(sm_count(), 1)));
}

}  // namespace

extern "C" {

int mxs_validate_lens(const int32_t* valid_lens, int64_t n, int64_t l_pad, int64_t* bad_index, int64_t* bad_value,
                      void* stream) {
  if (bad_index) *bad_index = -1;
  if (bad_value) *bad_value = 0;
  if (!valid_lens || n < 0 || l_pad < 1) return fail(MXS_INVALID_ARGUMENT, "mxs_validate_lens: bad arguments");
  if (n == 0) return MXS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long h[2] = {~0ull, 0ull};
  int s = run_check(st, h, [&](unsigned long long* d) {
    check_lens_kernel<<<checks_grid(n), 256, 0, st>>>(valid_lens, n, l_pad, d);
  });
  if (s != MXS_OK || h[0] == ~0ull) return s;
  int32_t v = 0;
  if (cudaMemcpy(&v, valid_lens + h[0], sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(MXS_CUDA_ERROR, "mxs_validate_lens: read-back failed");
  if (bad_index) *bad_index = (int64_t)h[0];
  if (bad_value) *bad_value = v;
  if (v < 1) return fail(MXS_EMPTY_DOCUMENT, "%lld", (long long)h[0]);
  return fail(MXS_SHAPE_MISMATCH, "valid_len %d exceeds document rows %lld", v, (long long)l_pad);
}

int mxs_validate_cu_seqlens(const int64_t* cu_seqlens, int64_t n_docs, int64_t n_tokens, int64_t* bad_index,
                            int64_t* bad_value, void* stream) {
  if (bad_index) *bad_index = -1;
  if (bad_value) *bad_value = 0;
  if (!cu_seqlens || n_docs < 1 || n_tokens < 0) return fail(MXS_INVALID_ARGUMENT, "mxs_validate_cu_seqlens: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long h[2] = {~0ull, 0ull};
  int s = run_check(st, h, [&](unsigned long long* d) {
    check_cu_kernel<<<checks_grid(n_docs), 256, 0, st>>>((const long long*)cu_seqlens, n_docs, n_tokens, d);
  });
  if (s != MXS_OK) return s;
  if (h[1] & 1ull)
    return fail(MXS_SHAPE_MISMATCH, "cu_seqlens must be 1-D with cu[0] = 0 and one entry per document plus one");
  if (h[0] != ~0ull) {
    if (bad_index) *bad_index = (int64_t)h[0];
    return fail(MXS_EMPTY_DOCUMENT, "%lld", (long long)h[0]);
  }
  if (h[1] & 2ull) {
    int64_t end = 0;
    cudaMemcpy(&end, cu_seqlens + n_docs, sizeof(end), cudaMemcpyDeviceToHost);
    if (bad_value) *bad_value = end;
    return fail(MXS_SHAPE_MISMATCH, "cu_seqlens end %lld does not match token count %lld", (long long)end,
                (long long)n_tokens);
  }
  return MXS_OK;
}

}  // extern "C"

extern "C" {

int mxs_softmax_ce(const double* scores, int64_t n_q, int64_t b, int64_t col0, int64_t ncols, double* loss, float* g,
                   void* stream) {
  if (!scores || !loss || (!g && ncols > 0)) return fail(MXS_INVALID_ARGUMENT, "mxs_softmax_ce: null pointer");
  if (n_q < 1 || b < n_q || col0 < 0 || ncols < 0 || col0 + ncols > b || b >= (1LL << 31))
    return fail(MXS_SHAPE_MISMATCH, "mxs_softmax_ce: scores [%lld, %lld] with positives on the diagonal, columns "
                "[%lld, %lld)", (long long)n_q, (long long)b, (long long)col0, (long long)(col0 + ncols));
  mxs::softmax_ce_kernel<<<1, mxs::kLossThreads, 0, (cudaStream_t)stream>>>(scores, (int)n_q, (int)b, (int)col0,
                                                                           (int)ncols, loss, g);
  return check_launch("softmax_ce_kernel");
}

}  // extern "C"

