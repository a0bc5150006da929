/*
 * maxsim_b200.h -- C-ABI of the B200-native Flash-MaxSim operator.
 *
 * Conventions (all entry points):
 *   - every pointer argument is a DEVICE pointer unless stated otherwise; the caller owns
 *     every output buffer (the only internal allocation is a stream-ordered cudaMallocAsync
 *     row-maxima scratch when a forward needs a separate S4 pass and rowmax is NULL);
 *   - `stream` is a cudaStream_t passed as void*; every call is stream-ordered and returns
 *     as soon as the work is enqueued;
 *   - the return value is an mxs_status; MXS_OK == 0.  mxs_last_error() returns a
 *     thread-local human-readable message for the most recent failure on this thread.
 *   - status codes map 1:1 onto the reference's typed errors (maxsim/errors.py:8-78).
 *
 * Each entry point cites the reference interface it replaces (paths relative to
 * /root/reference/pkg/src).
 */
#ifndef MAXSIM_B200_H
#define MAXSIM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MXS_OK = 0,
  MXS_DIM_MISMATCH = 1,       /* maxsim/errors.py:13 DimMismatch */
  MXS_SHAPE_MISMATCH = 2,     /* maxsim/errors.py:35 ShapeMismatch */
  MXS_EMPTY_DOCUMENT = 3,     /* maxsim/errors.py:29 EmptyDocument */
  MXS_INDEX_OUT_OF_RANGE = 4, /* maxsim/errors.py:43 IndexOutOfRange */
  MXS_STALE_CSR = 5,          /* maxsim/errors.py:47 StaleCsr */
  MXS_K_TOO_LARGE = 6,        /* maxsim/errors.py:55 KTooLarge */
  MXS_NAN_INPUT = 7,          /* maxsim/errors.py:21 NaNInput */
  MXS_BAD_TILE_CONFIG = 8,    /* maxsim/errors.py:39 BadTileConfig */
  MXS_UNSUPPORTED = 9,        /* shape/dtype outside what the sm_100a kernels accept */
  MXS_CUDA_ERROR = 10,        /* launch or driver failure */
  MXS_INVALID_ARGUMENT = 11,  /* null pointer / negative size */
  MXS_IO_ERROR = 12,          /* maxsim/errors.py:60 IoError */
  MXS_BAD_MAGIC = 13,         /* maxsim/errors.py:64 BadMagic */
  MXS_VERSION_UNSUPPORTED = 14, /* maxsim/errors.py:68 VersionUnsupported */
  MXS_TRUNCATED_PAYLOAD = 15, /* maxsim/errors.py:74 TruncatedPayload */
  MXS_STALE_ARGMIN = 16       /* maxsim/errors.py:49 StaleArgmin */
} mxs_status;

typedef enum { MXS_F32 = 0, MXS_F16 = 1, MXS_BF16 = 2, MXS_I8 = 3 } mxs_dtype;

/*
 * Input validation that needs the data (synchronous on `stream`: one small kernel + a 16-byte
 * read-back).  Replaces the checks of maxsim/forward.py:173-176 / maxsim/types.py:97-98
 * (valid_len < 1 -> EmptyDocument(index), valid_len > rows -> ShapeMismatch) and
 * maxsim/varlen.py:35-41 (cu[0] != 0 or cu[B] != n_tokens -> ShapeMismatch, a non-increasing
 * step -> EmptyDocument(index)).  *bad_index (host pointer, may be NULL) receives the first
 * offending index (-1 if none); *bad_value (host, may be NULL) the offending entry.
 */
int mxs_validate_lens(const int32_t* valid_lens, int64_t n, int64_t l_pad, int64_t* bad_index, int64_t* bad_value,
                      void* stream);
int mxs_validate_cu_seqlens(const int64_t* cu_seqlens, int64_t n_docs, int64_t n_tokens, int64_t* bad_index,
                            int64_t* bad_value, void* stream);

/* Library identification. */
const char* mxs_version(void);
const char* mxs_status_string(int status);
const char* mxs_last_error(void);
/* Number of SMs of the current device (grid sizing), or -1 on error. */
int mxs_device_sm_count(void);

/*
 * Dense all-pairs forward.  Replaces maxsim/forward.py:221 fused_score_batch (and
 * maxsim/forward.py:158 fused_score_pair for n_q = n_docs = 1).
 *   Q          [n_q, l_q, dim]        elements of `dtype`
 *   D          [n_docs, l_pad, dim]   zero-padded documents (maxsim/types.py:80 DocBatch)
 *   valid_lens [n_docs] int32, or NULL for "all rows valid"; every entry in [1, l_pad]
 *   scores     [n_q, n_docs] float64  (S4: sequential f64 sum of fp32 row maxima)
 *   argmax     [n_q, n_docs, l_q] int32, document-local, lowest index on ties; may be NULL:
 *              "rerank mode" -- the tensor-core kernels then keep only a running max per row
 *              (no index tracking; identical score bits, ~15 % faster at the ColPali shape)
 *   rowmax     [n_q, n_docs, l_q] float32 per-token maxima, OPTIONAL (NULL: not materialised).
 *              The tensor-core kernels fold S4 into their epilogue (score warp + cluster DSMEM)
 *              whenever one CTA cluster holds a whole query (l_q <= 2048 for bf16/fp16 d = 128);
 *              other shapes and the exact kernels run a separate S4 pass over the row maxima
 *              (a stream-ordered scratch when rowmax is NULL).
 *   exact      0: tcgen05 tensor-core path (MXS_BF16 / MXS_F16; fp32 accumulation)
 *              1: bit-exact fp32 fold on CUDA cores (S1; any float dtype, required for MXS_F32)
 * The kernels clamp valid_lens into [0, l_pad] (memory safety); out-of-range entries are a
 * caller error detected by mxs_validate_lens (the reference raises, maxsim/forward.py:173-176).
 */
int mxs_fused_score_batch(int dtype, const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs,
                          int64_t l_pad, int64_t dim, const int32_t* valid_lens, double* scores, int32_t* argmax,
                          float* rowmax, int exact, void* stream);

/*
 * The fused tile kernel of mxs_fused_score_batch alone: per-row maxima (rowmax) and argmax,
 * no f64 score fold (call mxs_rowsum for it).  Same arguments minus `scores`.
 */
int mxs_fused_rowmax_batch(int dtype, const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs,
                           int64_t l_pad, int64_t dim, const int32_t* valid_lens, int32_t* argmax, float* rowmax,
                           int exact, void* stream);

/*
 * INT8 x INT8 dense forward with fused dequantisation.  Replaces maxsim/quant.py:128
 * fused_score_int8 (batched over documents and queries; the reference is per pair).
 *   Q [n_q, l_q, dim] int8, q_scale [n_q, l_q] f32; D [n_docs, l_pad, dim] int8,
 *   d_scale [n_docs, l_pad] f32.  sim = fl(fl(f32(int32 acc) * s_q) * s_d)  (S7).
 *   argmax may be NULL (rerank mode: dim <= 128 runs the three-epilogue-set fwd_i8r kernel).
 */
int mxs_fused_score_int8(const int8_t* Q, const float* q_scale, int64_t n_q, int64_t l_q, const int8_t* D,
                         const float* d_scale, int64_t n_docs, int64_t l_pad, int64_t dim, const int32_t* valid_lens,
                         double* scores, int32_t* argmax, float* rowmax, void* stream);

/*
 * Padding-free forward over a packed corpus.  Replaces maxsim/varlen.py:88 fused_score_varlen
 * (generalised to n_q queries).
 *   tokens [n_tokens, dim] (concatenated document rows), cu_seqlens [n_docs + 1] int64 with
 *   cu[0] = 0, strictly increasing, cu[n_docs] = n_tokens (maxsim/varlen.py:22-63).
 *   scores [n_q, n_docs] f64; argmax [n_q, n_docs, l_q] int32 document-local; rowmax scratch.
 */
int mxs_fused_score_varlen(int dtype, const void* Q, int64_t n_q, int64_t l_q, const void* tokens,
                           const int64_t* cu_seqlens, int64_t n_docs, int64_t n_tokens, int64_t dim, double* scores,
                           int32_t* argmax, float* rowmax, int exact, void* stream);

/*
 * In-batch contrastive loss (positives on the diagonal) and its score gradient, fused.  Replaces
 * maxsim/cli.py:198 _softmax_ce for the C3 training step: scores f64 [n_q, b] (b >= n_q) ->
 * loss f64 [1] = mean_q(logsumexp(s[q]) - s[q, q]) and g f32 [n_q, ncols] = the columns
 * [col0, col0 + ncols) of (softmax(s) - eye) / n_q.
 */
int mxs_softmax_ce(const double* scores, int64_t n_q, int64_t b, int64_t col0, int64_t ncols, double* loss, float* g,
                   void* stream);

/* Sequential f64 row sum (S4) of rowmax [n_pairs, l_q] into scores [n_pairs]. */
int mxs_rowsum(const float* rowmax, int64_t n_pairs, int64_t l_q, double* scores, void* stream);

/*
 * Per-token symmetric quantisation.  Replaces maxsim/quant.py:104 quantize_per_token.
 *   x [rows, dim] of `dtype` (f32 / bf16 / f16) -> q [rows, dim] int8, scale [rows] f32 (S7).
 */
int mxs_quantize_per_token(int dtype, const void* x, int64_t rows, int64_t dim, int levels, int8_t* q, float* scale,
                           void* stream);

/*
 * Inverse-grid CSR of the saved argmax.  Replaces maxsim/backward.py:81 build_inverse_csr.
 *   argmax    [n_q, n_docs, l_q] int32 document-local winners
 *   dest_off  [n_docs] int64 first destination row of each document (maxsim/types.py:205-211:
 *             b * padded_len for a padded batch, prefix sums of doc_lens when packed)
 *   dest_len  [n_docs] int64 destination rows owned by each document (padded_len or doc_len)
 *   row_ptr   [n_dest + 1] int32, col_idx [n_q * n_docs * l_q] int32 (ascending source id per
 *             bucket, i.e. the reference's stable argsort)
 *   ws        unused (mxs_csr_workspace_bytes returns 0; kept for ABI stability, may be NULL):
 *             documents of up to ~14K rows build in one cluster-per-document kernel with
 *             shared-memory histograms, longer ones (Chamfer clouds) through a stable radix sort
 *             with stream-ordered scratch (cudaMallocAsync)
 *   dest ranges [dest_off[b], dest_off[b] + dest_len[b]) must tile [0, n_dest)
 */
size_t mxs_csr_workspace_bytes(int64_t n_q, int64_t n_dest);
int mxs_build_inverse_csr(const int32_t* argmax, int64_t n_q, int64_t n_docs, int64_t l_q, const int64_t* dest_off,
                          const int64_t* dest_len, int64_t n_dest, int64_t max_dest_len, int32_t* row_ptr,
                          int32_t* col_idx, void* ws, size_t ws_bytes, void* stream);

/*
 * FP32 inputs with the reference's exact arithmetic: float64 gradients, accumulated in the
 * reference's order with rounded f64 products and adds (bit-identical to maxsim/backward.py:135
 * grad_docs_csr and :218 grad_query).  g is float64 [n_q, n_docs]; dD [n_dest, dim] and
 * dQ [n_q, l_q, dim] are float64.  Same ownership rules as the entries below.
 */
int mxs_grad_docs_csr_f64(const int32_t* row_ptr, const int32_t* col_idx, int64_t n_dest, const double* g,
                          const float* Q, int64_t n_q, int64_t n_docs, int64_t l_q, int64_t dim, double* dD,
                          void* stream);
int mxs_grad_query_f64(const int32_t* argmax, const double* g, const float* D, const int64_t* doc_row_off, int64_t n_q,
                       int64_t n_docs, int64_t l_q, int64_t dim, double* dQ, void* stream);

/*
 * Destination-owned document gradient.  Replaces maxsim/backward.py:135 grad_docs_csr.
 *   dD[r] = sum_{s in bucket r} g[q(s), b(s)] * Q[q_row(s)]   (fp32 accumulation, no atomics)
 *   g [n_q, n_docs] f32; Q [n_q, l_q, dim] of `dtype`; dD [n_dest, dim] f32.
 */
int mxs_grad_docs_csr(int dtype, const int32_t* row_ptr, const int32_t* col_idx, int64_t n_dest, const float* g,
                      const void* Q, int64_t n_q, int64_t n_docs, int64_t l_q, int64_t dim, float* dD, void* stream);

/*
 * Query gradient (gather).  Replaces maxsim/backward.py:218 grad_query.
 *   dQ[q, i] = sum_b g[q, b] * D[doc_row_off[b] + argmax[q, b, i]]   (b ascending, fp32)
 *   D is the flat [rows, dim] document buffer (padded batch or packed tokens).
 */
int mxs_grad_query(int dtype, const int32_t* argmax, const float* g, const void* D, const int64_t* doc_row_off,
                   int64_t n_q, int64_t n_docs, int64_t l_q, int64_t dim, float* dQ, void* stream);

/*
 * Top-K selection with the reference ranking: score descending, document id ascending.
 * Replaces maxsim/streamio.py:230 TopKHeap (offer/ranked) and maxsim/cli.py:88 _ranked.
 *   scores [n] f64 -> top_s [k] f64, top_id [k] int64 (= position + id_offset).
 *   ws >= mxs_topk_workspace_bytes(n, k) bytes (may be NULL when that is 0: n <= 16384 for
 *   k <= 128, n <= 4096 above); k <= 2048.
 */
size_t mxs_topk_workspace_bytes(int64_t n, int64_t k);
int mxs_topk(const double* scores, int64_t n, int64_t k, int64_t id_offset, double* top_s, int64_t* top_id, void* ws,
             size_t ws_bytes, void* stream);
/*
 * Top-K over explicit (score, id) candidates, e.g. the all-gathered per-rank top-K lists of a
 * sharded corpus; entries with id < 0 are empty slots.  Same ordering as mxs_topk
 * (maxsim/streamio.py:255-262 TopKHeap.merge).  Slots beyond the valid candidates get id -1.
 * n <= 8192 for k <= 128 (n <= 4096 above).
 */
int mxs_topk_candidates(const double* scores, const int64_t* ids, int64_t n, int64_t k, double* top_s, int64_t* top_id,
                        void* stream);

/*
 * Chamfer distance (maxsim/chamfer.py:49-199), float32 bit-exact with the reference.
 *   mxs_sq_norms       X [rows, dim] f32 -> out [rows] f32 (maxsim/kernels.py:41 sq_norms)
 *   mxs_chamfer_nn     per point of A: min over B of |a|^2 + |b|^2 - 2<a,b> (reference order)
 *                      and the lowest argmin (maxsim/chamfer.py:49 _nearest_fold); dim <= 16
 *   mxs_chamfer_grad   one side of chamfer_backward (maxsim/chamfer.py:167): float64
 *                      dX[r] = c_gather (x_r - y_nn[r]) + sum over CSR bucket r of c_scatter (x_r - y_j)
 */
int mxs_sq_norms(const float* X, int64_t rows, int64_t dim, float* out, void* stream);
int mxs_chamfer_nn(const float* A, const float* a_norms, int64_t n, const float* B, const float* b_norms, int64_t m,
                   int64_t dim, float* best, int32_t* idx, void* stream);
int mxs_chamfer_grad(const float* X, int64_t nx, const float* Y, int64_t dim, const int32_t* nn,
                     const int32_t* row_ptr, const int32_t* col_idx, double c_gather, double c_scatter, double* dX,
                     void* stream);

/*
 * MXS1 embedding files (HOST side; maxsim/streamio.py:1-163).  Replaces _parse_header
 * (maxsim/streamio.py:103), read_embeddings (:136) and CorpusReader.read_block (:209).
 *   mxs_mxs1_open        parse + validate the header; *handle owns the file descriptor
 *   mxs_mxs1_info        elem (0 f32, 1 f16, 2 i8), layout (0 dense, 1 packed, 2 quantized),
 *                        n_docs, length (dense / quantized; 0 for packed), dim
 *   mxs_mxs1_cu_seqlens  packed only: copy the offset table [n_docs + 1] (int64) to host `out`
 *   mxs_mxs1_block_bytes payload bytes of documents [first, first + count)
 *   mxs_mxs1_read_block  copy those raw elements (file dtype) into HOST memory `dst`
 *   mxs_mxs1_read_scales quantized only: the [n_docs * length] f32 scales into HOST `dst`
 * Errors: MXS_IO_ERROR, MXS_BAD_MAGIC, MXS_VERSION_UNSUPPORTED, MXS_TRUNCATED_PAYLOAD (with the
 * reference's expected / actual byte counts in mxs_last_error()).
 */
int mxs_mxs1_open(const char* path, void** handle);
int mxs_mxs1_info(void* handle, int32_t* elem, int32_t* layout, int64_t* n_docs, int64_t* length, int64_t* dim);
int mxs_mxs1_cu_seqlens(void* handle, int64_t* out);
int64_t mxs_mxs1_block_bytes(void* handle, int64_t first, int64_t count);
int mxs_mxs1_read_block(void* handle, int64_t first, int64_t count, void* dst, size_t dst_bytes);
int mxs_mxs1_read_scales(void* handle, float* dst, size_t dst_bytes);
void mxs_mxs1_close(void* handle);

#ifdef __cplusplus
}
#endif

#endif /* MAXSIM_B200_H */
