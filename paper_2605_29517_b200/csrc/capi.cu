// extern "C" entry points of libmaxsim_b200.so (see include/maxsim_b200.h): forward dispatch,
// status strings and the MXS1 reader.  Kernels live in the launch_*.cu translation units.
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <string>

#include "host.h"
#include "mxs1_io.h"
#include <exception>

using namespace mxs_host;

namespace {
bool rerank_r3_opt_in() { return env_is("MXS_RERANK_IMPL", "r3"); }
bool use_ts_path() { return !env_is("MXS_FWD_IMPL", "ss"); }
}  // namespace

namespace {

// Row-maxima scratch for paths whose S4 sum runs as a separate pass when the caller did not ask
// for the row maxima (rowmax == NULL): stream-ordered allocation, freed after the rowsum pass.
struct RowmaxScratch {
  float* ptr = nullptr;
  cudaStream_t st = nullptr;
  int get(float* user, size_t n, cudaStream_t stream, float** out) {
    if (user || ptr) {
      *out = user ? user : ptr;
      return MXS_OK;
    }
    st = stream;
    if (int s = scratch_alloc((void**)&ptr, n * sizeof(float), stream)) return s;
    *out = ptr;
    return MXS_OK;
  }
  ~RowmaxScratch() {
    if (ptr) cudaFreeAsync(ptr, st);
  }
};

int check_dense_shapes(const char* what, int64_t n_q, int64_t l_q, int64_t n_docs, int64_t l_pad, int64_t dim) {
  if (n_q < 1 || n_docs < 1 || l_q < 1 || l_pad < 1 || dim < 1) return fail(MXS_SHAPE_MISMATCH, "%s: non-positive shape", what);
  if (n_q * l_q >= (1LL << 31) || n_docs * l_pad >= (1LL << 31) || n_q * n_docs * l_q >= (1LL << 40))
    return fail(MXS_UNSUPPORTED, "%s: problem too large for 32-bit row indices", what);
  return MXS_OK;
}

// bf16 / fp16 tensor-core dispatch: fwd_i8r (opt-in rerank) -> fwd_pair -> fwd_ts -> SS fwd_tc -> exact SIMT.
// On return *fused says whether `scores` was already written by the kernel's epilogue.
template <mxs::TcKind KIND>
int dispatch_float_tc(int dtype, const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad,
                      int64_t dim, const int32_t* valid_lens, int32_t* argmax, float* rowmax, double* scores,
                      int* fused, cudaStream_t st) {
  *fused = 0;
  // bf16 rerank: the three-slot kernel (2 resident Q blocks) measured 1.83 ms vs 1.76 ms for
  // fwd_ts at the C2 shape, so it is opt-in (MXS_RERANK_IMPL=r3)
  int s = (argmax || !rerank_r3_opt_in())
              ? MXS_UNSUPPORTED
              : launch_fwd_r3<KIND>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, nullptr, rowmax, scores,
                                    fused, st);
  // CTA-pair kernel (three accumulator slots) for 256 < L_q <= 1024, d <= 128; MXS_FWD_IMPL=ts
  // forces the single-CTA kernel
  if (s == MXS_UNSUPPORTED && use_ts_path() && !env_is("MXS_FWD_IMPL", "ts"))
    s = launch_fwd_pair<KIND>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, rowmax, argmax, scores, fused, st);
  if (s == MXS_UNSUPPORTED && use_ts_path())
    s = launch_fwd_ts<KIND>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, nullptr, rowmax, argmax, scores,
                            fused, st);
  if (!rowmax) return s;  // fused-sum attempt only: the kernels below need row maxima
  if (s == MXS_UNSUPPORTED)
    s = launch_fwd_tc<KIND>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, nullptr, rowmax, argmax, st);
  if (s == MXS_UNSUPPORTED)  // widths past the tensor-core tiles (d > 256 etc.): exact SIMT kernel on the GPU
    s = launch_fwd_exact(dtype, Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, rowmax, argmax, st);
  return s;
}

// rowmax must be non-null unless `scores` is (then the caller wants the row maxima only).
int fused_forward(int dtype, const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad,
                  int64_t dim, const int32_t* valid_lens, int32_t* argmax, float* rowmax, double* scores, int exact,
                  int* fused, cudaStream_t st) {
  *fused = 0;
  if (exact || dtype == MXS_F32) {
    if (dtype != MXS_F32 && dtype != MXS_BF16 && dtype != MXS_F16)
      return fail(MXS_UNSUPPORTED, "mxs_fused_score_batch: dtype %d not a float type", dtype);
    return launch_fwd_exact(dtype, Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, rowmax, argmax, st);
  }
  if (dtype == MXS_BF16)
    return dispatch_float_tc<mxs::TcKind::BF16>(dtype, Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, argmax, rowmax,
                                                scores, fused, st);
  if (dtype == MXS_F16)
    return dispatch_float_tc<mxs::TcKind::F16>(dtype, Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, argmax, rowmax,
                                               scores, fused, st);
  return fail(MXS_UNSUPPORTED, "mxs_fused_score_batch: dtype %d", dtype);
}

}  // namespace


extern "C" {

int mxs_fused_rowmax_batch(int dtype, const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs,
                           int64_t l_pad, int64_t dim, const int32_t* valid_lens, int32_t* argmax, float* rowmax,
                           int exact, void* stream);

const char* mxs_version(void) { return "maxsim_b200 0.1.0 (sm_100a)"; }

const char* mxs_status_string(int s) {
  switch (s) {
    case MXS_OK: return "ok";
    case MXS_DIM_MISMATCH: return "DimMismatch";
    case MXS_SHAPE_MISMATCH: return "ShapeMismatch";
    case MXS_EMPTY_DOCUMENT: return "EmptyDocument";
    case MXS_INDEX_OUT_OF_RANGE: return "IndexOutOfRange";
    case MXS_STALE_CSR: return "StaleCsr";
    case MXS_K_TOO_LARGE: return "KTooLarge";
    case MXS_NAN_INPUT: return "NaNInput";
    case MXS_BAD_TILE_CONFIG: return "BadTileConfig";
    case MXS_UNSUPPORTED: return "Unsupported";
    case MXS_CUDA_ERROR: return "CudaError";
    case MXS_INVALID_ARGUMENT: return "InvalidArgument";
    case MXS_IO_ERROR: return "IoError";
    case MXS_BAD_MAGIC: return "BadMagic";
    case MXS_VERSION_UNSUPPORTED: return "VersionUnsupported";
    case MXS_TRUNCATED_PAYLOAD: return "TruncatedPayload";
    case MXS_STALE_ARGMIN: return "StaleArgmin";
    default: return "unknown";
  }
}

const char* mxs_last_error(void) { return last_error(); }

int mxs_device_sm_count(void) { return sm_count(); }

int mxs_rowsum(const float* rowmax, int64_t n_pairs, int64_t l_q, double* scores, void* stream) {
  if (!rowmax || !scores || n_pairs < 0 || l_q < 1) return fail(MXS_INVALID_ARGUMENT, "mxs_rowsum: bad arguments");
  return launch_rowsum(rowmax, n_pairs, l_q, scores, (cudaStream_t)stream);
}

int mxs_fused_score_batch(int dtype, const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs,
                          int64_t l_pad, int64_t dim, const int32_t* valid_lens, double* scores, int32_t* argmax,
                          float* rowmax, int exact, void* stream) {
  if (!Q || !D || !scores) return fail(MXS_INVALID_ARGUMENT, "mxs_fused_score_batch: null pointer");
  int s = check_dense_shapes("mxs_fused_score_batch", n_q, l_q, n_docs, l_pad, dim);
  if (s != MXS_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  // try the fused epilogue first (no row maxima in HBM unless requested)
  int fused = 0;
  RowmaxScratch scratch;
  if (!rowmax && !exact && dtype != MXS_F32) {
    s = fused_forward(dtype, Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, argmax, nullptr, scores, 0, &fused, st);
    if (s == MXS_OK && fused) return MXS_OK;
    if (s != MXS_OK && s != MXS_UNSUPPORTED) return s;
    if (s == MXS_OK && !fused) return fail(MXS_CUDA_ERROR, "forward launched without row maxima or fused sum");
  }
  float* rm = nullptr;
  if ((s = scratch.get(rowmax, (size_t)(n_q * n_docs * l_q), st, &rm)) != MXS_OK) return s;
  s = fused_forward(dtype, Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, argmax, rm, scores, exact, &fused, st);
  if (s != MXS_OK || fused) return s;
  return launch_rowsum(rm, n_q * n_docs, l_q, scores, st);
}

int mxs_fused_rowmax_batch(int dtype, const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs,
                           int64_t l_pad, int64_t dim, const int32_t* valid_lens, int32_t* argmax, float* rowmax,
                           int exact, void* stream) {
  if (!Q || !D || !rowmax) return fail(MXS_INVALID_ARGUMENT, "mxs_fused_rowmax_batch: null pointer");
  int s = check_dense_shapes("mxs_fused_rowmax_batch", n_q, l_q, n_docs, l_pad, dim);
  if (s != MXS_OK) return s;
  int fused = 0;
  return fused_forward(dtype, Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, argmax, rowmax, nullptr, exact, &fused,
                       (cudaStream_t)stream);
}

int mxs_fused_score_int8(const int8_t* Q, const float* q_scale, int64_t n_q, int64_t l_q, const int8_t* D,
                         const float* d_scale, int64_t n_docs, int64_t l_pad, int64_t dim, const int32_t* valid_lens,
                         double* scores, int32_t* argmax, float* rowmax, void* stream) {
  if (!Q || !D || !q_scale || !d_scale || !scores) return fail(MXS_INVALID_ARGUMENT, "mxs_fused_score_int8: null pointer");
  int s = check_dense_shapes("mxs_fused_score_int8", n_q, l_q, n_docs, l_pad, dim);
  if (s != MXS_OK) return s;
  if (dim > 133000) return fail(MXS_SHAPE_MISMATCH, "dim %lld exceeds 133000 (int32 accumulation bound)", (long long)dim);
  cudaStream_t st = (cudaStream_t)stream;
  int fused = 0;
  // pass 0: fused epilogue sum, no row maxima; pass 1: row maxima (user buffer or scratch) + rowsum
  RowmaxScratch scratch;
  for (int pass = rowmax ? 1 : 0; pass < 2; ++pass) {
    float* rm = nullptr;
    if (pass == 1 && (s = scratch.get(rowmax, (size_t)(n_q * n_docs * l_q), st, &rm)) != MXS_OK) return s;
    s = argmax ? MXS_UNSUPPORTED
               : launch_fwd_r3<mxs::TcKind::I8>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, q_scale, d_scale, rm,
                                                scores, &fused, st);
    if (s == MXS_UNSUPPORTED && use_ts_path())
      s = launch_fwd_ts<mxs::TcKind::I8>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, q_scale, d_scale, rm, argmax,
                                         scores, &fused, st);
    if (pass == 0) {
      if (s == MXS_OK && fused) return MXS_OK;
      if (s != MXS_OK && s != MXS_UNSUPPORTED) return s;
      if (s == MXS_OK) return fail(MXS_CUDA_ERROR, "INT8 forward launched without row maxima or fused sum");
      continue;
    }
    if (s == MXS_UNSUPPORTED)
      s = launch_fwd_tc<mxs::TcKind::I8>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, q_scale, d_scale, rm, argmax,
                                         st);
    if (s == MXS_UNSUPPORTED)  // widths past the tensor-core tiles: exact SIMT kernel (still on the GPU)
      s = launch_fwd_exact_i8(Q, q_scale, n_q, l_q, D, d_scale, n_docs, l_pad, dim, valid_lens, rm, argmax, st);
    if (s != MXS_OK || fused) return s;
    return launch_rowsum(rm, n_q * n_docs, l_q, scores, st);
  }
  return MXS_OK;
}

int mxs_fused_score_varlen(int dtype, const void* Q, int64_t n_q, int64_t l_q, const void* tokens,
                           const int64_t* cu_seqlens, int64_t n_docs, int64_t n_tokens, int64_t dim, double* scores,
                           int32_t* argmax, float* rowmax, int exact, void* stream) {
  if (!Q || !tokens || !cu_seqlens || !scores) return fail(MXS_INVALID_ARGUMENT, "mxs_fused_score_varlen: null pointer");
  if (n_q < 1 || n_docs < 1 || l_q < 1 || dim < 1 || n_tokens < 1)
    return fail(MXS_SHAPE_MISMATCH, "mxs_fused_score_varlen: non-positive shape");
  cudaStream_t st = (cudaStream_t)stream;
  int s = MXS_UNSUPPORTED, fused = 0;
  RowmaxScratch scratch;
  if (!exact && (dtype == MXS_BF16 || dtype == MXS_F16)) {
    for (int pass = rowmax ? 1 : 0; pass < 2; ++pass) {
      float* rm = nullptr;
      if (pass == 1 && (s = scratch.get(rowmax, (size_t)(n_q * n_docs * l_q), st, &rm)) != MXS_OK) return s;
      s = dtype == MXS_BF16 ? launch_varlen_tc<mxs::TcKind::BF16>(Q, n_q, l_q, tokens, cu_seqlens, n_docs, n_tokens, dim,
                                                                  rm, argmax, scores, &fused, st)
                            : launch_varlen_tc<mxs::TcKind::F16>(Q, n_q, l_q, tokens, cu_seqlens, n_docs, n_tokens, dim,
                                                                 rm, argmax, scores, &fused, st);
      if (s == MXS_OK && fused) return MXS_OK;
      if (s != MXS_OK && s != MXS_UNSUPPORTED) return s;
      if (s == MXS_OK && pass == 0) return fail(MXS_CUDA_ERROR, "varlen forward launched without row maxima or fused sum");
      if (s == MXS_OK) return launch_rowsum(rm, n_q * n_docs, l_q, scores, st);
      if (pass == 0) continue;
      break;  // unsupported shape: exact SIMT path below (reuses the scratch)
    }
  }
  if (dtype != MXS_F32 && dtype != MXS_BF16 && dtype != MXS_F16)
    return fail(MXS_UNSUPPORTED, "mxs_fused_score_varlen: dtype %d", dtype);
  float* rm = nullptr;
  if ((s = scratch.get(rowmax, (size_t)(n_q * n_docs * l_q), st, &rm)) != MXS_OK) return s;
  s = launch_fwd_exact(dtype, Q, n_q, l_q, tokens, n_docs, 0, dim, nullptr, cu_seqlens, rm, argmax, st);
  if (s != MXS_OK) return s;
  return launch_rowsum(rm, n_q * n_docs, l_q, scores, st);
}

// ------------------------------------------------------------------ MXS1 files (host side)
static int mxs1_truncated(int64_t expected, int64_t actual) {
  return fail(MXS_TRUNCATED_PAYLOAD, "payload truncated: expected %lld bytes, file holds %lld", (long long)expected,
              (long long)actual);
}

static int mxs1_read_block_impl(void* handle, int64_t first, int64_t count, void* dst, size_t dst_bytes);

static int mxs1_open_impl(const char* path, void** handle) {
  if (!path || !handle) return fail(MXS_INVALID_ARGUMENT, "mxs_mxs1_open: null pointer");
  *handle = nullptr;
  const int fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0) return fail(MXS_IO_ERROR, "cannot read %s: %s", path, strerror(errno));
  auto* f = new mxs_io::Mxs1File();
  f->fd = fd;
  f->path = path;
  struct stat stt;
  f->file_size = (fstat(fd, &stt) == 0) ? (int64_t)stt.st_size : 0;
  auto bail = [&](int st) {
    ::close(fd);
    delete f;
    return st;
  };
  unsigned char head[8];
  if (mxs_io::pread_all(fd, head, 8, 0) != 8) return bail(fail(MXS_BAD_MAGIC, "file too short to hold a header"));
  if (memcmp(head, "MXS1", 4) != 0) {
    char m[64];
    snprintf(m, sizeof(m), "b'%c%c%c%c'", head[0], head[1], head[2], head[3]);
    return bail(fail(MXS_BAD_MAGIC, "bad magic %s", m));
  }
  const unsigned version = (unsigned)head[4] | ((unsigned)head[5] << 8);
  if (version != 1) return bail(fail(MXS_VERSION_UNSUPPORTED, "unsupported embedding file version %u", version));
  const int ec = head[6], lc = head[7];
  if (ec > 2 || lc > 2) return bail(fail(MXS_BAD_MAGIC, "unknown element/layout tags (%d, %d)", ec, lc));
  f->elem = ec;
  f->layout = lc;
  int64_t off = 8;
  auto u64 = [&](int64_t& out) -> bool {
    uint64_t v = 0;
    const int64_t got = mxs_io::pread_all(fd, &v, 8, off);
    if (got != 8) {
      mxs1_truncated(8, got < 0 ? 0 : got);
      return false;
    }
    off += 8;
    out = (int64_t)v;  // little-endian host (x86-64 / aarch64)
    return true;
  };
  // Header sizes come from an untrusted file: every count and byte product is checked against
  // the file size before anything is allocated (a hostile n_docs must raise TruncatedPayload the
  // way the reference's short read does, not abort the process with bad_alloc).
  if (lc == mxs_io::kDense || lc == mxs_io::kQuantized) {
    if (!u64(f->n_docs) || !u64(f->length) || !u64(f->dim)) return bail(MXS_TRUNCATED_PAYLOAD);
    const int64_t avail = f->file_size > off ? f->file_size - off : 0;
    int64_t need = 0;
    if (!mxs_io::payload_bytes(f->n_docs, f->length, f->dim, mxs_io::elem_size(ec), lc == mxs_io::kQuantized, &need))
      return bail(fail(MXS_TRUNCATED_PAYLOAD, "payload truncated: expected %llu bytes, file holds %lld",
                       (unsigned long long)UINT64_MAX, (long long)avail));
    (void)need;  // a short payload is reported lazily by the block reads (streaming reads a prefix)
  } else {
    if (!u64(f->n_docs) || !u64(f->dim)) return bail(MXS_TRUNCATED_PAYLOAD);
    const int64_t avail = f->file_size > off ? f->file_size - off : 0;
    // 8 * (n_docs + 1) offsets must fit in what is left of the file (n_docs < 0 = top bit set)
    if (f->n_docs < 0 || f->n_docs >= avail / 8) {
      const unsigned long long want = (f->n_docs < 0 || f->n_docs > (INT64_MAX / 8 - 1))
                                          ? (unsigned long long)UINT64_MAX
                                          : (unsigned long long)(8 * (f->n_docs + 1));
      return bail(fail(MXS_TRUNCATED_PAYLOAD, "payload truncated: expected %llu bytes, file holds %lld", want,
                       (long long)avail));
    }
    const int64_t need = 8 * (f->n_docs + 1);
    try {
      f->cu.resize((size_t)f->n_docs + 1);
    } catch (...) {
      return bail(fail(MXS_IO_ERROR, "cannot allocate the offset table of %lld documents", (long long)f->n_docs));
    }
    const int64_t got = mxs_io::pread_all(fd, f->cu.data(), need, off);
    if (got != need) return bail(mxs1_truncated(need, got < 0 ? 0 : got));
    off += need;
    // PackedCorpus invariants (maxsim/varlen.py:36-41): cu[0] = 0, strictly increasing, and the
    // token payload cu[B] * dim fits in the file
    if (f->cu[0] != 0)
      return bail(fail(MXS_SHAPE_MISMATCH, "cu_seqlens must be 1-D with cu[0] = 0 and one entry per document plus one"));
    for (int64_t b = 0; b < f->n_docs; ++b)
      if (f->cu[(size_t)b + 1] <= f->cu[(size_t)b]) return bail(fail(MXS_EMPTY_DOCUMENT, "document %lld has no valid tokens", (long long)b));
    const int64_t avail2 = f->file_size > off ? f->file_size - off : 0;
    int64_t need_t = 0;
    if (!mxs_io::payload_bytes(f->cu.back(), 1, f->dim, mxs_io::elem_size(ec), false, &need_t))
      return bail(fail(MXS_TRUNCATED_PAYLOAD, "payload truncated: expected %llu bytes, file holds %lld",
                       (unsigned long long)UINT64_MAX, (long long)avail2));
  }
  if (lc == mxs_io::kQuantized && ec != mxs_io::kI8)
    return bail(fail(MXS_BAD_MAGIC, "quantized layout requires the i8 element tag"));
  if (lc != mxs_io::kQuantized && ec == mxs_io::kI8)
    return bail(fail(MXS_BAD_MAGIC, "int8 elements require the quantized layout (scales are part of the data)"));
  f->payload_offset = off;
  *handle = f;
  return MXS_OK;
}

// The host-side reader allocates (the header object, the offset table) and spawns pread threads:
// no C++ exception may cross the extern "C" / ctypes boundary, so both entry points map one to a status.
int mxs_mxs1_open(const char* path, void** handle) {
  try {
    return mxs1_open_impl(path, handle);
  } catch (const std::exception& e) {
    return fail(MXS_IO_ERROR, "cannot read %s: %s", path ? path : "(null)", e.what());
  } catch (...) {
    return fail(MXS_IO_ERROR, "cannot read %s: unknown error", path ? path : "(null)");
  }
}

int mxs_mxs1_read_block(void* handle, int64_t first, int64_t count, void* dst, size_t dst_bytes) {
  try {
    return mxs1_read_block_impl(handle, first, count, dst, dst_bytes);
  } catch (const std::exception& e) {
    return fail(MXS_IO_ERROR, "mxs_mxs1_read_block: %s", e.what());
  } catch (...) {
    return fail(MXS_IO_ERROR, "mxs_mxs1_read_block: unknown error");
  }
}

int mxs_mxs1_info(void* handle, int32_t* elem, int32_t* layout, int64_t* n_docs, int64_t* length, int64_t* dim) {
  auto* f = static_cast<mxs_io::Mxs1File*>(handle);
  if (!f) return fail(MXS_INVALID_ARGUMENT, "mxs_mxs1_info: null handle");
  if (elem) *elem = f->elem;
  if (layout) *layout = f->layout;
  if (n_docs) *n_docs = f->n_docs;
  if (length) *length = f->length;
  if (dim) *dim = f->dim;
  return MXS_OK;
}

int mxs_mxs1_cu_seqlens(void* handle, int64_t* out) {
  auto* f = static_cast<mxs_io::Mxs1File*>(handle);
  if (!f || !out) return fail(MXS_INVALID_ARGUMENT, "mxs_mxs1_cu_seqlens: null pointer");
  if (f->layout != mxs_io::kPacked) return fail(MXS_SHAPE_MISMATCH, "offset table exists for packed files only");
  memcpy(out, f->cu.data(), f->cu.size() * sizeof(int64_t));
  return MXS_OK;
}

static bool mxs1_range(const mxs_io::Mxs1File* f, int64_t first, int64_t count, int64_t& off, int64_t& bytes) {
  if (first < 0 || count < 0 || first > f->n_docs) return false;
  count = std::min(count, f->n_docs - first);
  const int64_t es = mxs_io::elem_size(f->elem);
  if (f->layout == mxs_io::kPacked) {
    const int64_t t0 = f->cu[(size_t)first], t1 = f->cu[(size_t)(first + count)];
    off = f->payload_offset + t0 * f->dim * es;
    bytes = (t1 - t0) * f->dim * es;
  } else {
    off = f->payload_offset + first * f->length * f->dim * es;
    bytes = count * f->length * f->dim * es;
  }
  return true;
}

int64_t mxs_mxs1_block_bytes(void* handle, int64_t first, int64_t count) {
  auto* f = static_cast<mxs_io::Mxs1File*>(handle);
  int64_t off = 0, bytes = 0;
  if (!f || !mxs1_range(f, first, count, off, bytes)) return -1;
  return bytes;
}

static int mxs1_read_block_impl(void* handle, int64_t first, int64_t count, void* dst, size_t dst_bytes) {
  auto* f = static_cast<mxs_io::Mxs1File*>(handle);
  if (!f || !dst) return fail(MXS_INVALID_ARGUMENT, "mxs_mxs1_read_block: null pointer");
  int64_t off = 0, bytes = 0;
  if (!mxs1_range(f, first, count, off, bytes))
    return fail(MXS_INDEX_OUT_OF_RANGE, "block [%lld, +%lld) outside the %lld documents", (long long)first,
                (long long)count, (long long)f->n_docs);
  if ((int64_t)dst_bytes < bytes) return fail(MXS_INVALID_ARGUMENT, "mxs_mxs1_read_block: buffer too small");
  const int64_t got = mxs_io::pread_parallel(f->fd, dst, bytes, off);
  if (got < 0) return fail(MXS_IO_ERROR, "cannot read %s: %s", f->path.c_str(), strerror(errno));
  if (got != bytes) {
    // the reference reports the expected payload of the whole file for dense / packed loads
    return mxs1_truncated(bytes, got);
  }
  return MXS_OK;
}

int mxs_mxs1_read_scales(void* handle, float* dst, size_t dst_bytes) {
  auto* f = static_cast<mxs_io::Mxs1File*>(handle);
  if (!f || !dst) return fail(MXS_INVALID_ARGUMENT, "mxs_mxs1_read_scales: null pointer");
  if (f->layout != mxs_io::kQuantized) return fail(MXS_SHAPE_MISMATCH, "scales exist for quantized files only");
  const int64_t need_q = f->n_docs * f->length * f->dim, need_s = f->n_docs * f->length * 4;
  if ((int64_t)dst_bytes < need_s) return fail(MXS_INVALID_ARGUMENT, "mxs_mxs1_read_scales: buffer too small");
  const int64_t got = mxs_io::pread_all(f->fd, dst, need_s, f->payload_offset + need_q);
  if (got < 0) return fail(MXS_IO_ERROR, "cannot read %s: %s", f->path.c_str(), strerror(errno));
  if (got != need_s) return mxs1_truncated(need_q + need_s, got);
  return MXS_OK;
}

void mxs_mxs1_close(void* handle) {
  auto* f = static_cast<mxs_io::Mxs1File*>(handle);
  if (!f) return;
  if (f->fd >= 0) ::close(f->fd);
  delete f;
}

}  // extern "C"
