// extern "C" entry points of libmaxsim_b200.so (see include/maxsim_b200.h).
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/maxsim_b200.h"
#include "fwd_exact.cuh"
#include "fwd_tc.cuh"

namespace {

thread_local std::string g_err;

int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return status;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MXS_CUDA_ERROR, "%s: %s", what, cudaGetErrorString(e));
  return MXS_OK;
}

int sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  static int cache[64] = {0};
  if (dev < 64 && cache[dev]) return cache[dev];
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  if (dev < 64) cache[dev] = n;
  return n;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D row-major [rows, cols] tensor, box = 128 bytes x 128 rows, SWIZZLE_128B.
int make_tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem_bytes, int64_t cols,
                 int64_t rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(MXS_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(cols * elem_bytes)};
  cuuint32_t box[2] = {(cuuint32_t)(128 / elem_bytes), 128u};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MXS_CUDA_ERROR, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return MXS_OK;
}

int launch_rowsum(const float* rowmax, int64_t n_pairs, int64_t l_q, double* scores, cudaStream_t st) {
  if (n_pairs <= 0) return MXS_OK;
  const int threads = 256;
  const long long blocks = (n_pairs * 32 + threads - 1) / threads;
  mxs::rowsum_kernel<<<(unsigned)blocks, threads, 0, st>>>(rowmax, n_pairs, (int)l_q, scores);
  return check_launch("rowsum_kernel");
}

template <mxs::TcKind KIND>
int launch_fwd_tc(const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad, int64_t dim,
                  const int32_t* valid_lens, const float* q_scale, const float* d_scale, float* rowmax,
                  int32_t* argmax, cudaStream_t st) {
  const int eb = (KIND == mxs::TcKind::I8) ? 1 : 2;
  if ((dim * eb) % 16 != 0)
    return fail(MXS_UNSUPPORTED, "tensor-core path needs dim*elem_bytes %% 16 == 0 (dim=%lld)", (long long)dim);
  const int ka = (int)((dim * eb + 127) / 128);
  const int nmb = (int)((l_q + 127) / 128);
  int qb = nmb < mxs::kMaxQb ? nmb : mxs::kMaxQb;
  // shared-memory budget: (qb + stages) * ka * 16 KB <= ~225 KB
  const size_t max_smem = 232448;
  int stages = 0;
  for (;;) {
    stages = (int)((max_smem - 1024 - sizeof(mxs::FwdSmemHeader)) / ((size_t)ka * mxs::kAtomBytes)) - qb;
    if (stages > 8) stages = 8;
    if (stages >= 2 || qb == 1) break;
    --qb;
  }
  if (stages < 2) return fail(MXS_UNSUPPORTED, "dim %lld too large for the tensor-core tile", (long long)dim);
  mxs::FwdTcParams p;
  p.n_q = (int)n_q;
  p.l_q = (int)l_q;
  p.n_docs = (int)n_docs;
  p.l_pad = (int)l_pad;
  p.dim = (int)dim;
  p.ka = ka;
  p.qb = qb;
  p.n_groups = (nmb + qb - 1) / qb;
  p.stages = stages;
  p.n_units = (long long)n_q * p.n_groups * n_docs;
  p.valid_lens = valid_lens;
  p.q_scale = q_scale;
  p.d_scale = d_scale;
  p.rowmax = rowmax;
  p.argmax = argmax;
  {
    const char* dbg = getenv("MXS_DEBUG");
    p.debug = dbg ? atoi(dbg) : 0;
  }
  CUtensorMap tq, td;
  const CUtensorMapDataType dt = (KIND == mxs::TcKind::I8)     ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : (KIND == mxs::TcKind::BF16) ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                               : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  int s;
  if ((s = make_tmap_2d(&tq, Q, dt, eb, dim, n_q * l_q)) != MXS_OK) return s;
  if ((s = make_tmap_2d(&td, D, dt, eb, dim, n_docs * l_pad)) != MXS_OK) return s;
  const size_t smem = mxs::fwd_tc_smem_bytes(ka, qb, stages);
  auto kern = mxs::fwd_tc_kernel<KIND>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return fail(MXS_CUDA_ERROR, "cudaFuncSetAttribute(smem=%zu) failed", smem);
  const int nsm = sm_count();
  if (nsm <= 0) return fail(MXS_CUDA_ERROR, "no CUDA device");
  long long grid = p.n_units < nsm ? p.n_units : nsm;
  if (grid <= 0) return MXS_OK;
  kern<<<(unsigned)grid, mxs::kFwdThreads, smem, st>>>(tq, td, p);
  return check_launch("fwd_tc_kernel");
}

template <typename T>
int launch_fwd_exact(const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad,
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
  mxs::fwd_exact_kernel<T><<<(unsigned)grid, mxs::kExThreads, 0, st>>>(static_cast<const T*>(Q),
                                                                        static_cast<const T*>(D), p);
  return check_launch("fwd_exact_kernel");
}

}  // namespace

extern "C" {

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
    default: return "unknown";
  }
}

const char* mxs_last_error(void) { return g_err.c_str(); }

int mxs_device_sm_count(void) { return sm_count(); }

int mxs_rowsum(const float* rowmax, int64_t n_pairs, int64_t l_q, double* scores, void* stream) {
  if (!rowmax || !scores || n_pairs < 0 || l_q < 1) return fail(MXS_INVALID_ARGUMENT, "mxs_rowsum: bad arguments");
  return launch_rowsum(rowmax, n_pairs, l_q, scores, (cudaStream_t)stream);
}

int mxs_fused_score_batch(int dtype, const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs,
                          int64_t l_pad, int64_t dim, const int32_t* valid_lens, double* scores, int32_t* argmax,
                          float* rowmax, int exact, void* stream) {
  if (!Q || !D || !scores || !rowmax) return fail(MXS_INVALID_ARGUMENT, "mxs_fused_score_batch: null pointer");
  if (n_q < 1 || n_docs < 1 || l_q < 1 || l_pad < 1 || dim < 1)
    return fail(MXS_SHAPE_MISMATCH, "mxs_fused_score_batch: non-positive shape");
  if (n_q * l_q >= (1LL << 31) || n_docs * l_pad >= (1LL << 31) || n_q * n_docs * l_q >= (1LL << 40))
    return fail(MXS_UNSUPPORTED, "mxs_fused_score_batch: problem too large for 32-bit row indices");
  cudaStream_t st = (cudaStream_t)stream;
  int s;
  if (exact || dtype == MXS_F32) {
    if (dtype == MXS_F32)
      s = launch_fwd_exact<float>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, rowmax, argmax, st);
    else if (dtype == MXS_BF16)
      s = launch_fwd_exact<__nv_bfloat16>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, rowmax, argmax, st);
    else if (dtype == MXS_F16)
      s = launch_fwd_exact<__half>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, rowmax, argmax, st);
    else
      return fail(MXS_UNSUPPORTED, "mxs_fused_score_batch: dtype %d not a float type", dtype);
  } else if (dtype == MXS_BF16) {
    s = launch_fwd_tc<mxs::TcKind::BF16>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, nullptr, rowmax,
                                         argmax, st);
  } else if (dtype == MXS_F16) {
    s = launch_fwd_tc<mxs::TcKind::F16>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, nullptr, rowmax,
                                        argmax, st);
  } else {
    return fail(MXS_UNSUPPORTED, "mxs_fused_score_batch: dtype %d", dtype);
  }
  if (s != MXS_OK) return s;
  return launch_rowsum(rowmax, n_q * n_docs, l_q, scores, st);
}

int mxs_fused_score_int8(const int8_t* Q, const float* q_scale, int64_t n_q, int64_t l_q, const int8_t* D,
                         const float* d_scale, int64_t n_docs, int64_t l_pad, int64_t dim, const int32_t* valid_lens,
                         double* scores, int32_t* argmax, float* rowmax, void* stream) {
  if (!Q || !D || !q_scale || !d_scale || !scores || !rowmax)
    return fail(MXS_INVALID_ARGUMENT, "mxs_fused_score_int8: null pointer");
  if (n_q < 1 || n_docs < 1 || l_q < 1 || l_pad < 1 || dim < 1)
    return fail(MXS_SHAPE_MISMATCH, "mxs_fused_score_int8: non-positive shape");
  if (dim > 133000) return fail(MXS_SHAPE_MISMATCH, "dim %lld exceeds 133000 (int32 accumulation bound)", (long long)dim);
  cudaStream_t st = (cudaStream_t)stream;
  int s = launch_fwd_tc<mxs::TcKind::I8>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, q_scale, d_scale, rowmax,
                                         argmax, st);
  if (s != MXS_OK) return s;
  return launch_rowsum(rowmax, n_q * n_docs, l_q, scores, st);
}

}  // extern "C"
