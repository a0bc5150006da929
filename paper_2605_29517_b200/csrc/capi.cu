// extern "C" entry points of libmaxsim_b200.so (see include/maxsim_b200.h).
#include <cerrno>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <type_traits>
#include <string>

#include "../../include/maxsim_b200.h"
#include "fwd_exact.cuh"
#include "fwd_tc.cuh"
#include "fwd_ts.cuh"
#include "fwd_i8r.cuh"
#include "varlen_rows.cuh"
#include "csr.cuh"
#include "grad.cuh"
#include "quant.cuh"
#include "topk.cuh"
#include "mxs1_io.h"
#include "chamfer.cuh"

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

// Persistent cluster grids: as many clusters of `cl` CTAs as the device can keep resident at
// once (clusters of 4 do not tile every GPC, so nsm / 4 may over-subscribe and leave a tail
// wave); falls back to nsm / cl if the occupancy query fails.
template <typename KernT>
long long resident_clusters(KernT kern, int cl, int threads, size_t smem, int nsm) {
  if (cl <= 1) return nsm;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((nsm / cl) * cl));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (void*)kern, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    return nsm / cl;
  }
  return std::min<long long>(n, nsm / cl);
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
                 int64_t rows, int box_rows = 128) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(MXS_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(cols * elem_bytes)};
  cuuint32_t box[2] = {(cuuint32_t)(128 / elem_bytes), (cuuint32_t)box_rows};
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
    const char* spin = getenv("MXS_MMA_SPIN");
    p.mma_spin = spin ? atoi(spin) : 0;
  }
  CUtensorMap tq, td;
  const CUtensorMapDataType dt = (KIND == mxs::TcKind::I8)     ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : (KIND == mxs::TcKind::BF16) ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                               : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  int s;
  if ((s = make_tmap_2d(&tq, Q, dt, eb, dim, n_q * l_q)) != MXS_OK) return s;
  if ((s = make_tmap_2d(&td, D, dt, eb, dim, n_docs * l_pad)) != MXS_OK) return s;
  const size_t smem = mxs::fwd_tc_smem_bytes(ka, qb, stages);
  void (*kern)(const CUtensorMap, const CUtensorMap, const mxs::FwdTcParams) = nullptr;
  switch (ka) {
    case 1: kern = mxs::fwd_tc_kernel<KIND, 1>; break;
    case 2: kern = mxs::fwd_tc_kernel<KIND, 2>; break;
    case 3: kern = mxs::fwd_tc_kernel<KIND, 3>; break;
    case 4: kern = mxs::fwd_tc_kernel<KIND, 4>; break;
    default: return fail(MXS_UNSUPPORTED, "tensor-core path supports dim*elem_bytes <= 512 (dim=%lld)", (long long)dim);
  }
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return fail(MXS_CUDA_ERROR, "cudaFuncSetAttribute(smem=%zu) failed", smem);
  const int nsm = sm_count();
  if (nsm <= 0) return fail(MXS_CUDA_ERROR, "no CUDA device");
  long long grid = p.n_units < nsm ? p.n_units : nsm;
  if (grid <= 0) return MXS_OK;
  kern<<<(unsigned)grid, mxs::kFwdThreads, smem, st>>>(tq, td, p);
  return check_launch("fwd_tc_kernel");
}

// Rerank path (argmax not requested): three accumulator slots / three epilogue warp sets
// (fwd_i8r.cuh).  INT8 with d <= 128 (4 resident Q blocks), bf16 / fp16 with d <= 128 (2 resident
// Q blocks, 4-CTA clusters at L_q = 1024).  Returns MXS_UNSUPPORTED (without launching) otherwise.
template <mxs::TcKind KIND>
int launch_fwd_r3(const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad, int64_t dim,
                  const int32_t* valid_lens, const float* q_scale, const float* d_scale, float* rowmax,
                  cudaStream_t st) {
  constexpr bool kI8 = KIND == mxs::TcKind::I8;
  const int eb = kI8 ? 1 : 2;
  if (dim % 16 != 0 || dim > 128 || (kI8 && l_pad % 4 != 0)) return MXS_UNSUPPORTED;
  {
    const char* impl = getenv(kI8 ? "MXS_I8_IMPL" : "MXS_RERANK_IMPL");
    if (impl && strcmp(impl, "ts") == 0) return MXS_UNSUPPORTED;
  }
  constexpr int ka = kI8 ? 1 : 2;
  const int nmb = (int)((l_q + 127) / 128);
  const int qb = std::min(kI8 ? 4 : 2, nmb);
  const int n_groups = (nmb + qb - 1) / qb;
  const int cl = (n_groups == 2 || n_groups == 4) ? n_groups : 1;
  const size_t max_smem = 232448 - sizeof(mxs::R8SmemHeader);
  const size_t fixed = mxs::fwd_i8r_smem_bytes(ka, 0, kI8);
  int stages = (int)((max_smem - fixed) / ((size_t)ka * mxs::kAtomBytes));
  if (stages > 8) stages = 8;
  if (stages < 2) return MXS_UNSUPPORTED;
  mxs::FwdTcParams p = {};
  p.n_q = (int)n_q;
  p.l_q = (int)l_q;
  p.n_docs = (int)n_docs;
  p.l_pad = (int)l_pad;
  p.dim = (int)dim;
  p.ka = ka;
  p.qb = qb;
  p.n_groups = n_groups;
  p.stages = stages;
  p.n_units = (cl > 1) ? (long long)n_q * n_docs : (long long)n_q * n_groups * n_docs;
  p.valid_lens = valid_lens;
  p.q_scale = q_scale;
  p.d_scale = d_scale;
  p.rowmax = rowmax;
  p.argmax = nullptr;
  p.q_ptr = Q;
  {
    const char* dbg = getenv("MXS_DEBUG");  // 2: slots released unread; 3 (bf16/fp16): no drain wait
    p.debug = dbg ? atoi(dbg) : 0;
    if (kI8 && p.debug == 3) p.debug = 0;
  }
  const CUtensorMapDataType dt = kI8                         ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : KIND == mxs::TcKind::BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap td;
  int s;
  if ((s = make_tmap_2d(&td, D, dt, eb, dim, n_docs * l_pad, 128 / cl)) != MXS_OK) return s;
  const size_t smem = mxs::fwd_i8r_smem_bytes(ka, stages, kI8);
  using KernT = void (*)(const CUtensorMap, const mxs::FwdTcParams);
  KernT kern = cl == 4   ? mxs::fwd_i8r_kernel<KIND, ka, 4>
               : cl == 2 ? mxs::fwd_i8r_kernel<KIND, ka, 2>
                         : mxs::fwd_i8r_kernel<KIND, ka, 1>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return fail(MXS_CUDA_ERROR, "cudaFuncSetAttribute(smem=%zu) failed", smem);
  const int nsm = sm_count();
  if (nsm <= 0) return fail(MXS_CUDA_ERROR, "no CUDA device");
  long long workers = resident_clusters(kern, cl, mxs::kR8Threads, smem, nsm);
  if (p.n_units < workers) workers = p.n_units;
  if (workers <= 0) return MXS_OK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(workers * cl));
  cfg.blockDim = dim3(mxs::kR8Threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, td, p);
  if (e != cudaSuccess) return fail(MXS_CUDA_ERROR, "fwd_i8r_kernel launch: %s", cudaGetErrorString(e));
  return check_launch("fwd_i8r_kernel");
}

// v3 path: Q in TMEM, cluster multicast of document tiles, stash-based argmax.
// Returns MXS_UNSUPPORTED (without launching) when the shape needs the SS kernel.
template <mxs::TcKind KIND>
int launch_fwd_ts(const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad, int64_t dim,
                  const int32_t* valid_lens, const float* q_scale, const float* d_scale, float* rowmax,
                  int32_t* argmax, cudaStream_t st) {
  const int eb = (KIND == mxs::TcKind::I8) ? 1 : 2;
  if ((dim * eb) % 16 != 0) return MXS_UNSUPPORTED;
  const int ka = (int)((dim * eb + 127) / 128);
  if (ka > 4) return MXS_UNSUPPORTED;
  const int qb_max = std::min(mxs::kMaxQb, 256 / (ka * 32));
  const int nmb = (int)((l_q + 127) / 128);
  const int qb = std::min(qb_max, nmb);
  const int n_groups = (nmb + qb - 1) / qb;
  int cl = (n_groups == 2 || n_groups == 4) ? n_groups : 1;
  {
    const char* f = getenv("MXS_FWD_CL");  // profiling knob: force the cluster size (1 = no multicast)
    if (f && atoi(f) == 1) cl = 1;
  }
  const size_t max_smem = 232448 - sizeof(mxs::TsSmemHeader);  // static header comes out of the same 227 KB
  const bool scale_ring = (KIND == mxs::TcKind::I8) && (l_pad % 4 == 0);
  const bool bias = (KIND == mxs::TcKind::I8) && ka <= 2;  // fwd_ts_kernel's kBias
  const size_t fixed = mxs::fwd_ts_smem_bytes(0, qb, 0, scale_ring, bias);
  int stages = (int)((max_smem - fixed) / ((size_t)ka * mxs::kAtomBytes));
  if (stages > 8) stages = 8;
  if (stages < 2) return MXS_UNSUPPORTED;
  mxs::FwdTcParams p = {};
  p.n_q = (int)n_q;
  p.l_q = (int)l_q;
  p.n_docs = (int)n_docs;
  p.l_pad = (int)l_pad;
  p.dim = (int)dim;
  p.ka = ka;
  p.qb = qb;
  p.n_groups = n_groups;
  p.stages = stages;
  p.n_units = (cl > 1) ? (long long)n_q * n_docs : (long long)n_q * n_groups * n_docs;
  p.valid_lens = valid_lens;
  p.q_scale = q_scale;
  p.d_scale = d_scale;
  p.rowmax = rowmax;
  p.argmax = argmax;
  p.q_ptr = Q;
  {
    const char* dbg = getenv("MXS_DEBUG");
    p.debug = dbg ? atoi(dbg) : 0;
    const char* spin = getenv("MXS_MMA_SPIN");
    p.mma_spin = spin ? atoi(spin) : 0;
  }
  CUtensorMap td;
  const CUtensorMapDataType dt = (KIND == mxs::TcKind::I8)     ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : (KIND == mxs::TcKind::BF16) ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                               : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  int s;
  if ((s = make_tmap_2d(&td, D, dt, eb, dim, n_docs * l_pad, 128 / cl)) != MXS_OK) return s;
  const size_t smem = mxs::fwd_ts_smem_bytes(ka, qb, stages, scale_ring, bias);
  using KernT = void (*)(const CUtensorMap, const mxs::FwdTcParams);
  KernT kern = nullptr;
#define MXS_TS_CASE(KA_, CL_) \
  if (ka == KA_ && cl == CL_) kern = mxs::fwd_ts_kernel<KIND, KA_, CL_>;
  MXS_TS_CASE(1, 1) MXS_TS_CASE(1, 2) MXS_TS_CASE(1, 4) MXS_TS_CASE(2, 1) MXS_TS_CASE(2, 2) MXS_TS_CASE(2, 4)
  MXS_TS_CASE(3, 1) MXS_TS_CASE(3, 2) MXS_TS_CASE(3, 4) MXS_TS_CASE(4, 1) MXS_TS_CASE(4, 2) MXS_TS_CASE(4, 4)
#undef MXS_TS_CASE
  if (!kern) return MXS_UNSUPPORTED;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return fail(MXS_CUDA_ERROR, "cudaFuncSetAttribute(smem=%zu) failed", smem);
  const int nsm = sm_count();
  if (nsm <= 0) return fail(MXS_CUDA_ERROR, "no CUDA device");
  long long workers = resident_clusters(kern, cl, mxs::kTsThreads, smem, nsm);
  if (p.n_units < workers) workers = p.n_units;
  if (workers <= 0) return MXS_OK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(workers * cl));
  cfg.blockDim = dim3(mxs::kTsThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, td, p);
  if (e != cudaSuccess) return fail(MXS_CUDA_ERROR, "fwd_ts_kernel launch: %s", cudaGetErrorString(e));
  return check_launch("fwd_ts_kernel");
}

template <mxs::TcKind KIND>
int launch_varlen_tc(const void* Q, int64_t n_q, int64_t l_q, const void* tokens, const int64_t* cu, int64_t n_docs,
                     int64_t n_tokens, int64_t dim, float* rowmax, int32_t* argmax, cudaStream_t st) {
  static_assert(KIND != mxs::TcKind::I8, "varlen is a bf16 / f16 path");
  const int eb = 2;
  const long long rows = n_q * l_q;
  if ((dim * eb) % 16 != 0 || rows >= (1LL << 31)) return MXS_UNSUPPORTED;
  const int ka = (int)((dim * eb + 127) / 128);
  if (ka > 4) return MXS_UNSUPPORTED;
  const size_t max_smem = 232448 - sizeof(mxs::VrSmemHeader);
  const size_t fixed = mxs::varlen_rows_smem_bytes(ka, 0);
  int stages = (int)((max_smem - fixed) / ((size_t)ka * mxs::kAtomBytes));
  if (stages > 8) stages = 8;
  if (stages < 2) return MXS_UNSUPPORTED;
  void (*kern)(const CUtensorMap, const CUtensorMap, const mxs::VarlenRowsParams) = nullptr;
  switch (ka) {
    case 1: kern = mxs::varlen_rows_kernel<KIND, 1>; break;
    case 2: kern = mxs::varlen_rows_kernel<KIND, 2>; break;
    case 3: kern = mxs::varlen_rows_kernel<KIND, 3>; break;
    case 4: kern = mxs::varlen_rows_kernel<KIND, 4>; break;
    default: return MXS_UNSUPPORTED;
  }
  const size_t smem = mxs::varlen_rows_smem_bytes(ka, stages);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return fail(MXS_CUDA_ERROR, "cudaFuncSetAttribute(smem=%zu) failed", smem);
  const int nsm = sm_count();
  if (nsm <= 0) return fail(MXS_CUDA_ERROR, "no CUDA device");
  const long long grid = n_docs < nsm ? n_docs : nsm;
  const CUtensorMapDataType dt =
      (KIND == mxs::TcKind::BF16) ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tt;
  int s;
  if ((s = make_tmap_2d(&tt, tokens, dt, eb, dim, n_tokens)) != MXS_OK) return s;
  // More than 128 query rows (e.g. ColPali queries): one launch per 128-row group; every group
  // streams the token corpus once and writes its own (q, i) outputs.
  for (long long row0 = 0; row0 < rows; row0 += 128) {
    const long long n_cols = std::min(128LL, rows - row0);
    mxs::VarlenRowsParams p = {};
    p.n_q = (int)n_q;
    p.l_q = (int)l_q;
    p.n_cols = (int)n_cols;
    p.row0 = (int)row0;
    p.copies = n_cols <= 32 ? 4 : (n_cols <= 64 ? 2 : 1);  // query-row replication over TMEM quadrants
    p.n_docs = n_docs;
    p.n_tokens = n_tokens;
    p.dim = (int)dim;
    p.stages = stages;
    p.cu = (const long long*)cu;
    p.rowmax = rowmax;
    p.argmax = argmax;
    CUtensorMap tq;
    const void* q0 = static_cast<const uint8_t*>(Q) + row0 * dim * eb;
    // one box per row copy; rows >= n_cols read as 0
    if ((s = make_tmap_2d(&tq, q0, dt, eb, dim, n_cols, 128 / p.copies)) != MXS_OK) return s;
    kern<<<(unsigned)grid, mxs::kVrThreads, smem, st>>>(tt, tq, p);
    if ((s = check_launch("varlen_rows_kernel")) != MXS_OK) return s;
  }
  return MXS_OK;
}

bool rerank_r3_opt_in() {
  const char* impl = getenv("MXS_RERANK_IMPL");
  return impl && strcmp(impl, "r3") == 0;
}

bool use_ts_path() {
  const char* impl = getenv("MXS_FWD_IMPL");
  return !(impl && strcmp(impl, "ss") == 0);
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
  if constexpr (std::is_same<T, float>::value) {
    // double-buffered cp.async variant: 16-B aligned rows (dim % 4 == 0, aligned bases)
    if (dim % 4 == 0 && ((reinterpret_cast<uintptr_t>(Q) | reinterpret_cast<uintptr_t>(D)) & 15) == 0 &&
        !getenv("MXS_EXACT_V1")) {
      static std::once_flag once;
      std::call_once(once, [] {
        cudaFuncSetAttribute(mxs::fwd_exact_f32v_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)mxs::kExV4Smem);
      });
      mxs::fwd_exact_f32v_kernel<<<(unsigned)grid, mxs::kExThreads, mxs::kExV4Smem, st>>>(
          static_cast<const float*>(Q), static_cast<const float*>(D), p);
      return check_launch("fwd_exact_f32v_kernel");
    }
  }
  mxs::fwd_exact_kernel<T><<<(unsigned)grid, mxs::kExThreads, 0, st>>>(static_cast<const T*>(Q),
                                                                        static_cast<const T*>(D), p);
  return check_launch("fwd_exact_kernel");
}

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

const char* mxs_last_error(void) { return g_err.c_str(); }

int mxs_device_sm_count(void) { return sm_count(); }

int mxs_rowsum(const float* rowmax, int64_t n_pairs, int64_t l_q, double* scores, void* stream) {
  if (!rowmax || !scores || n_pairs < 0 || l_q < 1) return fail(MXS_INVALID_ARGUMENT, "mxs_rowsum: bad arguments");
  return launch_rowsum(rowmax, n_pairs, l_q, scores, (cudaStream_t)stream);
}

int mxs_fused_score_batch(int dtype, const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs,
                          int64_t l_pad, int64_t dim, const int32_t* valid_lens, double* scores, int32_t* argmax,
                          float* rowmax, int exact, void* stream) {
  if (!scores) return fail(MXS_INVALID_ARGUMENT, "mxs_fused_score_batch: null pointer");
  int s = mxs_fused_rowmax_batch(dtype, Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, argmax, rowmax, exact, stream);
  if (s != MXS_OK) return s;
  return launch_rowsum(rowmax, n_q * n_docs, l_q, scores, (cudaStream_t)stream);
}

int mxs_fused_rowmax_batch(int dtype, const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs,
                           int64_t l_pad, int64_t dim, const int32_t* valid_lens, int32_t* argmax, float* rowmax,
                           int exact, void* stream) {
  if (!Q || !D || !rowmax) return fail(MXS_INVALID_ARGUMENT, "mxs_fused_score_batch: null pointer");
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
    // bf16 rerank: the three-slot kernel (2 resident Q blocks) measured 1.83 ms vs 1.76 ms for
    // fwd_ts at the C2 shape, so it is opt-in (MXS_RERANK_IMPL=r3)
    s = (argmax || !rerank_r3_opt_in())
            ? MXS_UNSUPPORTED
            : launch_fwd_r3<mxs::TcKind::BF16>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, nullptr,
                                               rowmax, st);
    if (s == MXS_UNSUPPORTED)
      s = use_ts_path() ? launch_fwd_ts<mxs::TcKind::BF16>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr,
                                                           nullptr, rowmax, argmax, st)
                        : MXS_UNSUPPORTED;
    if (s == MXS_UNSUPPORTED)
      s = launch_fwd_tc<mxs::TcKind::BF16>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, nullptr, rowmax,
                                           argmax, st);
    if (s == MXS_UNSUPPORTED)  // widths past the tensor-core tiles (d > 256 etc.): exact SIMT kernel on the GPU
      s = launch_fwd_exact<__nv_bfloat16>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, rowmax, argmax, st);
  } else if (dtype == MXS_F16) {
    s = (argmax || !rerank_r3_opt_in())
            ? MXS_UNSUPPORTED
            : launch_fwd_r3<mxs::TcKind::F16>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, nullptr,
                                              rowmax, st);
    if (s == MXS_UNSUPPORTED)
      s = use_ts_path() ? launch_fwd_ts<mxs::TcKind::F16>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr,
                                                          nullptr, rowmax, argmax, st)
                        : MXS_UNSUPPORTED;
    if (s == MXS_UNSUPPORTED)
      s = launch_fwd_tc<mxs::TcKind::F16>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, nullptr, rowmax,
                                          argmax, st);
    if (s == MXS_UNSUPPORTED)  // widths past the tensor-core tiles (d > 256 etc.): exact SIMT kernel on the GPU
      s = launch_fwd_exact<__half>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, nullptr, rowmax, argmax, st);
  } else {
    return fail(MXS_UNSUPPORTED, "mxs_fused_score_batch: dtype %d", dtype);
  }
  return s;
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
  int s = argmax ? MXS_UNSUPPORTED
                 : launch_fwd_r3<mxs::TcKind::I8>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, q_scale, d_scale,
                                                  rowmax, st);
  if (s == MXS_UNSUPPORTED)
    s = use_ts_path() ? launch_fwd_ts<mxs::TcKind::I8>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, q_scale,
                                                         d_scale, rowmax, argmax, st)
                        : MXS_UNSUPPORTED;
  if (s == MXS_UNSUPPORTED)
    s = launch_fwd_tc<mxs::TcKind::I8>(Q, n_q, l_q, D, n_docs, l_pad, dim, valid_lens, q_scale, d_scale, rowmax,
                                       argmax, st);
  if (s == MXS_UNSUPPORTED)  // widths past the tensor-core tiles: exact SIMT kernel (still on the GPU)
    s = launch_fwd_exact_i8(Q, q_scale, n_q, l_q, D, d_scale, n_docs, l_pad, dim, valid_lens, rowmax, argmax, st);
  if (s != MXS_OK) return s;
  return launch_rowsum(rowmax, n_q * n_docs, l_q, scores, st);
}


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
    const long long want = (rows + 63) / 64;  // 32 groups x 2 rows per block pass (U = 4: 93 regs, slower)
    const long long sblocks = want < (long long)sm_count() * 8 ? want : (long long)sm_count() * 8;
    if (dtype == MXS_BF16)
      mxs::quantize128_stream_kernel<__nv_bfloat16, 2>
          <<<(unsigned)sblocks, 256, 0, st>>>((const __nv_bfloat16*)x, rows, levels, q, scale);
    else
      mxs::quantize128_stream_kernel<__half, 2><<<(unsigned)sblocks, 256, 0, st>>>((const __half*)x, rows, levels, q, scale);
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
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(mxs::csr_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(mxs::csr_place_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(mxs::csr_place_v2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(mxs::csr_count_w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(mxs::csr_place_w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  });
  const unsigned segs = (unsigned)(n_q * n_docs);
  // rows that belong to no document (never the case for padded / packed layouts) stay zero
  if (cudaMemsetAsync(ws, 0, mxs_csr_workspace_bytes(n_q, n_dest), st) != cudaSuccess)
    return fail(MXS_CUDA_ERROR, "memset");
  if (cudaMemsetAsync(row_ptr, 0, sizeof(int32_t) * (size_t)(n_dest + 1), st) != cudaSuccess)
    return fail(MXS_CUDA_ERROR, "memset");
  int s;
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
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(mxs::topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTopkSmem);
    cudaFuncSetAttribute(mxs::topk_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)std::max(select_smem(mxs::kSelChunkImplicit, mxs::kSelMaxK, false),
                                       select_smem(mxs::kSelChunkExplicit, mxs::kSelMaxK, true)));
  });
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

int mxs_fused_score_varlen(int dtype, const void* Q, int64_t n_q, int64_t l_q, const void* tokens,
                           const int64_t* cu_seqlens, int64_t n_docs, int64_t n_tokens, int64_t dim, double* scores,
                           int32_t* argmax, float* rowmax, int exact, void* stream) {
  if (!Q || !tokens || !cu_seqlens || !scores || !rowmax)
    return fail(MXS_INVALID_ARGUMENT, "mxs_fused_score_varlen: null pointer");
  if (n_q < 1 || n_docs < 1 || l_q < 1 || dim < 1 || n_tokens < 1)
    return fail(MXS_SHAPE_MISMATCH, "mxs_fused_score_varlen: non-positive shape");
  cudaStream_t st = (cudaStream_t)stream;
  int s = MXS_UNSUPPORTED;
  const long long* cu = (const long long*)cu_seqlens;
  if (!exact && dtype == MXS_BF16)
    s = launch_varlen_tc<mxs::TcKind::BF16>(Q, n_q, l_q, tokens, cu_seqlens, n_docs, n_tokens, dim, rowmax, argmax, st);
  else if (!exact && dtype == MXS_F16)
    s = launch_varlen_tc<mxs::TcKind::F16>(Q, n_q, l_q, tokens, cu_seqlens, n_docs, n_tokens, dim, rowmax, argmax, st);
  if (s == MXS_OK) return launch_rowsum(rowmax, n_q * n_docs, l_q, scores, st);
  if (s != MXS_UNSUPPORTED) return s;
  if (dtype == MXS_F32)
    s = launch_fwd_exact<float>(Q, n_q, l_q, tokens, n_docs, 0, dim, nullptr, cu, rowmax, argmax, st);
  else if (dtype == MXS_BF16)
    s = launch_fwd_exact<__nv_bfloat16>(Q, n_q, l_q, tokens, n_docs, 0, dim, nullptr, cu, rowmax, argmax, st);
  else if (dtype == MXS_F16)
    s = launch_fwd_exact<__half>(Q, n_q, l_q, tokens, n_docs, 0, dim, nullptr, cu, rowmax, argmax, st);
  else
    return fail(MXS_UNSUPPORTED, "mxs_fused_score_varlen: dtype %d", dtype);
  if (s != MXS_OK) return s;
  return launch_rowsum(rowmax, n_q * n_docs, l_q, scores, st);
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
  if (dim < 1 || dim > mxs::kChDimMax) return fail(MXS_UNSUPPORTED, "mxs_chamfer_nn: dim %lld outside [1, 16]", (long long)dim);
  if (m >= (1LL << 31)) return fail(MXS_UNSUPPORTED, "mxs_chamfer_nn: more than 2^31 points");
  const long long blocks = (n + mxs::kChThreads - 1) / mxs::kChThreads;
  cudaStream_t st = (cudaStream_t)stream;
  if (dim == 3)
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

// ------------------------------------------------------------------ MXS1 files (host side)
static int mxs1_truncated(int64_t expected, int64_t actual) {
  return fail(MXS_TRUNCATED_PAYLOAD, "payload truncated: expected %lld bytes, file holds %lld", (long long)expected,
              (long long)actual);
}

int mxs_mxs1_open(const char* path, void** handle) {
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
  if (lc == mxs_io::kDense || lc == mxs_io::kQuantized) {
    if (!u64(f->n_docs) || !u64(f->length) || !u64(f->dim)) return bail(MXS_TRUNCATED_PAYLOAD);
  } else {
    if (!u64(f->n_docs) || !u64(f->dim)) return bail(MXS_TRUNCATED_PAYLOAD);
    f->cu.resize((size_t)f->n_docs + 1);
    const int64_t need = 8 * (f->n_docs + 1);
    const int64_t got = mxs_io::pread_all(fd, f->cu.data(), need, off);
    if (got != need) return bail(mxs1_truncated(need, got < 0 ? 0 : got));
    off += need;
  }
  if (lc == mxs_io::kQuantized && ec != mxs_io::kI8)
    return bail(fail(MXS_BAD_MAGIC, "quantized layout requires the i8 element tag"));
  if (lc != mxs_io::kQuantized && ec == mxs_io::kI8)
    return bail(fail(MXS_BAD_MAGIC, "int8 elements require the quantized layout (scales are part of the data)"));
  f->payload_offset = off;
  *handle = f;
  return MXS_OK;
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

int mxs_mxs1_read_block(void* handle, int64_t first, int64_t count, void* dst, size_t dst_bytes) {
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
