// Launcher of the padding-free varlen_rows_kernel (cu_seqlens layout).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "varlen_rows.cuh"
#include "host.h"

namespace mxs_host {

template <mxs::TcKind KIND>
int launch_varlen_tc(const void* Q, int64_t n_q, int64_t l_q, const void* tokens, const int64_t* cu, int64_t n_docs,
                     int64_t n_tokens, int64_t dim, float* rowmax, int32_t* argmax, double* scores, int* fused,
                     cudaStream_t st) {
  *fused = 0;
  static_assert(KIND != mxs::TcKind::I8, "varlen is a bf16 / f16 path");
  const int eb = 2;
  const long long rows = n_q * l_q;
  // fused S4 score when a query's rows fit one warp's aligned lane segment (l_q divides 32)
  // (one launch of <= 32 rows: the fused kernel is compiled for the 4-copy layout only)
  const bool fuse = scores != nullptr && l_q <= 32 && (32 % l_q) == 0 && rows <= 32 && env_int("MXS_VARLEN_FUSE", 1) != 0;
  if (!fuse && !rowmax) return MXS_UNSUPPORTED;
  if ((dim * eb) % 16 != 0 || rows >= (1LL << 31)) return MXS_UNSUPPORTED;
  const int ka = (int)((dim * eb + 127) / 128);
  if (ka > 4) return MXS_UNSUPPORTED;
  const size_t max_smem = 232448 - sizeof(mxs::VrSmemHeader) - (fuse ? sizeof(mxs::VrRing) : 0);
  const size_t fixed = mxs::varlen_rows_smem_bytes(ka, 0);
  int stages = (int)((max_smem - fixed) / ((size_t)ka * mxs::kAtomBytes));
  if (stages > 8) stages = 8;
  if (stages < 2) return MXS_UNSUPPORTED;
  void (*kern)(const CUtensorMap, const CUtensorMap, const mxs::VarlenRowsParams) = nullptr;
  switch (ka) {
    case 1: kern = fuse ? mxs::varlen_rows_kernel<KIND, 1, true> : mxs::varlen_rows_kernel<KIND, 1, false>; break;
    case 2: kern = fuse ? mxs::varlen_rows_kernel<KIND, 2, true> : mxs::varlen_rows_kernel<KIND, 2, false>; break;
    case 3: kern = fuse ? mxs::varlen_rows_kernel<KIND, 3, true> : mxs::varlen_rows_kernel<KIND, 3, false>; break;
    case 4: kern = fuse ? mxs::varlen_rows_kernel<KIND, 4, true> : mxs::varlen_rows_kernel<KIND, 4, false>; break;
    default: return MXS_UNSUPPORTED;
  }
  const size_t smem = mxs::varlen_rows_smem_bytes(ka, stages);
  int s;
  if ((s = ensure_smem((const void*)kern, smem)) != MXS_OK) return s;
  const int nsm = sm_count();
  if (nsm <= 0) return fail(MXS_CUDA_ERROR, "no CUDA device");
  const long long grid = n_docs < nsm ? n_docs : nsm;
  const CUtensorMapDataType dt =
      (KIND == mxs::TcKind::BF16) ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tt;
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
    p.scores = fuse ? scores : nullptr;
    CUtensorMap tq;
    const void* q0 = static_cast<const uint8_t*>(Q) + row0 * dim * eb;
    // one box per row copy; rows >= n_cols read as 0
    if ((s = make_tmap_2d(&tq, q0, dt, eb, dim, n_cols, 128 / p.copies)) != MXS_OK) return s;
    kern<<<(unsigned)grid, mxs::kVrThreads, smem, st>>>(tt, tq, p);
    if ((s = check_launch("varlen_rows_kernel")) != MXS_OK) return s;
  }
  *fused = fuse ? 1 : 0;
  return MXS_OK;
}

template int launch_varlen_tc<mxs::TcKind::BF16>(const void*, int64_t, int64_t, const void*, const int64_t*, int64_t,
                                                 int64_t, int64_t, float*, int32_t*, double*, int*, cudaStream_t);
template int launch_varlen_tc<mxs::TcKind::F16>(const void*, int64_t, int64_t, const void*, const int64_t*, int64_t,
                                                int64_t, int64_t, float*, int32_t*, double*, int*, cudaStream_t);

}  // namespace mxs_host
