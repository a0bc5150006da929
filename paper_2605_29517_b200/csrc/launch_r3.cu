// Launcher of the three-slot rerank kernel fwd_i8r_kernel (INT8, and bf16 / fp16 opt-in).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "fwd_i8r.cuh"
#include "host.h"

namespace mxs_host {

// Rerank path (argmax not requested): three accumulator slots / three epilogue warp sets
// (fwd_i8r.cuh).  INT8 with d <= 128 (4 resident Q blocks), bf16 / fp16 with d <= 128 (2 resident
// Q blocks, 4-CTA clusters at L_q = 1024).  Returns MXS_UNSUPPORTED (without launching) otherwise.
template <mxs::TcKind KIND>
int launch_fwd_r3(const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad, int64_t dim,
                  const int32_t* valid_lens, const float* q_scale, const float* d_scale, float* rowmax,
                  double* scores, int* fused, cudaStream_t st) {
  *fused = 0;
  constexpr bool kI8 = KIND == mxs::TcKind::I8;
  const int eb = kI8 ? 1 : 2;
  if (dim % 16 != 0 || dim > 128 || (kI8 && l_pad % 4 != 0)) return MXS_UNSUPPORTED;
  if (env_is(kI8 ? "MXS_I8_IMPL" : "MXS_RERANK_IMPL", "ts")) return MXS_UNSUPPORTED;
  constexpr int ka = kI8 ? 1 : 2;
  const int nmb = (int)((l_q + 127) / 128);
  const int qb = std::min(kI8 ? 4 : 2, nmb);
  const int n_groups = (nmb + qb - 1) / qb;
  const int cl = (n_groups == 2 || n_groups == 4) ? n_groups : 1;
  const size_t max_smem = 232448 - sizeof(mxs::R8SmemHeader);
  const int dbg = env_int("MXS_DEBUG", 0);  // 2: slots released unread; 3 (bf16/fp16): no drain wait
  const bool fuse = scores != nullptr && cl == n_groups && !(!kI8 && dbg == 3) && env_int("MXS_FWD_FUSE", 1) != 0;
  if (!fuse && !rowmax) return MXS_UNSUPPORTED;
  const int sum_rows = fuse ? nmb * 128 : 0;
  const size_t fixed = mxs::fwd_i8r_smem_bytes(ka, 0, kI8, sum_rows);
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
  p.scores = fuse ? scores : nullptr;
  p.sum_rows = sum_rows;
  p.debug = (kI8 && dbg == 3) ? 0 : dbg;
  const CUtensorMapDataType dt = kI8                         ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : KIND == mxs::TcKind::BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap td;
  int s;
  if ((s = make_tmap_2d(&td, D, dt, eb, dim, n_docs * l_pad, 128 / cl)) != MXS_OK) return s;
  const size_t smem = mxs::fwd_i8r_smem_bytes(ka, stages, kI8, sum_rows);
  using KernT = void (*)(const CUtensorMap, const mxs::FwdTcParams);
  KernT kern = cl == 4   ? mxs::fwd_i8r_kernel<KIND, ka, 4>
               : cl == 2 ? mxs::fwd_i8r_kernel<KIND, ka, 2>
                         : mxs::fwd_i8r_kernel<KIND, ka, 1>;
  if ((s = ensure_smem((const void*)kern, smem)) != MXS_OK) return s;
  const int nsm = sm_count();
  if (nsm <= 0) return fail(MXS_CUDA_ERROR, "no CUDA device");
  long long workers = resident_clusters((const void*)kern, cl, mxs::kR8Threads, smem, nsm);
  if (p.n_units < workers) workers = p.n_units;
  if (workers <= 0) return MXS_OK;
  void* args[] = {(void*)&td, (void*)&p};
  if ((s = launch_cluster((const void*)kern, workers * cl, cl, mxs::kR8Threads, smem, st, args, "fwd_i8r_kernel")) !=
      MXS_OK)
    return s;
  *fused = fuse ? 1 : 0;
  return MXS_OK;
}

#define MXS_R3_INST(K)                                                                                         \
  template int launch_fwd_r3<mxs::TcKind::K>(const void*, int64_t, int64_t, const void*, int64_t, int64_t, int64_t, \
                                             const int32_t*, const float*, const float*, float*, double*, int*,     \
                                             cudaStream_t);
MXS_R3_INST(BF16)
MXS_R3_INST(F16)
MXS_R3_INST(I8)
#undef MXS_R3_INST

}  // namespace mxs_host
