// Launcher of the SS-form fwd_tc_kernel (Q and D both in shared memory): the fallback when Q does
// not fit the TMEM budget of fwd_ts (MXS_FWD_IMPL=ss forces it).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "fwd_tc.cuh"
#include "host.h"

namespace mxs_host {

template <mxs::TcKind KIND>
int launch_fwd_tc(const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad, int64_t dim,
                  const int32_t* valid_lens, const float* q_scale, const float* d_scale, float* rowmax,
                  int32_t* argmax, cudaStream_t st) {
  if (!rowmax) return fail(MXS_INVALID_ARGUMENT, "fwd_tc_kernel needs a row-maxima buffer");
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
  p.debug = env_int("MXS_DEBUG", 0);
  p.mma_spin = env_int("MXS_MMA_SPIN", 0);
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
  if ((s = ensure_smem((const void*)kern, smem)) != MXS_OK) return s;
  const int nsm = sm_count();
  if (nsm <= 0) return fail(MXS_CUDA_ERROR, "no CUDA device");
  long long grid = p.n_units < nsm ? p.n_units : nsm;
  if (grid <= 0) return MXS_OK;
  kern<<<(unsigned)grid, mxs::kFwdThreads, smem, st>>>(tq, td, p);
  return check_launch("fwd_tc_kernel");
}

#define MXS_SS_INST(K)                                                                                         \
  template int launch_fwd_tc<mxs::TcKind::K>(const void*, int64_t, int64_t, const void*, int64_t, int64_t, int64_t, \
                                             const int32_t*, const float*, const float*, float*, int32_t*, cudaStream_t);
MXS_SS_INST(BF16)
MXS_SS_INST(F16)
MXS_SS_INST(I8)
#undef MXS_SS_INST

}  // namespace mxs_host
