// Launcher of fwd_ts_kernel (instantiated once per operand kind by launch_ts_{bf16,f16,i8}.cu so
// the three heavy instantiations compile in parallel).
#pragma once
#include <algorithm>

#include "fwd_ts.cuh"
#include "host.h"

namespace mxs_host {

// v3 path: Q in TMEM, cluster multicast of document tiles, stash-based argmax.
// Returns MXS_UNSUPPORTED (without launching) when the shape needs the SS kernel.
template <mxs::TcKind KIND>
int launch_fwd_ts(const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad, int64_t dim,
                  const int32_t* valid_lens, const float* q_scale, const float* d_scale, float* rowmax,
                  int32_t* argmax, double* scores, int* fused, cudaStream_t st) {
  *fused = 0;
  const int eb = (KIND == mxs::TcKind::I8) ? 1 : 2;
  if ((dim * eb) % 16 != 0) return MXS_UNSUPPORTED;
  const int ka = (int)((dim * eb + 127) / 128);
  if (ka > 4) return MXS_UNSUPPORTED;
  const int qb_max = std::min(mxs::kMaxQb, 256 / (ka * 32));
  const int nmb = (int)((l_q + 127) / 128);
  const int qb = std::min(qb_max, nmb);
  const int n_groups = (nmb + qb - 1) / qb;
  int cl = (n_groups == 2 || n_groups == 4) ? n_groups : 1;
  if (env_int("MXS_FWD_CL", 0) == 1) cl = 1;  // profiling knob: force the cluster size (1 = no multicast)
  const size_t max_smem = 232448 - sizeof(mxs::TsSmemHeader);  // static header comes out of the same 227 KB
  const bool scale_ring = (KIND == mxs::TcKind::I8) && (l_pad % 4 == 0);
  const bool bias = (KIND == mxs::TcKind::I8) && ka <= 2;  // fwd_ts_kernel's kBias
  // fused S4 sum when one cluster holds a whole query (every Q row group of it) and the profiling
  // knob MXS_DEBUG=3 (no drain) is off
  const int dbg = env_int("MXS_DEBUG", 0);
  const bool fuse = scores != nullptr && cl == n_groups && !(KIND != mxs::TcKind::I8 && dbg == 3) &&
                    env_int("MXS_FWD_FUSE", 1) != 0;
  if (!fuse && !rowmax) return MXS_UNSUPPORTED;  // the caller supplies row maxima for the rowsum pass
  const int sum_rows = fuse ? nmb * 128 : 0;
  const size_t fixed = mxs::fwd_ts_smem_bytes(0, qb, 0, scale_ring, bias, argmax != nullptr, sum_rows);
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
  p.scores = fuse ? scores : nullptr;
  p.sum_rows = sum_rows;
  p.debug = dbg;
  p.mma_spin = env_int("MXS_MMA_SPIN", 0);
  CUtensorMap td;
  const CUtensorMapDataType dt = (KIND == mxs::TcKind::I8)     ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : (KIND == mxs::TcKind::BF16) ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                               : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  int s;
  if ((s = make_tmap_2d(&td, D, dt, eb, dim, n_docs * l_pad, 128 / cl)) != MXS_OK) return s;
  const size_t smem = mxs::fwd_ts_smem_bytes(ka, qb, stages, scale_ring, bias, argmax != nullptr, sum_rows);
  using KernT = void (*)(const CUtensorMap, const mxs::FwdTcParams);
  KernT kern = nullptr;
#define MXS_TS_CASE(KA_, CL_) \
  if (ka == KA_ && cl == CL_) kern = mxs::fwd_ts_kernel<KIND, KA_, CL_>;
  MXS_TS_CASE(1, 1) MXS_TS_CASE(1, 2) MXS_TS_CASE(1, 4) MXS_TS_CASE(2, 1) MXS_TS_CASE(2, 2) MXS_TS_CASE(2, 4)
  MXS_TS_CASE(3, 1) MXS_TS_CASE(3, 2) MXS_TS_CASE(3, 4) MXS_TS_CASE(4, 1) MXS_TS_CASE(4, 2) MXS_TS_CASE(4, 4)
#undef MXS_TS_CASE
  if (!kern) return MXS_UNSUPPORTED;
  if ((s = ensure_smem((const void*)kern, smem)) != MXS_OK) return s;
  const int nsm = sm_count();
  if (nsm <= 0) return fail(MXS_CUDA_ERROR, "no CUDA device");
  long long workers = resident_clusters((const void*)kern, cl, mxs::kTsThreads, smem, nsm);
  if (p.n_units < workers) workers = p.n_units;
  if (workers <= 0) return MXS_OK;
  void* args[] = {(void*)&td, (void*)&p};
  if ((s = launch_cluster((const void*)kern, workers * cl, cl, mxs::kTsThreads, smem, st, args, "fwd_ts_kernel")) !=
      MXS_OK)
    return s;
  *fused = fuse ? 1 : 0;
  return MXS_OK;
}

}  // namespace mxs_host
