// Launcher of the CTA-pair forward fwd_pair_kernel (fwd_pair.cuh): bf16 / fp16, d <= 128,
// 256 < L_q <= 1024 (two Q blocks per CTA, one or two pairs per cluster).
#include <algorithm>
#include <cstdio>

#include "fwd_pair.cuh"
#include "host.h"

namespace mxs_host {

template <mxs::TcKind KIND>
int launch_fwd_pair(const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad,
                    int64_t dim, const int32_t* valid_lens, float* rowmax, int32_t* argmax, double* scores, int* fused,
                    cudaStream_t st) {
  *fused = 0;
  if (dim % 8 != 0 || dim > 128) return MXS_UNSUPPORTED;
  const int ka = dim > 64 ? 2 : 1;
  const int nmb = (int)((l_q + 127) / 128);
  if (nmb < 3 || nmb > 8) return MXS_UNSUPPORTED;
  // one pair per cluster: two TMEM Q blocks per CTA up to L_q = 512, plus two SS blocks beyond;
  // MXS_PAIR_CL=4 selects two pairs of TMEM-only CTAs for L_q > 512 (4-CTA clusters: 132 SMs)
  const int cl = (nmb > 4 && env_int("MXS_PAIR_CL", 2) == 4) ? 4 : 2;
  const int qb = nmb <= 4 || cl == 4 ? 2 : 4;
  // QB = 4 rerank: all four Q blocks in shared memory (SS) leaves TMEM to FOUR accumulator slots
  // (MXS_PAIR_SS=1); the argmax stash does not fit next to them
  const int nts = (qb == 4 && argmax == nullptr && env_int("MXS_PAIR_SS", 0) == 1) ? 0 : 2;
  const int dbg = env_int("MXS_DEBUG", 0);
  const bool fuse = scores != nullptr && dbg != 3 && env_int("MXS_FWD_FUSE", 1) != 0;
  if (!fuse && !rowmax) return MXS_UNSUPPORTED;
  const int sum_rows = fuse ? cl * qb * 128 : 0;
  const size_t max_smem = 232448 - sizeof(mxs::PrSmemHeader);
  const size_t fixed = mxs::fwd_pair_smem_bytes(ka, qb, nts, 0, argmax != nullptr, sum_rows);
  int stages = (int)((max_smem - fixed) / ((size_t)ka * mxs::kPrHalfAtom));
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
  p.n_groups = cl;
  p.stages = stages;
  p.n_units = (long long)n_q * n_docs;
  p.valid_lens = valid_lens;
  p.rowmax = rowmax;
  p.argmax = argmax;
  p.q_ptr = Q;
  p.scores = fuse ? scores : nullptr;
  p.sum_rows = sum_rows;
  p.debug = dbg;
  p.mma_spin = env_int("MXS_MMA_SPIN", 0);
  CUtensorMap td;
  const CUtensorMapDataType dt =
      (KIND == mxs::TcKind::BF16) ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  int s;
  CUtensorMap tq;
  if ((s = make_tmap_2d(&td, D, dt, 2, dim, n_docs * l_pad, 64)) != MXS_OK) return s;
  if ((s = make_tmap_2d(&tq, Q, dt, 2, dim, n_q * l_q, 128)) != MXS_OK) return s;
  const size_t smem = mxs::fwd_pair_smem_bytes(ka, qb, nts, stages, argmax != nullptr, sum_rows);
  using KernT = void (*)(const CUtensorMap, const CUtensorMap, const mxs::FwdTcParams);
  KernT kern = nullptr;
  if (qb == 4 && nts == 0)
    kern = ka == 1 ? mxs::fwd_pair_kernel<KIND, 1, 2, 4, 0> : mxs::fwd_pair_kernel<KIND, 2, 2, 4, 0>;
  else if (qb == 4)
    kern = ka == 1 ? mxs::fwd_pair_kernel<KIND, 1, 2, 4, 2> : mxs::fwd_pair_kernel<KIND, 2, 2, 4, 2>;
  else if (cl == 2)
    kern = ka == 1 ? mxs::fwd_pair_kernel<KIND, 1, 2, 2, 2> : mxs::fwd_pair_kernel<KIND, 2, 2, 2, 2>;
  else
    kern = ka == 1 ? mxs::fwd_pair_kernel<KIND, 1, 4, 2, 2> : mxs::fwd_pair_kernel<KIND, 2, 4, 2, 2>;
  if ((s = ensure_smem((const void*)kern, smem)) != MXS_OK) return s;
  const int nsm = sm_count();
  if (nsm <= 0) return fail(MXS_CUDA_ERROR, "no CUDA device");
  long long workers = resident_clusters((const void*)kern, cl, mxs::kTsThreads, smem, nsm);
  if (env_int("MXS_PRINT_GRID", 0)) fprintf(stderr, "fwd_pair: cl=%d qb=%d nts=%d clusters=%lld stages=%d\n", cl, qb, nts, workers, stages);
  if (p.n_units < workers) workers = p.n_units;
  if (workers <= 0) return MXS_OK;
  void* args[] = {(void*)&td, (void*)&tq, (void*)&p};
  if ((s = launch_cluster((const void*)kern, workers * cl, cl, mxs::kTsThreads, smem, st, args, "fwd_pair_kernel")) !=
      MXS_OK)
    return s;
  *fused = fuse ? 1 : 0;
  return MXS_OK;
}

template int launch_fwd_pair<mxs::TcKind::BF16>(const void*, int64_t, int64_t, const void*, int64_t, int64_t, int64_t,
                                                const int32_t*, float*, int32_t*, double*, int*, cudaStream_t);
template int launch_fwd_pair<mxs::TcKind::F16>(const void*, int64_t, int64_t, const void*, int64_t, int64_t, int64_t,
                                               const int32_t*, float*, int32_t*, double*, int*, cudaStream_t);

}  // namespace mxs_host
