// Host-side plumbing shared by the launcher translation units of libmaxsim_b200.so:
// error reporting (thread-local message behind mxs_last_error), device queries, TMA descriptor
// encoding, per-device shared-memory opt-in, and the launcher prototypes.  No device code here.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/maxsim_b200.h"
#include "kinds.h"

namespace mxs_host {

int fail(int status, const char* fmt, ...);
const char* last_error();
int check_launch(const char* what);
int current_device();
int sm_count();
// cudaFuncAttributeMaxDynamicSharedMemorySize is per device/context: set it for the current
// device the first time a kernel needs `bytes` there (cached per (kernel, device)).
int ensure_smem(const void* kern, size_t bytes);
// cudaMallocAsync from the device's default pool, kept cached across synchronisations
int scratch_alloc(void** ptr, size_t bytes, cudaStream_t st);
int env_int(const char* name, int dflt);
bool env_is(const char* name, const char* value);

// 2-D row-major [rows, cols] tensor, box = 128 bytes x box_rows rows, SWIZZLE_128B.
int make_tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem_bytes, int64_t cols,
                 int64_t rows, int box_rows = 128);

// Persistent cluster grids: as many clusters of `cl` CTAs as the device keeps resident at once.
long long resident_clusters(const void* kern, int cl, int threads, size_t smem, int nsm);
int launch_cluster(const void* kern, long long ctas, int cl, int threads, size_t smem, cudaStream_t st, void** args,
                   const char* what);

// ---------------------------------------------------------------- launchers (one TU each)
int launch_rowsum(const float* rowmax, int64_t n_pairs, int64_t l_q, double* scores, cudaStream_t st);

// fwd_ts (launch_ts_*.cu).  scores != nullptr asks for the fused S4 sum; the launcher returns
// *fused = 1 when the kernel wrote the scores itself (else the caller runs the rowsum pass over rowmax).
template <mxs::TcKind KIND>
int launch_fwd_ts(const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad, int64_t dim,
                  const int32_t* valid_lens, const float* q_scale, const float* d_scale, float* rowmax,
                  int32_t* argmax, double* scores, int* fused, cudaStream_t st);
// fwd_tc SS fallback (launch_ss.cu)
template <mxs::TcKind KIND>
int launch_fwd_tc(const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad, int64_t dim,
                  const int32_t* valid_lens, const float* q_scale, const float* d_scale, float* rowmax,
                  int32_t* argmax, cudaStream_t st);
// three-slot rerank kernel (launch_r3.cu)
template <mxs::TcKind KIND>
int launch_fwd_r3(const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad, int64_t dim,
                  const int32_t* valid_lens, const float* q_scale, const float* d_scale, float* rowmax,
                  double* scores, int* fused, cudaStream_t st);
// CTA-pair forward (launch_pair.cu)
template <mxs::TcKind KIND>
int launch_fwd_pair(const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad,
                    int64_t dim, const int32_t* valid_lens, float* rowmax, int32_t* argmax, double* scores, int* fused,
                    cudaStream_t st);
// varlen rows kernel (launch_varlen.cu)
template <mxs::TcKind KIND>
int launch_varlen_tc(const void* Q, int64_t n_q, int64_t l_q, const void* tokens, const int64_t* cu, int64_t n_docs,
                     int64_t n_tokens, int64_t dim, float* rowmax, int32_t* argmax, double* scores, int* fused,
                     cudaStream_t st);
// exact SIMT kernels (launch_exact.cu); dtype = MXS_F32 / MXS_F16 / MXS_BF16
int launch_fwd_exact(int dtype, const void* Q, int64_t n_q, int64_t l_q, const void* D, int64_t n_docs, int64_t l_pad,
                     int64_t dim, const int32_t* valid_lens, const int64_t* cu, float* rowmax, int32_t* argmax,
                     cudaStream_t st);
int launch_fwd_exact_i8(const int8_t* Q, const float* qs, int64_t n_q, int64_t l_q, const int8_t* D, const float* ds,
                        int64_t n_docs, int64_t l_pad, int64_t dim, const int32_t* valid_lens, float* rowmax,
                        int32_t* argmax, cudaStream_t st);

// Device-side validation of valid_lens / cu_seqlens (launch_misc.cu): writes an error code to
// `status` (0 ok, 1 = entry < 1, 2 = entry > l_pad / non-increasing / wrong end) and the first bad index.
int launch_check_lens(const int32_t* valid_lens, int64_t n, int64_t l_pad, int32_t* status, cudaStream_t st);
int launch_check_cu(const int64_t* cu, int64_t n_docs, int64_t n_tokens, int32_t* status, cudaStream_t st);

}  // namespace mxs_host
