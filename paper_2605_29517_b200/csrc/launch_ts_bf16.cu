// fwd_ts_kernel instantiations for BF16 operands.
#include "launch_ts.cuh"

namespace mxs_host {
template int launch_fwd_ts<mxs::TcKind::BF16>(const void*, int64_t, int64_t, const void*, int64_t, int64_t, int64_t,
                                               const int32_t*, const float*, const float*, float*, int32_t*, double*,
                                               int*, cudaStream_t);
}  // namespace mxs_host
