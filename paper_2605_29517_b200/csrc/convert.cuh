// Element conversions shared by the SIMT kernels (exact widening of bf16 / fp16 to fp32).
#pragma once
#include "ptx.cuh"
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace mxs {

template <typename T>
MXS_DEV float to_f32(T x);
template <>
MXS_DEV float to_f32<float>(float x) { return x; }
template <>
MXS_DEV float to_f32<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <>
MXS_DEV float to_f32<__half>(__half x) { return __half2float(x); }

}  // namespace mxs
