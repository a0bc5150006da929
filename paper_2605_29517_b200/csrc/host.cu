// Host plumbing of libmaxsim_b200.so (see host.h).
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "host.h"

namespace mxs_host {

namespace {
thread_local std::string g_err;
}

int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return status;
}

const char* last_error() { return g_err.c_str(); }

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MXS_CUDA_ERROR, "%s: %s", what, cudaGetErrorString(e));
  return MXS_OK;
}

int current_device() {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  return dev;
}

int sm_count() {
  const int dev = current_device();
  if (dev < 0) return -1;
  static int cache[64] = {0};
  if (dev < 64 && cache[dev]) return cache[dev];
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  if (dev < 64) cache[dev] = n;
  return n;
}

// Stream-ordered scratch (cudaMallocAsync) comes from the device's default memory pool, whose
// default release threshold (0) hands memory back to the driver at every synchronisation -- the
// next allocation then maps fresh pages (~ms).  Keep the pool's memory cached instead (once per
// device); the scratch it holds is bounded by the largest request (row maxima, CSR temporaries).
int scratch_alloc(void** ptr, size_t bytes, cudaStream_t st) {
  const int dev = current_device();
  static std::mutex mu;
  static bool done[64] = {false};
  if (dev >= 0 && dev < 64) {
    std::lock_guard<std::mutex> g(mu);
    if (!done[dev]) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      cudaGetLastError();
      done[dev] = true;
    }
  }
  if (cudaMallocAsync(ptr, bytes, st) != cudaSuccess) {
    cudaGetLastError();
    *ptr = nullptr;
    return fail(MXS_CUDA_ERROR, "scratch allocation of %zu bytes failed", bytes);
  }
  return MXS_OK;
}

int ensure_smem(const void* kern, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  const int dev = current_device();
  if (dev < 0) return fail(MXS_CUDA_ERROR, "no CUDA device");
  const auto key = std::make_pair(kern, dev);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = done.find(key);
    if (it != done.end() && it->second >= bytes) return MXS_OK;
  }
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(MXS_CUDA_ERROR, "cudaFuncSetAttribute(smem=%zu) failed", bytes);
  }
  std::lock_guard<std::mutex> g(mu);
  size_t& v = done[key];
  v = std::max(v, bytes);
  return MXS_OK;
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

bool env_is(const char* name, const char* value) {
  const char* v = getenv(name);
  return v && strcmp(v, value) == 0;
}

namespace {
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
}  // namespace

int make_tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem_bytes, int64_t cols, int64_t rows,
                 int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(MXS_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(cols * elem_bytes)};
  cuuint32_t box[2] = {(cuuint32_t)(128 / elem_bytes), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MXS_CUDA_ERROR, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return MXS_OK;
}

// Clusters of 4 do not tile every GPC, so nsm / 4 may over-subscribe and leave a tail wave; the
// occupancy query gives the resident count (falls back to nsm / cl if it fails).
long long resident_clusters(const void* kern, int cl, int threads, size_t smem, int nsm) {
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
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    return nsm / cl;
  }
  return std::min<long long>(n, nsm / cl);
}

int launch_cluster(const void* kern, long long ctas, int cl, int threads, size_t smem, cudaStream_t st, void** args,
                   const char* what) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ctas);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelExC(&cfg, kern, args);
  if (e != cudaSuccess) return fail(MXS_CUDA_ERROR, "%s launch: %s", what, cudaGetErrorString(e));
  return check_launch(what);
}

}  // namespace mxs_host
