// L2 read roofline for the backward gathers (K7 / K8): how many bytes per second the B200's L2
// serves when the working set is L2-resident.
//   stream : every warp reads contiguous 16 B vectors of a 16 MB buffer, many passes
//   gather : every warp reads random 256 B rows (16 lanes x 16 B, 2 rows per warp step, 8 rows
//            in flight) of a 16 MB table -- the access pattern of grad_docs_rg / grad_query_rg
//            at C3 (bf16 rows of d = 128)
// Build + run on the box: nvcc -O3 -gencode arch=compute_100a,code=sm_100a l2_bw.cu -o /tmp/l2_bw && /tmp/l2_bw
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));          \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__global__ void stream_kernel(const uint4* __restrict__ buf, long long n_vec, int passes, float* sink) {
  float acc = 0.f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int p = 0; p < passes; ++p)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_vec; i += stride) {
      const uint4 v = __ldcg(buf + i);
      acc += __uint_as_float(v.x ^ v.y ^ v.z ^ v.w);
    }
  if (acc == 1.2345f) *sink = acc;
}

__global__ void gather_kernel(const uint4* __restrict__ table, int n_rows, const int* __restrict__ idx, long long n_idx,
                              float* sink) {
  // 16 lanes per 256 B row, 2 rows per warp step, 4 steps in flight
  const int lane = threadIdx.x & 31, h = lane >> 4, lp = lane & 15;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long n_warps = ((long long)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (long long base = warp * 8; base < n_idx; base += n_warps * 8) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long k = base + 2 * u + h;
      const int r = k < n_idx ? __ldg(idx + k) : 0;
      v[u] = __ldcg(table + (long long)r * 16 + lp);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += __uint_as_float(v[u].x ^ v[u].y ^ v[u].z ^ v[u].w);
  }
  if (acc == 1.2345f) *sink = acc;
}

int main() {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const long long bytes = 16ll << 20;
  uint4* buf;
  float* sink;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(buf, 1, bytes));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int bpsm : {4, 8, 16}) {
    const int passes = 64;
    stream_kernel<<<nsm * bpsm, 256>>>(buf, bytes / 16, 2, sink);
    cudaEventRecord(e0);
    stream_kernel<<<nsm * bpsm, 256>>>(buf, bytes / 16, passes, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("stream  blocks/SM=%2d : %.1f GB/s\n", bpsm, bytes * (double)passes / (ms * 1e-3) / 1e9);
  }
  // gather: 16 MB table of 256 B rows (65,536 rows), 4M random row ids (the C3 source count)
  const int n_rows = (int)(bytes / 256);
  const long long n_idx = 64ll * 64 * 1024;
  std::vector<int> h(n_idx);
  uint32_t s = 12345;
  for (auto& x : h) {
    s = s * 1664525u + 1013904223u;
    x = (int)(s % (uint32_t)n_rows);
  }
  int* idx;
  CK(cudaMalloc(&idx, n_idx * 4));
  CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
  for (int bpsm : {4, 8}) {
    gather_kernel<<<nsm * bpsm, 256>>>(buf, n_rows, idx, n_idx, sink);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) gather_kernel<<<nsm * bpsm, 256>>>(buf, n_rows, idx, n_idx, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double per = ms / 10;
    printf("gather  blocks/SM=%2d : %.1f us per 4M x 256 B rows = %.1f GB/s (rows) + index %.1f GB/s\n", bpsm,
           per * 1e3, n_idx * 256.0 / (per * 1e-3) / 1e9, n_idx * 4.0 / (per * 1e-3) / 1e9);
  }
  return 0;
}
