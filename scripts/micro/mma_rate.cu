// Microbenchmark: raw tcgen05.mma issue rate on one B200 (no TMA, no epilogue), to separate the
// MMA-shape ceiling from the forward kernel's pipeline.  One CTA per SM; one elected thread issues
// `iters` MMA chains of 8 K-steps (K = 16 bf16 each) into alternating accumulators.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_29517_b200/csrc scripts/micro/mma_rate.cu -o /tmp/mma_rate -lcuda
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
#include "fwd_tc.cuh"

using namespace mxs;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase;
  if (warp == 0) {
    constexpr uint32_t idesc = make_idesc(1, 1, 128, N);
    const uint64_t bdesc = sw128_kmajor_desc(smem_u32(sm));
    const uint64_t adesc = sw128_kmajor_desc(smem_u32(sm + 65536));
    const unsigned long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
        const uint32_t d = tb + (TS ? 256u : 0u) + (uint32_t)((it & 1) * (N == 256 ? 0 : N));
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t koff = (uint64_t)(((k >> 2) * 16384 + (k & 3) * 32) >> 4);
          if (TS)
            mma_f16_ts(d, tb + k * 8, bdesc + koff, idesc, k > 0 ? 1u : 0u);
          else
            mma_f16_ss(d, adesc + koff, bdesc + koff, idesc, k > 0 ? 1u : 0u);
        }
        if ((it & 15) == 15) mma_commit(&bar);
      }
      __syncwarp();
      if ((it & 15) == 15) {
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tb, 512);
  }
}

template <int N, bool TS>
void run(const char* name) {
  const int iters = 20000, blocks = 148;
  unsigned long long* d;
  cudaMalloc(&d, blocks * 8);
  auto k = mma_rate<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  k<<<blocks, 128, 140000>>>(100, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<blocks, 128, 140000>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d, blocks * 8, cudaMemcpyDeviceToHost);
  const double flops = 2.0 * 128 * N * 128 * (double)iters * blocks;
  const double per_clk = 2.0 * 128 * N * 128 * (double)iters / (double)h[0];
  printf("%-22s %8.3f ms  %7.1f TFLOP/s  %6.0f flop/clk/SM (8192 = nominal)  err=%s\n", name, ms,
         flops / ms / 1e9, per_clk, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<128, true>("TS  M128 N128 K16x8");
  run<128, false>("SS  M128 N128 K16x8");
  run<256, false>("SS  M128 N256 K16x8");
  run<64, true>("TS  M128 N64  K16x8");
  run<80, true>("TS  M128 N80  K16x8");
  run<96, true>("TS  M128 N96  K16x8");
  run<112, true>("TS  M128 N112 K16x8");
  return 0;
}
