// Inverse-grid CSR of the saved argmax (K6), on device, bit-identical to
// maxsim/backward.py:81-109 (bincount -> cumsum -> STABLE argsort of the flat destinations).
//
// Source s = (q * B + b) * L_q + i picks destination row dest_off[b] + argmax[s].  Every source
// of document b lands in b's rows, so b's bucket block starts at row_ptr = b * N_q * L_q and the
// problem splits per document.  Stability (ascending s inside each bucket) is ascending (q, i)
// within the document, obtained in three passes without global atomics:
//   1. csr_count_kernel   block (q, b): smem histogram of argmax[q, b, :] -> cnt[q][dest row]
//   2. csr_scan_kernel    block b: totals over q, exclusive scan over b's rows -> row_ptr;
//                         cnt[q][r] becomes the first slot of segment (q, b) inside bucket r
//   3. csr_place_kernel   block (q, b): stable in-segment ranks (warp match + warp-ordered
//                         cursor updates) -> col_idx[slot] = s
// Indices are int32 (n_src and n_dest < 2^31 are checked on the host).
#pragma once
#include "ptx.cuh"

namespace mxs {

struct CsrParams {
  const int32_t* argmax;    // [n_q, B, l_q]
  const long long* dest_off;  // [B] first destination row of each document
  const long long* dest_len;  // [B] destination rows owned by each document
  int n_q, n_docs, l_q;
  long long n_dest;
  int32_t* cnt;             // workspace [n_q][n_dest]
  int32_t* row_ptr;         // [n_dest + 1]
  int32_t* col_idx;         // [n_q * B * l_q]
};

__global__ void __launch_bounds__(256) csr_count_kernel(const CsrParams p) {
  extern __shared__ int32_t hist[];
  const int q = blockIdx.x / p.n_docs, b = blockIdx.x % p.n_docs;
  const long long off = p.dest_off[b];
  const int len = (int)p.dest_len[b];
  for (int t = threadIdx.x; t < len; t += blockDim.x) hist[t] = 0;
  __syncthreads();
  const int32_t* a = p.argmax + ((long long)q * p.n_docs + b) * p.l_q;
  for (int i = threadIdx.x; i < p.l_q; i += blockDim.x) {
    const int t = a[i];
    if (t >= 0 && t < len) atomicAdd(&hist[t], 1);
  }
  __syncthreads();
  int32_t* out = p.cnt + (long long)q * p.n_dest + off;
  for (int t = threadIdx.x; t < len; t += blockDim.x) out[t] = hist[t];
}

// One block per document: rows [off, off + len).  Padding rows between documents (padded
// layout) belong to the document before them and simply have zero count.
__global__ void __launch_bounds__(1024) csr_scan_kernel(const CsrParams p) {
  __shared__ int32_t warp_tot[32];
  __shared__ int32_t carry;
  const int b = blockIdx.x;
  const long long off = p.dest_off[b];
  const int len = (int)p.dest_len[b];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = (int32_t)((long long)b * p.n_q * p.l_q);
  __syncthreads();
  for (int t0 = 0; t0 < len; t0 += blockDim.x) {
    const int t = t0 + threadIdx.x;
    int tot = 0;
    if (t < len) {
#pragma unroll 16
      for (int q = 0; q < p.n_q; ++q) tot += p.cnt[(long long)q * p.n_dest + off + t];  // 16 loads in flight
    }
    // block exclusive scan of tot
    int x = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
      int v = (lane < (int)(blockDim.x >> 5)) ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      warp_tot[lane] = v;  // inclusive
    }
    __syncthreads();
    const int excl = carry + (w ? warp_tot[w - 1] : 0) + x - tot;
    if (t < len) {
      p.row_ptr[off + t] = excl;
      int run = excl;
      int q0 = 0;
      for (; q0 + 16 <= p.n_q; q0 += 16) {  // 16 independent loads, then the running prefix
        int v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = p.cnt[(long long)(q0 + u) * p.n_dest + off + t];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          p.cnt[(long long)(q0 + u) * p.n_dest + off + t] = run;
          run += v[u];
        }
      }
      for (int q = q0; q < p.n_q; ++q) {
        int32_t* c = p.cnt + (long long)q * p.n_dest + off + t;
        const int v = *c;
        *c = run;
        run += v;
      }
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + tot;
    __syncthreads();
  }
  if (b == p.n_docs - 1 && threadIdx.x == 0) p.row_ptr[p.n_dest] = (int32_t)((long long)p.n_docs * p.n_q * p.l_q);
}

// One block per (q, b) segment; warps take turns in source order so that the per-bucket
// cursor advances exactly as a sequential stable scatter would.
__global__ void __launch_bounds__(256) csr_place_kernel(const CsrParams p) {
  extern __shared__ int32_t cursor[];
  const int q = blockIdx.x / p.n_docs, b = blockIdx.x % p.n_docs;
  const long long off = p.dest_off[b];
  const int len = (int)p.dest_len[b];
  const int32_t* base = p.cnt + (long long)q * p.n_dest + off;
  for (int t = threadIdx.x; t < len; t += blockDim.x) cursor[t] = base[t];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const long long src0 = ((long long)q * p.n_docs + b) * p.l_q;
  const int32_t* a = p.argmax + src0;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int i0 = 0; i0 < p.l_q; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    const bool valid = i < p.l_q;
    const int key = valid ? a[i] : -1 - lane;  // distinct dummy keys never match real ones
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int rank = __popc(peers & lt_mask);
    for (int ww = 0; ww < nw; ++ww) {
      if (w == ww && valid) {
        p.col_idx[cursor[key] + rank] = (int32_t)(src0 + i);
      }
      __syncwarp();
      if (w == ww && valid && rank == 0) cursor[key] += __popc(peers);
      __syncthreads();
    }
  }
}

// Placement v2: one block per (q, b) segment, 8 warps on contiguous source chunks.  Per-warp
// bucket histograms in shared memory turn the cross-warp order into prefix offsets, so every
// warp places its chunk independently (in-warp order from __match_any_sync ranks) -- two block
// barriers per segment instead of one per warp turn.
constexpr int kCsrWarps = 8;
__global__ void __launch_bounds__(32 * kCsrWarps) csr_place_v2_kernel(const CsrParams p) {
  extern __shared__ int32_t hw[];  // [kCsrWarps][len]
  const int q = blockIdx.x / p.n_docs, b = blockIdx.x % p.n_docs;
  const long long off = p.dest_off[b];
  const int len = (int)p.dest_len[b];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < kCsrWarps * len; t += blockDim.x) hw[t] = 0;
  __syncthreads();
  const long long src0 = ((long long)q * p.n_docs + b) * p.l_q;
  const int32_t* a = p.argmax + src0;
  const int chunk = ((p.l_q + kCsrWarps - 1) / kCsrWarps + 31) & ~31;
  const int e0 = w * chunk, e1 = min(p.l_q, e0 + chunk);
  int32_t* h = hw + w * len;
  for (int e = e0 + lane; e < e1; e += 32) {
    const int key = __ldg(a + e);
    if (key >= 0 && key < len) atomicAdd(&h[key], 1);
  }
  __syncthreads();
  const int32_t* base = p.cnt + (long long)q * p.n_dest + off;  // first slot of (q, b) per bucket
  for (int r = threadIdx.x; r < len; r += blockDim.x) {
    int run = base[r];
#pragma unroll
    for (int ww = 0; ww < kCsrWarps; ++ww) {
      const int v = hw[ww * len + r];
      hw[ww * len + r] = run;
      run += v;
    }
  }
  __syncthreads();
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int e = e0; e < e1; e += 32) {
    const int i = e + lane;
    const bool valid = i < e1;
    int key = valid ? __ldg(a + i) : -1;
    const bool ok = valid && key >= 0 && key < len;
    if (!ok) key = -1 - lane;  // distinct dummy keys never match real ones
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int rank = __popc(peers & lt_mask);
    if (ok) p.col_idx[h[key] + rank] = (int32_t)(src0 + i);
    __syncwarp();
    if (ok && rank == 0) h[key] += __popc(peers);
    __syncwarp();
  }
}

// Warp-per-segment variants (used when every document has at most kCsrWarpLenMax rows): a
// block holds kCsrWW segments, each warp its own shared-memory histogram / cursor array, so a
// (q, b) segment needs no block barrier and all 4096 segments of C3 are resident in one wave
// (the block-per-segment kernels above ran ~4 waves of tiny blocks).
constexpr int kCsrWW = 8;
constexpr int kCsrWarpLenMax = 1536;  // 8 warps x 1536 x 4 B = 48 KB per block

__global__ void __launch_bounds__(32 * kCsrWW) csr_count_w_kernel(const CsrParams p, int hist_len) {
  extern __shared__ int32_t csr_sh[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long seg = (long long)blockIdx.x * kCsrWW + w;
  if (seg >= (long long)p.n_q * p.n_docs) return;  // warp-uniform; no block barrier below
  const int q = (int)(seg / p.n_docs), b = (int)(seg % p.n_docs);
  const long long off = p.dest_off[b];
  const int len = (int)p.dest_len[b];
  int32_t* hist = csr_sh + w * hist_len;
  for (int t = lane; t < len; t += 32) hist[t] = 0;
  __syncwarp();
  const int32_t* a = p.argmax + seg * p.l_q;
  for (int i = lane; i < p.l_q; i += 32) {
    const int key = __ldg(a + i);
    if (key >= 0 && key < len) atomicAdd(&hist[key], 1);
  }
  __syncwarp();
  int32_t* out = p.cnt + (long long)q * p.n_dest + off;
  for (int t = lane; t < len; t += 32) out[t] = hist[t];
}

// Stable placement, one warp per (q, b) segment: 32 sources per step in source order; ranks of
// equal keys inside the step from __match_any_sync, the bucket cursor advanced by the lowest lane
// of each key group after everyone has read it.  Keys are prefetched 8 steps at a time.
__global__ void __launch_bounds__(32 * kCsrWW) csr_place_w_kernel(const CsrParams p, int hist_len) {
  extern __shared__ int32_t csr_sh[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long seg = (long long)blockIdx.x * kCsrWW + w;
  if (seg >= (long long)p.n_q * p.n_docs) return;
  const int q = (int)(seg / p.n_docs), b = (int)(seg % p.n_docs);
  const long long off = p.dest_off[b];
  const int len = (int)p.dest_len[b];
  int32_t* cursor = csr_sh + w * hist_len;
  const int32_t* base = p.cnt + (long long)q * p.n_dest + off;  // first slot of (q, b) per bucket
  for (int t = lane; t < len; t += 32) cursor[t] = base[t];
  __syncwarp();
  const long long src0 = seg * p.l_q;
  const int32_t* a = p.argmax + src0;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int e0 = 0; e0 < p.l_q; e0 += 32 * 8) {
    int keys[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = e0 + 32 * u + lane;
      keys[u] = i < p.l_q ? __ldg(a + i) : -1;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = e0 + 32 * u + lane;
      if (e0 + 32 * u >= p.l_q) break;  // warp-uniform
      int key = keys[u];
      const bool ok = i < p.l_q && key >= 0 && key < len;
      if (!ok) key = -1 - lane;  // distinct dummy keys never match real ones
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      const int rank = __popc(peers & lt_mask);
      int slot = 0;
      if (ok) slot = cursor[key] + rank;
      __syncwarp();
      if (ok) {
        p.col_idx[slot] = (int32_t)(src0 + i);
        if (rank == 0) cursor[key] += __popc(peers);
      }
      __syncwarp();
    }
  }
}

}  // namespace mxs
