// Inverse-grid CSR of the saved argmax (K6), on device, bit-identical to
// maxsim/backward.py:81-109 (bincount -> cumsum -> STABLE argsort of the flat destinations).
//
// Source s = (q * B + b) * L_q + i picks destination row dest_off[b] + argmax[s].  Every source
// of document b lands in b's rows, so b's bucket block starts at row_ptr = b * N_q * L_q and the
// problem splits per document; inside a document, ascending s is ascending flat j = q * L_q + i.
//
// csr_doc_kernel -- ONE launch, no global workspace: a thread-block cluster of CL CTAs owns one
// document.  Its N_q * L_q sources (flat j) are cut into CL * W contiguous warp ranges, in order.
//   1. count:  every warp builds a shared-memory histogram of its range's destinations
//   2. prefix: per bucket, an exclusive prefix over the CTA's warps (in place) and the CTA total
//   3. cluster barrier; every CTA reads the other CTAs' totals through DSMEM: bucket base
//      (exclusive scan over the document's rows, one block scan) + the totals of lower ranks
//      -> each warp's first slot in every bucket.  Rank 0 writes row_ptr.
//   4. place:  every warp walks its range in source order, 32 keys per step; equal keys inside a
//      step find each other through a per-bucket lane-mask word (atomicOr, read back), are
//      ranked by lane, and the lowest lane of each group advances the bucket cursor.
// The CSR is therefore the stable counting sort the reference computes, with no atomics on
// global memory and one pass over argmax for the count plus one (L2-resident) for the placement.
//
// csr_sort_* -- the general path for destinations too long for shared-memory histograms
// (Chamfer clouds, documents beyond ~3K rows): a stable LSD radix sort of (dest row, source)
// pairs (cub::DeviceRadixSort, stable by construction) and row_ptr by binary search.
// Indices are int32 (n_src and n_dest < 2^31 are checked on the host).
#pragma once
#include "fastdiv.cuh"
#include "ptx.cuh"

namespace mxs {

// A lane's walk over the flat sources j = q * L_q + i of one document in steps of 32: the source
// id (which is also the argmax offset) advances incrementally (no division per step; L_q < 32
// wraps in a loop).
struct SrcWalk {
  int src;  // (q * B + b) * L_q + i
  int i;
  MXS_DEV void init(uint32_t j, const FastDiv& lq, int l_q, int n_docs, int b) {
    const uint32_t q = fdiv(j, lq);
    i = (int)(j - q * (uint32_t)l_q);
    src = (int)((q * (uint32_t)n_docs + (uint32_t)b) * (uint32_t)l_q) + i;
  }
  MXS_DEV void step32(int l_q, int wrap) {  // wrap = (B - 1) * L_q
    i += 32;
    src += 32;
    while (i >= l_q) {
      i -= l_q;
      src += wrap;
    }
  }
};

struct CsrParams {
  const int32_t* argmax;      // [n_q, B, l_q]
  const long long* dest_off;  // [B] first destination row of each document
  const long long* dest_len;  // [B] destination rows owned by each document
  int n_q, n_docs, l_q;
  long long n_dest;
  int hist_len;               // >= every dest_len, multiple of 4 (shared-memory row stride)
  FastDiv lq_div;             // division by l_q
  int32_t* row_ptr;           // [n_dest + 1]
  int32_t* col_idx;           // [n_q * B * l_q]
};

MXS_DEV uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
MXS_DEV int32_t ld_cluster_s32(uint32_t cluster_addr) {
  int32_t v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(cluster_addr) : "memory");
  return v;
}
MXS_DEV void cluster_arrive_release() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
MXS_DEV void cluster_wait_acquire() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

constexpr int kCsrMaxWarps = 16;

// Shared memory: hw[W][H] per-warp counts (then cursors), T[H] CTA totals (read by the other
// CTAs of the cluster), tot[H], bef[H] (document totals and lower-rank totals per bucket), then
// mk[W][H] per-warp key-group lane masks for the placement.
__global__ void __launch_bounds__(32 * kCsrMaxWarps) csr_doc_kernel(const CsrParams p) {
  extern __shared__ int32_t csr_sh[];
  __shared__ int32_t warp_sum[kCsrMaxWarps];
  const int nw = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = p.hist_len;
  const uint32_t cl = cluster_nctarank(), rank = cluster_ctarank();
  const int b = (int)(blockIdx.x / cl);
  const long long off = p.dest_off[b];
  const int len = (int)p.dest_len[b];
  int32_t* T = csr_sh + nw * H;
  int32_t* tot = T + H;
  int32_t* bef = tot + H;
  uint32_t* mk = reinterpret_cast<uint32_t*>(bef + H) + w * H;  // [W][H] per-step key-group lane masks
  for (int x = threadIdx.x; x < nw * H; x += blockDim.x) csr_sh[x] = 0;
  for (int x = threadIdx.x; x < nw * H; x += blockDim.x) reinterpret_cast<uint32_t*>(bef + H)[x] = 0u;
  __syncthreads();

  const long long n_src = (long long)p.n_q * p.l_q;  // sources of this document (flat j)
  const long long nwt = (long long)cl * nw;
  const long long chunk = (((n_src + nwt - 1) / nwt) + 31) & ~31LL;
  const long long j0 = min(n_src, (long long)(rank * nw + w) * chunk), j1 = min(n_src, j0 + chunk);
  int32_t* h = csr_sh + w * H;

  // 1. count (8 loads in flight per lane)
  const int wrap = (p.n_docs - 1) * p.l_q;
  SrcWalk wk;
  if (j0 < j1) wk.init((uint32_t)(j0 + lane), p.lq_div, p.l_q, p.n_docs, b);
  for (long long e0 = j0; e0 < j1; e0 += 32 * 8) {
    int keys[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      keys[u] = (e0 + 32 * u + lane < j1) ? __ldg(p.argmax + wk.src) : -1;
      wk.step32(p.l_q, wrap);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (keys[u] >= 0 && keys[u] < len) atomicAdd(&h[keys[u]], 1);
  }
  __syncthreads();
  // 2. exclusive prefix over this CTA's warps (in place) and the CTA totals
  for (int t = threadIdx.x; t < len; t += blockDim.x) {
    int run = 0;
    for (int ww = 0; ww < nw; ++ww) {
      const int v = csr_sh[ww * H + t];
      csr_sh[ww * H + t] = run;
      run += v;
    }
    T[t] = run;
  }
  // 3. cluster exchange: document totals and the totals of lower ranks, per bucket
  if (cl > 1) {
    cluster_arrive_release();
    cluster_wait_acquire();
  } else {
    __syncthreads();
  }
  const uint32_t t_addr = smem_u32(T);
  const int per = (len + (int)blockDim.x - 1) / (int)blockDim.x;  // contiguous buckets per thread
  const int t0 = min(len, (int)threadIdx.x * per), t1 = min(len, t0 + per);
  int my_sum = 0;
  for (int t = t0; t < t1; ++t) {
    int s = 0, before = 0;
    for (uint32_t r = 0; r < cl; ++r) {
      const int v = (r == rank) ? T[t] : ld_cluster_s32(mapa_u32(t_addr + 4u * (uint32_t)t, r));
      if (r < rank) before += v;
      s += v;
    }
    tot[t] = s;
    bef[t] = before;
    my_sum += s;
  }
  if (cl > 1) cluster_arrive_release();  // done reading remote T (peers wait before exiting)
  // block-wide exclusive scan of the per-thread sums
  int x = my_sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sum[w] = x;
  __syncthreads();
  int wbase = 0;
  for (int ww = 0; ww < w; ++ww) wbase += warp_sum[ww];
  const long long doc_base = (long long)b * n_src;
  int run = wbase + x - my_sum;  // exclusive prefix of this thread's first bucket within the document
  for (int t = t0; t < t1; ++t) {
    const int base = (int)doc_base + run;
    if (rank == 0) p.row_ptr[off + t] = base;
    const int c = base + bef[t];
    for (int ww = 0; ww < nw; ++ww) csr_sh[ww * H + t] += c;
    run += tot[t];
  }
  if (rank == 0 && threadIdx.x == 0 && b == p.n_docs - 1) p.row_ptr[p.n_dest] = (int32_t)(doc_base + n_src);
  __syncthreads();

  // 4. stable placement, one warp per range in source order
  const unsigned lt_mask = (1u << lane) - 1u;
  if (j0 < j1) wk.init((uint32_t)(j0 + lane), p.lq_div, p.l_q, p.n_docs, b);
  for (long long e0 = j0; e0 < j1; e0 += 32 * 8) {
    int keys[8], srcs[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      keys[u] = (e0 + 32 * u + lane < j1) ? __ldg(p.argmax + wk.src) : -1;
      srcs[u] = wk.src;
      wk.step32(p.l_q, wrap);
    }
    // stable placement of the 8 steps in order.  Equal keys of a step find each other through a
    // per-warp lane-mask word per bucket: every lane ORs its bit in (atomic, so the shared word
    // has no unordered writers), reads the group mask back, and the group's lowest lane advances
    // the cursor and clears the word for the next step -- no MATCH.ANY, no ballot per key bit.
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (e0 + 32 * u >= j1) break;  // warp-uniform
      const int key = keys[u];
      const bool ok = key >= 0 && key < len;
      if (ok) atomicOr(&mk[key], 1u << lane);
      __syncwarp();
      const uint32_t pm = ok ? mk[key] : 0u;
      __syncwarp();
      const int rk = __popc(pm & lt_mask);
      int v = 0;
      if (ok && rk == 0) {  // the lowest lane of each key group advances the bucket cursor
        v = h[key];
        h[key] = v + __popc(pm);
        mk[key] = 0u;
      }
      v = __shfl_sync(0xffffffffu, v, ok ? __ffs(pm) - 1 : lane);
      if (ok) p.col_idx[v + rk] = srcs[u];
      __syncwarp();
    }
  }
  if (cl > 1) cluster_wait_acquire();  // keep T alive until every peer has read it
}

// ---------------------------------------------------------------- general path (radix sort)
// keys[s] = global destination row of source s (n_dest for an out-of-range argmax: sorts last,
// outside every row), vals[s] = s.
__global__ void __launch_bounds__(256) csr_sort_keys_kernel(const CsrParams p, int32_t* keys, int32_t* vals) {
  const long long n = (long long)p.n_q * p.n_docs * p.l_q;
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < n; s += (long long)gridDim.x * blockDim.x) {
    const int b = (int)((s / p.l_q) % p.n_docs);
    const int a = p.argmax[s];
    const long long len = p.dest_len[b];
    keys[s] = (a >= 0 && a < len) ? (int32_t)(p.dest_off[b] + a) : (int32_t)p.n_dest;
    vals[s] = (int32_t)s;
  }
}

// row_ptr[r] = first position of a key >= r in the sorted keys (r = 0 .. n_dest).
__global__ void __launch_bounds__(256) csr_sort_rowptr_kernel(const int32_t* sorted_keys, long long n, long long n_dest,
                                                              int32_t* row_ptr) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r <= n_dest;
       r += (long long)gridDim.x * blockDim.x) {
    long long lo = 0, hi = n;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (sorted_keys[mid] < r)
        lo = mid + 1;
      else
        hi = mid;
    }
    row_ptr[r] = (int32_t)lo;
  }
}

}  // namespace mxs
