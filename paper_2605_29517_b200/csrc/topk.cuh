// Device top-K with the reference ranking (K9): score descending, document id ascending
// (maxsim/streamio.py:230-262 TopKHeap, maxsim/cli.py:88-92 _ranked).
//
// (score, id) pairs are totally ordered (ids are unique), so a sorting network under that order
// reproduces the heap's result exactly, ties included.
#pragma once
#include "ptx.cuh"

namespace mxs {

MXS_DEV bool better(double s1, long long i1, double s2, long long i2) {
  return s1 > s2 || (s1 == s2 && i1 < i2);
}

constexpr int kTopkThreads = 1024;
constexpr int kTopkSlice = 4096;  // elements sorted per block (64 KB of shared memory)

// Each block sorts one slice of (score, id) pairs with a bitonic network under the reference
// order (score desc, id asc; invalid slots -- past the end, NaN, id < 0 -- sort last) and keeps
// the first k.  Repeated over the surviving candidates until one slice remains.
// in_ids == nullptr means ids are positions + id_offset.
__global__ void __launch_bounds__(kTopkThreads) topk_kernel(const double* __restrict__ in_s,
                                                            const long long* __restrict__ in_ids, long long n, int k,
                                                            long long chunk, long long id_offset,
                                                            double* __restrict__ out_s, long long* __restrict__ out_ids) {
  extern __shared__ uint8_t tk_smem[];
  double* ss = reinterpret_cast<double*>(tk_smem);
  long long* si = reinterpret_cast<long long*>(tk_smem + kTopkSlice * sizeof(double));
  const long long lo = (long long)blockIdx.x * chunk;
  const long long hi = min(n, lo + chunk);
  for (int e = threadIdx.x; e < kTopkSlice; e += blockDim.x) {
    double s = -INFINITY;
    long long id = LLONG_MAX;
    const long long g = lo + e;
    if (g < hi) {
      const double v = in_s[g];
      const long long i = in_ids ? in_ids[g] : g + id_offset;
      if (v == v && i >= 0) {
        s = v;
        id = i;
      }
    }
    ss[e] = s;
    si[e] = id;
  }
  __syncthreads();
  for (int size = 2; size <= kTopkSlice; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < kTopkSlice / 2; t += blockDim.x) {
        const int a = 2 * t - (t & (stride - 1));  // first element of the pair
        const int b = a + stride;
        const bool desc_block = (a & size) == 0;   // this run is sorted "best first"
        const double sa = ss[a], sb = ss[b];
        const long long ia = si[a], ib = si[b];
        // b strictly better than a under (score desc, id asc, invalid last)?
        const bool b_first = (ib != LLONG_MAX) && (ia == LLONG_MAX || better(sb, ib, sa, ia));
        if (b_first == desc_block) {
          ss[a] = sb;
          ss[b] = sa;
          si[a] = ib;
          si[b] = ia;
        }
      }
      __syncthreads();
    }
  }
  for (int r = threadIdx.x; r < k; r += blockDim.x) {
    const long long id = si[r];
    out_s[(long long)blockIdx.x * k + r] = (id == LLONG_MAX) ? -INFINITY : ss[r];
    out_ids[(long long)blockIdx.x * k + r] = (id == LLONG_MAX) ? -1 : id;
  }
}

}  // namespace mxs

namespace mxs {

// ----------------------------------------------------------------------------------------------
// Small-k selection (k <= kSelMaxK): warp tournaments instead of a full sort.
//
// A CTA stages its slice of scores in shared memory; every warp owns a contiguous sub-slice,
// keeps one "best so far" per lane, and runs k rounds of a warp-wide argmax under the
// reference order (score desc, id asc).  Only the winning lane removes its element (the score
// slot becomes NaN = empty) and rescans its own strided elements, so a round costs one 5-level
// shuffle reduction plus one short rescan.  The per-warp winners (k each) are re-selected by
// warp 0.  (score, id) is a total order over the valid entries, so the result is exactly the
// first k of the sorted order -- identical to the bitonic kernel above and to TopKHeap.
// Ids are implicit (position + id_offset, 8 B of smem per element) for a score vector and
// explicit (16 B per element) for candidate lists.
// ----------------------------------------------------------------------------------------------
constexpr int kSelMaxK = 128;
constexpr int kSelThreads = 512;
constexpr long long kSelChunkImplicit = 16384;  // 128 KB of scores
constexpr long long kSelChunkExplicit = 8192;   // 128 KB of (score, id)

MXS_DEV long long sel_id(const long long* ids, long long base, int j) { return ids ? ids[j] : base + j; }

MXS_DEV void sel_lane_best(const double* s, const long long* ids, long long base, int cnt, double& bs, long long& bi,
                           int& bj) {
  bs = -INFINITY;
  bi = LLONG_MAX;
  bj = -1;
  for (int j = (int)lane_id(); j < cnt; j += 32) {
    const double v = s[j];
    if (v != v) continue;  // empty / consumed
    const long long i = sel_id(ids, base, j);
    if (bj < 0 || better(v, i, bs, bi)) {
      bs = v;
      bi = i;
      bj = j;
    }
  }
}

// Warp-cooperative: writes the k best of s[0, cnt) (ids explicit or base + j) to (os, oi)[0, k)
// in order; missing entries become (empty_s, -1).  Consumes (NaN-marks) the selected entries.
MXS_DEV void sel_warp(double* s, const long long* ids, long long base, int cnt, int k, double* os, long long* oi,
                      double empty_s) {
  double bs;
  long long bi;
  int bj;
  sel_lane_best(s, ids, base, cnt, bs, bi, bj);
  for (int r = 0; r < k; ++r) {
    double ws = bs;
    long long wi = bi;
    int has = bj >= 0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double os_ = __shfl_xor_sync(0xffffffffu, ws, off);
      const long long oi_ = __shfl_xor_sync(0xffffffffu, wi, off);
      const int oh = __shfl_xor_sync(0xffffffffu, has, off);
      if (oh && (!has || better(os_, oi_, ws, wi))) {
        ws = os_;
        wi = oi_;
        has = 1;
      }
    }
    if (!has) {  // nothing valid left: this and the remaining slots are empty
      for (int rr = r + (int)lane_id(); rr < k; rr += 32) {
        os[rr] = empty_s;
        oi[rr] = -1;
      }
      break;
    }
    if (lane_id() == 0) {
      os[r] = ws;
      oi[r] = wi;
    }
    if (bj >= 0 && bi == wi) {  // this lane owned the winner (ids are unique among valid entries)
      s[bj] = __longlong_as_double(0x7ff8000000000000LL);
      sel_lane_best(s, ids, base, cnt, bs, bi, bj);
    }
  }
  __syncwarp();
}

// Valid-first order used by the sorting networks: valid entries (id != LLONG_MAX) by (score desc,
// id asc), then the empty ones.
MXS_DEV bool sel_before(double s1, long long i1, double s2, long long i2) {
  return i1 != LLONG_MAX && (i2 == LLONG_MAX || better(s1, i1, s2, i2));
}

constexpr int kSelSurvivors = 1024;  // threshold-filter capacity (one sort element per thread pair)

// Threshold filter for k <= kSelMaxK.  Every lane's maximum is a real element, so for k <= 32 the
// k-th largest lane maximum of ANY warp is a lower bound T on the k-th largest score of the slice
// (the largest such bound over the warps is used); for larger k, the k-th largest of all the
// block's lane maxima.  Only elements with score >= T can be in the top k; they
// are compacted (typically k .. a few k of them) and sorted with a bitonic network under the
// reference order.  Returns false (nothing written) if more than kSelSurvivors survive -- e.g.
// massive ties at the threshold -- and the caller falls back to the warp tournaments.
MXS_DEV bool sel_threshold(const double* ss, const long long* si, long long base, int m, int k, double* out_s,
                           long long* out_ids, double* sv_s, long long* sv_i, double* wbound, int* counter) {
  constexpr int kWarps = kSelThreads / 32;
  const int w = (int)warp_id_uniform();
  const int lane = (int)lane_id();
  const int per = (m + kWarps - 1) / kWarps;
  const int b0 = min(m, w * per), b1 = min(m, b0 + per);
  // 1. lane maxima (NaN = empty never wins: the comparison is false)
  double lm = -INFINITY;
  for (int j = b0 + lane; j < b1; j += 32) lm = fmax(lm, ss[j]);
  double T = -INFINITY;
  if (k <= 32) {
    // 2. k-th largest lane maximum of this warp: bitonic sort of 32 values (descending)
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, lm, stride);
        const bool lower = (lane & stride) == 0;
        const bool desc = (lane & size) == 0 || size == 32;
        // in a descending run the lower lane keeps the max
        lm = (lower == desc) ? fmax(lm, o) : fmin(lm, o);
      }
    }
    const double kth = __shfl_sync(0xffffffffu, lm, k - 1);
    if (lane == 0) wbound[w] = kth;
    if (threadIdx.x == 0) *counter = 0;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kWarps; ++i) T = fmax(T, wbound[i]);
  } else {
    // 2'. k in (32, kSelThreads]: the k-th largest of ALL the block's lane maxima (distinct real
    //     elements, so again a lower bound), by a bitonic sort of the kSelThreads lane maxima
    sv_s[threadIdx.x] = lm;
    if (threadIdx.x == 0) *counter = 0;
    __syncthreads();
    for (int size = 2; size <= kSelThreads; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = threadIdx.x; t < kSelThreads / 2; t += blockDim.x) {
          const int a = 2 * t - (t & (stride - 1));
          const int b = a + stride;
          const bool desc = (a & size) == 0 || size == kSelThreads;
          const double va = sv_s[a], vb = sv_s[b];
          if ((vb > va) == desc) {
            sv_s[a] = vb;
            sv_s[b] = va;
          }
        }
        __syncthreads();
      }
    }
    T = sv_s[k - 1];
    __syncthreads();  // sv_s is reused for the survivors below
  }
  // 3. compact the survivors (score >= T); with T = -inf (fewer than k valid entries in every
  //    warp) everything valid survives and the capacity check decides
  for (int j = b0 + lane; j < b1; j += 32) {
    const double v = ss[j];
    if (v >= T) {
      const int pos = atomicAdd(counter, 1);
      if (pos < kSelSurvivors) {
        sv_s[pos] = v;
        sv_i[pos] = si ? si[j] : base + j;
      }
    }
  }
  __syncthreads();
  const int cnt = *counter;
  if (cnt > kSelSurvivors) return false;
  int P = 32;
  while (P < cnt) P <<= 1;
  for (int e = cnt + (int)threadIdx.x; e < P; e += blockDim.x) {
    sv_s[e] = -INFINITY;
    sv_i[e] = LLONG_MAX;
  }
  __syncthreads();
  // 4. bitonic sort of P <= 1024 survivors (one pair per thread per stage)
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < P / 2; t += blockDim.x) {
        const int a = 2 * t - (t & (stride - 1));
        const int b = a + stride;
        const bool first_block = (a & size) == 0 || size == P;  // sorted "best first"
        const double sa = sv_s[a], sb = sv_s[b];
        const long long ia = sv_i[a], ib = sv_i[b];
        if (sel_before(sb, ib, sa, ia) == first_block) {
          sv_s[a] = sb;
          sv_s[b] = sa;
          sv_i[a] = ib;
          sv_i[b] = ia;
        }
      }
      __syncthreads();
    }
  }
  for (int r = threadIdx.x; r < k; r += blockDim.x) {
    const bool ok = sv_i[r] != LLONG_MAX;
    out_s[r] = ok ? sv_s[r] : -INFINITY;
    out_ids[r] = ok ? sv_i[r] : -1;
  }
  return true;
}

// One launch: every CTA selects the k best of its slice [blockIdx.x * chunk, ... + chunk).
// in_ids == nullptr means ids are positions + id_offset; NaN scores and ids < 0 are empty, and
// empty output slots are (-inf, -1) -- so a pass's output is a valid input for the next pass.
__global__ void __launch_bounds__(kSelThreads) topk_select_kernel(const double* __restrict__ in_s,
                                                                  const long long* __restrict__ in_ids, long long n,
                                                                  int k, long long chunk, long long id_offset,
                                                                  double* __restrict__ out_s,
                                                                  long long* __restrict__ out_ids) {
  extern __shared__ __align__(16) uint8_t sel_smem[];
  constexpr int kWarps = kSelThreads / 32;
  __shared__ double wbound[kWarps];
  __shared__ int counter;
  const double kNaN = __longlong_as_double(0x7ff8000000000000LL);
  double* ss = reinterpret_cast<double*>(sel_smem);
  long long* si = in_ids ? reinterpret_cast<long long*>(ss + chunk) : nullptr;
  double* cs = reinterpret_cast<double*>(sel_smem + chunk * (in_ids ? 16 : 8));
  long long* ci = reinterpret_cast<long long*>(cs + kWarps * kSelMaxK);
  double* sv_s = reinterpret_cast<double*>(ci + kWarps * kSelMaxK);
  long long* sv_i = reinterpret_cast<long long*>(sv_s + kSelSurvivors);
  const long long lo = (long long)blockIdx.x * chunk;
  const int m = (int)max(0LL, min(n, lo + chunk) - lo);
  // the slice -> shared memory with many loads in flight per thread (a dependent load -> store
  // loop paid one L2 round trip per element and dominated the kernel)
  if (in_ids) {
#pragma unroll 4
    for (int e = threadIdx.x; e < m; e += blockDim.x) {
      const double v = in_s[lo + e];
      const long long i = in_ids[lo + e];
      ss[e] = (i >= 0) ? v : kNaN;
      si[e] = i;
    }
  } else {
    const double* src = in_s + lo;
    int e = threadIdx.x;
    for (; e + 7 * (int)blockDim.x < m; e += 8 * (int)blockDim.x) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(src + e + u * (int)blockDim.x);
#pragma unroll
      for (int u = 0; u < 8; ++u) ss[e + u * (int)blockDim.x] = v[u];
    }
    for (; e < m; e += blockDim.x) ss[e] = __ldg(src + e);
  }
  __syncthreads();
  double* os = out_s + (long long)blockIdx.x * k;
  long long* oi = out_ids + (long long)blockIdx.x * k;
  if (k <= kSelMaxK && sel_threshold(ss, si, lo + id_offset, m, k, os, oi, sv_s, sv_i, wbound, &counter)) return;
  const int w = (int)warp_id_uniform();
  const int per = (m + kWarps - 1) / kWarps;
  const int b0 = min(m, w * per), b1 = min(m, b0 + per);
  sel_warp(ss + b0, si ? si + b0 : nullptr, lo + b0 + id_offset, b1 - b0, k, cs + (long long)w * k,
           ci + (long long)w * k, kNaN);
  __syncthreads();
  if (w == 0) sel_warp(cs, ci, 0, kWarps * k, k, os, oi, -INFINITY);
}

}  // namespace mxs
