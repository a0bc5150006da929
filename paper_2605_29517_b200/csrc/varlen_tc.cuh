// Padding-free (cu_seqlens) MaxSim forward on tcgen05 (K5) -- maxsim/varlen.py:88-131.
//
// Operand roles are swapped relative to the dense kernel: A = a tile of 128 consecutive packed
// document tokens (TMA from the [total_tokens, dim] buffer, no padding anywhere), B = all query
// rows of the call (N = n_q * l_q <= 128 columns, resident in shared memory).  The accumulator
// tile is [128 tokens (TMEM lanes) x N query rows (columns)]; documents start and end at any
// token, so the row max over a document's tokens is a SEGMENTED column reduction:
//   1. each epilogue thread (= one token) writes its N similarities to a padded smem tile;
//   2. thread (column c, token quarter h) scans its 32 tokens in order, keeping (max, argmax) per
//      document piece (strict >, ascending token order => lowest index on ties, S3);
//   3. documents that end inside the quarter are final; the first / last piece of each quarter
//      is merged in order by a carry that also crosses tiles.
// CTA c owns a contiguous document range balanced by token count (binary search of cu_seqlens on
// the device), so every document is reduced by exactly one CTA -- no atomics, no second pass.
// The path is HBM-bound (L_q = 32 gives 32 FLOP/B); the MMA is a small fraction of the tile time.
#pragma once
#include "fwd_tc.cuh"

namespace mxs {

struct VarlenParams {
  int n_q, l_q, n_cols;  // n_cols = n_q * l_q (<= 128), padded to a multiple of 16 for the MMA
  int n_cols_pad;
  long long n_docs, n_tokens;
  int dim;
  int stages;
  const long long* cu;  // [n_docs + 1] device
  float* rowmax;        // [n_q, n_docs, l_q]
  int32_t* argmax;      // [n_q, n_docs, l_q] or nullptr
};

constexpr int kVlEpiWarps = 4;
constexpr int kVlThreads = 32 * (2 + kVlEpiWarps);  // warp 0 TMA, warp 1 MMA + TMEM alloc, 2..5 epilogue
constexpr int kVlTilePad = 33;                        // floats per token row of the transpose tile

struct VlSmemHeader {
  uint64_t full[8];
  uint64_t empty[8];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint64_t qfull;
  uint32_t tmem_base;
  int32_t doc_begin, doc_end;
  int32_t pad;
  long long tok_begin, tok_end;
  float tile[128 * kVlTilePad];     // transposed similarities of one 32-column chunk
  int32_t tok_doc[128];             // document of each token in the tile
  float hm[4][32];                  // per quarter / column: head piece (max, arg, doc)
  long long ha[4][32];
  int32_t hd[4][32];
  float tm[4][32];                  // tail piece
  long long ta[4][32];
  int32_t td[4][32];
};

__host__ __device__ inline size_t varlen_smem_bytes(int ka, int stages, int n_cols_pad) {
  return 1024 + (size_t)stages * ka * kAtomBytes + (size_t)ka * n_cols_pad * 128 + sizeof(VlSmemHeader);
}

// first document d in [lo, hi) with cu[d + 1] > tok (i.e. the document containing token tok)
MXS_DEV long long doc_of_token(const long long* cu, long long lo, long long hi, long long tok) {
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (__ldg(cu + mid + 1) > tok)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

MXS_DEV void vl_emit(const VarlenParams& p, int col, long long doc, float m, long long arg_tok) {
  if (doc < 0 || col >= p.n_cols) return;
  const int q = col / p.l_q, i = col % p.l_q;
  const long long o = ((long long)q * p.n_docs + doc) * p.l_q + i;
  p.rowmax[o] = m;
  if (p.argmax) p.argmax[o] = (int32_t)(arg_tok - __ldg(p.cu + doc));
}

template <TcKind KIND, int KA>
__global__ void __launch_bounds__(kVlThreads, 1)
    varlen_tc_kernel(const __grid_constant__ CUtensorMap tmT, const __grid_constant__ CUtensorMap tmQ,
                     const VarlenParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sT = smem;                                           // token tiles
  uint8_t* sQ = sT + (size_t)p.stages * KA * kAtomBytes;        // all query rows (B operand)
  VlSmemHeader* hdr = reinterpret_cast<VlSmemHeader*>(sQ + (size_t)KA * p.n_cols_pad * 128);
  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();

  if (threadIdx.x == 0) {
    // token-balanced contiguous document range of this CTA
    const long long total = __ldg(p.cu + p.n_docs);
    const long long t0 = total * blockIdx.x / gridDim.x;
    const long long t1 = total * (blockIdx.x + 1) / gridDim.x;
    const long long d0 = (blockIdx.x == 0) ? 0 : doc_of_token(p.cu, 0, p.n_docs, t0 - 1) + 1;
    const long long d1 = (blockIdx.x + 1 == gridDim.x) ? p.n_docs : doc_of_token(p.cu, 0, p.n_docs, t1 - 1) + 1;
    hdr->doc_begin = (int32_t)d0;
    hdr->doc_end = (int32_t)(d1 > d0 ? d1 : d0);
    hdr->tok_begin = __ldg(p.cu + d0);
    hdr->tok_end = __ldg(p.cu + hdr->doc_end);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&hdr->full[s], 1);
      mbar_init(&hdr->empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&hdr->tfull[s], 1);
      mbar_init(&hdr->tempty[s], kVlEpiWarps);
    }
    mbar_init(&hdr->qfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&hdr->tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = hdr->tmem_base;
  const long long tok_begin = hdr->tok_begin, tok_end = hdr->tok_end;
  const int n_tiles = (int)((tok_end - tok_begin + 127) / 128);
  constexpr int kElemsPerAtom = (KIND == TcKind::I8) ? 128 : 64;
  const int ncc = (p.n_cols + 31) / 32;  // 32-column chunks of the accumulator

  if (warp == 0) {
    if (lane == 0 && n_tiles > 0) {
      tma_prefetch_desc(&tmT);
      mbar_arrive_expect_tx(&hdr->qfull, (uint32_t)(KA * p.n_cols_pad * 128));
      for (int a = 0; a < KA; ++a)
        tma_load_2d(&tmQ, &hdr->qfull, sQ + (size_t)a * p.n_cols_pad * 128, a * kElemsPerAtom, 0, kEvictLast);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < n_tiles; ++t) {
        mbar_wait(&hdr->empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&hdr->full[stage], (uint32_t)(KA * kAtomBytes));
        for (int a = 0; a < KA; ++a)
          tma_load_2d(&tmT, &hdr->full[stage], sT + (size_t)(stage * KA + a) * kAtomBytes, a * kElemsPerAtom,
                      (int)(tok_begin + (long long)t * 128), kEvictFirst);
        if (++stage == p.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (n_tiles > 0) {
      const uint32_t idesc = (KIND == TcKind::I8) ? make_idesc(2, 1, 128, (uint32_t)p.n_cols_pad)
                             : (KIND == TcKind::BF16) ? make_idesc(1, 1, 128, (uint32_t)p.n_cols_pad)
                                                      : make_idesc(1, 0, 128, (uint32_t)p.n_cols_pad);
      mbar_wait(&hdr->qfull, 0);
      tc_fence_after();
      const uint64_t tdesc0 = sw128_kmajor_desc(smem_u32(sT));
      const uint64_t qdesc0 = sw128_kmajor_desc(smem_u32(sQ));
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < n_tiles; ++t) {
        const int slot = t & 1;
        const uint32_t sph = (uint32_t)(t >> 1) & 1u;
        mbar_wait(&hdr->full[stage], phase);
        mbar_wait(&hdr->tempty[slot], sph ^ 1u);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t ad0 = tdesc0 + (uint64_t)((stage * KA * kAtomBytes) >> 4);
          const uint32_t dcol = tmem_base + (uint32_t)(slot * 256);
#pragma unroll
          for (int k = 0; k < KA * 4; ++k) {
            const uint64_t aoff = (uint64_t)(((k >> 2) * kAtomBytes + (k & 3) * 32) >> 4);
            const uint64_t boff = (uint64_t)(((k >> 2) * p.n_cols_pad * 128 + (k & 3) * 32) >> 4);
            if constexpr (KIND == TcKind::I8)
              mma_i8_ss(dcol, ad0 + aoff, qdesc0 + boff, idesc, k > 0 ? 1u : 0u);
            else
              mma_f16_ss(dcol, ad0 + aoff, qdesc0 + boff, idesc, k > 0 ? 1u : 0u);
          }
          mma_commit(&hdr->tfull[slot]);
          mma_commit(&hdr->empty[stage]);
        }
        __syncwarp();
        if (++stage == p.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue: segmented max
    const int ew = (int)warp - 2;                // 0..3 == token quarter
    const int quad = (int)(warp & 3);            // TMEM lane quadrant of this warp
    const int tid = ew * 32 + (int)lane;          // 0..127
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const int my_tok = quad * 32 + (int)lane;    // token (TMEM lane) this thread loads
    // carry (merge threads: ew == 0, one column per lane per chunk)
    float cm[4];
    long long ca[4];
    long long cd[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      cm[c] = -INFINITY;
      ca[c] = 0;
      cd[c] = -1;
    }
    long long d_lo = hdr->doc_begin;  // first document that can own tokens of the current tile
    for (int t = 0; t < n_tiles; ++t) {
      const long long p0 = tok_begin + (long long)t * 128;
      // ---- document of every token of the tile (start marks + inclusive max scan)
      {
        // token 0 belongs to d_lo unless a later document starts exactly at p0 (written after
        // the barrier, so the two writes never race)
        const long long d = d_lo + tid;
        hdr->tok_doc[tid] = (tid == 0) ? (int32_t)d_lo : -1;
        named_bar_sync(1, 128);
        if (d < hdr->doc_end) {
          const long long s = __ldg(p.cu + d) - p0;
          if (s >= 0 && s < 128) hdr->tok_doc[s] = (int32_t)d;
        }
        named_bar_sync(1, 128);
        int v = hdr->tok_doc[tid];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, v, o);
          if ((int)lane >= o) v = max(v, y);
        }
        if (lane == 31) hdr->td[0][ew] = v;  // scratch for the cross-warp carry
        named_bar_sync(1, 128);
        for (int w = 0; w < ew; ++w) v = max(v, hdr->td[0][w]);
        if (p0 + tid >= tok_end) v = -1;  // tokens past this CTA's range belong to nobody here
        named_bar_sync(1, 128);
        hdr->tok_doc[tid] = v;
      }
      const int slot = t & 1;
      mbar_wait(&hdr->tfull[slot], (uint32_t)(t >> 1) & 1u);
      tc_fence_after();
      for (int cc = 0; cc < ncc; ++cc) {
        uint32_t r[32];
        tmem_ld32(tmem_base + lane_base + (uint32_t)(slot * 256 + cc * 32), r);
        tmem_ld_wait();
        if (cc == ncc - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&hdr->tempty[slot]);
        }
        float* trow = hdr->tile + my_tok * kVlTilePad;
#pragma unroll
        for (int j = 0; j < 32; ++j) trow[j] = __uint_as_float(r[j]);
        named_bar_sync(1, 128);
        // ---- scan: column c = lane, tokens of quarter ew
        const int c = (int)lane;
        float m = -INFINITY;
        long long a = 0;
        int cur = -2;
        int first_doc = -2;
        bool head_done = false;
        for (int k = 0; k < 32; ++k) {
          const int tau = ew * 32 + k;
          const int d = hdr->tok_doc[tau];
          if (d != cur) {
            if (cur != -2) {
              if (!head_done) {
                hdr->hm[ew][c] = m;
                hdr->ha[ew][c] = a;
                hdr->hd[ew][c] = cur;
                head_done = true;
              } else if (cur >= 0) {
                vl_emit(p, cc * 32 + c, cur, m, a);  // complete inside this quarter
              }
            } else {
              first_doc = d;
            }
            cur = d;
            m = -INFINITY;
            a = 0;
          }
          const float v = hdr->tile[tau * kVlTilePad + c];
          if (v > m) {
            m = v;
            a = p0 + tau;
          }
        }
        if (!head_done) {  // the whole quarter is one piece: head == tail
          hdr->hm[ew][c] = m;
          hdr->ha[ew][c] = a;
          hdr->hd[ew][c] = cur;
          hdr->td[ew][c] = -3;  // marker: no separate tail
        } else {
          hdr->tm[ew][c] = m;
          hdr->ta[ew][c] = a;
          hdr->td[ew][c] = cur;
        }
        (void)first_doc;
        named_bar_sync(1, 128);
        // ---- ordered merge of the quarter pieces with the carry (warp ew == 0)
        if (ew == 0) {
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int hd = hdr->hd[h][c];
            const float hmv = hdr->hm[h][c];
            const long long hav = hdr->ha[h][c];
            if (hd == cd[cc]) {
              if (hmv > cm[cc]) {  // the carry holds earlier tokens: strict > keeps it on ties
                cm[cc] = hmv;
                ca[cc] = hav;
              }
            } else {
              if (cd[cc] >= 0) vl_emit(p, cc * 32 + c, cd[cc], cm[cc], ca[cc]);
              cd[cc] = hd;
              cm[cc] = hmv;
              ca[cc] = hav;
            }
            const int tdv = hdr->td[h][c];
            if (tdv != -3) {  // a document ended inside quarter h; the tail starts a new carry
              if (cd[cc] >= 0) vl_emit(p, cc * 32 + c, cd[cc], cm[cc], ca[cc]);
              cd[cc] = tdv;
              cm[cc] = hdr->tm[h][c];
              ca[cc] = hdr->ta[h][c];
            }
          }
        }
        named_bar_sync(1, 128);
      }
      // next tile starts inside the document of this tile's last token (or the next one)
      {
        const int last = hdr->tok_doc[127];
        if (last >= 0) d_lo = last;
      }
      named_bar_sync(1, 128);
    }
    if (ew == 0) {
      for (int cc = 0; cc < ncc; ++cc)
        if (cd[cc] >= 0) vl_emit(p, cc * 32 + (int)lane, cd[cc], cm[cc], ca[cc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace mxs
