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

constexpr int kVlSets = 2;                            // epilogue warp sets, alternate tiles
constexpr int kVlEpiWarps = 4 * kVlSets;
constexpr int kVlThreads = 32 * (2 + kVlEpiWarps);  // warp 0 TMA, warp 1 MMA + TMEM alloc, 2..9 epilogue
constexpr int kVlTilePad = 36;                        // floats per token row (16-B rows, conflict-free STS.128)

struct VlSmemHeader {
  uint64_t full[8];
  uint64_t empty[8];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint64_t qfull;
  uint64_t carry_ready;  // phase t completes when the ordered merge of tile t is done
  uint32_t tmem_base;
  int32_t doc_begin, doc_end;
  int32_t pad;
  long long tok_begin, tok_end;
};

// Epilogue scratch in dynamic shared memory, one per warp set (set s owns tiles t = s mod 2).
constexpr int kVlCuCache = 1280;  // cached cu_seqlens window (documents)
struct VlPieces {
  float hm[4][32];
  float tm[4][32];
  int32_t hd[4][32];
  int32_t td[4][32];
  long long ha[4][32];
  long long ta[4][32];
};
struct VlSetScratch {
  float tile[128 * kVlTilePad];   // transposed similarities of one 32-column chunk
  int32_t tok_doc[128];           // document of every token of the tile
  VlPieces pieces[4];             // per column chunk
  long long cu_cache[kVlCuCache]; // cu[c0 + j]
};
struct VlCarry {                   // ordered-merge state handed from set to set
  float m[4][32];
  long long a[4][32];
  long long d[4][32];
};
struct VlScratch {
  VlSetScratch set[kVlSets];
  VlCarry carry;
};

// dynamic shared memory (the small header is static shared memory)
__host__ __device__ inline size_t varlen_smem_bytes(int ka, int stages, int n_cols_pad) {
  return 1024 + (size_t)stages * ka * kAtomBytes + (size_t)ka * n_cols_pad * 128 + sizeof(VlScratch);
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

// arg is already document-local
MXS_DEV void vl_emit(const VarlenParams& p, int col, long long doc, float m, long long arg) {
  if (doc < 0 || col >= p.n_cols) return;
  const int q = col / p.l_q, i = col % p.l_q;
  const long long o = ((long long)q * p.n_docs + doc) * p.l_q + i;
  p.rowmax[o] = m;
  if (p.argmax) p.argmax[o] = (int32_t)arg;
}

template <TcKind KIND, int KA>
__global__ void __launch_bounds__(kVlThreads, 1)
    varlen_tc_kernel(const __grid_constant__ CUtensorMap tmT, const __grid_constant__ CUtensorMap tmQ,
                     const VarlenParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment by offsetting the __shared__ array itself (keeps the shared address space,
  // so accesses compile to LDS/STS rather than generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sT = smem;                                           // token tiles
  uint8_t* sQ = sT + (size_t)p.stages * KA * kAtomBytes;        // all query rows (B operand)
  __shared__ VlSmemHeader vl_hdr;  // static shared: keeps every access on the LDS/STS path
  VlSmemHeader* hdr = &vl_hdr;
  VlScratch* scr = reinterpret_cast<VlScratch*>(sQ + (size_t)KA * p.n_cols_pad * 128);
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
      mbar_init(&hdr->tempty[s], 4);  // the four warps of the set owning the slot
    }
    mbar_init(&hdr->qfull, 1);
    mbar_init(&hdr->carry_ready, 1);
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
    const int set = ((int)warp - 2) >> 2;        // warp set: tiles t with t % 2 == set, TMEM slot set
    const int ew = ((int)warp - 2) & 3;          // token quarter of the scan
    const int quad = (int)(warp & 3);            // TMEM lane quadrant of this warp
    const int tid = ew * 32 + (int)lane;          // 0..127 within the set
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const int my_tok = quad * 32 + (int)lane;    // token (TMEM lane) this thread loads
    const long long doc_end = hdr->doc_end;
    const uint32_t bar_id = 1u + (uint32_t)set;  // named barrier of this set (128 threads)
    VlSetScratch& S = scr->set[set];
    VlCarry& C = scr->carry;
    if (set == 0 && ew == 0) {
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        C.m[cc][lane] = -INFINITY;
        C.a[cc][lane] = 0;
        C.d[cc][lane] = -1;
      }
    }
    long long lb = hdr->doc_begin;  // lower bound: document of a token at or before this tile
    long long c0 = -(1LL << 40);    // first document held by this set's cu cache
    for (int t = set; t < n_tiles; t += kVlSets) {
      const long long p0 = tok_begin + (long long)t * 128;
      // ---- cu cache refill (uniform within the set; one global round trip per ~1000 docs)
      if (lb + 260 > c0 + kVlCuCache) {
        c0 = lb;
        for (int j = tid; j < kVlCuCache; j += 128) {
          const long long d = c0 + j;
          S.cu_cache[j] = (d <= p.n_docs) ? __ldg(p.cu + d) : LLONG_MAX;
        }
        named_bar_sync(bar_id, 128);
      }
      // ---- document of this thread's token: binary search of the cached window (no barrier).
      // At most 257 documents start between the last token of tile t-2 and the end of tile t.
      {
        const long long tok = p0 + tid;
        int dsel = -1;
        if (tok < tok_end) {
          long long lo = lb, hi = min(lb + 258, doc_end);  // answer in [lo, hi)
          while (hi - lo > 1) {
            const long long mid = (lo + hi) >> 1;
            if (S.cu_cache[mid - c0] <= tok)
              lo = mid;
            else
              hi = mid;
          }
          dsel = (int)lo;
        }
        S.tok_doc[tid] = dsel;
      }
      int last_doc = -1;
      const int slot = set;
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
        float4* trow = reinterpret_cast<float4*>(S.tile + my_tok * kVlTilePad);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          trow[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
        named_bar_sync(bar_id, 128);  // (A) transpose tile + token documents visible
        // read now: after the last barrier of this tile a fast warp may already be rewriting
        // tok_doc for this set's next tile
        if (cc == 0) last_doc = S.tok_doc[127];
        // ---- scan: column c = lane over the 32 tokens of quarter ew, in order
        const int c = (int)lane;
        VlPieces& pc = S.pieces[cc];
        const float* tile = S.tile;
        const int d_first = S.tok_doc[ew * 32], d_last = S.tok_doc[ew * 32 + 31];
        if (d_first == d_last) {
          // fast path (same for all lanes): the quarter lies inside one document -> one piece,
          // branch-free strict-> fold in token order
          float m = -INFINITY;
          int kbest = 0;
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const float v = tile[(ew * 32 + k) * kVlTilePad + c];
            const bool up = v > m;
            m = up ? v : m;
            kbest = up ? k : kbest;
          }
          pc.hm[ew][c] = m;
          pc.ha[ew][c] = (d_first >= 0) ? p0 + ew * 32 + kbest - S.cu_cache[d_first - c0] : 0;
          pc.hd[ew][c] = d_first;
          pc.td[ew][c] = -3;  // marker: no separate tail
        } else {
          float m = -INFINITY;
          long long a = 0;
          int cur = -2;
          bool head_done = false;
          for (int k = 0; k < 32; ++k) {
            const int tau = ew * 32 + k;
            const int d = S.tok_doc[tau];
            const float v = tile[tau * kVlTilePad + c];
            if (d != cur) {
              if (cur != -2) {
                const long long al = (cur >= 0) ? a - S.cu_cache[cur - c0] : 0;
                if (!head_done) {
                  pc.hm[ew][c] = m;
                  pc.ha[ew][c] = al;
                  pc.hd[ew][c] = cur;
                  head_done = true;
                } else if (cur >= 0) {
                  vl_emit(p, cc * 32 + c, cur, m, al);  // document complete inside this quarter
                }
              }
              cur = d;
              m = -INFINITY;
              a = 0;
            }
            if (v > m) {  // strict: the earliest token wins ties
              m = v;
              a = p0 + tau;
            }
          }
          const long long al_last = (cur >= 0) ? a - S.cu_cache[cur - c0] : 0;
          pc.tm[ew][c] = m;  // head_done is always true here (the document changed)
          pc.ta[ew][c] = al_last;
          pc.td[ew][c] = cur;
        }
        named_bar_sync(bar_id, 128);  // (B) pieces of every quarter visible; tile buffer free
        // ---- ordered merge (first warp of the set), after the merge of tile t - 1
        if (ew == 0) {
          if (t > 0) mbar_wait(&hdr->carry_ready, (uint32_t)(t - 1) & 1u);
          float cm = C.m[cc][c];
          long long ca = C.a[cc][c], cd = C.d[cc][c];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int hd = pc.hd[h][c];
            const float hmv = pc.hm[h][c];
            const long long hav = pc.ha[h][c];
            if (hd == cd) {
              if (hmv > cm) {  // the carry holds earlier tokens: strict > keeps it on ties
                cm = hmv;
                ca = hav;
              }
            } else {
              if (cd >= 0) vl_emit(p, cc * 32 + c, cd, cm, ca);
              cd = hd;
              cm = hmv;
              ca = hav;
            }
            const int tdv = pc.td[h][c];
            if (tdv != -3) {  // a document ended inside quarter h; its tail starts the new carry
              if (cd >= 0) vl_emit(p, cc * 32 + c, cd, cm, ca);
              cd = tdv;
              cm = pc.tm[h][c];
              ca = pc.ta[h][c];
            }
          }
          C.m[cc][c] = cm;
          C.a[cc][c] = ca;
          C.d[cc][c] = cd;
          if (cc == ncc - 1) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&hdr->carry_ready);  // phase t: merge of tile t done
          }
        }
      }
      // this set's next tile starts at or after the document of this tile's last token
      if (last_doc >= 0) lb = last_doc;
    }
    // the merge of the last tile flushes the carry
    if (ew == 0 && n_tiles > 0 && set == ((n_tiles - 1) & 1)) {
      for (int cc = 0; cc < ncc; ++cc)
        if (C.d[cc][lane] >= 0) vl_emit(p, cc * 32 + (int)lane, C.d[cc][lane], C.m[cc][lane], C.a[cc][lane]);
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
