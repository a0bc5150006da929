// Flash-MaxSim dense forward on CTA PAIRS (tcgen05 cta_group::2) -- the bf16 / fp16 fold of
// maxsim/forward.py:108-155 (_fold_pair; S2 masking, S3 strict-> / lowest index) with the fused
// S4 score (maxsim/forward.py:216), same contract and epilogue as fwd_ts.cuh.
//
// Why.  fwd_ts keeps a 512-row Q group resident in TMEM (256 columns) and has room for only two
// 128-column accumulator slots, so the MMA of Q block n + 2 waits for the drain of block n: the
// commit -> epilogue -> release -> re-issue round trip outlasts one 512-cycle block and costs ~8 %
// (MXS_DEBUG=2 vs 3 in DESIGN.md §5).  Here two SMs cooperate on every MMA (M = 256 = 128 Q rows
// of each CTA, A read from each CTA's own TMEM), so a CTA keeps only two Q blocks resident
// (128 columns) and the freed TMEM holds a THIRD accumulator slot: two blocks of MMA work (1024
// cycles) stay queued behind every drain.  Each CTA holds only its half of the document tile
// (N = 128 split 64 / 64, the pair's MMA reads both halves), so the L2 -> SM traffic per MMA
// cycle is unchanged.
//
// Layouts (leader = even cluster rank of each pair):
//   * QB = 2, CL = 2 (256 < L_q <= 512): CTA r holds Q blocks 2r, 2r + 1 in TMEM (TS MMAs);
//   * QB = 4, CL = 2 (512 < L_q <= 1024): CTA r holds Q blocks 4r .. 4r + 3 -- blocks 0, 1 in
//     TMEM (TS) and blocks 2, 3 in shared memory (SS, loaded by TMA), because four TMEM-resident
//     blocks would leave room for two slots only.  (Two pairs per 4-CTA cluster with two TMEM
//     blocks each also works, but clusters of 4 tile only 132 of the 148 SMs.)
// Per pair:
//   * TMA (both CTAs): tokens [64 h, 64 h + 64) of every 128-token tile (and the CTA's SS Q
//     blocks) into the CTA's own shared memory, completing on the LEADER's barrier (cta_group::2
//     form); the leader posts the pair's expected bytes.  Stage reuse: each CTA waits on its own
//     empty barrier, which the leader's MMA commit arrives on in both CTAs (multicast).
//   * MMA (leader only): per tile, blocks 0 .. QB - 1 into slot n % 3 (n = accumulator number);
//     tfull[slot] in both CTAs via a multicast commit; tempty[slot] lives in the leader and counts
//     the four draining warps of each CTA (remote arrive from the follower).
//   * epilogue (both CTAs): warp set j drains blocks j, j + 2 of every tile from slot n % 3 of its
//     own TMEM, exactly like fwd_ts (register fold, argmax stash, CTA-local fused-score buffers).
#pragma once
#include "fwd_ts.cuh"

namespace mxs {

constexpr int kPrMaxSlots = 4;
#ifndef MXS_PAIR_ARGMAX_PIPE
#define MXS_PAIR_ARGMAX_PIPE 1  // software-pipelined argmax drain (C3 forward 0.767 -> 0.753 ms)
#endif
#ifndef MXS_PAIR_RERANK_PIPE
#define MXS_PAIR_RERANK_PIPE 1  // the same for the rerank drain (C2 1.626 -> 1.620 ms)
#endif
#ifndef MXS_PR_SCORE_BUFS
#define MXS_PR_SCORE_BUFS 2
#endif
constexpr int kPrScoreBufs = MXS_PR_SCORE_BUFS;  // fused-score row buffers (documents in flight)
// TMEM: NTS Q blocks x KA * 32 columns (<= 128), then the accumulator slots (4 when no Q block is
// TMEM-resident, else 3) of 128 columns
__host__ __device__ constexpr int pr_slots(int nts) { return nts == 0 ? 4 : 3; }
constexpr int kPrHalfAtom = 64 * 128;  // one 64-row x 128-byte SW128 atom (half a document tile)

struct PrSmemHeader {
  uint64_t full[8];
  uint64_t empty[8];
  uint64_t tfull[kPrMaxSlots];
  uint64_t tempty[kPrMaxSlots];
  uint64_t qfull;
  uint64_t qsfull;  // QB = 4: the SS Q blocks of both CTAs have landed (leader)
  uint64_t qempty;
  uint64_t sready[kPrScoreBufs];
  uint64_t sfree[kPrScoreBufs];
  uint64_t speer[kPrScoreBufs];
  uint64_t sdone[kPrScoreBufs];
  uint32_t tmem_base;
  uint32_t pad;
};

// dynamic smem: SS Q blocks (QB = 4: 2 blocks x KA atoms of 128 rows x 128 B) | document
// half-tile ring | argmax stash (QB blocks x 128 rows x kStashPadStride floats) | fused-score row buffers
__host__ __device__ inline size_t fwd_pair_smem_bytes(int ka, int qb, int nts, int stages, bool stash, int sum_rows) {
  return 1024 + (size_t)(qb - nts) * ka * kAtomBytes + (size_t)stages * ka * kPrHalfAtom +
         (stash ? (size_t)qb * 128 * kStashPadStride * sizeof(float) : 0) + (size_t)kPrScoreBufs * sum_rows * sizeof(float) +
         (sum_rows ? (size_t)kPrScoreBufs * 4 * kPartialsPerRank * sizeof(ScorePartial) : 0);
}

MXS_DEV void tmem_alloc_pair(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
MXS_DEV void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
// D[tmem, both CTAs] (+)= A[tmem, both CTAs] * B[smem halves of both CTAs]^T, M = 256.
MXS_DEV void mma_f16_ts_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
MXS_DEV void mma_f16_ss_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// Completion of this thread's prior pair MMAs arrives once on the barrier at the same offset in
// every CTA of cta_mask.
MXS_DEV void mma_commit_pair_mc(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}
// TMA 2-D load into this CTA's shared memory whose transaction bytes complete on the barrier at
// cluster address `bar_cluster` (the pair leader's).
MXS_DEV void tma_load_2d_pair(const void* tmap, uint32_t bar_cluster, void* smem_dst, int32_t c0, int32_t c1,
                              uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_cluster), "r"(c0), "r"(c1), "l"(cache_hint)
      : "memory");
}

template <TcKind KIND, int KA, int CL, int QB, int NTS>
__global__ void __launch_bounds__(kTsThreads, 1)
    fwd_pair_kernel(const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmQ,
                    const FwdTcParams p) {
  static_assert(KIND != TcKind::I8 && (CL == 2 || CL == 4) && KA >= 1 && KA <= 2, "bf16 / fp16, d <= 128");
  static_assert(QB == 2 || (QB == 4 && CL == 2), "QB = 4 (SS blocks) with single-pair clusters");
  static_assert(NTS == 2 || (NTS == 0 && QB == 4), "TMEM-resident Q blocks: 2, or 0 (all SS)");
  constexpr int kSlots = pr_slots(NTS);
  constexpr int kAccCol0 = NTS * KA * 32;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;  // QB = 4: SS Q blocks 2, 3
  uint8_t* sD = sQ + (size_t)(QB - NTS) * KA * kAtomBytes;
  float* sBest = reinterpret_cast<float*>(sD + (size_t)p.stages * KA * kPrHalfAtom);
  float* sSum = sBest + (p.argmax ? (size_t)QB * 128 * kStashPadStride : 0);
  ScorePartial* sPart = reinterpret_cast<ScorePartial*>(sSum + (size_t)kPrScoreBufs * p.sum_rows);
  const bool fuse = p.scores != nullptr && p.debug != 3;
  __shared__ PrSmemHeader pr_hdr;
  PrSmemHeader* hdr = &pr_hdr;

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const int crank = (int)cluster_ctarank();
  const int half = crank & 1;
  const uint32_t leader = (uint32_t)(crank & ~1);
  const uint16_t pair_mask = (uint16_t)(3u << leader);
  constexpr int kQCols = KA * 32;

  const long long n_workers = gridDim.x / CL;
  const long long worker = blockIdx.x / CL;
  const long long per = p.n_units / n_workers, rem = p.n_units % n_workers;
  const long long u_begin = worker * per + min(worker, rem);
  const long long u_end = u_begin + per + (worker < rem ? 1 : 0);
  auto decode = [&](long long u, int& q, int& g, int& b) {
    b = (int)(u % p.n_docs);
    q = (int)(u / p.n_docs);
    g = crank;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmD);
    if constexpr (QB == 4) tma_prefetch_desc(&tmQ);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&hdr->full[s], 1);   // leader: its producer's expect_tx arrive (+ both CTAs' bytes)
      mbar_init(&hdr->empty[s], 1);  // the leader's multicast commit
    }
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&hdr->tfull[s], 1);
      mbar_init(&hdr->tempty[s], 8);  // leader: 4 draining warps of each CTA of the pair
    }
    mbar_init(&hdr->qfull, 2 * kEpiWarps);  // leader: every epilogue warp of the pair
    mbar_init(&hdr->qsfull, 1);             // leader: its TMA warp's expect_tx arrive
    mbar_init(&hdr->qempty, 1);
    for (int s = 0; s < kPrScoreBufs; ++s) {
      mbar_init(&hdr->sready[s], 32 * kEpiWarps);
      mbar_init(&hdr->sfree[s], 1);
      mbar_init(&hdr->speer[s], 1);  // rank 0's expect_tx arrive + the other ranks' bulk-copy bytes
      mbar_init(&hdr->sdone[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair(&hdr->tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = hdr->tmem_base;
  constexpr uint32_t kIdesc = (KIND == TcKind::BF16) ? make_idesc(1, 1, 256, 128) : make_idesc(1, 0, 256, 128);
  constexpr int kElemsPerAtom = 64;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0, qeph = 0;
      long long cur_key = -1;
      for (long long u = u_begin; u < u_end; ++u) {
        int q, g, b;
        decode(u, q, g, b);
        if constexpr (QB == 4) {
          if ((long long)q != cur_key) {  // this CTA's SS Q blocks 2, 3 -> shared memory
            if (cur_key >= 0) {
              mbar_wait_idle(&hdr->qempty, qeph);  // every MMA reading the old blocks has completed
              qeph ^= 1;
            }
            if (half == 0) mbar_arrive_expect_tx(&hdr->qsfull, (uint32_t)(2 * (QB - NTS) * KA * kAtomBytes));
            const uint32_t qbar = mapa_u32(smem_u32(&hdr->qsfull), leader);
#pragma unroll
            for (int j = 0; j < QB - NTS; ++j)
#pragma unroll
              for (int a = 0; a < KA; ++a)
                tma_load_2d_pair(&tmQ, qbar, sQ + (size_t)(j * KA + a) * kAtomBytes, a * 64,
                                 q * p.l_q + (g * QB + NTS + j) * kTileRows, kEvictLast);
            cur_key = q;
          }
        }
        const int vl = doc_valid_len(p, b);
        const int ntiles = (vl + kTileRows - 1) / kTileRows;
        for (int t = 0; t < ntiles; ++t) {
          mbar_wait_idle(&hdr->empty[stage], phase ^ 1);
          if (half == 0) mbar_arrive_expect_tx(&hdr->full[stage], (uint32_t)(2 * KA * kPrHalfAtom));
          const uint32_t fbar = mapa_u32(smem_u32(&hdr->full[stage]), leader);
          const int row0 = b * p.l_pad + t * kTileRows + half * 64;
#pragma unroll
          for (int a = 0; a < KA; ++a)
            tma_load_2d_pair(&tmD, fbar, sD + (size_t)(stage * KA + a) * kPrHalfAtom, a * kElemsPerAtom, row0,
                             kEvictFirst);
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (pair leader)
    if (half == 0) {
      int stage = 0;
      uint32_t phase = 0, qphase = 0, nacc = 0;
      long long cur_key = -1;
      const uint64_t ddesc0 = sw128_kmajor_desc(smem_u32(sD));
      const uint64_t qdesc0 = sw128_kmajor_desc(smem_u32(sQ));
      for (long long u = u_begin; u < u_end; ++u) {
        int q, g, b;
        decode(u, q, g, b);
        const long long key = q;
        if (key != cur_key) {
          if (cur_key >= 0) {
            if (elect_one()) mma_commit_pair_mc(&hdr->qempty, pair_mask);
            __syncwarp();
          }
          mbar_wait(&hdr->qfull, qphase);  // both CTAs' Q blocks are in TMEM
          if constexpr (QB == 4) mbar_wait(&hdr->qsfull, qphase);  // and their SS blocks in smem
          qphase ^= 1;
          tc_fence_after();
          cur_key = key;
        }
        const int vl = doc_valid_len(p, b);
        const int ntiles = (vl + kTileRows - 1) / kTileRows;
        for (int t = 0; t < ntiles; ++t) {
          mbar_wait(&hdr->full[stage], phase);
          tc_fence_after();
          const uint64_t bd0 = ddesc0 + (uint64_t)((stage * KA * kPrHalfAtom) >> 4);
#pragma unroll
          for (int mb = 0; mb < QB; ++mb, ++nacc) {
            const uint32_t slot = nacc % kSlots, use = nacc / kSlots;
            // MXS_DEBUG=3: never wait for the drain (raw MMA + TMA rate; results garbage)
            if (p.debug != 3) {
              if (p.mma_spin)
                mbar_wait(&hdr->tempty[slot], (use & 1u) ^ 1u);
              else
                mbar_wait_idle(&hdr->tempty[slot], (use & 1u) ^ 1u);
            }
            tc_fence_after();
            if (elect_one()) {
              const uint32_t acol = tmem_base + (uint32_t)(mb * kQCols);
              const uint32_t dcol = tmem_base + (uint32_t)(kAccCol0 + slot * 128);
#pragma unroll
              for (int k = 0; k < KA * 4; ++k) {
                const uint64_t koff = (uint64_t)(((k >> 2) * kPrHalfAtom + (k & 3) * 32) >> 4);
                if (mb < NTS) {
                  mma_f16_ts_pair(dcol, acol + k * 8, bd0 + koff, kIdesc, k > 0 ? 1u : 0u);
                } else {
                  const uint64_t qoff = (uint64_t)((((mb - NTS) * KA + (k >> 2)) * kAtomBytes + (k & 3) * 32) >> 4);
                  mma_f16_ss_pair(dcol, qdesc0 + qoff, bd0 + koff, kIdesc, k > 0 ? 1u : 0u);
                }
              }
              mma_commit_pair_mc(&hdr->tfull[slot], pair_mask);
            }
            __syncwarp();
          }
          if (elect_one()) mma_commit_pair_mc(&hdr->empty[stage], pair_mask);
          __syncwarp();
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (p.debug == 3) {  // nobody drained: wait for the last MMAs before TMEM is freed
        if (elect_one()) mma_commit_pair_mc(&hdr->qempty, pair_mask);
        __syncwarp();
        mbar_wait(&hdr->qempty, qphase ^ 1u);
      }
    }
  } else if (warp == kTsSumWarp) {
    // ------------------------------------------------------------------ fused S4 score
    // profiling knob MXS_DEBUG=6: no score warp and no hand-off (scores invalid)
    if (fuse && p.debug != 6 && p.debug < 8) fused_score_warp<CL, kPrScoreBufs, true>(p, hdr->sready, hdr->sfree, hdr->speer, hdr->sdone, sSum, u_begin, u_end, decode,
                                   crank, lane, sPart);
  } else {
    // ------------------------------------------------------------------ epilogue (+ Q -> TMEM)
    // warp w in [2, 10): TMEM lane quadrant w % 4, set j = (w - 2) / 4 owns Q blocks j (TMEM) and
    // j + 2 (QB = 4, shared memory); it writes block j into TMEM and drains both.
    constexpr int kNB = QB / 2;  // blocks per set
    const int wset = ((int)warp - kTsEpiWarp0) >> 2;
    const int quad = (int)(warp & 3);
    const int row_local = quad * 32 + (int)lane;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    constexpr int swz = -1;  // padded argmax stash (see stash_chunk)
    const int row_bytes = p.dim * 2;
    const uint32_t qfull_leader = mapa_u32(smem_u32(&hdr->qfull), leader);
    uint32_t qeph = 0, ndoc = 0, nt = 0;  // nt: tiles drained so far (accumulator n = QB nt + mb)
    long long cur_key = -1;
    // At the end of a document each warp folds its rows into an integer fixed-point partial
    // (store_score_partial; deferring it past the next document's first slot release measured the
    // same) and arrives; the score warp combines the partials.
    int pend_sb = -1;  // row buffer of the document whose partial is pending, -1: none
    auto flush_partial = [&]() {
      if (pend_sb >= 0) {
        if (p.debug != 8 && p.debug != 9) {  // profiling knobs (scores invalid): 8 = no partial, no fence; 9 = no partial
          float pm[kNB];  // this thread's row maxima, back from the row buffer (no registers held across the drain)
          bool pv[kNB];
#pragma unroll
          for (int i = 0; i < kNB; ++i) {
            const int row = (crank * QB + wset + 2 * i) * kTileRows + row_local;
            pv[i] = row < p.l_q;
            pm[i] = pv[i] ? sSum[pend_sb * p.sum_rows + row] : 0.f;
          }
          store_score_partial<kNB>(pm, pv, sPart + (pend_sb * CL + crank) * kPartialsPerRank + ((int)warp - kTsEpiWarp0),
                                   lane, p.l_q);
        }
        if (p.debug != 8) fence_proxy_async();  // rows + partial travel to cluster rank 0 by bulk (async-proxy) copy
        if (p.debug != 6 && p.debug < 8) mbar_arrive(&hdr->sready[pend_sb]);  // every lane (release of its stores)
        pend_sb = -1;
      }
    };
    for (long long u = u_begin; u < u_end; ++u) {
      int q, g, b;
      decode(u, q, g, b);
      if ((long long)q != cur_key) {
        if (cur_key >= 0) {
          mbar_wait(&hdr->qempty, qeph);  // every MMA reading the old Q block has completed
          qeph ^= 1;
        }
        const int row = (g * QB + wset) * kTileRows + row_local;
        const uint8_t* src = static_cast<const uint8_t*>(p.q_ptr) + ((long long)q * p.l_q + row) * row_bytes;
#pragma unroll
        for (int a = 0; a < KA; ++a) {
          uint32_t r[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int off = a * 128 + c * 16;
            uint4 w = make_uint4(0u, 0u, 0u, 0u);
            if (row < p.l_q && off < row_bytes) w = __ldg(reinterpret_cast<const uint4*>(src + off));
            r[4 * c] = w.x;
            r[4 * c + 1] = w.y;
            r[4 * c + 2] = w.z;
            r[4 * c + 3] = w.w;
          }
          if constexpr (NTS > 0) tmem_st32(tmem_base + lane_base + (uint32_t)(wset * kQCols + a * 32), r);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(qfull_leader);
        cur_key = q;
      }
      const int vl = doc_valid_len(p, b);
      const int ntiles = (vl + kTileRows - 1) / kTileRows;
      if (p.debug == 3) {  // no drain (see the MMA issuer)
        nt += ntiles;
        continue;
      }
      float m[kNB];
      int cb[kNB];
#pragma unroll
      for (int i = 0; i < kNB; ++i) {
        m[i] = -INFINITY;
        cb[i] = 0;
      }
      for (int t = 0; t < ntiles; ++t, ++nt) {
        const int base = t * kTileRows;
#pragma unroll
        for (int i = 0; i < kNB; ++i) {
          const int mb = wset + 2 * i;
          const uint32_t n = (uint32_t)QB * nt + (uint32_t)mb;
          const uint32_t slot = n % kSlots;
          mbar_wait(&hdr->tfull[slot], (n / kSlots) & 1u);
          tc_fence_after();
          const uint32_t taddr = tmem_base + lane_base + (uint32_t)(kAccCol0 + slot * 128);
          const uint32_t tempty_leader = mapa_u32(smem_u32(&hdr->tempty[slot]), leader);
          if (p.debug == 2) {  // profiling knob: release the slot unread (finite maxima for the fused sum)
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty_leader);
            m[i] = 0.f;
            continue;
          }
          float* stash = p.argmax ? sBest + ((size_t)mb * 128 + row_local) * kStashPadStride : nullptr;
          uint32_t ra[32], rb[32], rc[32], rd[32];
#if MXS_PAIR_ARGMAX_PIPE
          if (stash && base + kTileRows <= vl) {
            // argmax drain, software-pipelined: chunks 2-3 load while chunks 0-1 are folded; the
            // slot is released once they have landed
            tmem_ld32(taddr, ra);
            tmem_ld32(taddr + 32, rb);
            tmem_ld_wait_regs(ra);
            tmem_ld_wait_regs(rb);
            tmem_ld32(taddr + 64, rc);
            tmem_ld32(taddr + 96, rd);
            ts_chunk_full<KIND, true>(ra, base, 1.f, m[i], cb[i], stash, swz, nullptr);
            ts_chunk_full<KIND, true>(rb, base + 32, 1.f, m[i], cb[i], stash, swz, nullptr);
            tmem_ld_wait_regs(rc);
            tmem_ld_wait_regs(rd);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty_leader);
            ts_chunk_full<KIND, true>(rc, base + 64, 1.f, m[i], cb[i], stash, swz, nullptr);
            ts_chunk_full<KIND, true>(rd, base + 96, 1.f, m[i], cb[i], stash, swz, nullptr);
            continue;
          }
#endif
#if MXS_PAIR_RERANK_PIPE
          if (!stash && base + kTileRows <= vl) {
            tmem_ld32(taddr, ra);
            tmem_ld32(taddr + 32, rb);
            tmem_ld_wait_regs(ra);
            tmem_ld_wait_regs(rb);
            tmem_ld32(taddr + 64, rc);
            tmem_ld32(taddr + 96, rd);
            ts_chunk_full<KIND, false>(ra, base, 1.f, m[i], cb[i], nullptr, swz, nullptr);
            ts_chunk_full<KIND, false>(rb, base + 32, 1.f, m[i], cb[i], nullptr, swz, nullptr);
            tmem_ld_wait_regs(rc);
            tmem_ld_wait_regs(rd);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty_leader);
            ts_chunk_full<KIND, false>(rc, base + 64, 1.f, m[i], cb[i], nullptr, swz, nullptr);
            ts_chunk_full<KIND, false>(rd, base + 96, 1.f, m[i], cb[i], nullptr, swz, nullptr);
            continue;
          }
#endif
          tmem_ld32(taddr, ra);
          tmem_ld32(taddr + 32, rb);
          tmem_ld32(taddr + 64, rc);
          tmem_ld32(taddr + 96, rd);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(tempty_leader);
          if (base + kTileRows <= vl) {
            if (stash) {
              ts_chunk_full<KIND, true>(ra, base, 1.f, m[i], cb[i], stash, swz, nullptr);
              ts_chunk_full<KIND, true>(rb, base + 32, 1.f, m[i], cb[i], stash, swz, nullptr);
              ts_chunk_full<KIND, true>(rc, base + 64, 1.f, m[i], cb[i], stash, swz, nullptr);
              ts_chunk_full<KIND, true>(rd, base + 96, 1.f, m[i], cb[i], stash, swz, nullptr);
            } else {
              ts_chunk_full<KIND, false>(ra, base, 1.f, m[i], cb[i], nullptr, swz, nullptr);
              ts_chunk_full<KIND, false>(rb, base + 32, 1.f, m[i], cb[i], nullptr, swz, nullptr);
              ts_chunk_full<KIND, false>(rc, base + 64, 1.f, m[i], cb[i], nullptr, swz, nullptr);
              ts_chunk_full<KIND, false>(rd, base + 96, 1.f, m[i], cb[i], nullptr, swz, nullptr);
            }
          } else {
            ts_chunk<KIND>(ra, base, vl, p, b, 1.f, m[i], cb[i], stash, swz);
            ts_chunk<KIND>(rb, base + 32, vl, p, b, 1.f, m[i], cb[i], stash, swz);
            ts_chunk<KIND>(rc, base + 64, vl, p, b, 1.f, m[i], cb[i], stash, swz);
            ts_chunk<KIND>(rd, base + 96, vl, p, b, 1.f, m[i], cb[i], stash, swz);
          }
        }
      }
      if (fuse) {  // row maxima -> this CTA's row buffer, then every lane arrives (CTA scope)
        const uint32_t sb = ndoc % kPrScoreBufs;
        // profiling knob MXS_DEBUG=6: no hand-off at all (scores invalid)
        if (p.debug != 6 && p.debug < 8) mbar_wait(&hdr->sfree[sb], ((ndoc / kPrScoreBufs) & 1u) ^ 1u);
#pragma unroll
        for (int i = 0; i < kNB; ++i) {
          const int row = (g * QB + wset + 2 * i) * kTileRows + row_local;
          if (row < p.l_q) sSum[sb * p.sum_rows + row] = m[i];
        }
        pend_sb = (int)sb;
        flush_partial();  // this warp's fixed-point partial, then the rows + partial are ready for the score warp
        ++ndoc;
      }
#pragma unroll
      for (int i = 0; i < kNB; ++i) {
        const int mb = wset + 2 * i;
        const int row = (g * QB + mb) * kTileRows + row_local;
        if (row < p.l_q) {
          const long long o = ((long long)q * p.n_docs + b) * p.l_q + row;
          if (p.rowmax) p.rowmax[o] = m[i];
          if (p.argmax) {
            float w[32];
            unstash_chunk(sBest + ((size_t)mb * 128 + row_local) * kStashPadStride, w, swz);
            p.argmax[o] = ntiles ? cb[i] + first_argmax32_chain(w, m[i]) : 0;  // 0: empty (invalid) doc
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

}  // namespace mxs
