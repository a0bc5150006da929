// Forward in RERANK mode (argmax not requested): scores only -- maxsim/forward.py:108-155 and
// maxsim/quant.py:128-182 with the per-token maxima reduced to the f64 score, no index tracking.
//
// Three accumulator slots instead of two.  With two, the MMA of Q block n + 2 waits until the
// accumulator of block n has been committed, drained and released -- a handshake that outlasts
// the 512-cycle MMA of block n + 1 (measured: the bf16 forward ran at ~70 % of the raw TS-MMA rate
// with the epilogue disabled).  With three, two blocks of work are always queued.  TMEM holds
// 128 columns of resident Q (4 INT8 blocks, or 2 bf16/fp16 blocks -- bf16 then uses 4-CTA
// clusters) plus 3 x 128 accumulator columns.  THREE epilogue warp sets also give the
// issue-bound INT8 epilogue (the reference's dequantise-before-max, S7, ~3 issued instructions
// per similarity) more warps.  Without argmax tracking the running row maximum is order-free
// (max is exact and commutative), which is what makes the split legal:
//   * the MMA issuer numbers every (tile, Q block) accumulator it produces, n = 0, 1, 2, ...;
//     accumulator n lands in TMEM slot n % 3 and is drained by epilogue set n % 3, so each set
//     consumes its own slot in order (no mbarrier phase aliasing);
//   * each set keeps, per Q block, a partial maximum over the tiles it happened to drain; at the
//     end of a document the three partials of every row are max-combined through shared memory
//     (double-buffered by document parity) and written once;
//   * fused S4 score: the combiner of each quadrant stores the combined maxima straight into
//     cluster rank 0's row buffer (DSMEM) and arrives there; rank 0's score warp folds them.
//     (Unlike fwd_ts, only 4 combiner warps per CTA and document pay the cluster-scope
//     release; the CTA-local variant with per-rank score warps made ptxas spill in this
//     register-capped kernel.)
// Everything else (TS MMA with Q resident in TMEM, cluster multicast of document tiles,
// TMA-staged INT8 scales, magic-number s32 -> f32) is fwd_ts.cuh's.
#pragma once
#include "fwd_ts.cuh"

namespace mxs {

constexpr int kR8Sets = 3;
constexpr int kR8EpiWarps = 4 * kR8Sets;
constexpr int kR8SumWarp = 2 + kR8EpiWarps;          // warp 14: fused S4 score (as in fwd_ts.cuh)
constexpr int kR8Threads = 32 * (kR8SumWarp + 1);  // warp 0 TMA, warp 1 MMA + TMEM, 2..13 epilogue
constexpr int kR8AccCol0 = 128;

constexpr int kR8PartBufs = 4;  // per-document partial-maximum buffers in flight

struct R8SmemHeader {
  uint32_t pcnt[kR8PartBufs][4];  // sets (warps) of a quadrant that have published doc partials
  uint64_t pdone[kR8PartBufs][4];  // all lanes of the three set warps of a quadrant published
  uint64_t pfree[kR8PartBufs][4];  // the combiner warp has read the buffer (it may be refilled)
  uint64_t full[8];
  uint64_t empty[8];
  uint64_t tfull[kR8Sets];
  uint64_t tempty[kR8Sets];
  uint64_t qfull;
  uint64_t qempty;
  uint64_t sfull[kScaleSlots];
  uint64_t sempty[kScaleSlots];
  uint64_t sready[2];  // fused score: the combiners of every CTA stored document n's maxima in rank 0's buffer [n & 1]
  uint64_t sfree[2];   // fused score: rank 0's score warp consumed buffer [n & 1]
  uint32_t tmem_base;
  uint32_t pad;
};

// dynamic smem: document tiles + per-document partial maxima [4 docs][3 sets][4 blocks][128 rows]
// + (INT8) the scale ring and the bias tile + the fused-score row buffers (2 x sum_rows floats)
__host__ __device__ inline size_t fwd_i8r_smem_bytes(int ka, int stages, bool i8, int sum_rows) {
  return 1024 + (size_t)stages * ka * kAtomBytes + (size_t)kR8PartBufs * kR8Sets * 4 * 128 * sizeof(float) +
         (i8 ? (size_t)kScaleSlots * kTileRows * sizeof(float) + kBiasTileBytes : 0) + (size_t)2 * sum_rows * sizeof(float);
}

template <TcKind KIND, int KA, int CL>
__global__ void __launch_bounds__(kR8Threads, 1)
    fwd_i8r_kernel(const __grid_constant__ CUtensorMap tmD, const FwdTcParams p) {
  static_assert(KA * 32 * (KIND == TcKind::I8 ? 4 : 2) <= 128, "resident Q must fit 128 TMEM columns");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sD = smem;
  float* sPart = reinterpret_cast<float*>(sD + (size_t)p.stages * KA * kAtomBytes);
  float* sScale = sPart + (size_t)kR8PartBufs * kR8Sets * 4 * 128;
  uint8_t* sBias = reinterpret_cast<uint8_t*>(sScale + kScaleSlots * kTileRows);  // 1024-B aligned
  float* sSum = (KIND == TcKind::I8) ? reinterpret_cast<float*>(sBias + kBiasTileBytes) : sScale;
  const bool fuse = p.scores != nullptr && !(KIND != TcKind::I8 && p.debug == 3);
  __shared__ R8SmemHeader r8_hdr;
  R8SmemHeader* hdr = &r8_hdr;

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const int crank = (CL > 1) ? (int)cluster_ctarank() : 0;
  constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1u);
  constexpr int kQCols = KA * 32;
  constexpr bool kI8 = KIND == TcKind::I8;
  constexpr int kElemsPerAtom = kI8 ? 128 : 64;

  const long long n_workers = gridDim.x / CL;
  const long long worker = blockIdx.x / CL;
  const long long per = p.n_units / n_workers, rem = p.n_units % n_workers;
  const long long u_begin = worker * per + min(worker, rem);
  const long long u_end = u_begin + per + (worker < rem ? 1 : 0);
  const int nmb_total = (p.l_q + kTileRows - 1) / kTileRows;
  auto decode = [&](long long u, int& q, int& g, int& b) {
    if (CL > 1) {
      b = (int)(u % p.n_docs);
      q = (int)(u / p.n_docs);
      g = crank;
    } else {
      decode_unit(u, p, q, g, b);
    }
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmD);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&hdr->full[s], 1);
      mbar_init(&hdr->empty[s], CL);
    }
    for (int s = 0; s < kR8Sets; ++s) {
      mbar_init(&hdr->tfull[s], 1);
      mbar_init(&hdr->tempty[s], 4);
    }
    mbar_init(&hdr->qfull, kR8EpiWarps);
    mbar_init(&hdr->qempty, 1);
    for (int s = 0; s < kScaleSlots; ++s) {
      mbar_init(&hdr->sfull[s], 1);
      mbar_init(&hdr->sempty[s], kR8EpiWarps);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&hdr->sready[s], 32 * 4 * CL);  // the four quadrant combiners of every CTA, all lanes
      mbar_init(&hdr->sfree[s], 1);
    }
    fence_mbar_init();
  }
  if (threadIdx.x < kR8PartBufs * 4) {
    (&hdr->pcnt[0][0])[threadIdx.x] = 0u;
    mbar_init(&hdr->pdone[0][0] + threadIdx.x, 32 * kR8Sets);
    mbar_init(&hdr->pfree[0][0] + threadIdx.x, 32);
  }
  if (threadIdx.x == 0) fence_mbar_init();
  if (warp == 1) tmem_alloc(&hdr->tmem_base, 512);
  if constexpr (KIND == TcKind::I8) {
    fill_bias_tile(sBias, (int)threadIdx.x, kR8Threads);
    fence_proxy_async();  // generic-proxy writes -> tensor-core (async proxy) reads
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = hdr->tmem_base;
  constexpr uint32_t kIdesc = kI8 ? make_idesc(2, 1, 128, 128)
                                  : (KIND == TcKind::BF16 ? make_idesc(1, 1, 128, 128) : make_idesc(1, 0, 128, 128));

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0, sc_n = 0;
      constexpr int kRowsPer = kTileRows / CL;
      for (long long u = u_begin; u < u_end; ++u) {
        int q, g, b;
        decode(u, q, g, b);
        const int vl = doc_valid_len(p, b);
        const int ntiles = (vl + kTileRows - 1) / kTileRows;
        for (int t = 0; t < ntiles; ++t) {
          if constexpr (kI8) {
            const int ss = (int)(sc_n % kScaleSlots);
            mbar_wait_idle(&hdr->sempty[ss], ((sc_n / kScaleSlots) & 1u) ^ 1u);
            const uint32_t bytes = (uint32_t)min(kTileRows, p.l_pad - t * kTileRows) * 4u;
            mbar_arrive_expect_tx(&hdr->sfull[ss], bytes);
            bulk_load_1d(&hdr->sfull[ss], sScale + ss * kTileRows,
                         p.d_scale + (long long)b * p.l_pad + t * kTileRows, bytes, kEvictFirst);
            ++sc_n;
          }
          mbar_wait_idle(&hdr->empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&hdr->full[stage], (uint32_t)(KA * kAtomBytes));
          const int row0 = b * p.l_pad + t * kTileRows + crank * kRowsPer;
#pragma unroll
          for (int a = 0; a < KA; ++a) {
            uint8_t* dst = sD + (size_t)(stage * KA + a) * kAtomBytes + crank * kRowsPer * 128;
            if (CL > 1)
              tma_load_2d_mc(&tmD, &hdr->full[stage], dst, a * kElemsPerAtom, row0, kMask, kEvictFirst);
            else
              tma_load_2d(&tmD, &hdr->full[stage], dst, a * kElemsPerAtom, row0, kEvictFirst);
          }
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (TS)
    int stage = 0;
    uint32_t phase = 0, qphase = 0;
    uint32_t nblk = 0;  // accumulators produced so far: slot = nblk % 3
    long long cur_key = -1;
    const uint64_t ddesc0 = sw128_kmajor_desc(smem_u32(sD));
    const uint64_t bias_desc = sw128_kmajor_desc(smem_u32(sBias));
    constexpr uint32_t kBiasIdesc = make_idesc(1, 1, 128, 128);  // f32 <- bf16 x bf16
    for (long long u = u_begin; u < u_end; ++u) {
      int q, g, b;
      decode(u, q, g, b);
      const long long key = (long long)q * p.n_groups + g;
      if (key != cur_key) {
        if (cur_key >= 0) {
          if (elect_one()) mma_commit(&hdr->qempty);
          __syncwarp();
        }
        mbar_wait_idle(&hdr->qfull, qphase);
        qphase ^= 1;
        tc_fence_after();
        cur_key = key;
      }
      const int qbv = min(p.qb, nmb_total - g * p.qb);
      const int vl = doc_valid_len(p, b);
      const int ntiles = (vl + kTileRows - 1) / kTileRows;
      for (int t = 0; t < ntiles; ++t) {
        mbar_wait_idle(&hdr->full[stage], phase);
        tc_fence_after();
        const uint64_t bd0 = ddesc0 + (uint64_t)((stage * KA * kAtomBytes) >> 4);
        for (int mb = 0; mb < qbv; ++mb, ++nblk) {
          const uint32_t slot = nblk % kR8Sets, use = nblk / kR8Sets;
          if (p.debug != 3) mbar_wait_idle(&hdr->tempty[slot], (use & 1u) ^ 1u);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t acol = tmem_base + (uint32_t)(mb * kQCols);
            const uint32_t dcol = tmem_base + (uint32_t)(kR8AccCol0 + slot * 128);
            if constexpr (kI8) mma_f16_ss(dcol, bias_desc, bias_desc, kBiasIdesc, 0u);  // TMEM = kMagicF
#pragma unroll
            for (int k = 0; k < KA * 4; ++k) {
              const uint64_t koff = (uint64_t)(((k >> 2) * kAtomBytes + (k & 3) * 32) >> 4);
              if constexpr (kI8)
                mma_i8_ts(dcol, acol + k * 8, bd0 + koff, kIdesc, 1u);
              else
                mma_f16_ts(dcol, acol + k * 8, bd0 + koff, kIdesc, k > 0 ? 1u : 0u);
            }
            if constexpr (kI8 && MXS_I8_TC_UNBIAS)  // TMEM = f32(acc) exactly (see i2f2_biased)
              mma_f16_ss(dcol, bias_desc, bias_desc, kBiasIdesc | kIdescNegA, 1u);
            mma_commit(&hdr->tfull[slot]);
          }
          __syncwarp();
        }
        if (elect_one()) {
          if (CL > 1)
            mma_commit_mc(&hdr->empty[stage], kMask);
          else
            mma_commit(&hdr->empty[stage]);
        }
        __syncwarp();
        if (++stage == p.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    if (p.debug == 3) {  // nobody drained: wait for the last MMAs before TMEM is freed
      if (elect_one()) mma_commit(&hdr->qempty);
      __syncwarp();
      mbar_wait(&hdr->qempty, qphase ^ 1u);
    }
  } else if (warp == kR8SumWarp) {
    // ------------------------------------------------------------------ fused S4 score (rank 0)
    if (fuse && crank == 0) {
      uint32_t n = 0;
      for (long long u = u_begin; u < u_end; ++u, ++n) {
        int q, g, b;
        decode(u, q, g, b);
        const uint32_t sb = n & 1u;
        mbar_wait_cl_idle<CL>(&hdr->sready[sb], (n >> 1) & 1u);
        const double sc = warp_score_sum(sSum + sb * p.sum_rows, p.l_q);
        if (lane == 0) p.scores[(long long)q * p.n_docs + b] = sc;
        __syncwarp();
        if (lane < (uint32_t)CL) mbar_arrive_rank<CL>(&hdr->sfree[sb], lane);  // release: buffer reusable
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue sets
    const int set = ((int)warp - 2) >> 2;
    const int quad = (int)(warp & 3);
    const int row_local = quad * 32 + (int)lane;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const uint32_t taddr = tmem_base + lane_base + (uint32_t)(kR8AccCol0 + set * 128);
    uint32_t nblk = 0, uses = 0, qeph = 0, sc_n = 0, ndoc = 0;
    long long cur_key = -1;
    for (long long u = u_begin; u < u_end; ++u) {
      int q, g, b;
      decode(u, q, g, b);
      const int qbv = min(p.qb, nmb_total - g * p.qb);
      const long long key = (long long)q * p.n_groups + g;
      if (key != cur_key) {
        if (cur_key >= 0) {
          mbar_wait(&hdr->qempty, qeph);
          qeph ^= 1;
        }
        // Q block mb is written by set mb % 3 (each warp its quadrant's 32 rows)
        const int row_bytes = p.dim * (kI8 ? 1 : 2);
        for (int mb = set; mb < qbv; mb += kR8Sets) {
          const int row = (g * p.qb + mb) * kTileRows + row_local;
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
            tmem_st32(tmem_base + lane_base + (uint32_t)(mb * kQCols + a * 32), r);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&hdr->qfull);
        cur_key = key;
      }
      if (!kI8 && p.debug == 3) continue;  // profiling: no drain, no output
      const int vl = doc_valid_len(p, b);
      const int ntiles = (vl + kTileRows - 1) / kTileRows;
      float part[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      float sq[4];
#pragma unroll
      for (int mb = 0; mb < 4; ++mb) {
        const int row = (g * p.qb + mb) * kTileRows + row_local;
        sq[mb] = (kI8 && mb < qbv && row < p.l_q) ? __ldg(p.q_scale + (long long)q * p.l_q + row) : 1.f;
      }
      for (int t = 0; t < ntiles; ++t) {
        const int ss = (int)(sc_n % kScaleSlots);
        if constexpr (kI8) mbar_wait(&hdr->sfull[ss], (sc_n / kScaleSlots) & 1u);
        const float* sdt = kI8 ? sScale + ss * kTileRows : nullptr;
        const int base = t * kTileRows;
        const bool full = base + kTileRows <= vl;
        // this set's blocks of the tile (one or two of the four); a rolled loop keeps the code
        // small enough for the instruction cache -- the per-block state is selected by value
        const int first = (int)((kR8Sets + set - (int)(nblk % kR8Sets)) % kR8Sets);
#pragma unroll 1
        for (int mb = first; mb < qbv; mb += kR8Sets) {
          float pm = mb == 0 ? part[0] : mb == 1 ? part[1] : mb == 2 ? part[2] : part[3];
          const float sqm = mb == 0 ? sq[0] : mb == 1 ? sq[1] : mb == 2 ? sq[2] : sq[3];
          mbar_wait(&hdr->tfull[set], uses & 1u);
          ++uses;
          tc_fence_after();
          uint32_t ra[32], rb[32];
          int cbd = 0;
          if (p.debug == 2) {  // profiling knob: release the slot unread (MMA + handshake bound)
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&hdr->tempty[set]);
          } else if (full) {
            // software-pipelined drain: the TMEM load of chunk c + 1 is in flight while chunk c
            // is folded (two 32-register buffers; the slot is released once chunk 3 has landed)
            tmem_ld32(taddr, ra);
            tmem_ld_wait_regs(ra);
            tmem_ld32(taddr + 32, rb);
            ts_chunk_full<KIND, false, kI8>(ra, base, sqm, pm, cbd, nullptr, 0, sdt);
            tmem_ld_wait_regs(rb);
            tmem_ld32(taddr + 64, ra);
            ts_chunk_full<KIND, false, kI8>(rb, base + 32, sqm, pm, cbd, nullptr, 0, kI8 ? sdt + 32 : nullptr);
            tmem_ld_wait_regs(ra);
            tmem_ld32(taddr + 96, rb);
            ts_chunk_full<KIND, false, kI8>(ra, base + 64, sqm, pm, cbd, nullptr, 0, kI8 ? sdt + 64 : nullptr);
            tmem_ld_wait_regs(rb);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&hdr->tempty[set]);
            ts_chunk_full<KIND, false, kI8>(rb, base + 96, sqm, pm, cbd, nullptr, 0, kI8 ? sdt + 96 : nullptr);
          } else {
            tmem_ld32(taddr, ra);
            tmem_ld32(taddr + 32, rb);
            tmem_ld_wait();
            ts_chunk<KIND, true, kI8>(ra, base, vl, p, b, sqm, pm, cbd, nullptr, 0, sdt);
            ts_chunk<KIND, true, kI8>(rb, base + 32, vl, p, b, sqm, pm, cbd, nullptr, 0, kI8 ? sdt + 32 : nullptr);
            tmem_ld32(taddr + 64, ra);
            tmem_ld32(taddr + 96, rb);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&hdr->tempty[set]);
            ts_chunk<KIND, true, kI8>(ra, base + 64, vl, p, b, sqm, pm, cbd, nullptr, 0, kI8 ? sdt + 64 : nullptr);
            ts_chunk<KIND, true, kI8>(rb, base + 96, vl, p, b, sqm, pm, cbd, nullptr, 0, kI8 ? sdt + 96 : nullptr);
          }
          part[0] = mb == 0 ? pm : part[0];
          part[1] = mb == 1 ? pm : part[1];
          part[2] = mb == 2 ? pm : part[2];
          part[3] = mb == 3 ? pm : part[3];
        }
        nblk += (uint32_t)qbv;
        if constexpr (kI8) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&hdr->sempty[ss]);
        }
        ++sc_n;
      }
      // ---- combine the three sets' partial maxima of this document without waiting for the
      // slowest set: every warp publishes its partials into the document's buffer (all lanes
      // arrive on pdone) and counts itself in; the last of the three warps of a quadrant (one per
      // set) max-combines the quadrant's rows and writes them.  A set can run several documents
      // ahead of another (small documents), so a buffer is refilled only after its previous
      // document's combiner released it (pfree; rarely waits).
      const uint32_t pb = ndoc % kR8PartBufs, gen = ndoc / kR8PartBufs;
      if (gen > 0) mbar_wait(&hdr->pfree[pb][quad], (gen - 1u) & 1u);
      float* buf = sPart + (size_t)pb * kR8Sets * 4 * 128;
#pragma unroll
      for (int mb = 0; mb < 4; ++mb) buf[(set * 4 + mb) * 128 + row_local] = part[mb];
      mbar_arrive(&hdr->pdone[pb][quad]);
      uint32_t arrived = 0;
      if (lane == 0) arrived = atomicAdd(&hdr->pcnt[pb][quad], 1u);
      arrived = __shfl_sync(0xffffffffu, arrived, 0);
      if (arrived == kR8Sets - 1) {
        mbar_wait(&hdr->pdone[pb][quad], gen & 1u);  // complete: the other two arrived before counting in
        const long long obase = ((long long)q * p.n_docs + b) * p.l_q;
        const uint32_t sb = ndoc & 1u;
        if (fuse) mbar_wait_cl<CL>(&hdr->sfree[sb], ((ndoc >> 1) & 1u) ^ 1u);
        for (int mb = 0; mb < qbv; ++mb) {
          const int row = (g * p.qb + mb) * kTileRows + row_local;
          const float m = fmaxf(fmaxf(buf[(0 * 4 + mb) * 128 + row_local], buf[(1 * 4 + mb) * 128 + row_local]),
                                buf[(2 * 4 + mb) * 128 + row_local]);
          if (row < p.l_q) {
            if (p.rowmax) p.rowmax[obase + row] = m;
            if (fuse) st_rank0_f32<CL>(sSum + sb * p.sum_rows + row, m);
          }
        }
        if (fuse) mbar_arrive_rank<CL>(&hdr->sready[sb], 0u);
        if (lane == 0) hdr->pcnt[pb][quad] = 0u;
        __syncwarp();
        mbar_arrive(&hdr->pfree[pb][quad]);  // every lane: its reads of the buffer are done
      }
      ++ndoc;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace mxs
