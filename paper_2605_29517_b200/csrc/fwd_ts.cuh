// Flash-MaxSim dense forward, v3: query resident in TMEM (tcgen05 "TS" MMA), document tiles
// multicast across a CTA cluster, per-row best-chunk stash for the argmax.
//
// Same contract as fwd_tc.cuh (maxsim/forward.py:108-155 _fold_pair; S2 masking, S3 strict-> /
// lowest index) -- only the data movement differs:
//   * Q row group (<= 4 blocks x 128 rows) lives in TMEM columns [0, 256): the MMA reads A
//     from TMEM and only the document tile B from shared memory (half the smem feed of SS);
//   * accumulators: two 128-column slots in TMEM columns [256, 512), slot = Q block parity;
//   * a cluster of CL CTAs (one per Q row group) scores the same documents in lockstep; each
//     CTA TMA-loads 128/CL rows of every 128-token document tile and multicasts them to the
//     whole cluster, so a document byte leaves L2 once (not once per Q row group);
//   * argmax: the epilogue keeps only a running max per row plus, for lanes that improve, a
//     copy of the improving 32-column chunk in shared memory.  The lowest index attaining the
//     final max is resolved once per (row, document) from that copy -- no per-chunk rescans
//     across the warp.
//   * fused S4 score: at the end of a document every epilogue thread stores its row maxima into a
//     double-buffered row array in its OWN shared memory and arrives on a CTA-local mbarrier (no
//     cluster-scope operation on the epilogue's critical path).  A score warp per CTA forwards
//     readiness to cluster rank 0, whose score warp reads the other ranks' rows through DSMEM,
//     folds the L_q maxima with the certified f64 sum (score_sum.cuh) and writes the score, so
//     the [N_q, B, L_q] row maxima never reach HBM (they are written only on request).
#pragma once
#include "fwd_tc.cuh"
#include "score_sum.cuh"

namespace mxs {

constexpr int kTsAccCol0 = 256;  // accumulator slots start here
constexpr int kTsSlots = 2;
constexpr int kTsEpiWarp0 = 2;                               // warps 2..9: epilogue
constexpr int kTsSumWarp = kTsEpiWarp0 + kEpiWarps;          // warp 10: fused S4 score
constexpr int kTsThreads = 32 * (kTsSumWarp + 1);  // warp 0 TMA, warp 1 MMA + TMEM alloc
constexpr int kScaleSlots = 8;  // INT8: ring of per-tile document scales (128 f32 each) in smem

struct TsSmemHeader {
  uint64_t full[8];
  uint64_t empty[8];
  uint64_t tfull[kTsSlots];
  uint64_t tempty[kTsSlots];
  uint64_t qfull;
  uint64_t qempty;
  uint64_t sfull[kScaleSlots];   // INT8 scale ring: TMA bulk copy landed
  uint64_t sempty[kScaleSlots];  // INT8 scale ring: all 8 epilogue warps done with the tile
  uint64_t sready[2];            // fused score: this CTA's row maxima of document n are in row buffer [n & 1]
  uint64_t sfree[2];             // fused score: row buffer [n & 1] may be refilled (local score warp)
  uint64_t speer[2];             // fused score, rank 0: the other ranks' buffers [n & 1] are ready
  uint64_t sdone[2];             // fused score, rank != 0: rank 0 has read buffer [n & 1]
  uint32_t tmem_base;
  uint32_t pad;
};

// INT8 accumulators start from the f32 bits of kMagicF instead of zero, so the epilogue's exact
// s32 -> f32 is one FADD2 per pair (i2f2_biased) rather than two IADDs and an FADD2 -- a third of
// the issue slots of the issue-bound INT8 epilogue.  The bias is written by the tensor core, not
// by tcgen05.st: one kind::f16 MMA (enable_input_d = 0) of a constant bf16 tile against itself,
// K = 16, every 16-byte chunk of which is {2048, 1024, 1024, 0, 0, 0, 0, 0}, so each output is
// 2 * (2^22 + 2^20 + 2^20) = 1.5 * 2^23 exactly -- the f32 kMagicF whose bits are kMagicI2F --
// whatever the swizzle.  The kind::i8 MMAs then accumulate (s32, enable_input_d = 1) on top:
// TMEM = kMagicI2F + acc, |acc| <= 2^21 for d <= 128.  A second K = 16 kind::f16 MMA of the same
// tile with the negate-A bit then adds -kMagicF to the accumulator read as f32 (MXS_I8_TC_UNBIAS,
// see i2f2_biased), leaving f32(acc) exactly, so the epilogue does no conversion at all.  Cost: two
// K = 16 bf16 MMAs per accumulator (+50 % tensor-pipe time: measured raw TMA + MMA rate 0.82 ms ->
// 1.14 ms at C4) on an epilogue-bound kernel (C4 rerank 1.61 -> 1.51 ms).
constexpr int kBiasTileBytes = 128 * 128;  // one SW128 K-major bf16 atom, 128 rows x 128 B
#ifndef MXS_TS_I8_PIPE
#define MXS_TS_I8_PIPE 1  // software-pipelined INT8 argmax drain (C4 +argmax 2.476 -> 2.396 ms)
#endif
MXS_DEV void fill_bias_tile(uint8_t* tile, int tid, int nthreads) {
  const uint4 chunk = make_uint4(0x44804500u, 0x00004480u, 0u, 0u);  // bf16 {2048, 1024 | 1024, 0 | 0, 0 | 0, 0}
  uint4* t4 = reinterpret_cast<uint4*>(tile);
  for (int i = tid; i < kBiasTileBytes / 16; i += nthreads) t4[i] = chunk;
}


// dynamic shared memory (the header is static shared memory): document-tile ring | argmax stash
// (`stash`: kStashPadStride = 36 floats per Q row) | INT8 scale ring (`scales`, or reserved when `bias`) | INT8 bias
// tile (`bias`) | fused-score row buffers (2 x `sum_rows` floats)
__host__ __device__ inline size_t fwd_ts_smem_bytes(int ka, int qb, int stages, bool scales, bool bias, bool stash,
                                                    int sum_rows) {
  return 1024 + (size_t)stages * ka * kAtomBytes + (stash ? (size_t)qb * 128 * 36 * 4 : 0) +
         ((scales || bias) ? (size_t)kScaleSlots * kTileRows * sizeof(float) : 0) + (bias ? kBiasTileBytes : 0) +
         (size_t)2 * sum_rows * sizeof(float);
}

// Stash layout: 32 floats (8 x 16 B) per (Q block, row); 16-byte pieces XOR-swizzled by lane so
// that a warp's predicated stores spread over all banks.
// swz < 0 (a compile-time constant at the call site): padded layout instead -- rows 144 B apart
// (kStashPadStride floats), which is bank-conflict free for STS.128 and needs no per-store address
// arithmetic (immediate offsets; the XOR form cost ~3 integer instructions per store).
constexpr int kStashPadStride = 36;
MXS_DEV void stash_chunk(float* row128, const float (&v)[32], int swz) {
  float4* dst = reinterpret_cast<float4*>(row128);
#pragma unroll
  for (int i = 0; i < 8; ++i)
    dst[swz < 0 ? i : (i ^ swz)] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}
MXS_DEV void unstash_chunk(const float* row128, float (&v)[32], int swz) {
  const float4* src = reinterpret_cast<const float4*>(row128);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float4 t = src[swz < 0 ? i : (i ^ swz)];
    v[4 * i] = t.x;
    v[4 * i + 1] = t.y;
    v[4 * i + 2] = t.z;
    v[4 * i + 3] = t.w;
  }
}

template <TcKind KIND, bool kMagic = false, bool kBiased = false>
MXS_DEV void ts_chunk(const uint32_t (&r)[32], int base, int vl, const FwdTcParams& p, int b, float sq, float& m,
                      int& cb, float* stash_row, int swz, const float* sd_smem = nullptr) {
  if (base >= vl) return;
  float v[32];
  if constexpr (KIND == TcKind::I8) {
    // fl(fl(f32(acc) * s_q) * s_d) in the order of maxsim/quant.py:174-176 (S7).
    const float* sd = p.d_scale + (long long)b * p.l_pad + base;
    const bool vec = (base + 32 <= p.l_pad) && ((p.l_pad & 3) == 0);
    float sdv[32];
    if (sd_smem) {  // this chunk's 32 scales, staged by the TMA warp (broadcast LDS.128)
      const float4* s4 = reinterpret_cast<const float4*>(sd_smem);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 t = s4[c];
        sdv[4 * c] = t.x;
        sdv[4 * c + 1] = t.y;
        sdv[4 * c + 2] = t.z;
        sdv[4 * c + 3] = t.w;
      }
    } else if (vec) {
      const float4* sd4 = reinterpret_cast<const float4*>(sd);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 t = __ldg(sd4 + c);
        sdv[4 * c] = t.x;
        sdv[4 * c + 1] = t.y;
        sdv[4 * c + 2] = t.z;
        sdv[4 * c + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) sdv[j] = (base + j < p.l_pad) ? __ldg(sd + j) : 1.f;
    }
    // f32(acc): exact either way -- the magic-number form (IADD + FADD2) when |acc| <= 2^22
    // (d <= 256 for any int8 input), else cvt.rn on the XU pipe, which is 4x narrower and
    // was the bottleneck of this epilogue (ncu: XU 129% of sustained peak).  Both multiplies as
    // packed FMUL2 pairs (each lane of the pair rounds exactly like the scalar fl(x * y)).
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      float c0, c1, t0, t1;
      if constexpr (kBiased) {
        i2f2_biased(c0, c1, r[j], r[j + 1]);
      } else if constexpr (kMagic) {
        i2f2_magic(c0, c1, r[j], r[j + 1]);
      } else {
        c0 = __int2float_rn((int)r[j]);
        c1 = __int2float_rn((int)r[j + 1]);
      }
      fmul2_rn(t0, t1, c0, c1, sq, sq);
      fmul2_rn(v[j], v[j + 1], t0, t1, sdv[j], sdv[j + 1]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  }
  if (base + 32 > vl) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (base + j >= vl) v[j] = -INFINITY;
  }
  const float cmax = max32(v);
  if (stash_row == nullptr) {  // scores only (argmax not requested): the running max is all
    m = fmaxf(m, cmax);
    return;
  }
  if (cmax > m) {  // predicated stash (see ts_chunk_full)
    m = cmax;
    cb = base;
    stash_chunk(stash_row, v, swz);
  }
}

// Fast path of ts_chunk for a chunk that lies entirely inside the document (no masking), with
// the INT8 scales already in shared memory and the argmax decision made at compile time: no
// per-chunk bounds checks or pointer tests, so the compiler sees one straight-line block.
template <TcKind KIND, bool kArgmax, bool kBiased = false>
MXS_DEV void ts_chunk_full(const uint32_t (&r)[32], int base, float sq, float& m, int& cb, float* stash_row, int swz,
                           const float* sd_smem) {
  float v[32];
  if constexpr (KIND == TcKind::I8) {
    const float4* s4 = reinterpret_cast<const float4*>(sd_smem);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 t = s4[c];
      float c0, c1, c2, c3, t0, t1, t2, t3;
      if constexpr (kBiased) {
        i2f2_biased(c0, c1, r[4 * c], r[4 * c + 1]);
        i2f2_biased(c2, c3, r[4 * c + 2], r[4 * c + 3]);
      } else {
        i2f2_magic(c0, c1, r[4 * c], r[4 * c + 1]);
        i2f2_magic(c2, c3, r[4 * c + 2], r[4 * c + 3]);
      }
      fmul2_rn(t0, t1, c0, c1, sq, sq);
      fmul2_rn(t2, t3, c2, c3, sq, sq);
      fmul2_rn(v[4 * c], v[4 * c + 1], t0, t1, t.x, t.y);
      fmul2_rn(v[4 * c + 2], v[4 * c + 3], t2, t3, t.z, t.w);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  }
  const float cmax = max32(v);
  if constexpr (!kArgmax) {
    m = fmaxf(m, cmax);
  } else {
    // improving lanes stash their chunk (predicated stores; guarding them with a warp vote and a
    // branch was 5 % slower at C2 +argmax -- nearly every chunk has an improving lane)
    if (cmax > m) {
      m = cmax;
      cb = base;
      stash_chunk(stash_row, v, swz);
    }
  }
}

// Score warp of the fused S4 epilogue (fwd_ts_kernel, fwd_pair_kernel).  The CTA's producers store
// the row maxima of document n into row buffer [n & 1] of their OWN shared memory, fence them to
// the async proxy and arrive on sready[n & 1] (CTA scope) -- nothing cluster-wide on the
// epilogue's critical path.  The score warp of rank r != 0 ships its rows into rank 0's buffer
// with ONE bulk copy (cp.async.bulk shared::cta -> shared::cluster, completing as transaction
// bytes on rank 0's speer) once rank 0 has consumed that buffer's previous document (sdone); rank
// 0's score warp arms speer with the other ranks' bytes, then holds all L_q maxima locally,
// computes the certified f64 sum and writes the score.  sfree[n & 1] re-arms a CTA's own buffer.
// (Round 2 first pushed the rows with per-lane st.shared::cluster stores and release.cluster
// arrives: their GPU-scope fences stalled the SM's tensor pipeline, 9 % of the C2 forward.)
MXS_DEV void bulk_copy_to_cluster(uint32_t dst_cluster, const void* src, uint32_t bytes, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_cluster),
      "r"(smem_u32(src)), "r"(bytes), "r"(bar_cluster)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
MXS_DEV void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// Rows [r0, r1) of rank r's share of a fused-score row buffer, padded to whole 16-byte chunks
// (the buffers hold whole 128-row blocks, so the padding stays inside them).
MXS_DEV uint32_t score_rows_bytes(int r0, int r1) { return (uint32_t)(((r1 - r0) + 3) & ~3) * 4u; }
// The score warps mostly wait: suspending waits keep them off the epilogue warps' issue slots
// (spinning measured the same).
MXS_DEV void score_wait(uint64_t* bar, uint32_t parity) { mbar_wait_idle(bar, parity); }
MXS_DEV void score_wait_cluster(uint64_t* bar, uint32_t parity) { mbar_wait_cluster_idle(bar, parity); }
// Certified partial of one epilogue warp's row maxima (PART mode of fused_score_warp), 16 bytes, in
// INTEGER fixed point: k = sum of the values in units of 2^(emax - 150 - S) (emax = the warp's
// largest biased exponent, S = 29 - ceil(log2 L_q)), plus the exponent range and finiteness for the
// certificate (score_sum.cuh).  Under the certificate (emax - emin <= S over the whole document)
// every value is an exact integer multiple of that unit, every partial and the total are exact
// int64 sums, and re-basing a partial to the document's emax is an exact right shift (its lowest
// set bit sits at >= emin - emax_doc + S >= 0) -- so the result is the exact sum, i.e. the
// reference's sequential f64 sum bit for bit.
// No FP64 instruction runs per value: on this B200 the FP64 form of the same fold (F2F + DADD per
// value) cost 5 % of the C2 forward's tensor throughput wherever it ran (score warp or epilogue).
struct ScorePartial {
  long long k;
  uint32_t e;  // emin | emax << 8 | finite << 16
  uint32_t pad;
};
constexpr int kPartialsPerRank = 8;  // one per epilogue warp
static_assert(sizeof(ScorePartial) == 16, "partial layout");
MXS_DEV long long warp_sum_i64(long long x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
// Every lane of an epilogue warp: fold its row maxima v[0..K) (rows >= L_q excluded by the caller)
// into the warp's partial; lane 0 stores it.
template <int K>
MXS_DEV void store_score_partial(const float (&v)[K], const bool (&valid)[K], ScorePartial* dst, uint32_t lane,
                                 int n_values) {
  int emin = 255, emax = 0;
  bool fin = true;
  uint32_t bits[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    bits[i] = valid[i] ? __float_as_uint(v[i]) : 0u;
    exp_range(bits[i], emin, emax, fin);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    emin = min(emin, __shfl_xor_sync(0xffffffffu, emin, o));
    emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  }
  fin = __all_sync(0xffffffffu, fin);
  const int S = fix_shift(n_values);  // the document's L_q fixes the unit for every partial
  long long k = 0;
#pragma unroll
  for (int i = 0; i < K; ++i) k += fix_term(bits[i], emax, S);
  k = warp_sum_i64(k);
  if (lane == 0) *dst = ScorePartial{k, (uint32_t)emin | ((uint32_t)emax << 8) | ((fin ? 1u : 0u) << 16), 0u};
}
// Whole warp (the score warp): combine np <= 32 partials into the S4 score; `fallback` gives the
// sequential chain when the certificate fails (or every value is +-0, whose sign only the chain
// reproduces).
template <typename Fallback>
MXS_DEV double combine_score_partials(const ScorePartial* part, int np, int n_values, Fallback fallback) {
  const int lane = (int)(threadIdx.x & 31u);
  long long k = 0;
  int emin = 255, emax = 0;
  bool fin = true;
  if (lane < np) {
    const ScorePartial e = part[lane];
    k = e.k;
    emin = (int)(e.e & 0xffu);
    emax = (int)((e.e >> 8) & 0xffu);
    fin = (e.e >> 16) & 1u;
  }
  int gmin = emin, gmax = emax;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    gmin = min(gmin, __shfl_xor_sync(0xffffffffu, gmin, o));
    gmax = max(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
  }
  fin = __all_sync(0xffffffffu, fin);
  if (!certified(gmin, gmax, fin, n_values)) return fallback();
  const long long total = warp_sum_i64(emax ? (k >> (gmax - emax)) : 0ll);  // exact re-basing (see above)
  // total * 2^(gmax - 150 - S): the int64 -> f64 conversion is exact (the certificate makes the sum
  // representable) and the scale is a power of two
  return fix_to_double(total, gmax, fix_shift(n_values));
}

// PART = false: the score warp folds the L_q row maxima itself; PART = true: every epilogue warp
// has already folded its rows into a certified partial (store_score_partial, spread over the four
// SM sub-partitions) and the score warp only combines CL x 8 partials -- the same certificate
// covers every subset sum, so the result is the same exact sum; the raw rows still travel for the
// rare sequential fallback.
template <int CL, int NB = 2, bool PART = false, typename Decode>
MXS_DEV void fused_score_warp(const FwdTcParams& p, uint64_t* sready, uint64_t* sfree, uint64_t* speer,
                              uint64_t* sdone, float* sSum, long long u_begin, long long u_end, Decode decode,
                              int crank, uint32_t lane, ScorePartial* sPart = nullptr) {
  const int rows_per_rank = p.qb * kTileRows;
  uint32_t peer_bytes = 0;  // rank 0: bytes the other ranks ship per document
  for (int r = 1; r < CL; ++r) {
    const int r0 = r * rows_per_rank, r1 = min(p.l_q, r0 + rows_per_rank);
    if (r1 > r0) peer_bytes += score_rows_bytes(r0, r1) + (PART ? kPartialsPerRank * sizeof(ScorePartial) : 0);
  }
  uint32_t n = 0;
  for (long long u = u_begin; u < u_end; ++u, ++n) {
    const uint32_t sb = n % NB, ph = (n / NB) & 1u;  // NB row buffers in flight
    float* buf = sSum + sb * p.sum_rows;
    score_wait(&sready[sb], ph);  // this CTA's rows are in
    if (crank == 0) {
      int q, g, b;
      decode(u, q, g, b);
      if constexpr (CL > 1) {
        if (lane == 0) mbar_arrive_expect_tx(&speer[sb], peer_bytes);
        score_wait(&speer[sb], ph);  // and every other rank's (bulk copies landed)
      }
      double sc;
      if constexpr (PART) {
        sc = combine_score_partials(sPart + sb * CL * kPartialsPerRank, CL * kPartialsPerRank, p.l_q,
                                    [&]() { return warp_score_sum(buf, p.l_q); });  // fallback: the sequential chain
      } else {
        sc = p.debug == 7 ? 0.0 : warp_score_sum(buf, p.l_q);  // 7: profiling, no sum
      }
      if (lane == 0) p.scores[(long long)q * p.n_docs + b] = sc;
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfree[sb]);
      if constexpr (CL > 1) {  // rank `lane` may refill our buffer [sb] (our reads are done: sc depends on them)
        if (lane >= 1 && lane < (uint32_t)CL) mbar_arrive_remote(mapa_u32(smem_u32(&sdone[sb]), lane));
      }
    } else if constexpr (CL > 1) {
      const int r0 = crank * rows_per_rank, r1 = min(p.l_q, r0 + rows_per_rank);
      if (lane == 0) {
        score_wait_cluster(&sdone[sb], ph ^ 1u);  // rank 0 consumed its buffer [sb] NB documents ago
        if (r1 > r0) {
          bulk_copy_to_cluster(mapa_u32(smem_u32(buf + r0), 0u), buf + r0, score_rows_bytes(r0, r1),
                               mapa_u32(smem_u32(&speer[sb]), 0u));
          if constexpr (PART) {
            ScorePartial* part = sPart + sb * CL * kPartialsPerRank + crank * kPartialsPerRank;
            bulk_copy_to_cluster(mapa_u32(smem_u32(part), 0u), part, kPartialsPerRank * sizeof(ScorePartial),
                                 mapa_u32(smem_u32(&speer[sb]), 0u));
          }
          bulk_wait_read_all();  // our buffer has been read: it may be refilled
        }
        mbar_arrive(&sfree[sb]);
      }
      __syncwarp();
    }
  }
}

template <TcKind KIND, int KA, int CL>
__global__ void __launch_bounds__(kTsThreads, 1)
    fwd_ts_kernel(const __grid_constant__ CUtensorMap tmD, const FwdTcParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment by offsetting the __shared__ array itself (keeps the shared address space,
  // so accesses compile to LDS/STS rather than generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sD = smem;
  float* sBest = reinterpret_cast<float*>(sD + (size_t)p.stages * KA * kAtomBytes);
  // INT8 scale ring (only when d_scale rows are 16-B aligned: l_pad % 4 == 0)
  float* sScale = sBest + (p.argmax ? (size_t)p.qb * 128 * kStashPadStride : 0);
  const bool scale_ring = (KIND == TcKind::I8) && ((p.l_pad & 3) == 0);
  // INT8 with |acc| <= 2^22 (d <= 256): accumulators pre-biased to kMagicF (see fill_bias_tile)
  constexpr bool kBias = (KIND == TcKind::I8) && (KA <= 2);
  uint8_t* sBias = reinterpret_cast<uint8_t*>(sScale + ((scale_ring || kBias) ? kScaleSlots * kTileRows : 0));
  float* sSum = reinterpret_cast<float*>(sBias + (kBias ? kBiasTileBytes : 0));
  // fused S4 score (the profiling knob MXS_DEBUG=3 skips the drain, so it has nothing to sum)
  const bool fuse = p.scores != nullptr && !(KIND != TcKind::I8 && p.debug == 3);
  __shared__ TsSmemHeader ts_hdr;  // static shared: keeps barrier / bookkeeping accesses on LDS/STS
  TsSmemHeader* hdr = &ts_hdr;

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const int crank = (CL > 1) ? (int)cluster_ctarank() : 0;
  constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1u);
  constexpr int kQCols = KA * 32;  // TMEM columns per Q block (128 B atoms / 4 B per column)

  // unit ranges: with a cluster, units are (q, b) and the Q row group is the CTA rank
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
    for (int s = 0; s < kTsSlots; ++s) {
      mbar_init(&hdr->tfull[s], 1);
      mbar_init(&hdr->tempty[s], 4);
    }
    mbar_init(&hdr->qfull, kEpiWarps);
    mbar_init(&hdr->qempty, 1);
    for (int s = 0; s < kScaleSlots; ++s) {
      mbar_init(&hdr->sfull[s], 1);
      mbar_init(&hdr->sempty[s], kEpiWarps);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&hdr->sready[s], 32 * kEpiWarps);  // every epilogue lane of this CTA
      mbar_init(&hdr->sfree[s], 1);
      mbar_init(&hdr->speer[s], 1);  // rank 0's expect_tx arrive + the other ranks' bulk-copy bytes
      mbar_init(&hdr->sdone[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&hdr->tmem_base, 512);
  if constexpr (kBias) {
    fill_bias_tile(sBias, (int)threadIdx.x, kTsThreads);
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = hdr->tmem_base;

  constexpr uint32_t kIdesc = (KIND == TcKind::I8) ? make_idesc(2, 1, 128, 128)
                              : (KIND == TcKind::BF16) ? make_idesc(1, 1, 128, 128)
                                                       : make_idesc(1, 0, 128, 128);
  constexpr int kElemsPerAtom = (KIND == TcKind::I8) ? 128 : 64;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t sc_n = 0;  // tiles issued on the scale ring
      constexpr int kRowsPer = kTileRows / CL;
      for (long long u = u_begin; u < u_end; ++u) {
        int q, g, b;
        decode(u, q, g, b);
        const int vl = doc_valid_len(p, b);
        const int ntiles = (vl + kTileRows - 1) / kTileRows;
        for (int t = 0; t < ntiles; ++t) {
          if (scale_ring) {
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
    // Accumulator slot = Q block parity, so each epilogue warp set (which owns the blocks of
    // one parity) consumes every phase of its own slot in order -- a waiter can never be two
    // phases behind and alias an mbarrier parity.
    int stage = 0;
    uint32_t phase = 0, qphase = 0;
    uint32_t sbits = 0;  // bit s = parity of slot s's next use
    long long cur_key = -1;
    const uint64_t ddesc0 = sw128_kmajor_desc(smem_u32(sD));
    const uint64_t bias_desc = sw128_kmajor_desc(smem_u32(sBias));
    for (long long u = u_begin; u < u_end; ++u) {
      int q, g, b;
      decode(u, q, g, b);
      const long long key = (long long)q * p.n_groups + g;
      if (key != cur_key) {
        if (cur_key >= 0) {
          if (elect_one()) mma_commit(&hdr->qempty);
          __syncwarp();
        }
        mbar_wait(&hdr->qfull, qphase);
        qphase ^= 1;
        tc_fence_after();
        cur_key = key;
      }
      const int qbv = min(p.qb, nmb_total - g * p.qb);
      const int vl = doc_valid_len(p, b);
      const int ntiles = (vl + kTileRows - 1) / kTileRows;
      for (int t = 0; t < ntiles; ++t) {
        mbar_wait(&hdr->full[stage], phase);
        tc_fence_after();
        const uint64_t bd0 = ddesc0 + (uint64_t)((stage * KA * kAtomBytes) >> 4);
        for (int mb = 0; mb < qbv; ++mb) {
          const int slot = mb & 1;
          // profiling knob MXS_DEBUG=3 (bf16/fp16 only): never wait for the drain -- the raw
          // MMA + TMA rate of this pipeline (accumulators overwritten, results garbage)
          if (p.debug != 3) {
            if (p.mma_spin)
              mbar_wait(&hdr->tempty[slot], ((sbits >> slot) & 1u) ^ 1u);
            else
              mbar_wait_idle(&hdr->tempty[slot], ((sbits >> slot) & 1u) ^ 1u);
          }
          tc_fence_after();
          if (elect_one()) {
            const uint32_t acol = tmem_base + (uint32_t)(mb * kQCols);
            const uint32_t dcol = tmem_base + (uint32_t)(kTsAccCol0 + slot * 128);
            if constexpr (kBias) mma_f16_ss(dcol, bias_desc, bias_desc, make_idesc(1, 1, 128, 128), 0u);
#pragma unroll
            for (int k = 0; k < KA * 4; ++k) {
              const uint64_t koff = (uint64_t)(((k >> 2) * kAtomBytes + (k & 3) * 32) >> 4);
              if constexpr (KIND == TcKind::I8)
                mma_i8_ts(dcol, acol + k * 8, bd0 + koff, kIdesc, (kBias || k > 0) ? 1u : 0u);
              else
                mma_f16_ts(dcol, acol + k * 8, bd0 + koff, kIdesc, k > 0 ? 1u : 0u);
            }
            if constexpr (kBias && MXS_I8_TC_UNBIAS)  // TMEM = kMagicF + acc - kMagicF (see i2f2_biased)
              mma_f16_ss(dcol, bias_desc, bias_desc, make_idesc(1, 1, 128, 128) | kIdescNegA, 1u);
            mma_commit(&hdr->tfull[slot]);
          }
          __syncwarp();
          sbits ^= 1u << slot;
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
  } else if (warp == kTsSumWarp) {
    // ------------------------------------------------------------------ fused S4 score
    if (fuse) fused_score_warp<CL>(p, hdr->sready, hdr->sfree, hdr->speer, hdr->sdone, sSum, u_begin, u_end, decode,
                                   crank, lane);
  } else {
    // ------------------------------------------------------------------ epilogue (+ Q -> TMEM)
    // warp w in [2, 10): TMEM lane quadrant w % 4 (hardware rule), set (w - 2) / 4.
    const int wset = ((int)warp - kTsEpiWarp0) >> 2;
    const int quad = (int)(warp & 3);
    const int row_local = quad * 32 + (int)lane;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    constexpr int swz = -1;  // padded argmax stash (see stash_chunk)
    const int eb = (KIND == TcKind::I8) ? 1 : 2;
    const int row_bytes = p.dim * eb;
    uint32_t sph = 0, qeph = 0;  // this set's slot is `wset`; sph = parity of its next use
    uint32_t sc_n = 0;           // tiles consumed from the scale ring
    uint32_t ndoc = 0;           // documents finished (fused-score row buffer = ndoc & 1)
    long long cur_key = -1;
    for (long long u = u_begin; u < u_end; ++u) {
      int q, g, b;
      decode(u, q, g, b);
      const int qbv = min(p.qb, nmb_total - g * p.qb);
      const long long key = (long long)q * p.n_groups + g;
      if (key != cur_key) {
        if (cur_key >= 0) {
          mbar_wait(&hdr->qempty, qeph);  // every MMA reading the old Q block has completed
          qeph ^= 1;
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int mb = 2 * i + wset;
          if (mb >= qbv) break;
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
      if (KIND != TcKind::I8 && p.debug == 3) continue;  // no drain (see the MMA issuer)
      const int vl = doc_valid_len(p, b);
      const int ntiles = (vl + kTileRows - 1) / kTileRows;
      float m[2], sq[2];
      int cb[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        m[i] = -INFINITY;
        cb[i] = 0;
        sq[i] = 1.f;
        if constexpr (KIND == TcKind::I8) {
          const int mb = 2 * i + wset;
          const int row = (g * p.qb + mb) * kTileRows + row_local;
          if (mb < qbv && row < p.l_q) sq[i] = __ldg(p.q_scale + (long long)q * p.l_q + row);
        }
      }
      for (int t = 0; t < ntiles; ++t) {
        const float* sdt = nullptr;  // this tile's staged scales
        if (scale_ring) {
          const int ss = (int)(sc_n % kScaleSlots);
          mbar_wait(&hdr->sfull[ss], (sc_n / kScaleSlots) & 1u);
          sdt = sScale + ss * kTileRows;
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int mb = 2 * i + wset;
          if (mb >= qbv) break;
          const uint32_t slot = (uint32_t)wset;
          mbar_wait(&hdr->tfull[slot], sph);
          sph ^= 1u;
          tc_fence_after();
          const uint32_t taddr = tmem_base + lane_base + (uint32_t)(kTsAccCol0 + slot * 128);
          // argmax not requested (rerank: scores only) -> no index tracking at all
          float* stash = p.argmax ? sBest + ((size_t)mb * 128 + row_local) * kStashPadStride : nullptr;
          const int base = t * kTileRows;
          if (p.debug == 2) {  // profiling knob: drain the slot without folding
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&hdr->tempty[slot]);
          } else if (KIND == TcKind::I8 && KA <= 2 && sdt != nullptr && base + kTileRows <= vl) {
            // full tile, staged scales: straight-line chunks, argmax tracking decided at compile time
            uint32_t ra[32], rb[32];
#if MXS_TS_I8_PIPE
            // software-pipelined drain (as fwd_i8r): the load of chunk c + 1 is in flight while
            // chunk c is folded; the slot is released once chunk 3 has landed
            if (stash) {
              tmem_ld32(taddr, ra);
              tmem_ld_wait_regs(ra);
              tmem_ld32(taddr + 32, rb);
              ts_chunk_full<KIND, true, kBias>(ra, base, sq[i], m[i], cb[i], stash, swz, sdt);
              tmem_ld_wait_regs(rb);
              tmem_ld32(taddr + 64, ra);
              ts_chunk_full<KIND, true, kBias>(rb, base + 32, sq[i], m[i], cb[i], stash, swz, sdt + 32);
              tmem_ld_wait_regs(ra);
              tmem_ld32(taddr + 96, rb);
              ts_chunk_full<KIND, true, kBias>(ra, base + 64, sq[i], m[i], cb[i], stash, swz, sdt + 64);
              tmem_ld_wait_regs(rb);
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&hdr->tempty[slot]);
              ts_chunk_full<KIND, true, kBias>(rb, base + 96, sq[i], m[i], cb[i], stash, swz, sdt + 96);
              continue;
            }
#endif
            tmem_ld32(taddr, ra);
            tmem_ld32(taddr + 32, rb);
            tmem_ld_wait();
            if (stash) {
              ts_chunk_full<KIND, true, kBias>(ra, base, sq[i], m[i], cb[i], stash, swz, sdt);
              ts_chunk_full<KIND, true, kBias>(rb, base + 32, sq[i], m[i], cb[i], stash, swz, sdt + 32);
            } else {
              ts_chunk_full<KIND, false, kBias>(ra, base, sq[i], m[i], cb[i], stash, swz, sdt);
              ts_chunk_full<KIND, false, kBias>(rb, base + 32, sq[i], m[i], cb[i], stash, swz, sdt + 32);
            }
            tmem_ld32(taddr + 64, ra);
            tmem_ld32(taddr + 96, rb);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&hdr->tempty[slot]);
            if (stash) {
              ts_chunk_full<KIND, true, kBias>(ra, base + 64, sq[i], m[i], cb[i], stash, swz, sdt + 64);
              ts_chunk_full<KIND, true, kBias>(rb, base + 96, sq[i], m[i], cb[i], stash, swz, sdt + 96);
            } else {
              ts_chunk_full<KIND, false, kBias>(ra, base + 64, sq[i], m[i], cb[i], stash, swz, sdt + 64);
              ts_chunk_full<KIND, false, kBias>(rb, base + 96, sq[i], m[i], cb[i], stash, swz, sdt + 96);
            }
          } else if constexpr (KIND == TcKind::I8) {
            // the dequantisation needs extra registers: two chunks in flight at a time
            uint32_t ra[32], rb[32];
            tmem_ld32(taddr, ra);
            tmem_ld32(taddr + 32, rb);
            tmem_ld_wait();
            ts_chunk<KIND, (KA <= 2), kBias>(ra, base, vl, p, b, sq[i], m[i], cb[i], stash, swz, sdt);
            ts_chunk<KIND, (KA <= 2), kBias>(rb, base + 32, vl, p, b, sq[i], m[i], cb[i], stash, swz, sdt ? sdt + 32 : sdt);
            tmem_ld32(taddr + 64, ra);
            tmem_ld32(taddr + 96, rb);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&hdr->tempty[slot]);
            ts_chunk<KIND, (KA <= 2), kBias>(ra, base + 64, vl, p, b, sq[i], m[i], cb[i], stash, swz, sdt ? sdt + 64 : sdt);
            ts_chunk<KIND, (KA <= 2), kBias>(rb, base + 96, vl, p, b, sq[i], m[i], cb[i], stash, swz, sdt ? sdt + 96 : sdt);
          } else if (KIND != TcKind::I8 && base + kTileRows <= vl) {
            uint32_t ra[32], rb[32], rc[32], rd[32];
            tmem_ld32(taddr, ra);
            tmem_ld32(taddr + 32, rb);
            tmem_ld32(taddr + 64, rc);
            tmem_ld32(taddr + 96, rd);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&hdr->tempty[slot]);
            if (stash) {
              ts_chunk_full<KIND, true, kBias>(ra, base, sq[i], m[i], cb[i], stash, swz, nullptr);
              ts_chunk_full<KIND, true, kBias>(rb, base + 32, sq[i], m[i], cb[i], stash, swz, nullptr);
              ts_chunk_full<KIND, true, kBias>(rc, base + 64, sq[i], m[i], cb[i], stash, swz, nullptr);
              ts_chunk_full<KIND, true, kBias>(rd, base + 96, sq[i], m[i], cb[i], stash, swz, nullptr);
            } else {
              ts_chunk_full<KIND, false, kBias>(ra, base, sq[i], m[i], cb[i], stash, swz, nullptr);
              ts_chunk_full<KIND, false, kBias>(rb, base + 32, sq[i], m[i], cb[i], stash, swz, nullptr);
              ts_chunk_full<KIND, false, kBias>(rc, base + 64, sq[i], m[i], cb[i], stash, swz, nullptr);
              ts_chunk_full<KIND, false, kBias>(rd, base + 96, sq[i], m[i], cb[i], stash, swz, nullptr);
            }
          } else {
            uint32_t ra[32], rb[32], rc[32], rd[32];
            tmem_ld32(taddr, ra);
            tmem_ld32(taddr + 32, rb);
            tmem_ld32(taddr + 64, rc);
            tmem_ld32(taddr + 96, rd);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&hdr->tempty[slot]);
            ts_chunk<KIND, (KA <= 2), kBias>(ra, base, vl, p, b, sq[i], m[i], cb[i], stash, swz);
            ts_chunk<KIND, (KA <= 2), kBias>(rb, base + 32, vl, p, b, sq[i], m[i], cb[i], stash, swz);
            ts_chunk<KIND, (KA <= 2), kBias>(rc, base + 64, vl, p, b, sq[i], m[i], cb[i], stash, swz);
            ts_chunk<KIND, (KA <= 2), kBias>(rd, base + 96, vl, p, b, sq[i], m[i], cb[i], stash, swz);
          }
        }
        if (scale_ring) {  // this warp is done with the tile's scales
          __syncwarp();
          if (lane == 0) mbar_arrive(&hdr->sempty[sc_n % kScaleSlots]);
          ++sc_n;
        }
      }
      if (fuse) {  // row maxima -> this CTA's row buffer, then every lane arrives (CTA scope)
        const uint32_t sb = ndoc & 1u;
        mbar_wait(&hdr->sfree[sb], ((ndoc >> 1) & 1u) ^ 1u);
        float* dst = sSum + sb * p.sum_rows;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int mb = 2 * i + wset;
          const int row = (g * p.qb + mb) * kTileRows + row_local;
          if (mb < qbv && row < p.l_q) dst[row] = m[i];
        }
        fence_proxy_async();  // the row maxima are shipped to cluster rank 0 by a bulk (async-proxy) copy
        mbar_arrive(&hdr->sready[sb]);
        ++ndoc;
      }
      const long long obase = ((long long)q * p.n_docs + b) * p.l_q;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int mb = 2 * i + wset;
        if (mb >= qbv) break;
        const int row = (g * p.qb + mb) * kTileRows + row_local;
        if (row < p.l_q) {
          if (p.rowmax) p.rowmax[obase + row] = m[i];
          if (p.argmax) {
            float w[32];
            unstash_chunk(sBest + ((size_t)mb * 128 + row_local) * kStashPadStride, w, swz);
            p.argmax[obase + row] = ntiles ? cb[i] + first_argmax32_chain(w, m[i]) : 0;  // 0: empty (invalid) doc
          }
        }
      }
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
