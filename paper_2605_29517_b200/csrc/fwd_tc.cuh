// Flash-MaxSim dense forward on tcgen05 (sm_100a).
//
// Follows the reference fold `maxsim/forward.py:108-155` (_fold_pair) and the tie / masking
// contract of `maxsim/kernels.py:69-93` (fold_extreme) and `maxsim/forward.py:153-154`:
//   sim[i, j]  = <Q_i, D_j>                      (tensor core, fp32 / s32 accumulators in TMEM)
//   padding    : columns j >= valid_len are -inf before the row reduction (S2)
//   rowmax[i]  = max_j sim[i, j], argmax = lowest j attaining it (strict > in column order, S3)
// The [L_q, L_d] similarity tile only ever exists in TMEM; HBM sees Q, D and the per-row
// (max, argmax) outputs.  The f64 per-pair score is folded by mxs_rowsum_kernel (S4).
//
// Work decomposition: unit = (query q, Q-row group g, document b), b fastest.  A CTA owns a
// contiguous unit range; its Q row group (<= 4 blocks of 128 rows) stays resident in shared
// memory while document tiles of 128 tokens stream through a TMA ring.  Per document tile
// the single MMA thread issues one 128x128xdim MMA chain per Q block into one of 4 TMEM
// accumulator slots (128 columns each); 8 epilogue warps drain the slots with tcgen05.ld and
// fold them into register-resident running (max, argmax) per Q row.
#pragma once
#include "ptx.cuh"
#include "kinds.h"

namespace mxs {


struct FwdTcParams {
  int n_q, l_q, n_docs, l_pad, dim;
  int ka;          // 128-byte K atoms per row (dim * elem_bytes / 128, rounded up)
  int qb;          // Q blocks (128 rows) per CTA group, <= 4
  int n_groups;    // Q row groups per query
  int stages;      // document-tile ring depth
  long long n_units;
  const int32_t* valid_lens;  // [n_docs] or nullptr (= l_pad)
  const float* q_scale;       // I8 only: [n_q * l_q]
  const float* d_scale;       // I8 only: [n_docs * l_pad]
  float* rowmax;              // [n_q, n_docs, l_q]
  int32_t* argmax;            // [n_q, n_docs, l_q] or nullptr
  int debug;                  // profiling knobs (MXS_DEBUG env): 1 = skip fold, 2 = skip TMEM loads too
  int mma_spin;               // MXS_MMA_SPIN=1: the MMA issuer spins (no suspend) on accumulator-slot waits
  const void* q_ptr;          // Q rows in global memory (TS kernel loads them into TMEM)
  double* scores;             // [n_q, n_docs]: fused S4 sum in the epilogue (fwd_ts / fwd_i8r), or nullptr
  int sum_rows;               // row capacity of each shared-memory row-maxima buffer (fused sum)
};

constexpr int kTileRows = 128;     // rows per Q block and per document tile
constexpr int kAtomBytes = 16384;  // 128 rows x 128 B
constexpr int kSlots = 4;          // TMEM accumulator slots of 128 columns
constexpr int kEpiWarps = 8;
constexpr int kFwdThreads = 128 + 32 * kEpiWarps;  // warp0 TMA, warp1 MMA, warp2 TMEM alloc, warp3 spare
constexpr int kMaxQb = 4;

struct FwdSmemHeader {
  uint64_t full[8];
  uint64_t empty[8];
  uint64_t tfull[kSlots];
  uint64_t tempty[kSlots];
  uint64_t qfull;
  uint64_t qempty;
  uint32_t tmem_base;
  uint32_t pad;
};

// dynamic shared memory (the header is static shared memory)
__host__ __device__ inline size_t fwd_tc_smem_bytes(int ka, int qb, int stages) {
  return 1024 /*align slack*/ + (size_t)(qb + stages) * ka * kAtomBytes;
}

MXS_DEV void decode_unit(long long u, const FwdTcParams& p, int& q, int& g, int& b) {
  b = (int)(u % p.n_docs);
  long long r = u / p.n_docs;
  g = (int)(r % p.n_groups);
  q = (int)(r / p.n_groups);
}

MXS_DEV int doc_valid_len(const FwdTcParams& p, int b) {
  // clamped into [0, l_pad] so that unvalidated input can never address another document's rows
  return p.valid_lens ? min(max(__ldg(p.valid_lens + b), 0), p.l_pad) : p.l_pad;
}

// max of 32 values as a 3-input tree (FMNMX3): 15 ALU instructions, depth 4.
MXS_DEV float max32(const float (&v)[32]) {
  float t[11];
#pragma unroll
  for (int j = 0; j < 10; ++j) t[j] = fmax3(v[3 * j], v[3 * j + 1], v[3 * j + 2]);
  t[10] = fmaxf(v[30], v[31]);
  const float a = fmax3(t[0], t[1], t[2]);
  const float b = fmax3(t[3], t[4], t[5]);
  const float c = fmax3(t[6], t[7], t[8]);
  return fmax3(fmax3(a, b, c), t[9], t[10]);
}

// Lowest j with v[j] == c, assuming c = max(v) and 2^-60 <= |c| <= 2^27.
// d_j = c - v_j >= 0 is exactly 0 iff v_j == c; otherwise d_j >= 2^-84, so
// w_j = d_j * 2^100 + j is j for the winners and >= 2^16 for everyone else.  Two FMA-pipe
// instructions per element and a min tree, all independent (no serial select chain).
MXS_DEV int first_argmax32_fast(const float (&v)[32], float c) {
  float w[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) w[j] = __fmaf_rn(__fsub_rn(c, v[j]), 0x1p100f, (float)j);
  float t[11];
#pragma unroll
  for (int j = 0; j < 10; ++j) t[j] = fmin3(w[3 * j], w[3 * j + 1], w[3 * j + 2]);
  t[10] = fminf(w[30], w[31]);
  const float a = fmin3(t[0], t[1], t[2]);
  const float b = fmin3(t[3], t[4], t[5]);
  const float d = fmin3(t[6], t[7], t[8]);
  return (int)fmin3(fmin3(a, b, d), t[9], t[10]);
}

// Exact fallback for extreme magnitudes: equality bitmask, first set bit.
MXS_DEV int first_argmax32_exact(const float (&v)[32], float c) {
  uint32_t bits = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) bits |= (v[j] == c) ? (1u << j) : 0u;
  return __ffs(bits) - 1;
}

// Fold one 32-column chunk into the running (m, ix) of this thread's row: chunk max first,
// index search only when some lane of the warp improves (strict >, so earlier columns win ties).
MXS_DEV int first_argmax32_chain(const float (&v)[32], float c) {
  int jj = 31;
#pragma unroll
  for (int j = 30; j >= 0; --j) jj = (v[j] == c) ? j : jj;
  return jj;
}

MXS_DEV void fold_chunk(float (&v)[32], int base, int vl, float& m, int& ix, int variant = 0) {
  if (base + 32 > vl) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (base + j >= vl) v[j] = -INFINITY;
  }
  const float cmax = max32(v);
  const bool upd = cmax > m;
  if (variant == 3) {  // profiling knob: max only
    if (upd) m = cmax;
    return;
  }
  if (variant == 10 || variant == 11) {
    if (__any_sync(0xffffffffu, upd)) {
      const int jj = variant == 10 ? first_argmax32_chain(v, cmax) : first_argmax32_exact(v, cmax);
      if (upd) {
        m = cmax;
        ix = base + jj;
      }
    }
    return;
  }
  if (__any_sync(0xffffffffu, upd)) {
    const float ac = fabsf(cmax);
    const bool odd = upd && !(ac >= 0x1p-60f && ac <= 0x1p27f);
    int jj;
    if (__any_sync(0xffffffffu, odd))
      jj = first_argmax32_exact(v, cmax);
    else
      jj = first_argmax32_fast(v, cmax);
    if (upd) {
      m = cmax;
      ix = base + jj;
    }
  }
}

// Convert one 32-column TMEM chunk to fp32 similarities and fold it.
template <TcKind KIND>
MXS_DEV void epi_chunk(const uint32_t (&r)[32], int base, int vl, const FwdTcParams& p, int b, float sq, float& m,
                       int& ix) {
  const int variant = p.debug >= 3 ? p.debug : 0;
  float v[32];
  if constexpr (KIND == TcKind::I8) {
    // f32(int32 acc) rounds to nearest even like numpy's int32->float32 cast; then
    // fl(fl(acc * s_q) * s_d) in the order of maxsim/quant.py:174-176 (S7).
    const float* sd = p.d_scale + (long long)b * p.l_pad + base;
    const bool full = base + 32 <= p.l_pad;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float sdj = (full || base + j < p.l_pad) ? __ldg(sd + j) : 1.f;
      v[j] = __fmul_rn(__fmul_rn(__int2float_rn((int)r[j]), sq), sdj);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  }
  if (base < vl) fold_chunk(v, base, vl, m, ix, variant);
}

template <TcKind KIND, int KA>
__global__ void __launch_bounds__(kFwdThreads, 1)
    fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmD,
                  const FwdTcParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment by offsetting the __shared__ array itself (keeps the shared address space,
  // so accesses compile to LDS/STS rather than generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;
  uint8_t* sD = smem + (size_t)p.qb * KA * kAtomBytes;
  __shared__ FwdSmemHeader tc_hdr;
  FwdSmemHeader* hdr = &tc_hdr;

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();

  const long long per = p.n_units / gridDim.x, rem = p.n_units % gridDim.x;
  const long long u_begin = blockIdx.x * per + min((long long)blockIdx.x, rem);
  const long long u_end = u_begin + per + (blockIdx.x < rem ? 1 : 0);
  const int nmb_total = (p.l_q + kTileRows - 1) / kTileRows;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmD);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&hdr->full[s], 1);
      mbar_init(&hdr->empty[s], 1);
    }
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&hdr->tfull[s], 1);
      mbar_init(&hdr->tempty[s], 4);
    }
    mbar_init(&hdr->qfull, 1);
    mbar_init(&hdr->qempty, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(&hdr->tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = hdr->tmem_base;

  constexpr uint32_t kIdesc = (KIND == TcKind::I8) ? make_idesc(2, 1, 128, 128)
                              : (KIND == TcKind::BF16) ? make_idesc(1, 1, 128, 128)
                                                       : make_idesc(1, 0, 128, 128);

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0, qphase = 0;
      long long cur_key = -1;
      for (long long u = u_begin; u < u_end; ++u) {
        int q, g, b;
        decode_unit(u, p, q, g, b);
        const long long key = (long long)q * p.n_groups + g;
        if (key != cur_key) {
          if (cur_key >= 0) {
            mbar_wait(&hdr->qempty, qphase);
            qphase ^= 1;
          }
          const int qbv = min(p.qb, nmb_total - g * p.qb);
          mbar_arrive_expect_tx(&hdr->qfull, (uint32_t)(qbv * KA * kAtomBytes));
          for (int mb = 0; mb < qbv; ++mb)
            for (int a = 0; a < KA; ++a)
              tma_load_2d(&tmQ, &hdr->qfull, sQ + (size_t)(mb * KA + a) * kAtomBytes, a * 128 / (KIND == TcKind::I8 ? 1 : 2),
                          q * p.l_q + (g * p.qb + mb) * kTileRows, kEvictLast);
          cur_key = key;
        }
        const int vl = doc_valid_len(p, b);
        const int ntiles = (vl + kTileRows - 1) / kTileRows;
        for (int t = 0; t < ntiles; ++t) {
          mbar_wait(&hdr->empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&hdr->full[stage], (uint32_t)(KA * kAtomBytes));
          for (int a = 0; a < KA; ++a)
            tma_load_2d(&tmD, &hdr->full[stage], sD + (size_t)(stage * KA + a) * kAtomBytes,
                        a * 128 / (KIND == TcKind::I8 ? 1 : 2), b * p.l_pad + t * kTileRows, kEvictNormal);
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    // The whole warp walks the schedule (warp-uniform state, uniform registers); one elected
    // lane issues each MMA chain.  Descriptors are a base plus compile-time K offsets, so the
    // issue loop is a handful of uniform adds per tcgen05.mma.
    // Q block mb belongs to epilogue set (mb & 1); that set alternates between its two slots
    // {set, set + 2}, so every slot's phases are consumed in order by one set (no parity aliasing).
    int stage = 0;
    uint32_t phase = 0, qphase = 0;
    uint32_t uses[2] = {0u, 0u};
    long long cur_key = -1;
    const uint64_t qdesc0 = sw128_kmajor_desc(smem_u32(sQ));
    const uint64_t ddesc0 = sw128_kmajor_desc(smem_u32(sD));
    for (long long u = u_begin; u < u_end; ++u) {
      int q, g, b;
      decode_unit(u, p, q, g, b);
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
          const int set = mb & 1;
          const int slot = set + 2 * (int)(uses[set] & 1u);
          const uint32_t sphase = (uses[set] >> 1) & 1u;
          ++uses[set];
          mbar_wait(&hdr->tempty[slot], sphase ^ 1);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t ad0 = qdesc0 + (uint64_t)((mb * KA * kAtomBytes) >> 4);
            const uint32_t dcol = tmem_base + (uint32_t)(slot * 128);
#pragma unroll
            for (int k = 0; k < KA * 4; ++k) {
              const uint64_t koff = (uint64_t)(((k >> 2) * kAtomBytes + (k & 3) * 32) >> 4);
              if constexpr (KIND == TcKind::I8)
                mma_i8_ss(dcol, ad0 + koff, bd0 + koff, kIdesc, k > 0 ? 1u : 0u);
              else
                mma_f16_ss(dcol, ad0 + koff, bd0 + koff, kIdesc, k > 0 ? 1u : 0u);
            }
            mma_commit(&hdr->tfull[slot]);
          }
          __syncwarp();
        }
        if (elect_one()) mma_commit(&hdr->empty[stage]);
        __syncwarp();
        if (++stage == p.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ epilogue
    // Warp set `wset` (warps 4-7 or 8-11) owns the Q blocks mb with (mb & 1) == wset; warp
    // (warp & 3) of a set reads TMEM lanes [32*(warp&3), +32), i.e. one Q row per thread.
    const int wset = ((int)warp - 4) >> 2;
    const int quad = (int)(warp & 3);
    const int row_local = quad * 32 + (int)lane;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    uint32_t uses = 0;  // slot uses by this set: slot = wset + 2 * (uses & 1), parity = (uses >> 1) & 1
    for (long long u = u_begin; u < u_end; ++u) {
      int q, g, b;
      decode_unit(u, p, q, g, b);
      const int qbv = min(p.qb, nmb_total - g * p.qb);
      const int vl = doc_valid_len(p, b);
      const int ntiles = (vl + kTileRows - 1) / kTileRows;
      float m[2];
      int ix[2];
      float sq[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        m[i] = -INFINITY;
        ix[i] = 0;
        sq[i] = 1.f;
        if constexpr (KIND == TcKind::I8) {
          const int mb = 2 * i + wset;
          const int row = (g * p.qb + mb) * kTileRows + row_local;
          if (mb < qbv && row < p.l_q) sq[i] = __ldg(p.q_scale + (long long)q * p.l_q + row);
        }
      }
      for (int t = 0; t < ntiles; ++t) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int mb = 2 * i + wset;
          if (mb >= qbv) break;
          const uint32_t slot = (uint32_t)wset + 2u * (uses & 1u), sphase = (uses >> 1) & 1u;
          ++uses;
          mbar_wait(&hdr->tfull[slot], sphase);
          tc_fence_after();
          const uint32_t taddr = tmem_base + lane_base + slot * 128u;
          const int base = t * kTileRows;
          if (p.debug == 1 || p.debug == 2) {
            if (p.debug == 1) {
              uint32_t ra[32], rb[32];
              tmem_ld32(taddr, ra);
              tmem_ld32(taddr + 32, rb);
              tmem_ld32(taddr + 64, ra);
              tmem_ld32(taddr + 96, rb);
              tmem_ld_wait();
              m[i] = fmaxf(m[i], __uint_as_float(ra[0] ^ rb[31]));
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&hdr->tempty[slot]);
          } else if constexpr (KIND == TcKind::I8) {
            // lower register pressure: two chunks in flight at a time
            uint32_t ra[32], rb[32];
            tmem_ld32(taddr, ra);
            tmem_ld32(taddr + 32, rb);
            tmem_ld_wait();
            epi_chunk<KIND>(ra, base, vl, p, b, sq[i], m[i], ix[i]);
            epi_chunk<KIND>(rb, base + 32, vl, p, b, sq[i], m[i], ix[i]);
            tmem_ld32(taddr + 64, ra);
            tmem_ld32(taddr + 96, rb);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&hdr->tempty[slot]);
            epi_chunk<KIND>(ra, base + 64, vl, p, b, sq[i], m[i], ix[i]);
            epi_chunk<KIND>(rb, base + 96, vl, p, b, sq[i], m[i], ix[i]);
          } else {
            uint32_t ra[32], rb[32], rc[32], rd[32];
            tmem_ld32(taddr, ra);
            tmem_ld32(taddr + 32, rb);
            tmem_ld_wait();
            tmem_ld32(taddr + 64, rc);
            tmem_ld32(taddr + 96, rd);
            epi_chunk<KIND>(ra, base, vl, p, b, sq[i], m[i], ix[i]);
            epi_chunk<KIND>(rb, base + 32, vl, p, b, sq[i], m[i], ix[i]);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&hdr->tempty[slot]);
            epi_chunk<KIND>(rc, base + 64, vl, p, b, sq[i], m[i], ix[i]);
            epi_chunk<KIND>(rd, base + 96, vl, p, b, sq[i], m[i], ix[i]);
          }
        }
      }
      const long long obase = ((long long)q * p.n_docs + b) * p.l_q;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int mb = 2 * i + wset;
        if (mb >= qbv) break;
        const int row = (g * p.qb + mb) * kTileRows + row_local;
        if (row < p.l_q) {
          p.rowmax[obase + row] = m[i];
          if (p.argmax) p.argmax[obase + row] = ix[i];
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace mxs
