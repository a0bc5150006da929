// Padding-free (cu_seqlens) MaxSim forward on tcgen05, v2 (K5) -- maxsim/varlen.py:88-131.
//
// Query rows live in the TMEM lanes, packed document tokens in the TMEM columns:
//   A = the n_cols = n_q * l_q (<= 128) query rows, replicated C = 128 / round_up(n_cols) times
//       (C = 4 for ColBERT's L_q = 32) so that every TMEM lane quadrant holds real rows;
//   B = a tile of 128 consecutive packed tokens (TMA from the [total_tokens, dim] buffer);
//   D = [128 lanes x 128 tokens] fp32 in one of four TMEM slots (slot = tile % 4, so each scan
//       set double-buffers and the MMA runs up to two tiles ahead of the drain).
// Copy k of the rows scans token range k of the tile (128 / C tokens): each epilogue thread owns
// one query row and folds the range's tokens IN ORDER straight out of its registers
// (tcgen05.ld), keeping (max, first argmax) per document piece -- strict >, so the earliest
// token wins ties (S3).  No transpose, no cross-thread scan.
// Document boundaries are warp-uniform (every row sees the same tokens).  A dedicated warp
// walks cu_seqlens ahead of the epilogue and publishes, per tile, the document holding the
// first token and a 128-bit "a document starts at this token" mask (one ballot per 32 docs).
// Pieces that cross a range edge are merged in token order (head pieces into the running
// carry, strict > so earlier tokens win) by one merge warp per 32 query rows, which walks all
// tiles in order and keeps the carry in registers; the two scan warp sets take alternate tiles.
// CTAs own contiguous, token-balanced document ranges (binary search of cu_seqlens on the
// device), so every document is finished by exactly one CTA: no atomics, no second pass.
// HBM-bound: L_q = 32 gives 32 FLOP/B; the MMA is a fraction of the per-tile HBM time.
// Fused S4 score (query length dividing 32): every emission site is warp-uniform and a warp holds
// 32 consecutive query rows, so the L_q maxima of a (query, document) pair meet in one warp and
// are folded there by a segmented certified f64 sum (score_sum.cuh) -- no row maxima in HBM.
#pragma once
#include "fwd_tc.cuh"
#include "score_sum.cuh"

namespace mxs {

struct VarlenRowsParams {
  int n_q, l_q, n_cols;  // this launch: flattened query rows [row0, row0 + n_cols), n_cols <= 128
  int row0;
  int copies;            // row replication C (4, 2 or 1)
  long long n_docs, n_tokens;
  int dim;
  int stages;
  const long long* cu;  // [n_docs + 1] device
  float* rowmax;        // [n_q, n_docs, l_q] or nullptr (fused score)
  int32_t* argmax;      // [n_q, n_docs, l_q] or nullptr
  double* scores;       // [n_q, n_docs]: fused S4 score (l_q divides 32), or nullptr
};

constexpr int kVrTile = 128;       // tokens per tile (MMA N)
constexpr int kVrThreads = 32 * 15;  // warp 0 TMA, 1 MMA + TMEM, 2..9 scan, 10 boundaries, 11..14 merge
constexpr int kVrSumWarp = 12;       // fused kernels (n_cols <= 32, merge warps 12..14 idle): S4 sum warp
constexpr int kVrSlotCols = 128;
constexpr int kVrSlots = 4;
constexpr int kVrInfoSlots = 16;
constexpr int kVrPieceBufs = 4;

struct VrInfo {  // per tile, written by the boundary warp
  long long d_first;       // document holding the tile's first token
  long long dstart_first;  // its first token
  uint32_t words[4];       // bit x: token p0 + x starts a document
};

struct VrShared {
  VrInfo info[kVrInfoSlots];
  // head / tail pieces of every (token range k, query row) of a tile at [k * 128 / C + row],
  // per set, in a ring of kVrPieceBufs buffers so that the scan runs ahead of the merge
  float hm[2][kVrPieceBufs][128];
  float tm[2][kVrPieceBufs][128];
  int16_t ha[2][kVrPieceBufs][128];  // token offset in the tile
  int16_t ta[2][kVrPieceBufs][128];
};

struct VrSmemHeader {
  uint64_t full[8];
  uint64_t empty[8];
  uint64_t tfull[kVrSlots];
  uint64_t tempty[kVrSlots];
  uint64_t qfull;
  uint64_t ifull[kVrInfoSlots];
  uint64_t iempty[kVrInfoSlots];
  uint64_t pfull[2][kVrPieceBufs];   // [set][buffer]: the set's scan warps wrote their pieces
  uint64_t pempty[2][kVrPieceBufs];  // [set][buffer]: the merge warps consumed them
  uint32_t tmem_base;
  int32_t pad;
  long long doc_begin, doc_end, tok_begin, tok_end;
};

__host__ __device__ inline size_t varlen_rows_smem_bytes(int ka, int stages) {
  return 1024 + (size_t)(stages + 1) * ka * kAtomBytes + sizeof(VrShared);
}

// first document d in [lo, hi) with cu[d + 1] > tok (the document containing token tok)
MXS_DEV long long vr_doc_of_token(const long long* cu, long long lo, long long hi, long long tok) {
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (__ldg(cu + mid + 1) > tok)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

// output offset of (query row, document 0); rows >= n_cols get -1 (nothing is written)
MXS_DEV long long vr_row_base(const VarlenRowsParams& p, int row) {
  if (row >= p.n_cols) return -1;
  const int r = p.row0 + row;
  const int q = r / p.l_q, i = r - q * p.l_q;
  return (long long)q * p.n_docs * p.l_q + i;
}
// Fused S4 ring (fused kernels only, n_cols <= 32: one emission = one document for ALL query
// rows).  The emitting scan / merge warp only stores its 32 row maxima into a slot of this ring
// and arrives on the slot's mbarrier (a few instructions); the sum warp folds the slots in
// allocation order, waiting on the mbarriers with the suspend hint so that it takes no issue slots
// from the scan / merge warps.  Putting the warp reduction itself at the emission sites cost the
// HBM-bound scan ~50 %.
constexpr int kVrRing = 32;
struct VrRing {
  float m[kVrRing][32];
  long long doc[kVrRing];
  uint64_t full[kVrRing];   // 32 arrivals: the emitting warp's lanes wrote slot k % kVrRing
  uint64_t empty[kVrRing];  // 1 arrival: the sum warp consumed it
  uint32_t tail;            // emissions allocated so far
};
__shared__ VrRing vr_ring;

MXS_DEV void vr_push(long long doc, float m) {
  if (doc < 0) return;  // warp-uniform
  const uint32_t lane = lane_id();
  uint32_t k = 0;
  if (lane == 0) k = atomicAdd(&vr_ring.tail, 1u);
  k = __shfl_sync(0xffffffffu, k, 0);
  const uint32_t s = k % kVrRing, gen = k / kVrRing;
  mbar_wait(&vr_ring.empty[s], (gen & 1u) ^ 1u);  // the slot's previous generation was consumed
  vr_ring.m[s][lane] = m;
  if (lane == 0) vr_ring.doc[s] = doc;
  mbar_arrive(&vr_ring.full[s]);  // release: orders this lane's stores
}

// Sum warp: the CTA's documents in emission order; per slot, the S4 score of every query whose
// l_q rows are lanes [k * l_q, (k + 1) * l_q) (l_q divides 32, rows = lanes < n_cols).
MXS_DEV void vr_sum_warp(const VarlenRowsParams& p, long long n_emit) {
  const int lane = (int)lane_id();
  const int seg = p.l_q;
  const bool valid = lane < p.n_cols;
  const bool lead = valid && (lane & (seg - 1)) == 0;
  for (long long n = 0; n < n_emit; ++n) {
    const uint32_t s = (uint32_t)(n % kVrRing), gen = (uint32_t)(n / kVrRing);
    mbar_wait_idle(&vr_ring.full[s], gen & 1u);
    const float m = vr_ring.m[s][lane];
    const long long doc = vr_ring.doc[s];
    // certified exact sum in integer fixed point (score_sum.cuh), per segment of seg lanes
    const uint32_t bits = valid ? __float_as_uint(m) : 0u;
    int emin = 255, emax = 0;
    bool finb = true;
    exp_range(bits, emin, emax, finb);
    int fin = finb ? 1 : 0;
    for (int o = seg >> 1; o; o >>= 1) {  // segmented butterfly: xor offsets < seg stay in the segment
      emin = min(emin, __shfl_xor_sync(0xffffffffu, emin, o));
      emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
      fin = min(fin, __shfl_xor_sync(0xffffffffu, fin, o));
    }
    const bool ex = certified(emin, emax, fin != 0, seg);
    const int S = fix_shift(seg);
    long long k = fix_term(bits, emax, S);
    for (int o = seg >> 1; o; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
    double sc = fix_to_double(k, emax, S);
    if (__any_sync(0xffffffffu, lead && !ex)) {  // sequential chain (rare): the reference order
      double t = 0.0;
      for (int i = 0; i < seg; ++i) {
        const float v = __shfl_sync(0xffffffffu, m, (lane & ~(seg - 1)) + i);
        t = (i == 0) ? (double)v : __dadd_rn(t, (double)v);
      }
      if (!ex) sc = t;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&vr_ring.empty[s]);  // every lane has consumed its value (c / sc above)
    if (lead) p.scores[(long long)((p.row0 + lane) / seg) * p.n_docs + doc] = sc;
  }
}

// FUSED is a compile-time choice: the non-fused kernels carry no trace of the warp reduction (its
// mere presence at the emission sites cost the HBM-bound scan ~40 % through code generation).
template <bool FUSED>
MXS_DEV void vr_emit(const VarlenRowsParams& p, long long rbase, long long doc, float m, long long arg_local) {
  if constexpr (FUSED) vr_push(doc, m);
  if (rbase < 0 || doc < 0) return;
  const long long o = rbase + doc * p.l_q;
  if (p.rowmax) p.rowmax[o] = m;
  if (p.argmax) p.argmax[o] = (int32_t)arg_local;
}

// bits of the 128-bit mask at positions [lo, hi) (0 <= lo <= hi <= 128)
MXS_DEV int vr_popc_range(const uint32_t (&w)[4], int lo, int hi) {
  int n = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int a = max(lo - 32 * i, 0), b = min(hi - 32 * i, 32);
    if (a < b) {
      const uint32_t mk = (b == 32 ? 0xffffffffu : ((1u << b) - 1u)) & ~((1u << a) - 1u);
      n += __popc(w[i] & mk);
    }
  }
  return n;
}
// highest set position in [lo, hi), or -1
MXS_DEV int vr_last_bit(const uint32_t (&w)[4], int lo, int hi) {
  int r = -1;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int a = max(lo - 32 * i, 0), b = min(hi - 32 * i, 32);
    if (a < b) {
      const uint32_t mk = (b == 32 ? 0xffffffffu : ((1u << b) - 1u)) & ~((1u << a) - 1u);
      const uint32_t x = w[i] & mk;
      if (x) r = 32 * i + 31 - __clz(x);
    }
  }
  return r;
}
MXS_DEV bool vr_bit(const uint32_t (&w)[4], int x) { return (w[x >> 5] >> (x & 31)) & 1u; }

// Scan warp (set, lane quadrant): token range k of the tiles t = set (mod 2), its 32 query rows.
// Documents that start and end inside the range are written out directly; the range's head
// piece (before its first document start) and tail piece (from its last start) go to shared
// memory for the merge warp.
template <TcKind KIND, int KA, int C, bool FUSED>
MXS_DEV void vr_scan(const VarlenRowsParams& p, VrSmemHeader* hdr, VrShared* sh, uint32_t tmem_base, int set,
                     int quad, uint32_t lane, int n_tiles, long long tok_begin, long long tok_end) {
  constexpr int L = kVrTile / C;        // tokens per range
  constexpr int QPC = 4 / C;            // lane quadrants per row copy
  const int k = quad / QPC;             // token range (row copy) of this warp
  const int j = quad % QPC;             // row block within the copy
  const int row = j * 32 + (int)lane;   // query row
  if (j * 32 >= p.n_cols) return;       // no real rows in this quadrant
  const long long rbase = vr_row_base(p, row);
  const int pidx = k * (kVrTile / C) + row;  // piece slot of (range k, row)
  const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
  const int x0 = k * L;
  for (int t = set; t < n_tiles; t += 2) {
    const long long p0 = tok_begin + (long long)t * kVrTile;
    const int ntok = (int)min((long long)kVrTile, tok_end - p0);
    const int islot = t % kVrInfoSlots;
    mbar_wait(&hdr->ifull[islot], ((uint32_t)t / kVrInfoSlots) & 1u);
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = sh->info[islot].words[i];
    const long long d_first = sh->info[islot].d_first;
    const long long dstart_first = sh->info[islot].dstart_first;
    __syncwarp();
    if (lane == 0) mbar_arrive(&hdr->iempty[islot]);
    const uint32_t slot = (uint32_t)t & (kVrSlots - 1);  // = set or set + 2
    const int pb = (t >> 1) % kVrPieceBufs;
    const int x1 = min(x0 + L, ntok);
    float m = -INFINITY, hm = -INFINITY;
    int a = 0, ha = 0;
    mbar_wait(&hdr->tfull[slot], ((uint32_t)t >> 2) & 1u);
    tc_fence_after();
    if (x0 < ntok) {
      long long doc = d_first + vr_popc_range(w, 1, x0 + 1);
      const int lb = vr_last_bit(w, 1, x0 + 1);
      long long dstart = (lb >= 0) ? p0 + lb : dstart_first;
      bool in_head = !vr_bit(w, x0);
      const uint32_t taddr = tmem_base + lane_base + slot * kVrSlotCols + (uint32_t)x0;
#pragma unroll
      for (int cc = 0; cc < L / 32; ++cc) {
        uint32_t r[32];
        tmem_ld32(taddr + cc * 32, r);
        tmem_ld_wait();
        if (cc == L / 32 - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&hdr->tempty[slot]);
        }
        const int xb = x0 + cc * 32;
        if (xb < x1) {
          uint32_t word = w[xb >> 5];
          if (cc == 0) word &= ~1u;  // a start at x0 itself is the range's own first document
          if (word == 0u && xb + 32 <= x1) {
#pragma unroll
            for (int q = 0; q < 32; ++q) {  // branch-free strict-> fold in token order
              const float v = __uint_as_float(r[q]);
              a = (v > m) ? xb + q : a;
              m = fmaxf(m, v);
            }
          } else {
            const int nv = min(32, x1 - xb);
            uint32_t starts = word & (nv >= 32 ? 0xffffffffu : ((1u << nv) - 1u));
            if (__popc(starts) <= 1) {
              // Common case (documents of >= 32 tokens): one start in the chunk.  Single in-order
              // pass; the document it closes is emitted after the unrolled loop, so the emission
              // code exists once.
              bool pend = false;
              float pm = -INFINITY;
              int pa = 0;
              long long pdoc = 0, pds = 0;
#pragma unroll
              for (int q = 0; q < 32; ++q) {
                if (q < nv) {
                  if ((starts >> q) & 1u) {  // token xb + q starts document doc + 1 (warp-uniform)
                    if (in_head) {
                      hm = m;
                      ha = a;
                      in_head = false;
                    } else {  // complete inside this range
                      pend = true;
                      pm = m;
                      pa = a;
                      pdoc = doc;
                      pds = dstart;
                    }
                    ++doc;
                    dstart = p0 + xb + q;
                    m = -INFINITY;
                    a = 0;
                  }
                  const float v = __uint_as_float(r[q]);
                  if (v > m) {
                    m = v;
                    a = xb + q;
                  }
                }
              }
              if (pend) vr_emit<FUSED>(p, rbase, pdoc, pm, p0 + pa - pds);
            } else {
              // Several starts (documents shorter than a range): one rolled iteration per piece,
              // tokens [s, e) folded in order by a predicated unrolled pass (r[] stays in
              // registers), then the document ending at start e is closed.
              int s = 0;
#pragma unroll 1
              for (;;) {
                const int e = starts ? __ffs((int)starts) - 1 : nv;
                const uint32_t seg = (e >= 32 ? 0xffffffffu : ((1u << e) - 1u)) & ~((1u << s) - 1u);
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                  const float v = __uint_as_float(r[q]);
                  if (((seg >> q) & 1u) && v > m) {
                    m = v;
                    a = xb + q;
                  }
                }
                if (!starts) break;
                if (in_head) {
                  hm = m;
                  ha = a;
                  in_head = false;
                } else {
                  vr_emit<FUSED>(p, rbase, doc, m, p0 + a - dstart);
                }
                ++doc;
                dstart = p0 + xb + e;
                m = -INFINITY;
                a = 0;
                starts &= starts - 1u;
                s = e;
              }
            }
          }
        }
      }
      if (in_head) {  // no document starts in this range: the whole range is one head piece
        hm = m;
        ha = a;
      }
    } else {
      // empty range (short last tile): still release the TMEM slot
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&hdr->tempty[slot]);
    }
    // hand the pieces to the merge warp (the buffer's previous tile must have been merged)
    const uint32_t use = ((uint32_t)t >> 1) / kVrPieceBufs;  // t = set + 2 * (pb + kVrPieceBufs * use)
    mbar_wait(&hdr->pempty[set][pb], (use & 1u) ^ 1u);
    sh->hm[set][pb][pidx] = hm;
    sh->ha[set][pb][pidx] = (int16_t)ha;
    sh->tm[set][pb][pidx] = m;
    sh->ta[set][pb][pidx] = (int16_t)a;
    mbar_arrive(&hdr->pfull[set][pb]);  // every lane (release of its own stores)
  }
}

// Fold the C token ranges of one tile for one query row, in token order, without the carry:
// the tile head (tokens before the tile's first document start) and the piece after its last
// start are returned; documents lying between two starts are written out here.
struct VrTileFold {
  bool seen = false;        // a document starts somewhere in the tile
  float thm = -INFINITY;    // tile head
  int tha = 0;
  float pm = -INFINITY;     // piece after the latest start
  int pa = 0, plast = 0;    // its max position and its start (tile offsets)
  long long pd = 0;         // its document
};
template <int C, bool FULL, bool FUSED>
MXS_DEV void vr_fold_ranges(VrTileFold& f, const float* hm, const int16_t* ha, const float* tm, const int16_t* ta,
                            const uint32_t (&w)[4], long long d_first, int ntok, int row, const VarlenRowsParams& p,
                            long long rbase) {
  constexpr int L = kVrTile / C;
  float h[C], tl[C];
  int hx[C], tx[C];
#pragma unroll
  for (int kk = 0; kk < C; ++kk) {  // all loads first (independent LDS)
    h[kk] = hm[kk * L + row];
    hx[kk] = ha[kk * L + row];
    tl[kk] = tm[kk * L + row];
    tx[kk] = ta[kk * L + row];
  }
#pragma unroll
  for (int kk = 0; kk < C; ++kk) {
    const int r0 = kk * L;
    if (!FULL && r0 >= ntok) break;
    const int r1 = FULL ? r0 + L : min(r0 + L, ntok);
    const bool st = vr_bit(w, r0);
    const bool nb = vr_popc_range(w, r0 + 1, r1) > 0;
    if (!st) {  // the range's head continues the current piece (strict >: earlier tokens win)
      if (!f.seen) {
        if (h[kk] > f.thm) {
          f.thm = h[kk];
          f.tha = hx[kk];
        }
      } else if (h[kk] > f.pm) {
        f.pm = h[kk];
        f.pa = hx[kk];
      }
    }
    if (st || nb) {  // the current piece ends at the range's first start
      if (f.seen) vr_emit<FUSED>(p, rbase, f.pd, f.pm, f.pa - f.plast);
      f.seen = true;
      f.plast = vr_last_bit(w, r0, r1);
      f.pd = d_first + vr_popc_range(w, 1, r1);
      f.pm = tl[kk];
      f.pa = tx[kk];
    }
  }
}

// Merge warp for query rows [32 j, 32 j + 32): walks ALL tiles in order, folds the ranges of each
// tile (token order, strict >) and carries the document still open at the tile's end in
// registers -- the only serial work of the kernel, ~100 instructions per tile.
template <int C, bool FUSED>
MXS_DEV void vr_merge(const VarlenRowsParams& p, VrSmemHeader* hdr, VrShared* sh, int j, uint32_t lane, int n_tiles,
                      long long tok_begin, long long tok_end) {
  constexpr int L = kVrTile / C;
  const int row = j * 32 + (int)lane;
  if (j * 32 >= p.n_cols) return;
  const long long rbase = vr_row_base(p, row);
  float cm = -INFINITY;
  long long ca = 0, cd = -1, cs = 0;
  for (int t = 0; t < n_tiles; ++t) {
    const long long p0 = tok_begin + (long long)t * kVrTile;
    const int ntok = (int)min((long long)kVrTile, tok_end - p0);
    const int islot = t % kVrInfoSlots;
    mbar_wait(&hdr->ifull[islot], ((uint32_t)t / kVrInfoSlots) & 1u);
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = sh->info[islot].words[i];
    const long long d_first = sh->info[islot].d_first;
    __syncwarp();
    if (lane == 0) mbar_arrive(&hdr->iempty[islot]);
    const int set = t & 1, pb = (t >> 1) % kVrPieceBufs;
    mbar_wait(&hdr->pfull[set][pb], (((uint32_t)t >> 1) / kVrPieceBufs) & 1u);
    VrTileFold f;
    if (ntok == kVrTile)
      vr_fold_ranges<C, true, FUSED>(f, sh->hm[set][pb], sh->ha[set][pb], sh->tm[set][pb], sh->ta[set][pb], w, d_first,
                              kVrTile, row, p, rbase);
    else
      vr_fold_ranges<C, false, FUSED>(f, sh->hm[set][pb], sh->ha[set][pb], sh->tm[set][pb], sh->ta[set][pb], w, d_first,
                               ntok, row, p, rbase);
    mbar_arrive(&hdr->pempty[set][pb]);  // every lane (its reads are done)
    if (!vr_bit(w, 0) && (f.thm > cm || cd < 0)) {  // the tile head continues the carried document
      cm = f.thm;
      ca = p0 + f.tha;
    }
    if (f.seen) {  // the carried document ended at the tile's first start
      vr_emit<FUSED>(p, rbase, cd, cm, ca - cs);
      cm = f.pm;
      ca = p0 + f.pa;
      cd = f.pd;
      cs = p0 + f.plast;
    }
  }
  if (n_tiles > 0) vr_emit<FUSED>(p, rbase, cd, cm, ca - cs);  // the CTA's last document ends at tok_end
}

template <TcKind KIND, int KA, bool FUSED>
__global__ void __launch_bounds__(kVrThreads, 1)
    varlen_rows_kernel(const __grid_constant__ CUtensorMap tmT, const __grid_constant__ CUtensorMap tmQ,
                       const VarlenRowsParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;                                       // A operand: 128 (replicated) query rows
  uint8_t* sT = sQ + (size_t)KA * kAtomBytes;               // token tile ring
  VrShared* sh = reinterpret_cast<VrShared*>(sT + (size_t)p.stages * KA * kAtomBytes);
  __shared__ VrSmemHeader vr_hdr;
  VrSmemHeader* hdr = &vr_hdr;
  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const int C = p.copies;
  const int n_merge = (p.n_cols + 31) >> 5;       // merge warps (one per 32 query rows)
  const int n_active = C * n_merge;               // scan warps per set holding real rows

  if (threadIdx.x == 0) {
    // token-balanced contiguous document range of this CTA
    const long long total = __ldg(p.cu + p.n_docs);
    const long long t0 = total * blockIdx.x / gridDim.x;
    const long long t1 = total * (blockIdx.x + 1) / gridDim.x;
    const long long d0 = (blockIdx.x == 0) ? 0 : vr_doc_of_token(p.cu, 0, p.n_docs, t0 - 1) + 1;
    long long d1 = (blockIdx.x + 1 == gridDim.x) ? p.n_docs : vr_doc_of_token(p.cu, 0, p.n_docs, t1 - 1) + 1;
    if (d1 < d0) d1 = d0;
    hdr->doc_begin = d0;
    hdr->doc_end = d1;
    hdr->tok_begin = __ldg(p.cu + d0);
    hdr->tok_end = __ldg(p.cu + d1);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&hdr->full[s], 1);
      mbar_init(&hdr->empty[s], 1);
    }
    for (int s = 0; s < kVrSlots; ++s) {
      mbar_init(&hdr->tfull[s], 1);
      mbar_init(&hdr->tempty[s], (uint32_t)n_active);
    }
    mbar_init(&hdr->qfull, 1);
    for (int s = 0; s < kVrInfoSlots; ++s) {
      mbar_init(&hdr->ifull[s], 1);
      mbar_init(&hdr->iempty[s], (uint32_t)(n_active + n_merge));  // scan warps of the set + merge warps
    }
    for (int s = 0; s < 2; ++s)
      for (int b = 0; b < kVrPieceBufs; ++b) {
        mbar_init(&hdr->pfull[s][b], 32u * (uint32_t)n_active);  // all lanes of the scan warps
        mbar_init(&hdr->pempty[s][b], 32u * (uint32_t)n_merge);  // all lanes of the merge warps
      }
    fence_mbar_init();
  }
  if constexpr (FUSED) {
    if (warp == kVrSumWarp) {
      mbar_init(&vr_ring.full[lane], 32);
      mbar_init(&vr_ring.empty[lane], 1);
      if (lane == 0) vr_ring.tail = 0u;
      fence_mbar_init();
    }
  }
  if (warp == 1) tmem_alloc(&hdr->tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = hdr->tmem_base;
  const long long tok_begin = hdr->tok_begin, tok_end = hdr->tok_end;
  const int n_tiles = (int)((tok_end - tok_begin + kVrTile - 1) / kVrTile);
  constexpr int kElemsPerAtom = 64;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0 && n_tiles > 0) {
      tma_prefetch_desc(&tmT);
      const int rpc = kVrTile / C;  // rows per copy
      mbar_arrive_expect_tx(&hdr->qfull, (uint32_t)(KA * kAtomBytes));
      for (int a = 0; a < KA; ++a)
        for (int c = 0; c < C; ++c)
          tma_load_2d(&tmQ, &hdr->qfull, sQ + (size_t)a * kAtomBytes + (size_t)c * rpc * 128, a * kElemsPerAtom, 0,
                      kEvictLast);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < n_tiles; ++t) {
        mbar_wait_idle(&hdr->empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&hdr->full[stage], (uint32_t)(KA * kAtomBytes));
        for (int a = 0; a < KA; ++a)
          tma_load_2d(&tmT, &hdr->full[stage], sT + (size_t)(stage * KA + a) * kAtomBytes, a * kElemsPerAtom,
                      (int)(tok_begin + (long long)t * kVrTile), kEvictFirst);
        if (++stage == p.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (n_tiles > 0) {
      constexpr uint32_t kIdesc = (KIND == TcKind::BF16) ? make_idesc(1, 1, 128, kVrTile)
                                                         : make_idesc(1, 0, 128, kVrTile);
      mbar_wait_idle(&hdr->qfull, 0);
      tc_fence_after();
      const uint64_t qdesc0 = sw128_kmajor_desc(smem_u32(sQ));
      const uint64_t tdesc0 = sw128_kmajor_desc(smem_u32(sT));
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < n_tiles; ++t) {
        const int slot = t & (kVrSlots - 1);
        mbar_wait_idle(&hdr->full[stage], phase);
        mbar_wait_idle(&hdr->tempty[slot], (((uint32_t)t >> 2) & 1u) ^ 1u);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t bd0 = tdesc0 + (uint64_t)((stage * KA * kAtomBytes) >> 4);
          const uint32_t dcol = tmem_base + (uint32_t)(slot * kVrSlotCols);
#pragma unroll
          for (int k = 0; k < KA * 4; ++k) {
            const uint64_t koff = (uint64_t)(((k >> 2) * kAtomBytes + (k & 3) * 32) >> 4);
            mma_f16_ss(dcol, qdesc0 + koff, bd0 + koff, kIdesc, k > 0 ? 1u : 0u);
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
  } else if (warp == 10) {
    // ------------------------------------------------------------------ boundary producer
    // Walks cu_seqlens once, ahead of the epilogue: per tile, the document holding its first
    // token and the 128-bit mask of document starts.  cu lines are reused across many tiles,
    // so the loads are L1 hits in the common case.
    const long long doc_end = hdr->doc_end;
    long long base = hdr->doc_begin;  // cu[base] <= first token of the next tile
    for (int t = 0; t < n_tiles; ++t) {
      const long long p0 = tok_begin + (long long)t * kVrTile;
      const long long pe = min(p0 + kVrTile, tok_end);
      const int islot = t % kVrInfoSlots;
      mbar_wait_idle(&hdr->iempty[islot], (((uint32_t)t / kVrInfoSlots) & 1u) ^ 1u);
      long long c;
      int n;
      for (;;) {  // document holding p0: last lane with cu <= p0
        const long long dd = base + lane;
        c = (dd <= doc_end) ? __ldg(p.cu + dd) : LLONG_MAX;
        n = __popc(__ballot_sync(0xffffffffu, c <= p0));  // >= 1
        if (n < 32) break;
        base += 31;
      }
      base += n - 1;
      const long long dstart = __shfl_sync(0xffffffffu, c, n - 1);
      uint32_t wd[4] = {0u, 0u, 0u, 0u};
      if (dstart == p0) wd[0] = 1u;
      // starts after p0: lanes >= n of this window, then further windows while all are inside
      bool more = true;
      bool first = true;
      long long wbase = base - (n - 1);
      while (more) {
        if (!first) {
          const long long dd = wbase + lane;
          c = (dd <= doc_end) ? __ldg(p.cu + dd) : LLONG_MAX;
        }
        const bool valid = first ? ((int)lane >= n) : true;
        const bool in = valid && c < pe && c > p0;
        const int pos = in ? (int)(c - p0) : 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          wd[i] |= __reduce_or_sync(0xffffffffu, (in && (pos >> 5) == i) ? (1u << (pos & 31)) : 0u);
        const long long last = __shfl_sync(0xffffffffu, c, 31);
        more = last < pe;  // the window ended inside the tile: more starts may follow
        wbase += 32;
        first = false;
      }
      if (lane == 0) {
        sh->info[islot].d_first = base;
        sh->info[islot].dstart_first = dstart;
#pragma unroll
        for (int i = 0; i < 4; ++i) sh->info[islot].words[i] = wd[i];
        mbar_arrive(&hdr->ifull[islot]);
      }
      __syncwarp();
    }
  } else if (FUSED && warp == kVrSumWarp) {
    // ------------------------------------------------------------------ fused S4 sum
    vr_sum_warp(p, hdr->doc_end - hdr->doc_begin);
  } else if (warp >= 11) {
    // ------------------------------------------------------------------ merge
    const int j = (int)warp - 11;
    if constexpr (FUSED) {  // fused kernels: n_cols <= 32 (C = 4) only
      vr_merge<4, true>(p, hdr, sh, j, lane, n_tiles, tok_begin, tok_end);
    } else {
      if (C == 4)
        vr_merge<4, false>(p, hdr, sh, j, lane, n_tiles, tok_begin, tok_end);
      else if (C == 2)
        vr_merge<2, false>(p, hdr, sh, j, lane, n_tiles, tok_begin, tok_end);
      else
        vr_merge<1, false>(p, hdr, sh, j, lane, n_tiles, tok_begin, tok_end);
    }
  } else {
    // ------------------------------------------------------------------ scan
    const int set = ((int)warp - 2) >> 2;  // tiles t with t % 2 == set, TMEM slots set and set + 2
    const int quad = (int)(warp & 3);      // TMEM lane quadrant (hardware rule: warp id % 4)
    if constexpr (FUSED) {
      vr_scan<KIND, KA, 4, true>(p, hdr, sh, tmem_base, set, quad, lane, n_tiles, tok_begin, tok_end);
    } else {
      if (C == 4)
        vr_scan<KIND, KA, 4, false>(p, hdr, sh, tmem_base, set, quad, lane, n_tiles, tok_begin, tok_end);
      else if (C == 2)
        vr_scan<KIND, KA, 2, false>(p, hdr, sh, tmem_base, set, quad, lane, n_tiles, tok_begin, tok_end);
      else
        vr_scan<KIND, KA, 1, false>(p, hdr, sh, tmem_base, set, quad, lane, n_tiles, tok_begin, tok_end);
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
