/*
 * maxsim_oracle.c -- CPU restatement of the reference Flash-MaxSim algorithm.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the sm_100a kernels; it is
 * loaded by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg, never by the
 * product path (paper_2605_29517_b200/ fails loudly without its CUDA library).
 *
 * Every function restates a reference function (paths relative to
 * /root/reference/pkg/src) with the same arithmetic order, so results are bit-identical to
 * the numpy reference on x86-64 (SSE scalar fp32/fp64, compiled with -ffp-contract=off):
 *   S1 sim[i,j]  = strict left-to-right fp32 fold of fp32 products (maxsim/kernels.py:29-38)
 *   S2 padding   = -inf before the row reduction (maxsim/forward.py:153-154)
 *   S3 argmax    = strict '>' in ascending column order, lowest index on ties (maxsim/kernels.py:69-93)
 *   S4 score     = sequential float64 sum of the fp32 row maxima (maxsim/kernels.py:22-26)
 *   S6 backward  = float64 accumulation in ascending flat source order (maxsim/backward.py:135-173)
 *   S7 int8      = fl32(maxabs/levels) (1e-12 for zero rows), rint-half-even, clamp;
 *                  sim = fl(fl(f32(acc) * s_q) * s_d) (maxsim/quant.py:104-120,171-176)
 * Pinned against golden vectors produced by the reference itself (tests/golden/).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* S1: one similarity, maxsim/kernels.py:29-38 (dot_block: out = q0*d0; out += qk*dk). */
static float dot_f32(const float* q, const float* d, int64_t dim) {
  float acc = q[0] * d[0];
  for (int64_t k = 1; k < dim; ++k) {
    float p = q[k] * d[k];
    acc = acc + p;
  }
  return acc;
}

/* S4: maxsim/kernels.py:22-26 seq_sum_f64 (np.add.accumulate in float64). */
static double seq_sum_f64(const float* v, int64_t n) {
  if (n <= 0) return 0.0;
  double s = (double)v[0];
  for (int64_t i = 1; i < n; ++i) s = s + (double)v[i];
  return s;
}

/*
 * One (query, document) pair: maxsim/forward.py:108-155 (_fold_pair) collapsed to its
 * tile-invariant result (maxsim/types.py:11-13: results are identical for every TileConfig).
 * rows = number of document rows present (l_pad for padded docs), vl = valid length.
 */
static void fold_pair_f32(const float* q, int64_t l_q, const float* d, int64_t vl, int64_t dim, float* m,
                          int32_t* arg) {
  for (int64_t i = 0; i < l_q; ++i) {
    float best = -INFINITY;
    int32_t bi = 0;
    for (int64_t j = 0; j < vl; ++j) {
      float s = dot_f32(q + i * dim, d + j * dim, dim);
      if (s > best) { /* strict replace: ties keep the earlier column */
        best = s;
        bi = (int32_t)j;
      }
    }
    m[i] = best;
    arg[i] = bi;
  }
}

/* maxsim/forward.py:221-265 fused_score_batch (padded DocBatch layout). */
int orc_fused_score_batch(const float* Q, int64_t n_q, int64_t l_q, const float* D, int64_t n_docs, int64_t l_pad,
                          int64_t dim, const int32_t* valid_lens, double* scores, int32_t* argmax) {
  float* m = (float*)malloc(sizeof(float) * (size_t)(l_q > 0 ? l_q : 1));
  int32_t* a = (int32_t*)malloc(sizeof(int32_t) * (size_t)(l_q > 0 ? l_q : 1));
  if (!m || !a) return -1;
  for (int64_t qi = 0; qi < n_q; ++qi)
    for (int64_t b = 0; b < n_docs; ++b) {
      int64_t vl = valid_lens ? valid_lens[b] : l_pad;
      fold_pair_f32(Q + qi * l_q * dim, l_q, D + b * l_pad * dim, vl, dim, m, a);
      scores[qi * n_docs + b] = seq_sum_f64(m, l_q);
      if (argmax) memcpy(argmax + (qi * n_docs + b) * l_q, a, sizeof(int32_t) * (size_t)l_q);
    }
  free(m);
  free(a);
  return 0;
}

/* maxsim/varlen.py:88-131 fused_score_varlen (packed tokens + cu_seqlens), for n_q queries. */
int orc_fused_score_varlen(const float* Q, int64_t n_q, int64_t l_q, const float* tokens, const int64_t* cu,
                           int64_t n_docs, int64_t dim, double* scores, int32_t* argmax) {
  float* m = (float*)malloc(sizeof(float) * (size_t)(l_q > 0 ? l_q : 1));
  int32_t* a = (int32_t*)malloc(sizeof(int32_t) * (size_t)(l_q > 0 ? l_q : 1));
  if (!m || !a) return -1;
  for (int64_t qi = 0; qi < n_q; ++qi)
    for (int64_t b = 0; b < n_docs; ++b) {
      fold_pair_f32(Q + qi * l_q * dim, l_q, tokens + cu[b] * dim, cu[b + 1] - cu[b], dim, m, a);
      scores[qi * n_docs + b] = seq_sum_f64(m, l_q);
      if (argmax) memcpy(argmax + (qi * n_docs + b) * l_q, a, sizeof(int32_t) * (size_t)l_q);
    }
  free(m);
  free(a);
  return 0;
}

/* maxsim/quant.py:104-120 quantize_per_token. */
int orc_quantize_per_token(const float* x, int64_t rows, int64_t dim, int levels, int8_t* q, float* scale) {
  if (levels < 1 || levels > 127) return -1;
  for (int64_t r = 0; r < rows; ++r) {
    const float* xr = x + r * dim;
    float mx = 0.0f;
    for (int64_t k = 0; k < dim; ++k) {
      float v = fabsf(xr[k]);
      if (v > mx) mx = v;
    }
    float s = mx / (float)levels;
    if (s == 0.0f) s = 1e-12f; /* ZERO_ROW_SCALE, maxsim/quant.py:27 */
    scale[r] = s;
    for (int64_t k = 0; k < dim; ++k) {
      float t = nearbyintf(xr[k] / s); /* np.round: half to even */
      if (t > (float)levels) t = (float)levels;
      if (t < -(float)levels) t = -(float)levels;
      q[r * dim + k] = (int8_t)t;
    }
  }
  return 0;
}

/* maxsim/quant.py:128-182 fused_score_int8, batched over queries and documents. */
int orc_fused_score_int8(const int8_t* Q, const float* q_scale, int64_t n_q, int64_t l_q, const int8_t* D,
                         const float* d_scale, int64_t n_docs, int64_t l_pad, int64_t dim, const int32_t* valid_lens,
                         double* scores, int32_t* argmax) {
  float* m = (float*)malloc(sizeof(float) * (size_t)(l_q > 0 ? l_q : 1));
  if (!m) return -1;
  for (int64_t qi = 0; qi < n_q; ++qi)
    for (int64_t b = 0; b < n_docs; ++b) {
      int64_t vl = valid_lens ? valid_lens[b] : l_pad;
      const int8_t* qb = Q + qi * l_q * dim;
      const int8_t* db = D + b * l_pad * dim;
      const float* sq = q_scale + qi * l_q;
      const float* sd = d_scale + b * l_pad;
      for (int64_t i = 0; i < l_q; ++i) {
        float best = -INFINITY;
        int32_t bi = 0;
        for (int64_t j = 0; j < vl; ++j) {
          int32_t acc = 0;
          for (int64_t k = 0; k < dim; ++k) acc += (int32_t)qb[i * dim + k] * (int32_t)db[j * dim + k];
          float f = (float)acc; /* int32 -> float32, round to nearest even */
          f = f * sq[i];
          f = f * sd[j];
          if (f > best) {
            best = f;
            bi = (int32_t)j;
          }
        }
        m[i] = best;
        if (argmax) argmax[(qi * n_docs + b) * l_q + i] = bi;
      }
      scores[qi * n_docs + b] = seq_sum_f64(m, l_q);
    }
  free(m);
  return 0;
}

/*
 * maxsim/backward.py:81-109 build_inverse_csr: bincount -> cumsum -> stable argsort of the
 * flat destinations (maxsim/types.py:213-216).  dest_off[b] = first destination row of doc b.
 */
int orc_build_inverse_csr(const int32_t* argmax, int64_t n_q, int64_t n_docs, int64_t l_q, const int64_t* dest_off,
                          int64_t n_dest, int64_t* row_ptr, int64_t* col_idx) {
  const int64_t n_src = n_q * n_docs * l_q;
  int64_t* cursor = (int64_t*)calloc((size_t)(n_dest + 1), sizeof(int64_t));
  if (!cursor) return -1;
  memset(row_ptr, 0, sizeof(int64_t) * (size_t)(n_dest + 1));
  for (int64_t s = 0; s < n_src; ++s) {
    int64_t b = (s / l_q) % n_docs;
    int64_t dst = dest_off[b] + argmax[s];
    if (dst < 0 || dst >= n_dest) {
      free(cursor);
      return -2;
    }
    row_ptr[dst + 1] += 1;
  }
  for (int64_t r = 0; r < n_dest; ++r) row_ptr[r + 1] += row_ptr[r];
  for (int64_t r = 0; r < n_dest; ++r) cursor[r] = row_ptr[r];
  for (int64_t s = 0; s < n_src; ++s) { /* ascending source order == stable sort */
    int64_t b = (s / l_q) % n_docs;
    int64_t dst = dest_off[b] + argmax[s];
    col_idx[cursor[dst]++] = s;
  }
  free(cursor);
  return 0;
}

/*
 * maxsim/backward.py:135-173 grad_docs_csr: dD[r] = sum over the bucket (ascending source
 * order) of g[q,b] * Q[q_row(s)], float64; q_row = (s // (B*L_q))*L_q + s % L_q.
 */
int orc_grad_docs_csr(const int64_t* row_ptr, const int64_t* col_idx, int64_t n_dest, const double* g,
                      const float* Q, int64_t n_q, int64_t n_docs, int64_t l_q, int64_t dim, double* out) {
  double* acc = (double*)malloc(sizeof(double) * (size_t)dim);
  if (!acc) return -1;
  for (int64_t r = 0; r < n_dest; ++r) {
    for (int64_t k = 0; k < dim; ++k) acc[k] = 0.0;
    for (int64_t t = row_ptr[r]; t < row_ptr[r + 1]; ++t) {
      int64_t s = col_idx[t];
      int64_t qi = s / (n_docs * l_q);
      int64_t b = (s / l_q) % n_docs;
      int64_t qrow = qi * l_q + s % l_q;
      double w = g[qi * n_docs + b];
      const float* qr = Q + qrow * dim;
      for (int64_t k = 0; k < dim; ++k) acc[k] = acc[k] + w * (double)qr[k];
    }
    memcpy(out + r * dim, acc, sizeof(double) * (size_t)dim);
  }
  free(acc);
  return 0;
}

/*
 * maxsim/backward.py:218-231 grad_query: dQ[q, s] += g[q, b] * D_b[argmax[q, b, s]], b
 * ascending, float64.  doc_row_off[b] = first row of doc b in D (padded: b*l_pad; packed: cu[b]).
 */
int orc_grad_query(const int32_t* argmax, const double* g, const float* D, const int64_t* doc_row_off, int64_t n_q,
                   int64_t n_docs, int64_t l_q, int64_t dim, double* out) {
  memset(out, 0, sizeof(double) * (size_t)(n_q * l_q * dim));
  for (int64_t qi = 0; qi < n_q; ++qi)
    for (int64_t b = 0; b < n_docs; ++b) {
      double w = g[qi * n_docs + b];
      for (int64_t s = 0; s < l_q; ++s) {
        const float* dr = D + (doc_row_off[b] + argmax[(qi * n_docs + b) * l_q + s]) * dim;
        double* o = out + (qi * l_q + s) * dim;
        for (int64_t k = 0; k < dim; ++k) o[k] = o[k] + w * (double)dr[k];
      }
    }
  return 0;
}

/*
 * Top-K with the TopKHeap / _ranked ordering (maxsim/streamio.py:230-262, maxsim/cli.py:88-92):
 * score descending, document id ascending.  Simple selection; k is small.
 */
int orc_topk(const double* scores, int64_t n, int64_t k, int64_t id_offset, double* top_s, int64_t* top_id) {
  if (k > n) return -1;
  unsigned char* taken = (unsigned char*)calloc((size_t)(n > 0 ? n : 1), 1);
  if (!taken) return -1;
  for (int64_t r = 0; r < k; ++r) {
    int64_t best = -1;
    for (int64_t i = 0; i < n; ++i) {
      if (taken[i]) continue;
      if (best < 0 || scores[i] > scores[best]) best = i; /* ascending scan keeps the lower id on ties */
    }
    taken[best] = 1;
    top_s[r] = scores[best];
    top_id[r] = best + id_offset;
  }
  free(taken);
  return 0;
}
