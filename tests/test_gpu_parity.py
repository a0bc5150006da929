"""GPU parity: every sm_100a kernel, called through the operator API / C-ABI, against the oracle.

Tolerances (BASELINE.json north_star):
  * fp32 exact kernel, INT8 scores, quantisation, all argmax / CSR indices: bit-exact
    (float argmax on the tensor-core path: rows whose oracle top-2 gap exceeds 1e-5 only);
  * BF16 / FP16 scores: within 1e-3 relative of the FP32 oracle fed the same rounded values;
  * gradients: within 1e-3 relative (max-norm) of the float64 oracle.
"""

import os

import numpy as np
import pytest
import torch

import paper_2605_29517_b200 as mx
from conftest import golden
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

REL = 1e-3
GAP = 1e-5


def cuda(x, dtype=None):
    t = torch.as_tensor(np.asarray(x)).cuda()
    return t.to(dtype) if dtype is not None else t


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def top2_gap(Q, D, valid_lens):
    """Per-(q, b, i) gap between the best and second-best similarity (float64)."""
    S = np.einsum("qid,bjd->qbij", Q.astype(np.float64), D.astype(np.float64))
    L = D.shape[1]
    mask = np.arange(L)[None, None, None, :] >= np.asarray(valid_lens)[None, :, None, None]
    S = np.where(mask, -np.inf, S)
    part = np.sort(S, axis=-1)
    gap = part[..., -1] - part[..., -2] if L > 1 else np.full(part.shape[:-1], np.inf)
    return np.where(np.isfinite(gap), gap, np.inf)


def varlen_top2_gap(Q, toks, cu):
    """float64 top-2 gap per (q, document, query row) of a packed corpus."""
    n_q, l_q, _ = Q.shape
    gap = np.full((n_q, cu.size - 1, l_q), np.inf)
    Q64 = Q.astype(np.float64)
    for d in range(cu.size - 1):
        S = np.einsum("qid,jd->qij", Q64, toks[cu[d]:cu[d + 1]].astype(np.float64))
        if S.shape[-1] > 1:
            part = np.sort(S, axis=-1)
            gap[:, d] = part[..., -1] - part[..., -2]
    return gap


@pytest.mark.parametrize("dim", [8, 16, 40, 200, 320, 512])
def test_forward_unusual_dims(dim):
    """Embedding widths off the 64-element atom (zero-filled K tail in TMA / TMEM) and past the
    resident-Q budget (d > 256 takes the SS kernel): scores within 1e-3 of the oracle, argmax
    identical where the oracle's top-2 gap is clear, rerank mode bit-identical to the argmax mode."""
    rng = np.random.default_rng(dim)
    l_q, n_docs, l_pad = 150, 20, 200
    Q = orc.make_queries(2, l_q, dim, seed=dim)
    lens = rng.integers(1, l_pad + 1, n_docs)
    D, vl = orc.padded(orc.make_corpus(n_docs, lens, dim, seed=dim + 1), l_pad)
    Qr, Dr = cuda(Q, torch.bfloat16), cuda(D, torch.bfloat16)
    sc, am, _ = mx.score_dense(Qr, Dr, cuda(vl))
    Qo, Do = Qr.float().cpu().numpy(), Dr.float().cpu().numpy()
    ref_s, ref_a = orc.fused_score_batch(Qo, Do, vl)
    assert rel_err(sc.cpu().numpy(), ref_s) < REL
    clear = top2_gap(Qo, Do, vl) > 1e-5
    assert np.array_equal(am.cpu().numpy()[clear], ref_a[clear])
    s2, _, _ = mx.score_dense(Qr, Dr, cuda(vl), want_argmax=False)
    assert torch.equal(s2, sc)


# ------------------------------------------------------------------ exact fp32 path (K10)
def test_exact_fp32_golden_bitwise():
    for name in ("fwd_ragged", "fwd_ties"):
        g = golden(name)
        docs = mx.DocBatch.from_dense(g["D"], g["valid_lens"])
        sc, am, rep = mx.fused_score_batch(cuda(g["Q"]), docs)
        assert np.array_equal(sc.numpy(), g["scores"]), name
        assert np.array_equal(am.numpy(), g["argmax"]), name
    g = golden("fwd_hand")
    s, a, _ = mx.fused_score_pair(g["q"], g["d"])
    assert s == 2.5 and a.tolist() == [0, 1]
    s, a, _ = mx.fused_score_pair(g["q"], g["d"], valid_len=1)
    assert s == 0.5 and a.tolist() == [0, 0]
    s, a, _ = mx.fused_score_pair(g["qn"], g["dn"], valid_len=2)
    assert s == -0.5 and a.tolist() == [1]


def test_exact_fp32_c1_config_bitwise_and_ledger():
    """configs[0] (ColBERT 1x1000, 32/180/128, FP32): bit-identical to the reference."""
    g = golden("fwd_c1")
    Q = orc.make_queries(1, 32, 128, seed=0)
    D, vl = orc.padded(orc.make_corpus(1000, np.full(1000, 180), 128, seed=1))
    sc, am, rep = mx.fused_score_batch(cuda(Q), mx.DocBatch.from_dense(D, vl))
    assert np.array_equal(sc.numpy(), g["scores"])
    assert np.array_equal(am.numpy(), g["argmax"])
    assert rep.mac_count == int(g["macs"]) and rep.bytes_read == int(g["bytes_read"])
    assert rep.bytes_written == int(g["bytes_written"])


# ------------------------------------------------------------------ tensor-core forward (K1/K2)
@pytest.mark.parametrize(
    "n_q,l_q,n_docs,l_pad,dim,dtype",
    [
        (1, 1024, 24, 1024, 128, torch.bfloat16),  # ColPali shape (C2 / C3 per-pair shape)
        (4, 300, 40, 260, 128, torch.bfloat16),    # ragged, not tile aligned
        (3, 32, 50, 180, 128, torch.bfloat16),     # ColBERT shape
        (2, 200, 30, 333, 64, torch.float16),
        (2, 520, 20, 400, 256, torch.bfloat16),
        (1, 130, 10, 129, 96, torch.bfloat16),
        (2, 1100, 6, 300, 128, torch.bfloat16),    # L_q > 1024: three Q row groups
        (1, 640, 30, 512, 128, torch.bfloat16),    # two groups (4 + 1 blocks), 2-CTA cluster
        (1, 384, 170, 256, 128, torch.bfloat16),   # one group of 3 blocks, more docs than SMs
    ],
)
def test_tensor_core_forward_vs_oracle(n_q, l_q, n_docs, l_pad, dim, dtype):
    rng = np.random.default_rng(n_q * 1000 + l_q)
    Q = orc.make_queries(n_q, l_q, dim, seed=int(rng.integers(1 << 30)))
    lens = rng.integers(1, l_pad + 1, n_docs)
    lens[0] = l_pad
    D, vl = orc.padded(orc.make_corpus(n_docs, lens, dim, seed=int(rng.integers(1 << 30))), l_pad)
    Qr = cuda(Q, dtype)
    Dr = cuda(D, dtype)
    sc, am, _ = mx.fused_score_batch(Qr, mx.DocBatch.from_dense(Dr, vl))
    # oracle fed the rounded values widened to fp32
    Qo = Qr.float().cpu().numpy()
    Do = Dr.float().cpu().numpy()
    ref_s, ref_a = orc.fused_score_batch(Qo, Do, vl)
    assert rel_err(sc.numpy(), ref_s) < REL
    safe = top2_gap(Qo, Do, vl) > GAP
    assert np.array_equal(am.numpy()[safe], ref_a[safe])
    assert safe.mean() > 0.99
    # rerank mode (no argmax): identical score bits
    s2, a2, _ = mx.score_dense(Qr, Dr, cuda(vl), want_argmax=False)
    assert a2 is None and np.array_equal(s2.cpu().numpy(), sc.numpy())


def test_tensor_core_top20_agreement_planted():
    """100% top-20 agreement with the fp32 oracle on a planted corpus (no boundary near-ties)."""
    q = orc.make_queries(1, 64, 128, seed=11)[0]
    docs = orc.planted_corpus(q, 200, 96, seed=12)
    D, vl = orc.padded(docs)
    sc, _, _ = mx.fused_score_batch(cuda(q[None], torch.bfloat16), mx.DocBatch.from_dense(cuda(D, torch.bfloat16), vl))
    ref, _ = orc.fused_score_batch(q[None], D, vl)
    top_gpu = np.lexsort((np.arange(200), -sc.numpy()[0]))[:20]
    top_ref = np.lexsort((np.arange(200), -ref[0]))[:20]
    assert list(top_gpu) == list(top_ref)


def test_forward_deterministic_and_shard_invariant():
    rng = np.random.default_rng(7)
    Q = cuda(orc.make_queries(2, 256, 128, seed=1), torch.bfloat16)
    D = cuda(rng.standard_normal((64, 256, 128)).astype(np.float32), torch.bfloat16)
    s1, a1, _ = mx.score_dense(Q, D)
    s2, a2, _ = mx.score_dense(Q, D)
    assert torch.equal(s1, s2) and torch.equal(a1, a2)
    # emulated corpus sharding: each shard scored alone gives the same bits
    parts = [mx.score_dense(Q, D[lo:lo + 16]) for lo in range(0, 64, 16)]
    assert torch.equal(torch.cat([p[0] for p in parts], dim=1), s1)
    assert torch.equal(torch.cat([p[1] for p in parts], dim=1), a1)
    # document permutation permutes the outputs bit-for-bit
    perm = torch.randperm(64, device="cuda")
    sp, ap, _ = mx.score_dense(Q, D[perm].contiguous())
    assert torch.equal(sp, s1[:, perm]) and torch.equal(ap, a1[:, perm])


def test_c2_scale_sampled_parity():
    """ColPali rerank at full size (10K docs): sampled oracle check + size-independent properties."""
    g = torch.Generator(device="cuda").manual_seed(3)
    nb = 10000
    Q = torch.randn(1, 1024, 128, device="cuda", generator=g)
    Q = (Q / Q.norm(dim=-1, keepdim=True)).bfloat16()
    D = torch.randn(nb, 1024, 128, device="cuda", generator=g, dtype=torch.bfloat16)
    sc, am, _ = mx.score_dense(Q, D)
    assert torch.isfinite(sc).all()
    assert int(am.min()) >= 0 and int(am.max()) < 1024
    idx = torch.tensor([0, 1, 4999, 7777, 9998, 9999], device="cuda")
    Qo = Q.float().cpu().numpy()
    Do = D.index_select(0, idx).float().cpu().numpy()
    ref_s, ref_a = orc.fused_score_batch(Qo, Do)
    assert rel_err(sc[:, idx].cpu().numpy(), ref_s) < REL
    safe = top2_gap(Qo, Do, [1024] * len(idx)) > GAP
    assert np.array_equal(am[:, idx].cpu().numpy()[safe], ref_a[safe])
    # the two Q row groups of one document are independent: splitting the query agrees exactly
    s_lo, a_lo, r_lo = mx.score_dense(Q[:, :512].contiguous(), D[:100], want_rowmax=True)
    _, _, r_full = mx.score_dense(Q, D[:100], want_rowmax=True)
    assert torch.equal(r_full[:, :, :512], r_lo)


# ------------------------------------------------------------------ INT8 (K3, K4)
def test_quantize_bitwise_against_golden():
    g = golden("quant")
    for x, key_q, key_s, lv in ((g["x"], "q127", "s127", 127), (g["x"], "q7", "s7", 7)):
        qm = mx.quantize_per_token(x, levels=lv)
        assert np.array_equal(qm.q.cpu().numpy(), g[key_q])
        assert np.array_equal(qm.scale.cpu().numpy(), g[key_s])
    qm = mx.quantize_per_token(np.array([[0.5, -1.0]], np.float32))
    assert qm.q.cpu().tolist() == [[64, -127]]
    z = mx.quantize_per_token(np.zeros((2, 3), np.float32))
    assert np.all(z.scale.cpu().numpy() == np.float32(1e-12))


@pytest.mark.parametrize("dim,dtype", [(128, torch.bfloat16), (128, torch.float16), (96, torch.bfloat16),
                                       (128, torch.float32)])
def test_quantize_half_way_quotients(dim, dtype):
    """Reciprocal fast path + exact-division fallback: quotients exactly on / next to k + 0.5."""
    rng = np.random.default_rng(dim)
    x = np.zeros((64, dim), np.float32)
    x[:, 0] = 127.0                                          # scale 1 (maxabs / 127)
    halves = rng.integers(-126, 126, (64, dim - 1)) + 0.5   # exact ties -> even
    x[:, 1:] = halves
    x[1::3, 1:] = np.nextafter(halves[1::3], np.inf)          # just above a tie
    x[2::3, 1:] = np.nextafter(halves[2::3], -np.inf)         # just below
    x[40:] *= rng.uniform(0.001, 30, (24, 1)).astype(np.float32)  # other scales
    xt = cuda(x, dtype)
    xr = xt.float().cpu().numpy()                             # the values the device sees
    q, sc = orc.quantize_per_token(xr)
    qm, sm = mx.quant.quantize_tensor(xt)
    assert np.array_equal(qm.cpu().numpy(), q) and np.array_equal(sm.cpu().numpy(), sc)


def test_quantize_random_bitwise_vs_oracle():
    rng = np.random.default_rng(8)
    x = (rng.standard_normal((777, 130)) * rng.uniform(0.01, 10, (777, 1))).astype(np.float32)
    x[5] = 0
    q, s = orc.quantize_per_token(x)
    qm = mx.quantize_per_token(x)
    assert np.array_equal(qm.q.cpu().numpy(), q) and np.array_equal(qm.scale.cpu().numpy(), s)
    xb = cuda(x, torch.bfloat16)
    qb, sb = mx.quant.quantize_tensor(xb)
    q2, s2 = orc.quantize_per_token(xb.float().cpu().numpy())
    assert np.array_equal(qb.cpu().numpy(), q2) and np.array_equal(sb.cpu().numpy(), s2)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_quantize_streaming_kernel_many_rows_bitwise(dtype):
    """The persistent d = 128 streaming quantiser (magic-number rounding, next row prefetched) on
    a row count that is not a multiple of any pass width, with zero rows and mixed scales, vs the
    oracle: every int8 and every scale bit-identical."""
    rng = np.random.default_rng(11)
    n = 100_003
    x = (rng.standard_normal((n, 128)) * rng.uniform(1e-3, 50, (n, 1))).astype(np.float32)
    x[::997] = 0
    x[7::1001, 3] = 127.0 * np.abs(x[7::1001]).max(axis=1)  # rows whose scale is exactly representable
    xt = cuda(x, dtype)
    q, sc = orc.quantize_per_token(xt.float().cpu().numpy())
    qm, sm = mx.quant.quantize_tensor(xt)
    assert np.array_equal(qm.cpu().numpy(), q) and np.array_equal(sm.cpu().numpy(), sc)


def test_int8_golden_bitwise():
    g = golden("int8")
    corpus = mx.QuantizedCorpus(g["d_q"], g["d_s"])
    sm, am, _ = mx.fused_score_int8_batch(mx.QuantizedMatrix(g["q_q"], g["q_s"]), corpus, valid_lens=g["valid_lens"])
    assert np.array_equal(sm.numpy()[0], g["scores"])
    assert np.array_equal(am.numpy()[0], g["argmax"])
    s, a = mx.fused_score_int8(mx.QuantizedMatrix(g["q_q"], g["q_s"]), corpus.doc(1), valid_len=13)
    assert s == g["scores"][1] and a.cpu().tolist() == list(g["argmax"][1])


@pytest.mark.parametrize("l_q,n_docs,l_pad,dim", [(1024, 12, 1024, 128), (33, 40, 200, 64), (300, 9, 517, 256),
                                                 (256, 30, 640, 128)])
def test_int8_random_bitwise_incl_ties(l_q, n_docs, l_pad, dim):
    rng = np.random.default_rng(l_q + dim)
    Qf = rng.standard_normal((2, l_q, dim)).astype(np.float32)
    Df = rng.standard_normal((n_docs, l_pad, dim)).astype(np.float32)
    Df[1] = Df[0]                       # identical documents
    Df[2, 1::2] = Df[2, 0::2][: Df[2, 1::2].shape[0]]  # duplicated rows -> exact ties
    lens = rng.integers(1, l_pad + 1, n_docs)
    qq, qs = mx.quant.quantize_tensor(cuda(Qf))
    dq, ds = mx.quant.quantize_tensor(cuda(Df))
    sc, am, _ = mx.score_int8(qq, qs, dq, ds, cuda(lens.astype(np.int32)))
    oq, os_ = orc.quantize_per_token(Qf.reshape(-1, dim))
    dq_o, ds_o = orc.quantize_per_token(Df.reshape(-1, dim))
    ref_s, ref_a = orc.fused_score_int8(oq.reshape(2, l_q, dim), os_.reshape(2, l_q), dq_o.reshape(n_docs, l_pad, dim),
                                        ds_o.reshape(n_docs, l_pad), lens)
    assert np.array_equal(sc.cpu().numpy(), ref_s)
    assert np.array_equal(am.cpu().numpy(), ref_a)
    # rerank mode (no argmax, max-only fast path): the same bits
    sc2, am2, _ = mx.score_int8(qq, qs, dq, ds, cuda(lens.astype(np.int32)), want_argmax=False)
    assert am2 is None and np.array_equal(sc2.cpu().numpy(), ref_s)


@pytest.mark.parametrize("dim", [128, 256, 384, 1100, 3000])
def test_int8_extreme_accumulators_bitwise(dim):
    """Raw int8 at the edges of the s32 range the kernels convert: all -128 x -128 at d = 256 gives
    acc = 2^22 exactly (the limit of the biased / magic-number s32 -> f32), -128 x 127 the most
    negative sums; d = 384 takes the cvt path, d = 1100 / 3000 (past the tensor-core tiles) the exact
    SIMT kernel, whose f32(acc) rounds once |acc| > 2^24.  Scores and argmax bit-identical to the oracle."""
    rng = np.random.default_rng(dim)
    l_q, n_docs, l_pad = 160, 6, 256
    qq = rng.integers(-128, 128, (1, l_q, dim)).astype(np.int8)
    dq = rng.integers(-128, 128, (n_docs, l_pad, dim)).astype(np.int8)
    qq[0, :40] = -128
    dq[0] = -128            # acc = dim * 2^14 for the first 40 query rows
    dq[1] = 127             # acc = -dim * 128 * 127
    dq[2, ::3] = -128
    qs = rng.uniform(0.001, 0.05, (1, l_q)).astype(np.float32)
    ds = rng.uniform(0.001, 0.05, (n_docs, l_pad)).astype(np.float32)
    lens = np.array([256, 255, 129, 128, 1, 77], dtype=np.int32)
    sc, am, _ = mx.score_int8(cuda(qq), cuda(qs), cuda(dq), cuda(ds), cuda(lens))
    ref_s, ref_a = orc.fused_score_int8(qq, qs, dq, ds, lens)
    assert np.array_equal(sc.cpu().numpy(), ref_s)
    assert np.array_equal(am.cpu().numpy(), ref_a)
    sc2, _, _ = mx.score_int8(cuda(qq), cuda(qs), cuda(dq), cuda(ds), cuda(lens), want_argmax=False)
    assert np.array_equal(sc2.cpu().numpy(), ref_s)


def test_two_stage_topk_matches_reference():
    g = golden("two_stage")
    D = g["D"]
    corpus_q = mx.quantize_corpus(cuda(D))
    top = mx.two_stage_topk(g["q"], corpus_q, mx.DocBatch.from_dense(D), k=5)
    assert [t[0] for t in top] == list(g["top_ids"])
    assert [t[1] for t in top] == list(g["top_scores"])
    with pytest.raises(mx.KTooLarge):
        mx.two_stage_topk(g["q"], corpus_q, mx.DocBatch.from_dense(D), k=31)


# ------------------------------------------------------------------ varlen (K5)
def test_varlen_golden_bitwise():
    g = golden("varlen")
    pk = mx.PackedCorpus(g["tokens"], g["cu"])
    s, am, rep = mx.fused_score_varlen(g["q"], pk)
    assert np.array_equal(s.cpu().numpy(), g["scores"])
    assert np.array_equal(am.numpy(), g["argmax"])
    assert am.padded_len is None and rep.mac_count == int(g["macs"])


def test_varlen_equals_padded_bf16():
    rng = np.random.default_rng(9)
    lens = rng.integers(32, 513, 300)
    docs = orc.make_corpus(300, lens, 128, seed=4)
    q = orc.make_queries(1, 32, 128, seed=5)
    toks = cuda(np.concatenate(docs), torch.bfloat16)
    cu = np.concatenate([[0], np.cumsum(lens)])
    s_v, a_v, _ = mx.score_varlen(cuda(q, torch.bfloat16), toks, cuda(cu))
    D, vl = orc.padded(docs)
    s_p, a_p, _ = mx.score_dense(cuda(q, torch.bfloat16), cuda(D, torch.bfloat16), cuda(vl))
    ref_s, ref_a = orc.fused_score_varlen(cuda(q, torch.bfloat16).float().cpu().numpy(), toks.float().cpu().numpy(), cu)
    assert rel_err(s_v.cpu().numpy(), ref_s) < REL and rel_err(s_p.cpu().numpy(), ref_s) < REL
    # argmax: exact on every row whose oracle top-2 gap exceeds 1e-5
    safe = varlen_top2_gap(cuda(q, torch.bfloat16).float().cpu().numpy(), toks.float().cpu().numpy(), cu) > GAP
    assert safe.mean() > 0.99
    assert np.array_equal(a_v.cpu().numpy()[safe], ref_a[safe])
    assert np.array_equal(a_p.cpu().numpy()[safe], ref_a[safe])


# ------------------------------------------------------------------ backward (K6, K7, K8)
def test_csr_bitwise_against_golden_and_oracle():
    g = golden("csr")
    csr = mx.build_inverse_csr(mx.ArgmaxMap(g["h_argmax"], [2], padded_len=2))
    rp, ci = csr.to_numpy()
    assert list(rp) == [0, 1, 3] and list(ci) == [2, 0, 1]
    csr = mx.build_inverse_csr(mx.ArgmaxMap(np.zeros((3, 4, 5), np.int32), [6] * 4, padded_len=6))
    rp, ci = csr.to_numpy()
    assert np.array_equal(rp, g["hot_row_ptr"]) and np.array_equal(ci, g["hot_col_idx"])
    csr = mx.build_inverse_csr(mx.ArgmaxMap(g["p_argmax"], g["p_lens"], padded_len=None))
    rp, ci = csr.to_numpy()
    assert np.array_equal(rp, g["p_row_ptr"]) and np.array_equal(ci, g["p_col_idx"])
    assert np.array_equal(csr.destinations_per_source().cpu().numpy(),
                          mx.ArgmaxMap(g["p_argmax"], g["p_lens"]).flat_destinations().cpu().numpy())


def test_csr_random_maps_bitwise():
    """tests/test_acceptance.py:192-220 style: many random maps incl. all-hot and permutations."""
    rng = np.random.default_rng(10)
    for trial in range(60):
        n_q, b, l_q = rng.integers(1, 6), rng.integers(1, 7), rng.integers(1, 40)
        L = int(rng.integers(1, 50))
        lens = rng.integers(1, L + 1, b)
        if trial % 3 == 0:
            idx = np.zeros((n_q, b, l_q), np.int32)  # all hot
        else:
            idx = np.stack([np.stack([rng.integers(0, lens[j], l_q) for j in range(b)]) for _ in range(n_q)])
        packed = trial % 2 == 1
        am = mx.ArgmaxMap(idx.astype(np.int32), lens, padded_len=None if packed else L)
        rp, ci = mx.build_inverse_csr(am).to_numpy()
        orp, oci = orc.build_inverse_csr(idx, lens, None if packed else L)
        assert np.array_equal(rp, orp) and np.array_equal(ci, oci), trial


def test_csr_c3_scale_bitwise():
    rng = np.random.default_rng(12)
    idx = rng.integers(0, 1024, (64, 64, 1024)).astype(np.int32)
    idx[3, 5, :] = 7  # a hot token
    am = mx.ArgmaxMap(idx, [1024] * 64, padded_len=1024)
    rp, ci = mx.build_inverse_csr(am).to_numpy()
    orp, oci = orc.build_inverse_csr(idx, [1024] * 64, 1024)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)


@pytest.mark.parametrize("impl,per_warp", [("doc", "32"), ("doc", "1024"), ("doc", "100000"), ("sort", None)])
def test_csr_every_path_bitwise(monkeypatch, impl, per_warp):
    """Both CSR builders (cluster-per-document counting sort with 1..8 CTAs per cluster and 1..16
    warps per CTA, and the radix-sort path) against the oracle's stable argsort, on random,
    all-hot, packed and long-document maps (the reference's long_doc regime, L_d >= 2048)."""
    if impl == "sort":
        monkeypatch.setenv("MXS_CSR_IMPL", "sort")
    if per_warp:
        monkeypatch.setenv("MXS_CSR_SRC_PER_WARP", per_warp)
    rng = np.random.default_rng(31)
    cases = [(3, 5, 300, 77), (1, 1, 5000, 2048), (2, 3, 700, 4096), (64, 2, 1024, 1024), (1, 2, 40, 9000)]
    for trial, (n_q, b, l_q, L) in enumerate(cases):
        lens = rng.integers(1, L + 1, b)
        lens[0] = L
        idx = np.stack([np.stack([rng.integers(0, lens[j], l_q) for j in range(b)]) for _ in range(n_q)])
        if trial % 2:
            idx[..., : l_q // 3] = 0  # a hot bucket inside every segment
        packed = trial % 2 == 1
        am = mx.ArgmaxMap(idx.astype(np.int32), lens, padded_len=None if packed else L)
        rp, ci = mx.build_inverse_csr(am).to_numpy()
        orp, oci = orc.build_inverse_csr(idx, lens, None if packed else L)
        assert np.array_equal(rp, orp) and np.array_equal(ci, oci), (impl, per_warp, trial)


def test_csr_destination_beyond_shared_memory():
    """A single destination block far longer than a shared-memory histogram (Chamfer clouds of
    more than 51,200 points) takes the radix-sort path, still bit-identical."""
    rng = np.random.default_rng(32)
    n_src, n_dest = 70_000, 60_000
    idx = rng.integers(0, n_dest, (1, 1, n_src)).astype(np.int32)
    idx[0, 0, ::7] = 12345
    am = mx.ArgmaxMap(idx, [n_dest], padded_len=n_dest)
    rp, ci = mx.build_inverse_csr(am).to_numpy()
    orp, oci = orc.build_inverse_csr(idx, [n_dest], n_dest)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)


def test_backward_golden():
    g = golden("backward")
    docs = mx.DocBatch.from_dense(g["D"], g["valid_lens"])
    sc, am, _ = mx.fused_score_batch(cuda(g["Q"]), docs)
    assert np.array_equal(am.numpy(), g["argmax"])
    dq, dd = mx.backward_dispatch(am, g["g"], cuda(g["Q"]), docs)
    assert rel_err(dq.cpu().numpy(), g["dQ"]) < 1e-6
    assert rel_err(dd.cpu().numpy(), g["dD"]) < 1e-6
    flat = mx.grad_docs_csr(mx.build_inverse_csr(am), g["g"], cuda(g["Q"]))
    assert rel_err(flat.cpu().numpy(), g["flat_dD"]) < 1e-6
    with pytest.raises(mx.StaleCsr):
        mx.grad_docs_csr(mx.build_inverse_csr(am), np.ones((2, 3)), cuda(np.ones((2, 9, 8), np.float32)))


def test_inbatch_training_step_c3_shape_bf16():
    """C3: N_q = B = 64 at ColPali shape, bf16, CSR backward, vs the float64 oracle on the same argmax."""
    from paper_2605_29517_b200.parallel import inbatch_step

    gen = torch.Generator(device="cuda").manual_seed(5)
    Q = torch.randn(64, 1024, 128, device="cuda", generator=gen)
    Q = (Q / Q.norm(dim=-1, keepdim=True)).bfloat16()
    D = torch.randn(64, 1024, 128, device="cuda", generator=gen)
    D = (D / D.norm(dim=-1, keepdim=True)).bfloat16()
    loss, scores, dQ, dD = inbatch_step(Q, D, 0)
    _, am, _ = mx.score_dense(Q, D)
    l_ref, g_ref = orc.softmax_ce(scores.cpu().numpy())
    assert abs(float(loss) - l_ref) <= 1e-9 * abs(l_ref)
    Qo = Q.float().cpu().numpy()
    Do = D.float().cpu().numpy()
    a = am.cpu().numpy()
    dq_ref = orc.grad_query(a, g_ref, Do.reshape(-1, 128), np.arange(64) * 1024)
    rp, ci = orc.build_inverse_csr(a, [1024] * 64, 1024)
    dd_ref = orc.grad_docs_csr(rp, ci, g_ref, Qo, n_docs=64).reshape(64, 1024, 128)
    assert rel_err(dQ.cpu().numpy(), dq_ref) < REL
    assert rel_err(dD.cpu().numpy(), dd_ref) < REL


def test_inbatch_step_graph_replay_matches_eager():
    from paper_2605_29517_b200.parallel import InBatchStepGraph, inbatch_step

    rng = np.random.default_rng(12)
    Q = cuda(orc.make_queries(8, 256, 128, seed=1), torch.bfloat16)
    D = cuda(orc.make_queries(8, 200, 128, seed=2), torch.bfloat16)
    g = InBatchStepGraph(Q, D)
    for _ in range(2):
        loss, sc, dq, dd = g()
        el, es, edq, edd = inbatch_step(Q, D, 0)
        assert float(loss) == float(el) and torch.equal(sc, es)
        assert torch.equal(dq, edq) and torch.equal(dd, edd)
        D.add_(torch.from_numpy(rng.standard_normal(D.shape) * 0.01).cuda().bfloat16())  # in-place update


def test_autograd_matches_oracle_and_finite_differences():
    g = golden("inbatch")
    Q = cuda(g["Q"]).requires_grad_(True)
    D = cuda(g["D"]).requires_grad_(True)
    scores = mx.maxsim(Q, D)
    assert np.array_equal(scores.detach().cpu().numpy(), g["scores"])
    up = cuda(g["g"])
    (scores * up).sum().backward()
    assert rel_err(Q.grad.cpu().numpy(), g["dQ"]) < 1e-6
    assert rel_err(D.grad.cpu().numpy(), g["dD"]) < 1e-6


def test_autograd_varlen_matches_padded():
    rng = np.random.default_rng(14)
    lens = rng.integers(3, 20, 6)
    docs = [rng.standard_normal((int(n), 16)).astype(np.float32) for n in lens]
    Q = cuda(rng.standard_normal((2, 5, 16)).astype(np.float32)).requires_grad_(True)
    toks = cuda(np.concatenate(docs)).requires_grad_(True)
    cu = np.concatenate([[0], np.cumsum(lens)])
    up = cuda(rng.standard_normal((2, 6)))
    (mx.maxsim_varlen(Q, toks, cu) * up).sum().backward()
    D, vl = orc.padded(docs)
    s, a = orc.fused_score_varlen(Q.detach().cpu().numpy(), np.concatenate(docs), cu)
    dq_ref = orc.grad_query(a, up.cpu().numpy(), np.concatenate(docs), cu[:-1])
    rp, ci = orc.build_inverse_csr(a, lens, None)
    dt_ref = orc.grad_docs_csr(rp, ci, up.cpu().numpy(), Q.detach().cpu().numpy(), n_docs=6)
    assert rel_err(Q.grad.cpu().numpy(), dq_ref) < 1e-6
    assert rel_err(toks.grad.cpu().numpy(), dt_ref) < 1e-6


def test_training_drift_matches_reference_loop():
    """tests/test_acceptance.py:438-447 criterion c11 (shortened): SGD through the device path
    tracks the float64 oracle loop; loss drift <= 1e-4."""
    rng = np.random.default_rng(0)
    q = rng.standard_normal((4, 6, 8)).astype(np.float32)
    d = rng.standard_normal((4, 7, 8)).astype(np.float32)
    qo, do = q.copy(), d.copy()
    drift = 0.0
    for _ in range(30):
        Q = cuda(q).requires_grad_(True)
        D = cuda(d).requires_grad_(True)
        s = mx.maxsim(Q, D)
        from paper_2605_29517_b200.parallel import softmax_ce

        loss, g = softmax_ce(s.detach())
        (s * g).sum().backward()
        q = (q.astype(np.float64) - 0.05 * Q.grad.cpu().numpy()).astype(np.float32)
        d = (d.astype(np.float64) - 0.05 * D.grad.cpu().numpy()).astype(np.float32)
        so, ao = orc.fused_score_batch(qo, do)
        lo, go = orc.softmax_ce(so)
        dq = orc.grad_query(ao, go, do.reshape(-1, 8), np.arange(4) * 7)
        rp, ci = orc.build_inverse_csr(ao, [7] * 4, 7)
        dd = orc.grad_docs_csr(rp, ci, go, qo, n_docs=4).reshape(4, 7, 8)
        qo = (qo.astype(np.float64) - 0.05 * dq).astype(np.float32)
        do = (do.astype(np.float64) - 0.05 * dd).astype(np.float32)
        drift = max(drift, abs(float(loss) - lo) / abs(lo))
    assert drift <= 1e-4


def test_contrastive_drift_api():
    """maxsim/cli.py:209 contrastive_drift on the device: fused path vs dense path."""
    out = mx.contrastive_drift(n_docs=4, len_q=6, len_d=7, dim=8, steps=40, seed=3)
    assert out["steps"] == 40 and out["max_rel_drift"] <= 1e-4
    assert out["loss_last_fused"] < out["loss_first"]


@pytest.mark.parametrize("l_q", [200, 512, 1024])
def test_rerank_three_slot_kernel_matches(l_q, monkeypatch):
    """The opt-in three-slot rerank kernel (MXS_RERANK_IMPL=r3; 2 resident Q blocks, 4-CTA
    clusters at L_q = 1024) returns the same score bits as the default forward."""
    rng = np.random.default_rng(l_q)
    Q = cuda(orc.make_queries(1, l_q, 128, seed=5), torch.bfloat16)
    lens = rng.integers(1, 300, 160).astype(np.int32)
    D, vl = orc.padded(orc.make_corpus(160, lens, 128, seed=6), 300)
    Dt, vlt = cuda(D, torch.bfloat16), cuda(vl)
    s_ts, _, _ = mx.score_dense(Q, Dt, vlt, want_argmax=False)
    monkeypatch.setenv("MXS_RERANK_IMPL", "r3")
    s_r3, _, _ = mx.score_dense(Q, Dt, vlt, want_argmax=False)
    assert torch.equal(s_ts, s_r3)


def test_scores_without_argmax_are_identical():
    """The rerank mode (argmax not requested: max only, no index tracking) returns the same bits."""
    rng = np.random.default_rng(17)
    Q = cuda(orc.make_queries(2, 300, 128, seed=3), torch.bfloat16)
    lens = rng.integers(1, 400, 37).astype(np.int32)
    D, vl = orc.padded(orc.make_corpus(37, lens, 128, seed=4), 400)
    Dt, vlt = cuda(D, torch.bfloat16), cuda(vl)
    s1, a1, r1 = mx.score_dense(Q, Dt, vlt, want_rowmax=True)
    s2, a2, r2 = mx.score_dense(Q, Dt, vlt, want_argmax=False, want_rowmax=True)
    assert a2 is None and torch.equal(s1, s2) and torch.equal(r1, r2)
    s3, a3, r3 = mx.score_dense(Q, Dt, vlt, want_argmax=False)  # fused S4, no row maxima materialised
    assert r3 is None and torch.equal(s3, s1)


# ------------------------------------------------------------------ top-K (K9)
def test_topk_ties_and_chunking():
    g = golden("misc")
    ts, ti = mx.topk(cuda(g["tie_scores"]), 15)
    assert ti.cpu().tolist() == list(g["tie_ids"])
    rng = np.random.default_rng(6)
    s = np.round(rng.standard_normal(100_000), 2)  # > 8192: two-pass path, heavy ties
    ts, ti = mx.topk(cuda(s), 20, id_offset=500)
    os_, oi = orc.topk(s, 20, id_offset=500)
    assert ti.cpu().tolist() == oi.tolist() and ts.cpu().tolist() == os_.tolist()
    assert mx.ranked(cuda([0.0, 1.0, 0.5, 1.0]), 2) == [[1, 1.0], [3, 1.0]]
    with pytest.raises(mx.KTooLarge):
        mx.topk(cuda(s[:5]), 6)


@pytest.mark.parametrize("n,k", [(1, 1), (20, 20), (10_000, 20), (10_000, 1), (16_384, 128), (16_385, 128), (8193, 100),
                                 (2_000_000, 128), (50_000, 129), (10_000, 500), (300_000, 32)])
def test_topk_select_paths_match_oracle(n, k):
    """Warp-tournament selection (k <= 128, multi-pass above 8192) and the bitonic path (k > 128)."""
    rng = np.random.default_rng(n + k)
    s = np.round(rng.standard_normal(n), 3)  # heavy ties: exercises the id-ascending rule
    if n > 10:
        s[rng.integers(0, n, 5)] = np.nan  # NaN entries are never selected
    ts, ti = mx.topk(cuda(s), k, id_offset=7)
    os_, oi = orc.topk(np.where(np.isnan(s), -np.inf, s), k, id_offset=7)
    valid = ~np.isnan(s)
    if valid.sum() >= k:
        assert ti.cpu().tolist() == oi.tolist() and ts.cpu().tolist() == os_.tolist()


def test_sharded_rerank_merge_equals_global():
    from paper_2605_29517_b200.topk import select_candidates

    rng = np.random.default_rng(13)
    s = np.round(rng.standard_normal(50_000), 2)
    cand_s, cand_i = [], []
    for lo in range(0, 50_000, 12_500):  # four emulated ranks
        ts, ti = mx.topk(cuda(s[lo:lo + 12_500]), 20, id_offset=lo)
        cand_s.append(ts)
        cand_i.append(ti)
    ms, mi = select_candidates(torch.cat(cand_s), torch.cat(cand_i), 20)
    os_, oi = orc.topk(s, 20)
    assert mi.cpu().tolist() == oi.tolist() and ms.cpu().tolist() == os_.tolist()


@pytest.mark.parametrize(
    "n_docs,lo,hi,l_q,n_q",
    [(300, 32, 512, 32, 1), (1000, 1, 20, 32, 1), (50, 100, 2000, 32, 1), (200, 1, 300, 16, 4), (100, 5, 200, 128, 1),
     (7, 1, 3, 32, 1), (40, 5, 300, 48, 3), (30, 10, 100, 100, 3), (24, 50, 700, 1024, 1)],
)
def test_varlen_tensor_core_vs_exact_and_oracle(n_docs, lo, hi, l_q, n_q):
    """K5 (tcgen05 varlen): documents start/end anywhere in a 128-token tile, 1-token docs, docs
    spanning many tiles, multi-query column blocks, more than 128 query rows (one launch per
    128-row group, a query split across groups); vs the exact kernel and the oracle."""
    rng = np.random.default_rng(n_docs + l_q)
    lens = rng.integers(lo, hi + 1, n_docs)
    cu = np.concatenate([[0], np.cumsum(lens)])
    toks = cuda(np.concatenate(orc.make_corpus(n_docs, lens, 128, seed=int(rng.integers(1 << 30)))), torch.bfloat16)
    Q = cuda(orc.make_queries(n_q, l_q, 128, seed=int(rng.integers(1 << 30))), torch.bfloat16)
    s_tc, a_tc, _ = mx.score_varlen(Q, toks, cuda(cu))
    s_ex, a_ex, _ = mx.score_varlen(Q, toks, cuda(cu), exact=True)
    ref_s, ref_a = orc.fused_score_varlen(Q.float().cpu().numpy(), toks.float().cpu().numpy(), cu)
    assert np.array_equal(s_ex.cpu().numpy(), ref_s) and np.array_equal(a_ex.cpu().numpy(), ref_a)
    assert rel_err(s_tc.cpu().numpy(), ref_s) < REL
    safe = varlen_top2_gap(Q.float().cpu().numpy(), toks.float().cpu().numpy(), cu) > GAP
    print(f"varlen: {int((~safe).sum())} of {safe.size} rows excluded (top-2 gap <= {GAP})")
    assert safe.mean() > 0.98
    assert np.array_equal(a_tc.cpu().numpy()[safe], ref_a[safe])


@pytest.mark.parametrize("dtype,dim", [(torch.bfloat16, 128), (torch.float32, 40), (torch.float32, 7), (torch.float16, 64)])
def test_gather_rows_written_exactly_once(monkeypatch, dtype, dim):
    """Ownership ledger of the destination-owned gathers (MXS_DEBUG_WRITES=1): every dD row and
    every dQ row is stored by exactly one warp -- the reference's WriteTracking assertion
    (tests/test_backward.py:94-108) -- on ragged, all-hot and packed maps, through every gather
    variant (row-group, vectorised, scalar)."""
    monkeypatch.setenv("MXS_DEBUG_WRITES", "1")
    rng = np.random.default_rng(dim)
    Q = torch.from_numpy(rng.standard_normal((3, 70, dim)).astype(np.float32)).cuda().to(dtype)
    lens = np.array([33, 1, 128, 77], np.int32)
    D = torch.from_numpy(rng.standard_normal((4, 128, dim)).astype(np.float32)).cuda().to(dtype)
    g = rng.standard_normal((3, 4))
    docs = mx.DocBatch.from_dense(D, torch.from_numpy(lens))
    _, am, _ = mx.fused_score_batch(Q, docs)
    dq, dd = mx.backward_dispatch(am, g, Q, docs)
    assert torch.isfinite(dq).all() and torch.isfinite(dd).all()
    hot = mx.ArgmaxMap(np.zeros((3, 4, 70), np.int32), lens, padded_len=128)  # every source on row 0
    dq, dd = mx.backward_dispatch(hot, g, Q, docs)
    assert torch.isfinite(dd).all()
    packed = mx.ArgmaxMap(am.numpy(), lens, padded_len=None)
    flat = mx.grad_docs_csr(mx.build_inverse_csr(packed), g, Q)
    assert flat.shape == (int(lens.sum()), dim)


@pytest.mark.parametrize("knob,value", [("MXS_FWD_IMPL", "ss"), ("MXS_RERANK_IMPL", "r3"), ("MXS_FWD_IMPL", "ts"),
                                        ("MXS_FWD_IMPL", "pair"), ("MXS_PAIR_SS", "1"), ("MXS_PAIR_CL", "4")])
def test_alternate_forward_kernels_vs_oracle(monkeypatch, knob, value):
    """The SS-form kernel (fwd_tc: Q streamed through shared memory instead of resident in TMEM),
    the three-slot rerank kernel, the single-CTA TS kernel (fwd_ts), the CTA-pair kernel (fwd_pair)
    and its all-shared-memory-Q (four slots) and 4-CTA-cluster variants on bf16, forced by their
    run-time knobs on the ColPali pair shape, a 2-pair-cluster
    ragged shape, a 1-pair shape and a ragged ColBERT shape: scores within 1e-3 of the oracle,
    clear-gap argmax exact, rerank bits equal to the argmax mode."""
    monkeypatch.setenv(knob, value)
    rng = np.random.default_rng(41)
    for n_q, l_q, n_docs, l_pad in ((1, 1024, 6, 1024), (2, 777, 9, 300), (2, 300, 7, 260), (3, 32, 40, 180)):
        Q = orc.make_queries(n_q, l_q, 128, seed=int(rng.integers(1 << 30)))
        lens = rng.integers(1, l_pad + 1, n_docs)
        lens[0] = l_pad
        D, vl = orc.padded(orc.make_corpus(n_docs, lens, 128, seed=int(rng.integers(1 << 30))), l_pad)
        Qr, Dr = cuda(Q, torch.bfloat16), cuda(D, torch.bfloat16)
        Qo, Do = Qr.float().cpu().numpy(), Dr.float().cpu().numpy()
        ref_s, ref_a = orc.fused_score_batch(Qo, Do, vl)
        sc, am, _ = mx.score_dense(Qr, Dr, cuda(vl))
        assert rel_err(sc.cpu().numpy(), ref_s) < REL
        safe = top2_gap(Qo, Do, vl) > GAP
        assert np.array_equal(am.cpu().numpy()[safe], ref_a[safe])
        s2, _, _ = mx.score_dense(Qr, Dr, cuda(vl), want_argmax=False)
        assert rel_err(s2.cpu().numpy(), ref_s) < REL


@pytest.mark.parametrize("n,col0,ncols", [(64, 0, 64), (64, 16, 32), (7, 3, 4), (300, 100, 200)])
def test_fused_softmax_ce_vs_reference_formula(n, col0, ncols):
    """mxs_softmax_ce (the C3 step's fused loss, maxsim/cli.py:198-206) vs the float64 restatement
    on the same scores: loss to 1e-12 relative, the fp32 gradient slice to fp32 rounding."""
    from paper_2605_29517_b200.parallel import softmax_ce, softmax_ce_device

    rng = np.random.default_rng(n + col0)
    s = torch.from_numpy(rng.standard_normal((n, n)) * 30).cuda()
    loss_ref, g_ref = softmax_ce(s)
    loss, g = softmax_ce_device(s, col0, ncols)
    assert abs(float(loss) - float(loss_ref)) <= 1e-12 * abs(float(loss_ref))
    gr = g_ref[:, col0:col0 + ncols].to(torch.float32)
    assert torch.allclose(g, gr, rtol=2e-7, atol=1e-30)
    # the reference's numpy formula on the host
    sn = s.cpu().numpy()
    shifted = sn - sn.max(axis=1, keepdims=True)
    lse = np.log(np.exp(shifted).sum(axis=1)) + sn.max(axis=1)
    assert abs(float(loss) - float(np.mean(lse - np.diag(sn)))) <= 1e-12 * abs(float(loss))


def test_sharded_step_graphs_equal_eager_step():
    """ShardedInBatchStepGraph (G1 forward | eager all_gather | G2 loss + CSR + dQ | eager async
    all_reduce | G3 dD) at world 1 reproduces inbatch_step bit for bit, replay after replay, and
    follows in-place updates of Q / D."""
    from paper_2605_29517_b200.parallel import ShardedInBatchStepGraph, inbatch_step

    g = torch.Generator(device="cuda").manual_seed(5)
    Q = torch.randn(8, 300, 128, device="cuda", generator=g).bfloat16()
    D = torch.randn(8, 260, 128, device="cuda", generator=g).bfloat16()
    step = ShardedInBatchStepGraph(Q, D, 0)
    for it in range(3):
        if it == 2:  # in-place parameter update between steps
            Q.mul_(-0.5)
            D.add_(0.25)
        loss, scores, dQ, dD = step()
        rl, rs, rq, rd = inbatch_step(Q, D, 0)
        torch.cuda.synchronize()
        assert torch.equal(scores, rs) and torch.equal(loss, rl)
        assert torch.equal(dQ, rq) and torch.equal(dD, rd)


def _sharded_graph_worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_2605_29517_b200.parallel import ShardedInBatchStepGraph, inbatch_step

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda").manual_seed(9)
    Q = torch.randn(8, 200, 128, device="cuda", generator=g).bfloat16()
    D = torch.randn(8, 150, 128, device="cuda", generator=g).bfloat16()
    lo, hi = 4 * rank, 4 * rank + 4
    D_loc = D[lo:hi].contiguous()
    step = ShardedInBatchStepGraph(Q, D_loc, lo)
    ok = True
    for _ in range(2):
        loss, scores, dQ, dD = step()
        rl, rs, rq, rd = inbatch_step(Q, D_loc, lo)
        torch.cuda.synchronize()
        ok &= bool(torch.equal(scores, rs) and torch.equal(loss, rl) and torch.equal(dQ, rq) and torch.equal(dD, rd))
    out[rank] = ok
    dist.destroy_process_group()


def test_sharded_step_graphs_two_ranks_equal_eager():
    """World 2 (two processes on cuda:0 over gloo, B sharded 4 + 4): the graph step with the
    eager all_gather / async all_reduce between replays equals the eager sharded step bit for bit."""
    import socket

    import torch.multiprocessing as tmp

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    out = tmp.Manager().dict()
    tmp.spawn(_sharded_graph_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] and out[1]
