"""Known-answer cases of the reference's own test suite, restated against the device API.

Each test names the reference test it mirrors.  fp32 inputs take the exact kernel,
so the reference's exact-equality assertions carry over unchanged; INT8 is bit-exact too.
"""

import numpy as np
import pytest
import torch

import paper_2605_29517_b200 as mx
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def em(rows):
    return mx.EmbeddingMatrix(torch.tensor(rows, dtype=torch.float32).cuda())


def test_padding_never_wins_with_all_negative_sims():
    """tests/test_forward.py:40-48: valid sims all negative, zero padding would win unmasked."""
    q = em([[1.0, 0.0]])
    d = em([[-1.0, 0.0], [-0.5, 0.0], [0.0, 0.0], [0.0, 0.0]])
    for tile in (mx.TileConfig(bq=1, bd=2, qchunk=1), mx.DEFAULT_TILE):
        s, a, _ = mx.fused_score_pair(q, d, valid_len=2, tile=tile)
        assert s == -0.5 and int(a[0]) == 1
    docs = mx.DocBatch([mx.EmbeddingMatrix(d.data[:2])], padded_len=4)
    rs, ra = mx.dense_score(q, docs)
    assert float(rs[0]) == -0.5 and int(ra.indices[0, 0, 0]) == 1


def test_hand_pair_valid_len_one():
    """tests/test_reference.py:18-24: the 2x2 hand pair cut to one document row."""
    q = em([[1.0, 0.0], [0.0, 1.0]])
    d = em([[0.5, 0.0], [0.0, 2.0]])
    s, a, _ = mx.fused_score_pair(q, d, valid_len=1)
    assert s == 0.5 and a.cpu().tolist() == [0, 0]


def test_results_are_tile_invariant():
    """tests/test_acceptance.py:109-135: every TileConfig gives the same bits (tiles are a host knob;
    the device kernels choose their own)."""
    rng = np.random.default_rng(0)
    Q = orc.make_queries(2, 37, 24, seed=1)
    lens = rng.integers(1, 60, 9)
    D, vl = orc.padded(orc.make_corpus(9, lens, 24, seed=2), 60)
    qs = [mx.EmbeddingMatrix(torch.from_numpy(Q[i]).cuda()) for i in range(2)]
    docs = mx.DocBatch.from_dense(torch.from_numpy(D).cuda(), torch.from_numpy(vl))
    outs = [mx.fused_score_batch(qs, docs, tile=mx.TileConfig(bq=bq, bd=bd, qchunk=qc))
            for bq, bd, qc in ((1, 1, 1), (4, 7, 8), (32, 64, 128), (16, 16, 64))]
    for s, a, _ in outs[1:]:
        assert np.array_equal(s.numpy(), outs[0][0].numpy()) and np.array_equal(a.numpy(), outs[0][1].numpy())
    assert np.array_equal(np.asarray(outs[0][0]), outs[0][0].numpy())  # numpy interop of the result types
    ref_s, ref_a = orc.fused_score_batch(Q, D, vl)
    assert np.array_equal(outs[0][0].numpy(), ref_s) and np.array_equal(outs[0][1].numpy(), ref_a)


def test_query_chunks_sum_to_the_whole():
    """tests/test_forward.py:144-166: chunk scores sum to the whole-query score."""
    q = mx.EmbeddingMatrix(torch.from_numpy(orc.make_queries(1, 100, 8, seed=5)[0]).cuda())
    d = mx.EmbeddingMatrix(torch.from_numpy(orc.make_queries(1, 35, 8, seed=6)[0]).cuda())
    chunks = mx.query_chunk_decompose(q, 32)
    assert [c.rows for c in chunks] == [32, 32, 32, 4]
    whole, _, _ = mx.fused_score_pair(q, d)
    total = sum(mx.fused_score_pair(c, d)[0] for c in chunks)
    assert total == pytest.approx(whole, rel=1e-12)
    two = mx.query_chunk_decompose(mx.EmbeddingMatrix(q.data[:4]), 2)
    assert sum(mx.fused_score_pair(c, d)[0] for c in two) == mx.fused_score_pair(mx.EmbeddingMatrix(q.data[:4]), d)[0]
    assert len(mx.query_chunk_decompose(q, 999)) == 1


def lossless(rng, rows, dim):
    """Integer embeddings with a +-127 entry in every row: per-token quantisation is exact."""
    x = rng.integers(-120, 121, (rows, dim)).astype(np.float32)
    x[np.arange(rows), rng.integers(0, dim, rows)] = 127.0 * rng.choice([-1.0, 1.0], rows)
    return x


def test_lossless_int8_equals_full_precision_exactly():
    """tests/test_quant.py:60-65 and :73-77: INT8 on exactly quantisable inputs == fp32, masking too."""
    rng = np.random.default_rng(7)
    q = mx.EmbeddingMatrix(torch.from_numpy(lossless(rng, 6, 16)).cuda())
    d = mx.EmbeddingMatrix(torch.from_numpy(lossless(rng, 9, 16)).cuda())
    s_full, a_full, _ = mx.fused_score_pair(q, d)
    s_int, a_int = mx.fused_score_int8(mx.quantize_per_token(q), mx.quantize_per_token(d))
    assert s_int == s_full and np.array_equal(np.asarray(a_int.cpu()), a_full.cpu().numpy())
    s5, _, _ = mx.fused_score_pair(q, d, valid_len=5)
    s5i, a5i = mx.fused_score_int8(mx.quantize_per_token(q), mx.quantize_per_token(d), valid_len=5)
    assert s5i == s5 and bool(((a5i >= 0) & (a5i < 5)).all())
    with pytest.raises(mx.EmptyDocument):
        mx.fused_score_int8(mx.quantize_per_token(q), mx.quantize_per_token(d), valid_len=0)


def test_int8_ranking_fidelity_on_planted_corpus():
    """tests/test_quant.py:84-95: Spearman rho >= 0.99 and identical top-20 vs full precision."""
    from scipy import stats

    query = orc.make_queries(1, 24, 64, seed=17)[0]
    corpus = orc.planted_corpus(query, 256, 32, seed=18)
    D, vl = orc.padded(corpus, 32)
    Qt = torch.from_numpy(query).cuda()
    full, _, _ = mx.fused_score_batch(Qt, mx.DocBatch.from_dense(torch.from_numpy(D).cuda(), torch.from_numpy(vl)))
    qq, qs = mx.quant.quantize_tensor(Qt[None])
    dq, ds = mx.quant.quantize_tensor(torch.from_numpy(D).cuda())
    coarse, _, _ = mx.score_int8(qq, qs, dq, ds, torch.from_numpy(vl).cuda(), want_argmax=False)
    f, c = full.numpy()[0], coarse.cpu().numpy()[0]
    assert stats.spearmanr(f, c).statistic >= 0.99
    assert set(np.argsort(-f)[:20]) == set(np.argsort(-c)[:20])


def test_two_stage_exhaustive_and_shortlist_recall():
    """tests/test_quant.py:125-140: k = n is the exhaustive full-precision ranking (score desc, id
    asc); a 4x shortlist recovers the true top-10; k = 0 is empty."""
    query = orc.make_queries(1, 16, 32, seed=29)[0]
    corpus = orc.planted_corpus(query, 256, 20, seed=30)
    D, vl = orc.padded(corpus, 20)
    docs = mx.DocBatch.from_dense(torch.from_numpy(D).cuda(), torch.from_numpy(vl))
    corpus_q = mx.quantize_corpus(torch.from_numpy(D).cuda())
    q = torch.from_numpy(query).cuda()
    full, _, _ = mx.fused_score_batch(q, docs)
    f = full.numpy()[0]
    got = mx.two_stage_topk(q, corpus_q, docs, k=len(corpus))
    order = np.lexsort((np.arange(len(corpus)), -f))
    assert got == [(int(b), float(f[b])) for b in order]
    top10 = mx.two_stage_topk(q, corpus_q, docs, k=10, shortlist_factor=4)
    assert {i for i, _ in top10} == set(np.argsort(-f)[:10])
    assert [s for _, s in top10] == sorted((s for _, s in top10), reverse=True)
    assert mx.two_stage_topk(q, corpus_q, docs, k=0) == []


def test_varlen_mac_count_and_per_doc_bits():
    """tests/test_varlen.py:55-65 and :77-82: packed scoring equals per-document scoring bit for bit
    and counts exactly 2 * L_q * sum(L_d) * d MACs."""
    rng = np.random.default_rng(11)
    lens = rng.integers(1, 30, 6)
    docs = orc.make_corpus(6, lens, 4, seed=12)
    q = orc.make_queries(1, 7, 4, seed=13)[0]
    packed = mx.pack([mx.EmbeddingMatrix(torch.from_numpy(d).cuda()) for d in docs])
    s, a, rep = mx.fused_score_varlen(mx.EmbeddingMatrix(torch.from_numpy(q).cuda()), packed)
    assert rep.mac_count == 2 * 7 * int(lens.sum()) * 4
    for b, d in enumerate(docs):
        sb, ab, _ = mx.fused_score_pair(torch.from_numpy(q).cuda(), torch.from_numpy(d).cuda())
        assert float(s[b]) == sb  # scores stay on the device (f64 [B])
        assert np.array_equal(a.indices[0, b].cpu().numpy(), ab.cpu().numpy())


def test_gradient_paths_agree():
    """tests/test_backward.py:195-205: the CSR and scatter contracts give the same dD, and the
    dispatcher picks CSR once a bucket exceeds the threshold."""
    rng = np.random.default_rng(21)
    Q = orc.make_queries(3, 12, 8, seed=22)
    D, vl = orc.padded(orc.make_corpus(4, rng.integers(3, 10, 4), 8, seed=23), 10)
    qs = [mx.EmbeddingMatrix(torch.from_numpy(Q[i]).cuda()) for i in range(3)]
    docs = mx.DocBatch.from_dense(torch.from_numpy(D).cuda(), torch.from_numpy(vl))
    _, am, _ = mx.fused_score_batch(qs, docs)
    g = rng.standard_normal((3, 4))
    d_csr = mx.grad_docs_csr(mx.build_inverse_csr(am), g, qs)
    d_sc = mx.grad_docs_scatter(am, g, qs)
    assert torch.allclose(torch.as_tensor(d_csr).double(), torch.as_tensor(d_sc).double(), rtol=1e-6, atol=1e-9)
    assert mx.choose_gradient_path(am, threshold=0) == "csr"
    assert mx.choose_gradient_path(am, threshold=10 ** 9) == "scatter"
