"""Drop-in check with the REAL reference objects: inputs are built by the unmodified reference
package (`baseline/_ref/maxsim`: its synth generators, EmbeddingMatrix, DocBatch, ArgmaxMap,
QuantizedMatrix, PackedCorpus, PointSet, MXS1 writer), passed unconverted into this package's
API, and the results are compared with what the reference itself returns for the same call --
the switch a reference user makes.

The reference runs here as the checker only (CPU, small shapes).  Skipped when the reference
install (`baseline/_ref`) is absent.
"""

import importlib
import os
import sys

import numpy as np
import pytest
import torch

import paper_2605_29517_b200 as mx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "maxsim")), reason="baseline/_ref not installed")]


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF)
    try:
        m = importlib.import_module("maxsim")
        for sub in ("synth", "backward", "quant", "varlen", "streamio", "chamfer"):
            importlib.import_module("maxsim." + sub)
        yield m
    finally:
        sys.path.remove(REF)


def host(x):
    if hasattr(x, "numpy") and not isinstance(x, torch.Tensor):
        return np.asarray(x.numpy())
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def _ragged_batch(ref, n_docs, max_len, dim, seed):
    lens = ref.synth.doc_lengths("uniform", n_docs, max_len, seed)
    return ref.synth.padded_batch(ref.synth.make_corpus(n_docs, lens, dim, seed + 1), max_len)


def test_forward_pair_and_batch_bitwise(ref):
    queries = ref.synth.make_queries(3, 24, 32, seed=5)
    docs = _ragged_batch(ref, 9, 40, 32, seed=6)
    assert isinstance(docs, ref.DocBatch)
    rs, ra, rrep = ref.fused_score_batch(queries, docs)
    s, a, rep = mx.fused_score_batch(queries, docs)  # reference objects, unconverted
    assert np.array_equal(host(s), host(rs.values)) and np.array_equal(host(a.indices), host(ra.indices))
    assert rep.mac_count == rrep.mac_count
    # explicit conversion path
    ours = mx.DocBatch.from_reference(docs)
    assert np.array_equal(ours.valid_lens_host, np.asarray(docs.valid_lens))
    assert np.array_equal(host(ours.data), np.asarray(docs.data))
    sc, arg, _ = mx.fused_score_pair(queries[0], ref.EmbeddingMatrix(docs.data[2]), valid_len=int(docs.valid_lens[2]))
    rsc, rarg, _ = ref.fused_score_pair(queries[0], ref.EmbeddingMatrix(docs.data[2]), valid_len=int(docs.valid_lens[2]))
    assert float(sc) == float(rsc) and np.array_equal(host(arg), host(rarg))


def test_backward_with_reference_argmax(ref):
    queries = ref.synth.make_queries(2, 16, 24, seed=7)
    docs = _ragged_batch(ref, 5, 30, 24, seed=8)
    _, ra, _ = ref.fused_score_batch(queries, docs)
    g = np.random.default_rng(9).standard_normal((2, 5))
    rq, rd = ref.backward_dispatch(ra, g, queries, docs)
    dq, dd = mx.backward_dispatch(ra, g, queries, docs)  # the reference's own ArgmaxMap
    assert np.allclose(host(dq), rq, rtol=1e-5, atol=1e-6)
    assert np.allclose(host(dd).reshape(rd.shape), rd, rtol=1e-5, atol=1e-6)
    rc = ref.build_inverse_csr(ra)
    rp, ci = mx.build_inverse_csr(ra).to_numpy()
    assert np.array_equal(rp, rc.row_ptr) and np.array_equal(ci, rc.col_idx)


def test_int8_quantizer_and_scores_bitwise(ref):
    rng = np.random.default_rng(10)
    q = ref.EmbeddingMatrix(rng.standard_normal((20, 64)).astype(np.float32))
    d = ref.EmbeddingMatrix(rng.standard_normal((33, 64)).astype(np.float32))
    rq, rdq = ref.quantize_per_token(q), ref.quantize_per_token(d)
    oq = mx.quantize_per_token(q)
    assert np.array_equal(host(oq.q), rq.q) and np.array_equal(host(oq.scale), rq.scale)
    rsc, rarg = ref.fused_score_int8(rq, rdq, valid_len=29)
    sc, arg = mx.fused_score_int8(rq, rdq, valid_len=29)  # the reference's QuantizedMatrix objects
    assert float(sc) == float(rsc) and np.array_equal(host(arg), rarg)


def test_varlen_with_reference_packed_corpus(ref):
    lens = ref.synth.doc_lengths("uniform", 12, 50, seed=11)
    packed = ref.pack(ref.synth.make_corpus(12, lens, 32, seed=12))
    assert isinstance(packed, ref.PackedCorpus)
    query = ref.synth.make_queries(1, 20, 32, seed=13)[0]
    rs, ra, rrep = ref.fused_score_varlen(query, packed)
    s, a, rep = mx.fused_score_varlen(query, packed)
    assert np.array_equal(host(s), rs) and np.array_equal(host(a.indices), host(ra.indices))
    assert rep.mac_count == rrep.mac_count


def test_two_stage_topk_with_reference_objects(ref):
    query = ref.synth.make_queries(1, 16, 32, seed=14)[0]
    docs = _ragged_batch(ref, 40, 24, 32, seed=15)
    # the reference's corpus form: one QuantizedMatrix per document (maxsim/quant.py:205-216)
    corpus_q = [ref.quantize_per_token(ref.EmbeddingMatrix(np.asarray(docs.data[b]))) for b in range(40)]
    rtop = ref.two_stage_topk(query, corpus_q, docs, k=5)
    top = mx.two_stage_topk(query, corpus_q, docs, k=5)
    assert [int(i) for i, _ in top] == [int(i) for i, _ in rtop]
    assert np.allclose([s for _, s in top], [s for _, s in rtop], rtol=0, atol=0)


def test_chamfer_with_reference_point_sets(ref):
    p, s = ref.synth.point_cloud(300, seed=16), ref.synth.point_cloud(250, seed=17)
    rcd, r1, r2 = ref.chamfer_forward(p, s)
    cd, a1, a2 = mx.chamfer_forward(p, s)
    assert cd == rcd and np.array_equal(host(a1), r1) and np.array_equal(host(a2), r2)
    rp, rs = ref.chamfer_backward(p, s, r1, r2, upstream=0.7)[:2]
    dp, ds = mx.chamfer_backward(p, s, a1, a2, upstream=0.7)
    assert np.array_equal(host(dp), rp) and np.array_equal(host(ds), rs)


def test_streaming_a_reference_written_file(ref, tmp_path):
    docs = ref.synth.padded_batch(ref.synth.make_corpus(30, [20] * 30, 16, seed=18), 20)
    path = str(tmp_path / "corpus.mxs1")
    ref.write_embeddings(path, docs)  # the reference's writer (dense files hold full-length documents)
    query = ref.synth.make_queries(1, 8, 16, seed=19)[0]
    rtop, _ = ref.stream_score_topk(query, ref.CorpusReader(path), block_docs=7, k=6)
    top, _ = mx.stream_score_topk(query, path, block_docs=7, k=6)
    assert [int(i) for i, _ in top] == [int(i) for i, _ in rtop]
    assert [float(v) for _, v in top] == [float(v) for _, v in rtop]
    # ragged corpora are written packed by the reference (write_embeddings refuses ragged dense)
    packed = ref.pack(ref.synth.make_corpus(30, ref.synth.doc_lengths("uniform", 30, 20, 20), 16, seed=21))
    ppath = str(tmp_path / "packed.mxs1")
    ref.write_embeddings(ppath, packed)
    rtop, _ = ref.stream_score_topk(query, ref.CorpusReader(ppath), block_docs=7, k=6)
    top, _ = mx.stream_score_topk(query, ppath, block_docs=7, k=6)
    assert [(int(i), float(v)) for i, v in top] == [(int(i), float(v)) for i, v in rtop]
