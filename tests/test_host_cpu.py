"""Host-side logic of the operator layer (types, validation, dispatch, ranking, sharding).

Runs without a GPU: tensors stay on the host, and every compute entry point must refuse to
run there (no CPU fallback).
"""

import numpy as np
import pytest
import torch

import paper_2605_29517_b200 as mx
from conftest import golden
from oracle import oracle as orc
from paper_2605_29517_b200.parallel import shard_bounds, softmax_ce


def test_embedding_matrix_validation():
    e = mx.EmbeddingMatrix(np.ones((3, 4), np.float32))
    assert (e.rows, e.dim, e.elem) == (3, 4, "f32")
    bad = np.ones((2, 3), np.float32)
    bad[1, 2] = np.nan
    with pytest.raises(mx.NaNInput) as ei:
        mx.EmbeddingMatrix(bad)
    assert ei.value.location == ("embeddings", 1, 2)
    with pytest.raises(mx.ShapeMismatch):
        mx.EmbeddingMatrix(np.ones(4, np.float32))
    with pytest.raises(mx.ShapeMismatch):
        mx.EmbeddingMatrix(np.ones((3, 0), np.float32))
    bf = mx.EmbeddingMatrix(torch.ones(2, 8, dtype=torch.bfloat16))
    assert bf.elem == "bf16"


def test_docbatch_padding_and_errors():
    docs = [np.ones((2, 4), np.float32), np.ones((5, 4), np.float32)]
    db = mx.DocBatch(docs)
    assert db.padded_len == 5 and list(db.valid_lens_host) == [2, 5]
    assert float(db.data[0, 2:].abs().sum()) == 0.0  # zero padding
    with pytest.raises(mx.EmptyDocument) as ei:
        mx.DocBatch([np.ones((2, 4), np.float32), np.zeros((0, 4), np.float32), np.ones((1, 4), np.float32)])
    assert ei.value.index == 1
    with pytest.raises(mx.DimMismatch):
        mx.DocBatch([np.ones((2, 4), np.float32), np.ones((2, 5), np.float32)])
    with pytest.raises(mx.ShapeMismatch):
        mx.DocBatch(docs, padded_len=3)
    with pytest.raises(mx.ShapeMismatch):
        mx.DocBatch([])
    fd = mx.DocBatch.from_dense(np.zeros((3, 6, 4), np.float32), valid_lens=[6, 1, 2])
    assert list(fd.valid_lens_host) == [6, 1, 2]
    with pytest.raises(mx.EmptyDocument):
        mx.DocBatch.from_dense(np.zeros((2, 6, 4), np.float32), valid_lens=[6, 0])


def test_argmax_map_destinations_match_reference():
    # tests/test_types.py:111-117: padded [1, 4] and packed [1, 2]
    am = mx.ArgmaxMap(np.array([[[1], [1]]], np.int32), [2, 3], padded_len=3)
    assert am.flat_destinations().tolist() == [1, 4]
    am = mx.ArgmaxMap(np.array([[[1], [0]]], np.int32), [2, 3], padded_len=None)
    assert am.flat_destinations().tolist() == [1, 2]
    assert am.n_dest_rows == 5 and am.n_sources == 2
    with pytest.raises(mx.IndexOutOfRange):
        mx.ArgmaxMap(np.array([[[2]]], np.int32), [2], padded_len=4)
    with pytest.raises(mx.IndexOutOfRange):
        mx.ArgmaxMap(np.array([[[-1]]], np.int32), [2], padded_len=4)
    with pytest.raises(mx.ShapeMismatch):
        mx.ArgmaxMap(np.zeros((1, 2), np.int32), [1, 1])
    # int32 indices near 2^31 (tests/test_types.py:104-109)
    big = mx.ArgmaxMap(np.array([[[2**31 - 2]]], np.int32), [2**31 - 1], padded_len=None)
    assert int(big.flat_destinations()[0]) == 2**31 - 2


def test_tile_config_and_dispatch():
    with pytest.raises(mx.BadTileConfig):
        mx.TileConfig(bq=0)
    with pytest.raises(mx.BadTileConfig):
        mx.TileConfig(bq=32, bd=64, qchunk=48)
    assert mx.dispatch(1, 10, 32, 180, 128).tag == "single_query_rerank"
    assert mx.dispatch(4, 10, 32, 180, 128).tag == "batched_multiquery"
    assert mx.dispatch(1, 10, 32, 180, 128, packed=True).tag == "varlen_packed"
    assert mx.dispatch(1, 10, 32, 180, 128, dtype="i8", packed=True).tag == "int8_two_stage"
    assert mx.dispatch(1, 10, 32, 4096, 128).tile.bd == 128
    with pytest.raises(ValueError):
        mx.dispatch(0, 1, 1, 1, 1)


def test_validate_pair():
    mx.validate_pair(np.ones((2, 3), np.float32), np.ones((4, 3), np.float32))
    with pytest.raises(mx.DimMismatch):
        mx.validate_pair(np.ones((2, 3), np.float32), np.ones((4, 5), np.float32))
    with pytest.raises(mx.ShapeMismatch):
        mx.validate_pair(np.ones((2, 3), np.int8), np.ones((4, 3), np.float32))


def test_topk_heap_tie_semantics():
    g = golden("misc")
    h = mx.TopKHeap(2)
    for i, s in [(3, 1.0), (1, 1.0), (2, 0.5), (4, 1.0)]:
        h.offer(i, s)
    assert [r[0] for r in h.ranked()] == list(g["heap_ids"])
    h2 = mx.TopKHeap(15)
    h2.offer_many(range(200), g["tie_scores"])
    assert [r[0] for r in h2.ranked()] == list(g["tie_ids"])
    a, b = mx.TopKHeap(3), mx.TopKHeap(3)
    a.offer_many([0, 1, 2], [1.0, 0.5, 0.25])
    b.offer_many([3, 4], [1.0, 0.75])
    a.merge(b)
    assert a.ranked() == [(0, 1.0), (3, 1.0), (4, 0.75)]


def test_select_candidates_has_no_host_path():
    """The candidate merge runs on the device only (no CPU fallback); the gloo tests inject their
    own CPU twin through merge_topk_across_ranks(select=...)."""
    from paper_2605_29517_b200.topk import select_candidates

    if torch.cuda.is_available():
        pytest.skip("host-only check")
    with pytest.raises(Exception):
        select_candidates(torch.tensor([1.0, 2.0]), torch.tensor([0, 1]), 1)


def test_shard_bounds_cover_and_balance():
    for n, w in ((10000, 8), (7, 3), (1, 2)):
        spans = [shard_bounds(n, w, r) for r in range(w)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
    lens = np.random.default_rng(0).integers(32, 513, 10000)
    spans = [shard_bounds(10000, 8, r, weights=lens) for r in range(8)]
    assert spans[0][0] == 0 and spans[-1][1] == 10000
    toks = [lens[lo:hi].sum() for lo, hi in spans]
    assert max(toks) / min(toks) < 1.01


def test_softmax_ce_matches_reference():
    g = golden("inbatch")
    loss, grad = softmax_ce(torch.tensor(g["scores"]))
    assert abs(float(loss) - float(g["loss"])) < 1e-12
    assert np.allclose(grad.numpy(), g["g"], rtol=0, atol=1e-15)


def test_traffic_report_and_byte_model():
    rep = mx.TrafficReport()
    rep.add_read(10)
    rep.add_macs(4)
    other = mx.TrafficReport()
    other.add_read(5)
    other.alloc(100)
    other.release(100)
    rep.merge(other)
    assert rep.as_dict() == {"bytes_read": 15, "bytes_written": 0, "peak_aux_bytes": 100, "mac_count": 4}
    g = golden("misc")
    tm = mx.model_traffic(1, 1000, 1024, 1024, 128, elem_bytes=2)
    assert [tm.fused_read, tm.fused_write, tm.naive_read, tm.naive_write] == list(g["traffic"])
    assert tm.naive_over_fused == tm.naive_total / tm.fused_total and tm.bytes("fused") == tm.fused_total
    with pytest.raises(ValueError):
        mx.model_traffic(0, 1, 1, 1, 1)


def test_compute_refuses_host_tensors():
    """No CPU fallback: the operators only run on CUDA tensors."""
    if torch.cuda.is_available():
        pytest.skip("host-only check")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mx.score_dense(torch.zeros(1, 4, 8), torch.zeros(2, 4, 8))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mx.fused_score_batch([np.ones((4, 8), np.float32)], mx.DocBatch([np.ones((3, 8), np.float32)]))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mx.quantize_per_token(np.ones((4, 8), np.float32))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mx.topk(torch.zeros(5, dtype=torch.float64), 2)


def test_packed_corpus_validation():
    pk = mx.pack([np.ones((2, 4), np.float32), np.ones((3, 4), np.float32)])
    assert list(pk.cu_seqlens) == [0, 2, 5] and pk.total_tokens == 5
    with pytest.raises(mx.EmptyDocument):
        mx.PackedCorpus(np.ones((5, 4), np.float32), [0, 2, 2, 5])
    with pytest.raises(mx.ShapeMismatch):
        mx.PackedCorpus(np.ones((5, 4), np.float32), [0, 2, 4])
    with pytest.raises(mx.ShapeMismatch):
        mx.PackedCorpus(np.ones((5, 4), np.float32), [1, 5])
    assert [d.rows for d in mx.unpack(pk)] == [2, 3]
