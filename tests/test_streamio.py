"""MXS1 files (native reader, our writer) and out-of-core streamed scoring.

CPU part (no GPU needed): the native reader parses the fixtures written by the REAL reference
writer (tests/golden/make_mxs1.py) bit for bit, reports the reference's error classes and
fields, and our writer reproduces those files byte for byte
(maxsim/streamio.py:57-163; tests/test_streamio.py:27-119 of the reference).

GPU part: stream_score_topk ranks exactly like in-memory scoring + top-K, and like the oracle
(bit-exact for f32 files, which take the exact fp32 kernel); GPU memory stays flat in corpus
size (maxsim/streamio.py:265-322; reference tests/test_acceptance.py:387-408).
"""

import os
import shutil
import struct

import numpy as np
import pytest
import torch

import paper_2605_29517_b200 as mx
from conftest import GOLDEN, cuda_ok
from oracle import oracle as orc
from paper_2605_29517_b200 import streamio

FIX = os.path.join(GOLDEN, "mxs1")


def expected():
    return np.load(os.path.join(FIX, "mxs1_expected.npz"))


def stand_in(name, **attrs):
    """Host-side object with a reference type name (the writer dispatches on the name)."""
    return type(name, (), attrs)()


# ------------------------------------------------------------------ reader (CPU)
@pytest.mark.parametrize("fname,elem", [("dense_f32", "f32"), ("dense_f16", "f16")])
def test_reader_dense_fixture(fname, elem):
    e = expected()
    with streamio.CorpusReader(os.path.join(FIX, fname + ".mxs1")) as r:
        assert (r.elem, r.layout, r.n_docs, r.length, r.dim) == (elem, "dense", 7, 9, 16)
        want = e["dense"].astype(np.float16) if elem == "f16" else e["dense"]
        whole, rel = r.read_block_host(0, 7)
        assert rel is None and np.array_equal(whole, want)
        part, _ = r.read_block_host(5, 10)  # clipped at the end like the reference
        assert np.array_equal(part, want[5:])
        assert r.block_bytes(2, 3) == 3 * 9 * 16 * (4 if elem == "f32" else 2)


@pytest.mark.parametrize("fname,elem", [("packed_f32", "f32"), ("packed_f16", "f16")])
def test_reader_packed_fixture(fname, elem):
    e = expected()
    with streamio.CorpusReader(os.path.join(FIX, fname + ".mxs1")) as r:
        assert (r.elem, r.layout, r.n_docs, r.dim) == (elem, "packed", 5, 16)
        assert np.array_equal(r.cu_seqlens, e["packed_cu"])
        toks = e["packed_tokens"].astype(np.float16) if elem == "f16" else e["packed_tokens"]
        blk, rel = r.read_block_host(1, 3)
        cu = e["packed_cu"]
        assert np.array_equal(rel, cu[1:5] - cu[1]) and np.array_equal(blk, toks[cu[1]:cu[4]])


def test_reader_quantized_fixture():
    e = expected()
    with pytest.raises(mx.ShapeMismatch):
        streamio.CorpusReader(os.path.join(FIX, "quant.mxs1"))  # streaming refuses quantized files
    r = streamio.CorpusReader(os.path.join(FIX, "quant.mxs1"), _allow_quantized=True)
    q, _ = r.read_block_host(0, r.n_docs)
    assert np.array_equal(q, e["quant_q"])
    s = np.empty(e["quant_scales"].shape, np.float32)
    mx._lib.check(mx._lib.load().mxs_mxs1_read_scales(r._h, s.ctypes.data, s.nbytes))
    assert np.array_equal(s, e["quant_scales"])
    r.close()


def _corrupt(tmp_path, name, mutate):
    p = tmp_path / name
    shutil.copy(os.path.join(FIX, "dense_f32.mxs1"), p)
    raw = bytearray(p.read_bytes())
    p.write_bytes(bytes(mutate(raw)))
    return str(p)


def test_reader_errors(tmp_path):
    with pytest.raises(mx.IoError):
        streamio.CorpusReader(str(tmp_path / "missing.mxs1"))
    with pytest.raises(mx.BadMagic, match="bad magic"):
        streamio.CorpusReader(_corrupt(tmp_path, "m", lambda b: b"NOPE" + b[4:]))
    with pytest.raises(mx.BadMagic, match="too short"):
        streamio.CorpusReader(_corrupt(tmp_path, "s", lambda b: b[:5]))
    with pytest.raises(mx.VersionUnsupported) as ei:
        streamio.CorpusReader(_corrupt(tmp_path, "v", lambda b: b[:4] + struct.pack("<H", 2) + b[6:]))
    assert ei.value.version == 2
    with pytest.raises(mx.BadMagic, match="unknown element/layout"):
        streamio.CorpusReader(_corrupt(tmp_path, "t", lambda b: b[:6] + bytes([7]) + b[7:]))
    with pytest.raises(mx.BadMagic, match="int8 elements require"):
        streamio.CorpusReader(_corrupt(tmp_path, "i", lambda b: b[:6] + bytes([2]) + b[7:]))
    with pytest.raises(mx.TruncatedPayload) as ei:
        streamio.CorpusReader(_corrupt(tmp_path, "h", lambda b: b[:20]))  # header field cut
    assert (ei.value.expected, ei.value.actual) == (8, 4)
    r = streamio.CorpusReader(_corrupt(tmp_path, "p", lambda b: b[:-100]))  # payload cut
    with pytest.raises(mx.TruncatedPayload) as ei:
        r.read_block_host(0, 7)
    assert ei.value.expected == 7 * 9 * 16 * 4 and ei.value.actual == 7 * 9 * 16 * 4 - 100
    assert isinstance(ei.value, mx.IoError)
    r.close()


def test_reader_hostile_headers(tmp_path):
    """Untrusted header counts raise the reference's error classes instead of aborting the
    process: the offset table of a packed file is sized against the file before it is allocated,
    products that overflow int64 are refused, and the PackedCorpus invariants
    (maxsim/varlen.py:36-41) hold for what the reader hands out."""
    head = b"MXS1" + struct.pack("<H", 1)

    def write(name, body):
        p = tmp_path / name
        p.write_bytes(body)
        return str(p)

    for n_docs in (1 << 40, (1 << 63) + 5, (1 << 64) - 1):  # huge, and top bit set (negative as int64)
        path = write(f"n{n_docs}", head + bytes([0, 1]) + struct.pack("<QQ", n_docs, 16) + b"\0" * 64)
        with pytest.raises(mx.TruncatedPayload) as ei:
            streamio.CorpusReader(path)
        assert ei.value.actual == 64 and ei.value.expected > 64
    # dense: n_docs * length * dim * 4 overflows int64
    with pytest.raises(mx.TruncatedPayload):
        streamio.CorpusReader(write("ovf", head + bytes([0, 0]) + struct.pack("<QQQ", 1 << 40, 1 << 20, 1 << 10)))
    # packed offset table: cu[0] != 0, an empty document, a decreasing offset
    for cu, err in (([1, 3, 5], mx.ShapeMismatch), ([0, 3, 3], mx.EmptyDocument), ([0, 3, 2], mx.EmptyDocument)):
        body = head + bytes([0, 1]) + struct.pack("<QQ", len(cu) - 1, 4) + struct.pack(f"<{len(cu)}Q", *cu)
        with pytest.raises(err) as ei:
            streamio.CorpusReader(write("cu", body + b"\0" * 80))
        if err is mx.EmptyDocument:
            assert ei.value.index == 1


# ------------------------------------------------------------------ writer (CPU)
def test_writer_reproduces_reference_files(tmp_path):
    e = expected()
    dense = e["dense"]
    lens = np.full(7, 9, np.int32)
    for elem in ("f32", "f16"):
        p = tmp_path / f"d_{elem}.mxs1"
        streamio.write_embeddings(str(p), stand_in("DocBatch", data=dense, valid_lens=lens), elem=elem)
        assert p.read_bytes() == open(os.path.join(FIX, f"dense_{elem}.mxs1"), "rb").read()
        p = tmp_path / f"p_{elem}.mxs1"
        streamio.write_embeddings(str(p), stand_in("PackedCorpus", tokens=e["packed_tokens"],
                                                   cu_seqlens=e["packed_cu"]), elem=elem)
        assert p.read_bytes() == open(os.path.join(FIX, f"packed_{elem}.mxs1"), "rb").read()
    p = tmp_path / "q.mxs1"
    streamio.write_embeddings(str(p), stand_in("QuantizedCorpus", q=e["quant_q"], scales=e["quant_scales"]))
    assert p.read_bytes() == open(os.path.join(FIX, "quant.mxs1"), "rb").read()
    with pytest.raises(mx.ShapeMismatch):
        streamio.write_embeddings(str(tmp_path / "x"), stand_in("DocBatch", data=dense, valid_lens=lens - 1))
    with pytest.raises(mx.ShapeMismatch):
        streamio.write_embeddings(str(tmp_path / "y"), stand_in("DocBatch", data=dense, valid_lens=lens), elem="i8")
    with pytest.raises(mx.ShapeMismatch):
        streamio.write_embeddings(str(tmp_path / "z"), object())


# ------------------------------------------------------------------ streaming (GPU)
def _write_dense(path, docs, elem):
    streamio.write_embeddings(path, stand_in("DocBatch", data=docs, valid_lens=np.full(len(docs), docs.shape[1])),
                              elem=elem)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a GPU")
def test_stream_dense_f16_equals_in_memory(tmp_path):
    rng = np.random.default_rng(21)
    q = orc.unit_tokens(rng, 32, 64).astype(np.float32)
    docs = np.stack([orc.unit_tokens(rng, 40, 64) for _ in range(300)]).astype(np.float32)
    path = str(tmp_path / "c.mxs1")
    _write_dense(path, docs, "f16")
    ranked, rep = mx.stream_score_topk(mx.EmbeddingMatrix(torch.from_numpy(q).cuda()), path, block_docs=64, k=20)
    s, _, _ = mx.score_dense(torch.from_numpy(q).cuda().half()[None], torch.from_numpy(docs).cuda().half())
    ts, ti = mx.topk(s[0], 20)
    assert [r[0] for r in ranked] == ti.cpu().tolist() and [r[1] for r in ranked] == ts.cpu().tolist()
    # and the oracle on the same f16-rounded values: scores within 1e-3 relative
    os_, _ = orc.fused_score_batch(q.astype(np.float16).astype(np.float32)[None],
                                   docs.astype(np.float16).astype(np.float32))
    got = np.array([r[1] for r in ranked])
    ref = os_[0][[r[0] for r in ranked]]
    assert np.max(np.abs(got - ref) / np.abs(ref)) < 1e-3
    assert rep.bytes_read == 32 * 64 * 2 + 300 * 40 * 64 * 2


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a GPU")
def test_stream_packed_f32_bit_exact_with_oracle(tmp_path):
    rng = np.random.default_rng(22)
    q = orc.unit_tokens(rng, 32, 64).astype(np.float32)
    lens = rng.integers(1, 60, 300)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    toks = orc.unit_tokens(rng, int(cu[-1]), 64).astype(np.float32)
    path = str(tmp_path / "p.mxs1")
    streamio.write_embeddings(path, stand_in("PackedCorpus", tokens=toks, cu_seqlens=cu))
    ranked, _ = mx.stream_score_topk(q, path, block_docs=37, k=25)
    ref, _ = orc.fused_score_varlen(q[None], toks, cu)
    oi = orc.topk(ref[0], 25)
    assert [r[0] for r in ranked] == oi[1].tolist() and [r[1] for r in ranked] == oi[0].tolist()
    with pytest.raises(mx.KTooLarge):
        mx.stream_score_topk(q, path, block_docs=37, k=301)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a GPU")
def test_stream_peak_memory_flat_in_corpus_size(tmp_path):
    rng = np.random.default_rng(23)
    q = torch.from_numpy(orc.unit_tokens(rng, 32, 128).astype(np.float32)).cuda()
    peaks = []
    for n in (256, 2048):
        docs = np.stack([orc.unit_tokens(rng, 64, 128) for _ in range(n)]).astype(np.float32)
        path = str(tmp_path / f"c{n}.mxs1")
        _write_dense(path, docs, "f16")
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        mx.stream_score_topk(q, path, block_docs=128, k=10)
        torch.cuda.synchronize()
        peaks.append(torch.cuda.max_memory_allocated() - base)
    assert peaks[1] <= peaks[0] * 1.05 + (1 << 16)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a GPU")
def test_read_embeddings_to_device():
    e = expected()
    d = mx.read_embeddings(os.path.join(FIX, "dense_f32.mxs1"))
    assert np.array_equal(d.data.cpu().numpy(), e["dense"])
    p = mx.read_embeddings(os.path.join(FIX, "packed_f16.mxs1"))
    assert np.array_equal(p.tokens.float().cpu().numpy(), e["packed_tokens"].astype(np.float16).astype(np.float32))
    qc = mx.read_embeddings(os.path.join(FIX, "quant.mxs1"))
    assert np.array_equal(qc.q.cpu().numpy(), e["quant_q"]) and np.array_equal(qc.scales.cpu().numpy(),
                                                                                e["quant_scales"])


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a GPU")
def test_stream_score_host_equals_device_scoring():
    rng = np.random.default_rng(24)
    q = torch.from_numpy(orc.unit_tokens(rng, 64, 128).astype(np.float32)).cuda().bfloat16()
    docs = torch.from_numpy(np.stack([orc.unit_tokens(rng, 96, 128) for _ in range(1030)]).astype(np.float32))
    docs = docs.bfloat16().pin_memory()
    scores, ts, ti = mx.stream_score_host(q, docs, k=17, block_docs=256)
    ref, _, _ = mx.score_dense(q[None], docs.cuda(), want_argmax=False)
    rs, ri = mx.topk(ref[0], 17)
    assert torch.equal(scores, ref[0]) and torch.equal(ts, rs) and torch.equal(ti, ri)
