"""Generate golden vectors from the REAL reference implementation (run in the build container).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports `maxsim` read-only from /root/reference/pkg/src and writes small .npz fixtures next
to this file.  Those fixtures pin the oracle restatement (oracle/) and, through it, the GPU
path: nothing on the GPU box reads /root/reference.  Each case cites the reference test or
function it comes from.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import maxsim  # noqa: E402
from maxsim import (  # noqa: E402
    ArgmaxMap,
    DocBatch,
    EmbeddingMatrix,
    TileConfig,
    TopKHeap,
    backward_dispatch,
    build_inverse_csr,
    dense_backward,
    fused_score_batch,
    fused_score_int8,
    fused_score_pair,
    fused_score_varlen,
    grad_docs_csr,
    grad_query,
    model_traffic,
    pack,
    quantize_per_token,
    two_stage_topk,
)
from maxsim import synth  # noqa: E402
from maxsim.cli import _softmax_ce  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}.npz  {os.path.getsize(path)} B  keys={sorted(arrays)}")


def padded_arrays(docs: DocBatch):
    return docs.data, docs.valid_lens


def forward_cases():
    # hand cases: tests/test_reference.py:11-24, tests/test_forward.py:33-48
    q = EmbeddingMatrix([[1.0, 0.0], [0.0, 1.0]])
    d = EmbeddingMatrix([[0.5, 0.0], [0.0, 2.0]])
    s1, a1, _ = fused_score_pair(q, d)
    s2, a2, _ = fused_score_pair(q, d, valid_len=1)
    qn = EmbeddingMatrix([[1.0, 0.0]])
    dn = EmbeddingMatrix([[-1.0, 0.0], [-0.5, 0.0], [0.0, 0.0], [0.0, 0.0]])
    s3, a3, _ = fused_score_pair(qn, dn, valid_len=2)
    save("fwd_hand", q=q.data, d=d.data, s_full=np.float64(s1), a_full=a1, s_vl1=np.float64(s2), a_vl1=a2,
         qn=qn.data, dn=dn.data, s_neg=np.float64(s3), a_neg=a3)

    # random ragged batch, not tile aligned (tests/test_forward.py:96-123)
    rng = np.random.default_rng(13)
    queries = [EmbeddingMatrix(rng.standard_normal((37, 12)).astype(np.float32)) for _ in range(3)]
    docs = DocBatch([EmbeddingMatrix(rng.standard_normal((int(n), 12)).astype(np.float32))
                     for n in rng.integers(1, 54, size=7)], padded_len=53)
    sc, am, rep = fused_score_batch(queries, docs)
    save("fwd_ragged", Q=np.stack([x.data for x in queries]), D=docs.data, valid_lens=docs.valid_lens,
         scores=sc.values, argmax=am.indices, macs=np.int64(rep.mac_count), bytes_read=np.int64(rep.bytes_read))

    # integer embeddings: exact ties everywhere (tests/test_forward.py:79-92)
    rng = np.random.default_rng(0)
    qi = [EmbeddingMatrix(rng.integers(-2, 3, size=(6, 4)).astype(np.float32)) for _ in range(2)]
    di = DocBatch([EmbeddingMatrix(rng.integers(-2, 3, size=(40, 4)).astype(np.float32)) for _ in range(3)])
    sc, am, _ = fused_score_batch(qi, di)
    save("fwd_ties", Q=np.stack([x.data for x in qi]), D=di.data, valid_lens=di.valid_lens, scores=sc.values,
         argmax=am.indices)

    # C1 (configs[0]): ColBERT rerank 1 x 1000, L_q=32, L_d=180, d=128, FP32
    qs = synth.make_queries(1, 32, 128, seed=0)
    corpus = synth.make_corpus(1000, np.full(1000, 180), 128, seed=1)
    batch = synth.padded_batch(corpus)
    sc, am, rep = fused_score_batch(qs, batch)
    save("fwd_c1", scores=sc.values, argmax=am.indices, macs=np.int64(rep.mac_count),
         bytes_read=np.int64(rep.bytes_read), bytes_written=np.int64(rep.bytes_written),
         q_head=qs[0].data[:2], d_head=batch.data[:2, :3])


def synth_cases():
    qs = synth.make_queries(2, 5, 16, seed=3)
    lens = synth.doc_lengths("hotpot", 20, 64, seed=4)
    lens_u = synth.doc_lengths("uniform", 20, 64, seed=4)
    lens_r = synth.doc_lengths("ragged", 30, 64, seed=4)
    corpus = synth.make_corpus(4, np.array([3, 7, 1, 5]), 16, seed=5)
    planted = synth.planted_corpus(qs[0], 3, 9, seed=6)
    save("synth", queries=np.stack([q.data for q in qs]), lens_hotpot=lens, lens_uniform=lens_u, lens_ragged=lens_r,
         corpus=np.concatenate([c.data for c in corpus]), planted=np.stack([p.data for p in planted]))


def backward_cases():
    # CSR hand case tests/test_backward.py:29-33
    am = ArgmaxMap(np.array([[[1, 1, 0]]], np.int32), [2], padded_len=2)
    csr = build_inverse_csr(am)
    hand = dict(h_argmax=am.indices, h_row_ptr=csr.row_ptr, h_col_idx=csr.col_idx)
    # all-hot extreme tests/test_acceptance.py:213-219
    hot = ArgmaxMap(np.zeros((3, 4, 5), np.int32), [6, 6, 6, 6], padded_len=6)
    csr_hot = build_inverse_csr(hot)
    # random maps, padded and packed
    rng = np.random.default_rng(5)
    idx = rng.integers(0, 8, size=(2, 3, 16)).astype(np.int32)
    am_r = ArgmaxMap(idx, [8, 8, 8], padded_len=8)
    csr_r = build_inverse_csr(am_r)
    lens_p = np.array([3, 9, 4], np.int64)
    idx_p = np.stack([np.stack([rng.integers(0, lens_p[b], size=7) for b in range(3)]) for _ in range(2)]).astype(np.int32)
    am_p = ArgmaxMap(idx_p, lens_p, padded_len=None)
    csr_p = build_inverse_csr(am_p)
    save("csr", **hand, hot_row_ptr=csr_hot.row_ptr, hot_col_idx=csr_hot.col_idx, r_argmax=idx,
         r_row_ptr=csr_r.row_ptr, r_col_idx=csr_r.col_idx, p_argmax=idx_p, p_lens=lens_p, p_row_ptr=csr_p.row_ptr,
         p_col_idx=csr_p.col_idx)

    # full backward on a forward argmax (tests/test_backward.py:83-92, 136-156)
    rng = np.random.default_rng(11)
    queries = [EmbeddingMatrix(rng.standard_normal((6, 8)).astype(np.float32)) for _ in range(2)]
    docs = DocBatch([EmbeddingMatrix(rng.standard_normal((int(n), 8)).astype(np.float32)) for n in (7, 5, 7)],
                    padded_len=7)
    g = rng.standard_normal((2, 3))
    sc, am, _ = fused_score_batch(queries, docs)
    d_q, d_d = backward_dispatch(am, g, queries, docs, threshold=0)  # force the CSR path
    csr = build_inverse_csr(am)
    flat = grad_docs_csr(csr, g, queries)
    ref_dq, ref_dd = dense_backward(queries, docs, g, am)
    save("backward", Q=np.stack([x.data for x in queries]), D=docs.data, valid_lens=docs.valid_lens, g=g,
         argmax=am.indices, dQ=d_q, dD=d_d, flat_dD=flat, dense_dQ=ref_dq, dense_dD=ref_dd,
         row_ptr=csr.row_ptr, col_idx=csr.col_idx)

    # in-batch contrastive upstream (maxsim/cli.py:198-206) on a C3-like small case
    rng = np.random.default_rng(7)
    qs = rng.standard_normal((4, 5, 8)).astype(np.float32)
    ds = rng.standard_normal((4, 6, 8)).astype(np.float32)
    sc, am, _ = fused_score_batch([EmbeddingMatrix(x) for x in qs], DocBatch([EmbeddingMatrix(x) for x in ds]))
    loss, grad = _softmax_ce(sc.values)
    dq, dd = backward_dispatch(am, grad, [EmbeddingMatrix(x) for x in qs], DocBatch([EmbeddingMatrix(x) for x in ds]))
    save("inbatch", Q=qs, D=ds, scores=sc.values, argmax=am.indices, loss=np.float64(loss), g=grad, dQ=dq, dD=dd)


def quant_cases():
    # tests/test_quant.py:34-42
    a = quantize_per_token(np.array([[0.5, -1.0]], np.float32))
    z = quantize_per_token(np.zeros((2, 3), np.float32))
    rng = np.random.default_rng(21)
    x = rng.standard_normal((50, 40)).astype(np.float32)
    x[3] = 0.0
    x[4, :5] = [0.5, -0.5, 1.5, 2.5, -2.5]  # half-way rounding cases after scaling
    full = quantize_per_token(x)
    coarse = quantize_per_token(x, levels=7)
    save("quant", a_q=a.q, a_s=a.scale, z_q=z.q, z_s=z.scale, x=x, q127=full.q, s127=full.scale, q7=coarse.q,
         s7=coarse.scale)

    # INT8 pair scoring incl. masking (tests/test_quant.py:60-77)
    rng = np.random.default_rng(22)
    qf = rng.standard_normal((9, 32)).astype(np.float32)
    qq = quantize_per_token(qf)
    docs = [rng.standard_normal((int(n), 32)).astype(np.float32) for n in (20, 13, 20, 1)]
    dq = [quantize_per_token(np.pad(d, ((0, 20 - d.shape[0]), (0, 0)))) for d in docs]
    scores, args = [], []
    for b, qm in enumerate(dq):
        s, a_ = fused_score_int8(qq, qm, valid_len=docs[b].shape[0])
        scores.append(s)
        args.append(a_)
    save("int8", qf=qf, q_q=qq.q, q_s=qq.scale, d_q=np.stack([m.q for m in dq]), d_s=np.stack([m.scale for m in dq]),
         valid_lens=np.array([d.shape[0] for d in docs], np.int32), scores=np.array(scores), argmax=np.stack(args))

    # two-stage top-K on a planted corpus (tests/test_quant.py:125-140)
    q = synth.make_queries(1, 8, 32, seed=1)[0]
    corpus = synth.planted_corpus(q, 30, 12, seed=2)
    batch = synth.padded_batch(corpus)
    cq = [quantize_per_token(c) for c in corpus]
    top = two_stage_topk(q, cq, batch, k=5)
    save("two_stage", q=q.data, D=batch.data, top_ids=np.array([t[0] for t in top]),
         top_scores=np.array([t[1] for t in top]))


def varlen_cases():
    rng = np.random.default_rng(31)
    q = EmbeddingMatrix(rng.standard_normal((7, 16)).astype(np.float32))
    docs = [rng.standard_normal((int(n), 16)).astype(np.float32) for n in (5, 1, 12, 3, 8)]
    pk = pack(docs)
    s, am, rep = fused_score_varlen(q, pk)
    save("varlen", q=q.data, tokens=pk.tokens, cu=pk.cu_seqlens, scores=s, argmax=am.indices,
         macs=np.int64(rep.mac_count))


def misc_cases():
    h = TopKHeap(2)
    for i, s in [(3, 1.0), (1, 1.0), (2, 0.5), (4, 1.0)]:
        h.offer(i, s)
    ranked = h.ranked()
    rng = np.random.default_rng(41)
    scores = np.round(rng.standard_normal(200), 1)  # many exact ties
    h2 = TopKHeap(15)
    for i, s in enumerate(scores):
        h2.offer(i, float(s))
    r2 = h2.ranked()
    tm = model_traffic(1, 1000, 1024, 1024, 128, elem_bytes=2)
    save("misc", heap_ids=np.array([r[0] for r in ranked]), heap_scores=np.array([r[1] for r in ranked]),
         tie_scores=scores, tie_ids=np.array([r[0] for r in r2]), tie_top=np.array([r[1] for r in r2]),
         traffic=np.array([tm.fused_read, tm.fused_write, tm.naive_read, tm.naive_write], np.int64))


def chamfer_cases():
    """maxsim/chamfer.py: hand case (tests/test_chamfer.py:36-42), random clouds vs the dense
    oracle (:51-63), ties (identical sets, :44-49), 5-D points, backward with upstream 1.7
    (:109-118) -- forward and backward outputs of the reference itself."""
    from maxsim import PointSet, chamfer_backward, chamfer_forward
    from maxsim.synth import point_cloud

    hp = PointSet([[0.0, 0.0, 0.0]])
    hs = PointSet([[1.0, 0.0, 0.0], [0.0, 2.0, 0.0]])
    hcd, ha1, ha2 = chamfer_forward(hp, hs)
    p, s = point_cloud(200, seed=23), point_cloud(300, seed=24)
    cd, a1, a2 = chamfer_forward(p, s)
    dp, ds = chamfer_backward(p, s, a1, a2, upstream=1.7)
    p5, s5 = point_cloud(70, seed=3, dim=5), point_cloud(45, seed=4, dim=5, scale=2.0)
    cd5, b1, b2 = chamfer_forward(p5, s5)
    dp5, ds5 = chamfer_backward(p5, s5, b1, b2)
    # exact ties: duplicated points in the second set (lowest index must win)
    rng = np.random.default_rng(8)
    base = np.round(rng.standard_normal((20, 3)), 1).astype(np.float32)
    tp = PointSet(base)
    ts = PointSet(np.concatenate([base[::-1], base]).astype(np.float32))
    cdt, t1, t2 = chamfer_forward(tp, ts)
    save("chamfer", h_p=hp.data, h_s=hs.data, h_cd=np.float64(hcd), h_a1=ha1, h_a2=ha2, p=p.data, s=s.data,
         cd=np.float64(cd), a1=a1, a2=a2, dp=dp, ds=ds, p5=p5.data, s5=s5.data, cd5=np.float64(cd5), b1=b1, b2=b2,
         dp5=dp5, ds5=ds5, tp=tp.data, ts=ts.data, cdt=np.float64(cdt), t1=t1, t2=t2)


if __name__ == "__main__":
    np.seterr(all="ignore")
    cases = {"forward": forward_cases, "synth": synth_cases, "backward": backward_cases, "quant": quant_cases,
             "varlen": varlen_cases, "misc": misc_cases, "chamfer": chamfer_cases}
    for name in (sys.argv[1:] or list(cases)):
        cases[name]()
    print("reference version", maxsim.__version__)
