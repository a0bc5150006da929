"""Pin the oracle restatement (oracle/) against golden vectors produced by the reference itself.

CPU only.  Every assertion is bit-exact: the oracle restates the reference's arithmetic order.
"""

import numpy as np

from conftest import golden
from oracle import oracle as orc


def test_forward_hand_cases():
    g = golden("fwd_hand")
    s, a = orc.fused_score_batch(g["q"][None], g["d"][None])
    assert s[0, 0] == g["s_full"] == 2.5 and list(a[0, 0]) == list(g["a_full"]) == [0, 1]
    s, a = orc.fused_score_batch(g["q"][None], g["d"][None], valid_lens=[1])
    assert s[0, 0] == g["s_vl1"] == 0.5 and list(a[0, 0]) == list(g["a_vl1"]) == [0, 0]
    s, a = orc.fused_score_batch(g["qn"][None], g["dn"][None], valid_lens=[2])
    assert s[0, 0] == g["s_neg"] == -0.5 and a[0, 0, 0] == g["a_neg"][0] == 1


def test_forward_ragged_bitwise():
    g = golden("fwd_ragged")
    s, a = orc.fused_score_batch(g["Q"], g["D"], g["valid_lens"])
    assert np.array_equal(s, g["scores"])
    assert np.array_equal(a, g["argmax"])


def test_forward_integer_ties_lowest_index():
    g = golden("fwd_ties")
    s, a = orc.fused_score_batch(g["Q"], g["D"], g["valid_lens"])
    assert np.array_equal(s, g["scores"]) and np.array_equal(a, g["argmax"])


def test_forward_c1_config_bitwise():
    """configs[0]: ColBERT 1x1000, L_q=32, L_d=180, d=128, FP32 -- the reference's own CPU case."""
    g = golden("fwd_c1")
    Q = orc.make_queries(1, 32, 128, seed=0)
    docs = orc.make_corpus(1000, np.full(1000, 180), 128, seed=1)
    D, vl = orc.padded(docs)
    assert np.array_equal(Q[0, :2], g["q_head"]) and np.array_equal(D[:2, :3], g["d_head"])
    s, a = orc.fused_score_batch(Q, D, vl)
    assert np.array_equal(s, g["scores"])
    assert np.array_equal(a, g["argmax"])
    # the reference ledger's FLOP count (maxsim/forward.py:152) and byte model
    assert int(g["macs"]) == 2 * 32 * 180 * 128 * 1000
    read, write = orc.model_traffic(1, 1000, 32, 180, 128)
    assert read == int(g["bytes_read"]) and write == int(g["bytes_written"])


def test_synth_restatement():
    g = golden("synth")
    assert np.array_equal(orc.make_queries(2, 5, 16, seed=3), g["queries"])
    assert np.array_equal(orc.doc_lengths("hotpot", 20, 64, seed=4), g["lens_hotpot"])
    assert np.array_equal(orc.doc_lengths("uniform", 20, 64, seed=4), g["lens_uniform"])
    assert np.array_equal(orc.doc_lengths("ragged", 30, 64, seed=4), g["lens_ragged"])
    c = orc.make_corpus(4, np.array([3, 7, 1, 5]), 16, seed=5)
    assert np.array_equal(np.concatenate(c), g["corpus"])
    p = orc.planted_corpus(g["queries"][0], 3, 9, seed=6)
    assert np.array_equal(np.stack(p), g["planted"])


def test_csr_cases():
    g = golden("csr")
    rp, ci = orc.build_inverse_csr(g["h_argmax"], [2], 2)
    assert list(rp) == [0, 1, 3] and list(ci) == [2, 0, 1]
    assert np.array_equal(rp, g["h_row_ptr"]) and np.array_equal(ci, g["h_col_idx"])
    rp, ci = orc.build_inverse_csr(np.zeros((3, 4, 5), np.int32), [6] * 4, 6)
    assert np.array_equal(rp, g["hot_row_ptr"]) and np.array_equal(ci, g["hot_col_idx"])
    rp, ci = orc.build_inverse_csr(g["r_argmax"], [8, 8, 8], 8)
    assert np.array_equal(rp, g["r_row_ptr"]) and np.array_equal(ci, g["r_col_idx"])
    rp, ci = orc.build_inverse_csr(g["p_argmax"], g["p_lens"], None)
    assert np.array_equal(rp, g["p_row_ptr"]) and np.array_equal(ci, g["p_col_idx"])


def test_backward_bitwise():
    g = golden("backward")
    s, a = orc.fused_score_batch(g["Q"], g["D"], g["valid_lens"])
    assert np.array_equal(a, g["argmax"])
    rp, ci = orc.build_inverse_csr(a, g["valid_lens"], g["D"].shape[1])
    assert np.array_equal(rp, g["row_ptr"]) and np.array_equal(ci, g["col_idx"])
    flat = orc.grad_docs_csr(rp, ci, g["g"], g["Q"], n_docs=3)
    assert np.array_equal(flat, g["flat_dD"])
    assert np.array_equal(flat.reshape(g["dD"].shape), g["dD"])
    assert np.array_equal(flat.reshape(g["dD"].shape), g["dense_dD"])
    B, L, d = g["D"].shape
    dq = orc.grad_query(a, g["g"], g["D"].reshape(B * L, d), np.arange(B) * L)
    assert np.array_equal(dq, g["dQ"]) and np.array_equal(dq, g["dense_dQ"])


def test_inbatch_softmax_ce_and_grads():
    g = golden("inbatch")
    s, a = orc.fused_score_batch(g["Q"], g["D"])
    assert np.array_equal(s, g["scores"]) and np.array_equal(a, g["argmax"])
    loss, grad = orc.softmax_ce(s)
    assert loss == float(g["loss"]) and np.array_equal(grad, g["g"])
    B, L, d = g["D"].shape
    rp, ci = orc.build_inverse_csr(a, [L] * B, L)
    dd = orc.grad_docs_csr(rp, ci, grad, g["Q"], n_docs=B).reshape(B, L, d)
    dq = orc.grad_query(a, grad, g["D"].reshape(B * L, d), np.arange(B) * L)
    assert np.array_equal(dd, g["dD"]) and np.array_equal(dq, g["dQ"])


def test_quantize_bitwise():
    g = golden("quant")
    q, s = orc.quantize_per_token(np.array([[0.5, -1.0]], np.float32))
    assert list(q[0]) == [64, -127] and s[0] == np.float32(1.0) / np.float32(127)
    assert np.array_equal(q, g["a_q"]) and np.array_equal(s, g["a_s"])
    q, s = orc.quantize_per_token(np.zeros((2, 3), np.float32))
    assert np.all(s == np.float32(1e-12)) and np.array_equal(q, g["z_q"])
    q, s = orc.quantize_per_token(g["x"])
    assert np.array_equal(q, g["q127"]) and np.array_equal(s, g["s127"])
    q, s = orc.quantize_per_token(g["x"], levels=7)
    assert np.array_equal(q, g["q7"]) and np.array_equal(s, g["s7"])


def test_int8_scores_bitwise():
    g = golden("int8")
    q, s = orc.quantize_per_token(g["qf"])
    assert np.array_equal(q, g["q_q"]) and np.array_equal(s, g["q_s"])
    sc, a = orc.fused_score_int8(g["q_q"][None], g["q_s"][None], g["d_q"], g["d_s"], g["valid_lens"])
    assert np.array_equal(sc[0], g["scores"])
    assert np.array_equal(a[0], g["argmax"])


def test_two_stage_topk_against_reference():
    g = golden("two_stage")
    q = g["q"]
    D = g["D"]
    B = D.shape[0]
    qq, qs = orc.quantize_per_token(q)
    dq = np.stack([orc.quantize_per_token(D[b])[0] for b in range(B)])
    ds = np.stack([orc.quantize_per_token(D[b])[1] for b in range(B)])
    coarse, _ = orc.fused_score_int8(qq[None], qs[None], dq, ds)
    order = np.lexsort((np.arange(B), -coarse[0]))[: 5 * 4]
    full, _ = orc.fused_score_batch(q[None], D[order])
    resc = sorted(zip(order.tolist(), full[0].tolist()), key=lambda t: (-t[1], t[0]))[:5]
    assert [r[0] for r in resc] == list(g["top_ids"])
    assert [r[1] for r in resc] == list(g["top_scores"])


def test_varlen_bitwise():
    g = golden("varlen")
    s, a = orc.fused_score_varlen(g["q"][None], g["tokens"], g["cu"])
    assert np.array_equal(s[0], g["scores"]) and np.array_equal(a, g["argmax"])
    assert int(g["macs"]) == 2 * 7 * int(g["cu"][-1]) * 16


def test_topk_tie_order():
    g = golden("misc")
    ts, ti = orc.topk(np.array([0.0, 1.0, 0.5, 1.0, 1.0]), 2)
    assert list(ti) == list(g["heap_ids"]) == [1, 3]
    ts, ti = orc.topk(g["tie_scores"], 15)
    assert list(ti) == list(g["tie_ids"]) and list(ts) == list(g["tie_top"])
    fr, fw = orc.model_traffic(1, 1000, 1024, 1024, 128, elem_bytes=2)
    assert fr == g["traffic"][0] and fw == g["traffic"][1]
