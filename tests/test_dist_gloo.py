"""World-size-2 gloo runs of the multi-GPU plumbing (corpus sharding, top-K merge, in-batch
training collectives) on CPU, with the oracle standing in for the device kernels."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def cpu_select(scores, ids, k):
    """CPU twin of topk.select_candidates (the reference order: score desc, id asc), for gloo."""
    s = scores.reshape(-1).to(torch.float64)
    i = ids.reshape(-1).to(torch.int64)
    keep = i >= 0
    s, i = s[keep], i[keep]
    order = sorted(range(s.numel()), key=lambda j: (-float(s[j]), int(i[j])))[:k]
    return s[order], i[order]


class OracleKernels:
    """CPU twin of parallel.DeviceKernels (f64 oracle arithmetic), for the collective logic only."""

    @staticmethod
    def score(Q, D, valid_lens):
        s, a = orc.fused_score_batch(Q.numpy(), D.numpy(), None if valid_lens is None else valid_lens.numpy())
        return torch.from_numpy(s), torch.from_numpy(a)

    @staticmethod
    def grad_docs(Q, argmax, g, l_pad):
        b = argmax.shape[1]
        rp, ci = orc.build_inverse_csr(argmax.numpy(), [l_pad] * b, l_pad)
        return torch.from_numpy(orc.grad_docs_csr(rp, ci, g.double().numpy(), Q.numpy(), n_docs=b))

    @staticmethod
    def grad_query(D, argmax, g):
        b, l, d = D.shape
        return torch.from_numpy(orc.grad_query(argmax.numpy(), g.double().numpy(), D.numpy().reshape(b * l, d),
                                               np.arange(b) * l))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_29517_b200.parallel import inbatch_step, shard_bounds
        from paper_2605_29517_b200.topk import merge_topk_across_ranks

        # ---- sharded rerank: per-rank top-K + all_gather merge == global ranking
        rng = np.random.default_rng(5)
        scores = np.round(rng.standard_normal(103), 1)  # many exact ties
        lo, hi = shard_bounds(103, world, rank)
        ls, li = cpu_select(torch.tensor(scores[lo:hi]), torch.arange(lo, hi), 7)
        ts, ti = merge_topk_across_ranks(ls, li, 7, select=cpu_select)
        os_, oi = orc.topk(scores, 7)
        ok_topk = ti.tolist() == oi.tolist() and ts.tolist() == os_.tolist()

        # ---- in-batch training step with B sharded (C3 decomposition)
        Q = torch.from_numpy(orc.make_queries(4, 5, 8, seed=1))
        D = torch.from_numpy(orc.make_queries(4, 6, 8, seed=2))
        lo, hi = shard_bounds(4, world, rank)
        loss, sc, dQ, dD = inbatch_step(Q, D[lo:hi].contiguous(), lo, kernels=OracleKernels)
        s_ref, a_ref = orc.fused_score_batch(Q.numpy(), D.numpy())
        l_ref, g_ref = orc.softmax_ce(s_ref)
        dq_ref = orc.grad_query(a_ref, g_ref, D.numpy().reshape(24, 8), np.arange(4) * 6)
        rp, ci = orc.build_inverse_csr(a_ref, [6] * 4, 6)
        dd_ref = orc.grad_docs_csr(rp, ci, g_ref, Q.numpy(), n_docs=4).reshape(4, 6, 8)
        ok_train = (
            np.array_equal(sc.numpy(), s_ref)
            and abs(float(loss) - l_ref) < 1e-12
            and np.allclose(dQ.numpy(), dq_ref, rtol=1e-5, atol=1e-6)
            and np.allclose(dD.numpy(), dd_ref[lo:hi], rtol=1e-5, atol=1e-6)
        )
        # ---- C5 decomposition: token-balanced contiguous document shards of a packed corpus,
        #      per-rank varlen scoring + top-K, all_gather merge == global oracle ranking
        rng = np.random.default_rng(9)
        lens = rng.integers(1, 40, 61)
        cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        toks = orc.unit_tokens(rng, int(cu[-1]), 8).astype(np.float32)
        qv = orc.unit_tokens(rng, 4, 8).astype(np.float32)
        lo, hi = shard_bounds(61, world, rank, weights=lens)
        loc_cu = cu[lo:hi + 1] - cu[lo]
        loc_s, _ = orc.fused_score_varlen(qv[None], toks[cu[lo]:cu[hi]], loc_cu)
        ls, li = cpu_select(torch.from_numpy(loc_s[0]), torch.arange(lo, hi), 9)
        ts, ti = merge_topk_across_ranks(ls, li, 9, select=cpu_select)
        g_s, _ = orc.fused_score_varlen(qv[None], toks, cu)
        os_, oi = orc.topk(g_s[0], 9)
        tok_share = (cu[hi] - cu[lo]) / cu[-1]
        ok_varlen = ti.tolist() == oi.tolist() and ts.tolist() == os_.tolist() and abs(tok_share - 0.5) < 0.2
        q.put((rank, ok_topk, ok_train and ok_varlen))
    finally:
        dist.destroy_process_group()


def test_world_size_2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] for r in res), res
    assert all(r[2] for r in res), res
