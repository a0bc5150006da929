"""The dense brute-force API twin (maxsim/reference.py) on the device: f32 precision matches the
exact fused kernel bit for bit (reference tests/test_reference.py:26-34), f64 is the tolerance
oracle, dense_backward agrees with the fused CSR backward, finite_diff_grad checks dQ."""

import numpy as np
import pytest
import torch

import paper_2605_29517_b200 as mx
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def test_dense_f32_bitwise_equals_exact_fused():
    rng = np.random.default_rng(3)
    qs = [mx.EmbeddingMatrix(torch.from_numpy(rng.standard_normal((7, 16)).astype(np.float32)).cuda())
          for _ in range(3)]
    lens = np.array([9, 1, 13, 5], np.int32)
    docs = mx.DocBatch.from_dense(torch.from_numpy(rng.standard_normal((4, 13, 16)).astype(np.float32)).cuda(),
                                  torch.from_numpy(lens))
    ds, da = mx.dense_score_batch(qs, docs)
    fs, fa, _ = mx.fused_score_batch(qs, docs)
    assert torch.equal(ds.cpu(), torch.as_tensor(np.asarray(fs.numpy())))
    assert np.array_equal(da.numpy(), fa.numpy())
    d64, _ = mx.dense_score_batch(qs, docs, precision="f64")
    assert torch.allclose(d64, ds, rtol=1e-5)
    with pytest.raises(ValueError):
        mx.dense_score(qs[0], docs, precision="f16")


def test_dense_backward_and_finite_differences():
    rng = np.random.default_rng(4)
    Q = rng.standard_normal((2, 5, 8)).astype(np.float32)
    D = rng.standard_normal((3, 6, 8)).astype(np.float32)
    g = rng.standard_normal((2, 3))
    qs = [mx.EmbeddingMatrix(torch.from_numpy(Q[i]).cuda()) for i in range(2)]
    docs = mx.DocBatch.from_dense(torch.from_numpy(D).cuda())
    _, am = mx.dense_score_batch(qs, docs)
    dq, dd = mx.dense_backward(qs, docs, g, am)
    fq, fd = mx.backward_dispatch(am, g, qs, docs)
    assert torch.allclose(dq, fq.double(), rtol=1e-5, atol=1e-6)
    assert torch.allclose(dd, fd.double().reshape(dd.shape), rtol=1e-5, atol=1e-6)

    def f(x):
        s, _ = orc.fused_score_batch(x.astype(np.float32)[None], D)
        return float(s[0] @ g[0])

    fdq = mx.finite_diff_grad(f, Q[0].astype(np.float64), eps=1e-3)
    assert np.allclose(dq[0].cpu().numpy(), fdq, rtol=1e-3, atol=1e-3)
    with pytest.raises(ValueError):
        mx.finite_diff_grad(f, Q[0], eps=0.0)
