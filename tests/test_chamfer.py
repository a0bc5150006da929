"""Chamfer distance (maxsim/chamfer.py) on the device against the REAL reference's outputs
(tests/golden/chamfer.npz, tests/golden/make_golden.py chamfer): forward distance and argmins
bit-identical (float32 arithmetic in the reference order, lowest index on ties), backward
bit-identical (float64, reference accumulation order through the shared inverse CSR)."""

import numpy as np
import pytest
import torch

import paper_2605_29517_b200 as mx
from conftest import golden

gpu = pytest.mark.gpu


def test_pointset_validation_host():
    with pytest.raises(mx.ShapeMismatch):
        mx.PointSet(np.zeros((0, 3), np.float32))
    with pytest.raises(mx.ShapeMismatch):
        mx.PointSet(np.zeros(3, np.float32))
    with pytest.raises(mx.NaNInput):
        mx.PointSet([[0.0, np.inf, 0.0]])


@gpu
def test_hand_case_and_ties():
    g = golden("chamfer")
    cd, a1, a2 = mx.chamfer_forward(g["h_p"], g["h_s"])
    assert cd == 3.5 == float(g["h_cd"])
    assert a1.cpu().tolist() == [0] and a2.cpu().tolist() == [0, 0]
    cd, a1, a2 = mx.chamfer_forward(g["tp"], g["ts"])
    assert cd == float(g["cdt"])
    assert np.array_equal(a1.cpu().numpy(), g["t1"]) and np.array_equal(a2.cpu().numpy(), g["t2"])
    p = mx.PointSet(g["p"][:40])
    cd, a1, a2 = mx.chamfer_forward(p, p)
    assert cd == 0.0 and np.array_equal(a1.cpu().numpy(), np.arange(40))


@gpu
@pytest.mark.parametrize("suffix", ["", "5"])
def test_forward_backward_bit_exact_with_reference(suffix):
    g = golden("chamfer")
    p, s = g["p" + suffix], g["s" + suffix]
    cd, a1, a2 = mx.chamfer_forward(p, s)
    assert cd == float(g["cd" + suffix])
    n1, n2 = ("a1", "a2") if not suffix else ("b1", "b2")
    assert np.array_equal(a1.cpu().numpy(), g[n1]) and np.array_equal(a2.cpu().numpy(), g[n2])
    up = 1.7 if not suffix else 1.0
    d_p, d_s = mx.chamfer_backward(p, s, a1, a2, upstream=up)
    assert np.array_equal(d_p.cpu().numpy(), g["dp" + suffix]) and np.array_equal(d_s.cpu().numpy(), g["ds" + suffix])
    # the dense reference paths agree (f64 oracle to tolerance, f32 path bit-identical)
    assert mx.dense_chamfer_forward(p, s)[0] == cd
    assert mx.dense_chamfer_forward(p, s, precision="f64")[0] == pytest.approx(cd, rel=1e-5)
    r_p, r_s = mx.dense_chamfer_backward(p, s, a1, a2, upstream=up)
    assert torch.allclose(d_p, r_p, rtol=1e-12, atol=0) and torch.allclose(d_s, r_s, rtol=1e-12, atol=0)


@gpu
def test_errors():
    g = golden("chamfer")
    with pytest.raises(mx.DimMismatch):
        mx.chamfer_forward(g["p"], g["p5"])
    _, a1, a2 = mx.chamfer_forward(g["p"], g["s"])
    with pytest.raises(mx.StaleArgmin):
        mx.chamfer_backward(g["p"], g["s"], a1[:-1], a2)
    bad = a1.clone()
    bad[0] = 10_000
    with pytest.raises(mx.StaleArgmin):
        mx.chamfer_backward(g["p"], g["s"], bad, a2)
    d_p, d_s = mx.chamfer_backward(g["p"], g["s"], a1, a2, upstream=0.0)
    assert not bool(d_p.any()) and not bool(d_s.any())


@gpu
def test_large_cloud_against_f64_oracle():
    rng = np.random.default_rng(31)
    p = rng.standard_normal((20_000, 3)).astype(np.float32)
    s = rng.standard_normal((30_000, 3)).astype(np.float32)
    cd, a1, a2 = mx.chamfer_forward(p, s)
    # f64 nearest neighbours on a subsample of rows
    P, S = torch.from_numpy(p).cuda().double(), torch.from_numpy(s).cuda().double()
    rows = torch.arange(0, 20_000, 97, device="cuda")
    d = ((P[rows, None, :] - S[None, :, :]) ** 2).sum(-1)
    best = d.min(dim=1).values
    got = ((P[rows] - S[a1[rows].long()]) ** 2).sum(-1)
    assert torch.allclose(got, best, rtol=1e-4, atol=1e-6)
    d_p, d_s = mx.chamfer_backward(p, s, a1, a2)
    assert d_p.shape == (20_000, 3) and d_s.shape == (30_000, 3)


def _numpy_nearest(a, b):
    """The reference's float32 arithmetic (maxsim/kernels.py:29-66 dot_block / sq_norms /
    sq_dist_block, fold_extreme strict <) restated with numpy on the whole pair grid."""
    def norms(x):
        out = x[:, 0] * x[:, 0]
        for k in range(1, x.shape[1]):
            out = out + x[:, k] * x[:, k]
        return out

    dot = a[:, 0, None] * b[None, :, 0]
    for k in range(1, a.shape[1]):
        dot = dot + a[:, k, None] * b[None, :, k]
    d = dot * np.float32(-2.0) + norms(a)[:, None] + norms(b)[None, :]
    return d.min(axis=1), d.argmin(axis=1)


def _numpy_chamfer_grad(x, y, nn_xy, nn_yx, c_gather, c_scatter):
    """maxsim/chamfer.py:179-199 for one side, in the reference's float64 order: the gather term
    c_gather * (x[r] - y[nn_xy[r]]) first, then for every source j with nn_yx[j] == r in
    ascending j, += c_scatter * (x[r] - y[j]) (vectorised over destinations per source rank)."""
    x64 = x.astype(np.float64)
    d = 0.0 + c_gather * (x64 - y[nn_xy].astype(np.float64))
    order = np.argsort(nn_yx, kind="stable")
    dest = nn_yx[order]
    starts = np.searchsorted(dest, np.arange(x.shape[0]))
    counts = np.bincount(nn_yx, minlength=x.shape[0])
    for t in range(int(counts.max(initial=0))):
        rows = np.nonzero(counts > t)[0]
        src = order[starts[rows] + t]
        d[rows] += c_scatter * (x64[rows] - y[src].astype(np.float64))
    return d


@gpu
@pytest.mark.parametrize("dim", [3, 17, 40])
def test_any_dimension_bit_exact(dim):
    """Chamfer is dimension-generic in the reference: wide embeddings (dim > 16) take the
    shared-memory-tiled kernel with the same fold, bit-identical distances and argmins."""
    rng = np.random.default_rng(dim)
    p = rng.standard_normal((301, dim)).astype(np.float32)
    s = rng.standard_normal((203, dim)).astype(np.float32)
    s[7] = p[11]  # an exact match and a duplicate (tie -> lowest index)
    s[9] = p[11]
    cd, a1, a2 = mx.chamfer_forward(p, s)
    b1, i1 = _numpy_nearest(p, s)
    b2, i2 = _numpy_nearest(s, p)
    assert np.array_equal(a1.cpu().numpy(), i1) and np.array_equal(a2.cpu().numpy(), i2)
    ref = float(np.add.accumulate(b1, dtype=np.float64)[-1]) / 301 + float(np.add.accumulate(b2, dtype=np.float64)[-1]) / 203
    assert cd == ref
    d_p, d_s = mx.chamfer_backward(p, s, a1, a2)
    r_p = _numpy_chamfer_grad(p, s, i1, i2, 2.0 / 301, 2.0 / 203)
    r_s = _numpy_chamfer_grad(s, p, i2, i1, 2.0 / 203, 2.0 / 301)
    # bit-identical to the reference's destination-owned, ascending-source loops
    # (a dense index_add scatter only agrees to rounding: order-free, and cancellation-prone)
    assert np.array_equal(d_p.cpu().numpy(), r_p) and np.array_equal(d_s.cpu().numpy(), r_s)


@gpu
def test_clouds_beyond_shared_memory_histograms():
    """More than 51,200 points per cloud: the backward's inverse CSR takes the
    radix-sort path and stays equal to the dense float64 scatter."""
    rng = np.random.default_rng(77)
    p = rng.standard_normal((60_000, 3)).astype(np.float32)
    s = rng.standard_normal((55_000, 3)).astype(np.float32)
    cd, a1, a2 = mx.chamfer_forward(p, s)
    d_p, d_s = mx.chamfer_backward(p, s, a1, a2, upstream=1.3)
    r_p, r_s = mx.dense_chamfer_backward(p, s, a1, a2, upstream=1.3)
    assert torch.allclose(d_p, r_p, rtol=1e-12, atol=1e-300) and torch.allclose(d_s, r_s, rtol=1e-12, atol=1e-300)
