"""The per-pair f64 score folded into the forward epilogues (no [N_q, B, L_q] row maxima in HBM)
and the input validation of the tensor-level APIs / C-ABI.

Fused S4 (score warp + cluster DSMEM, fwd_ts / fwd_i8r; segmented warp sum, varlen) must give
the SAME score bits as the separate rowsum pass over the materialised row maxima, which is the
reference's sequential f64 sum whenever the exactness certificate holds (score_sum.cuh) --
checked here against the oracle's own seq_sum_f64 of the kernel's row maxima.
"""

import ctypes

import numpy as np
import pytest
import torch

import paper_2605_29517_b200 as mx
from paper_2605_29517_b200 import _dev, _lib
from paper_2605_29517_b200.errors import EmptyDocument, ShapeMismatch
from paper_2605_29517_b200.quant import quantize_tensor

pytestmark = pytest.mark.gpu


def seq_sum_f64(rowmax):
    """maxsim/kernels.py:22-26: strict left-to-right float64 sum over the last axis."""
    r = rowmax.astype(np.float64)
    out = r[..., 0].copy()
    for i in range(1, r.shape[-1]):
        out = out + r[..., i]
    return out


def unit(g, shape, dtype=torch.bfloat16):
    x = torch.randn(*shape, device="cuda", generator=g)
    return (x / x.norm(dim=-1, keepdim=True)).to(dtype)


@pytest.mark.parametrize(
    "n_q,l_q,n_docs,l_pad,dim,want_argmax",
    [
        (1, 1024, 300, 1024, 128, False),  # C2 shape: 2-CTA cluster, fused (rerank)
        (1, 1024, 300, 1024, 128, True),   # C2 shape, argmax mode: fused with the stash
        (2, 2048, 40, 512, 128, False),    # 4-CTA cluster
        (3, 300, 200, 260, 128, True),     # one CTA per query (CL = 1), ragged
        (2, 1536, 30, 300, 128, False),    # three row groups: not fusable -> rowmax + rowsum pass
        (4, 32, 500, 180, 128, True),      # ColBERT shape
        (2, 200, 40, 333, 64, False),      # fp16 below
    ],
)
def test_fused_dense_equals_rowsum_pass(n_q, l_q, n_docs, l_pad, dim, want_argmax):
    g = torch.Generator(device="cuda").manual_seed(n_q * 7 + l_q)
    dt = torch.float16 if dim == 64 else torch.bfloat16
    Q = unit(g, (n_q, l_q, dim), dt)
    D = unit(g, (n_docs, l_pad, dim), dt)
    vl = torch.randint(1, l_pad + 1, (n_docs,), device="cuda", generator=g, dtype=torch.int32)
    vl[0] = l_pad
    s_f, a_f, r_f = mx.score_dense(Q, D, vl, want_argmax=want_argmax)
    assert r_f is None
    s_r, a_r, rm = mx.score_dense(Q, D, vl, want_argmax=want_argmax, want_rowmax=True)
    assert torch.equal(s_f, s_r)
    if want_argmax:
        assert torch.equal(a_f, a_r)
    assert np.array_equal(s_r.cpu().numpy(), seq_sum_f64(rm.cpu().numpy()))


@pytest.mark.parametrize("l_q,n_docs,l_pad", [(1024, 200, 1024), (130, 300, 256), (512, 64, 200)])
def test_fused_int8_equals_rowsum_pass(l_q, n_docs, l_pad):
    g = torch.Generator(device="cuda").manual_seed(l_q + n_docs)
    Q = unit(g, (1, l_q, 128), torch.float32)
    D = unit(g, (n_docs, l_pad, 128), torch.float32)
    qq, qs = quantize_tensor(Q)
    dq, ds = quantize_tensor(D)
    vl = torch.randint(1, l_pad + 1, (n_docs,), device="cuda", generator=g, dtype=torch.int32)
    for want_argmax in (False, True):
        s_f, a_f, _ = mx.score_int8(qq, qs, dq, ds, vl, want_argmax=want_argmax)
        s_r, a_r, rm = mx.score_int8(qq, qs, dq, ds, vl, want_argmax=want_argmax, want_rowmax=True)
        assert torch.equal(s_f, s_r)
        assert np.array_equal(s_r.cpu().numpy(), seq_sum_f64(rm.cpu().numpy()))


def test_fused_sum_certificate_fallback_is_sequential():
    """Row maxima spanning > 2^19 in magnitude fail the exactness certificate: the fused sum must
    then take the sequential chain and still equal the reference's seq_sum_f64 bit for bit."""
    g = torch.Generator(device="cuda").manual_seed(3)
    Q = unit(g, (1, 1024, 128), torch.float32)
    Q[0, ::7] *= 1e-7  # tiny rows -> tiny maxima next to O(1) ones
    D = unit(g, (64, 1024, 128), torch.float32)
    Qb, Db = Q.bfloat16(), D.bfloat16()
    s_f, _, _ = mx.score_dense(Qb, Db, want_argmax=False)
    _, _, rm = mx.score_dense(Qb, Db, want_argmax=False, want_rowmax=True)
    assert np.array_equal(s_f.cpu().numpy(), seq_sum_f64(rm.cpu().numpy()))


@pytest.mark.parametrize("l_q,n_q", [(32, 1), (16, 4), (8, 3), (1, 5), (32, 6)])
def test_fused_varlen_equals_rowsum_pass(l_q, n_q):
    rng = np.random.default_rng(l_q * 10 + n_q)
    lens = rng.integers(1, 400, 700)
    cu = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)])).cuda()
    g = torch.Generator(device="cuda").manual_seed(11)
    toks = unit(g, (int(lens.sum()), 128))
    Q = unit(g, (n_q, l_q, 128))
    s_f, a_f, r_f = mx.score_varlen(Q, toks, cu)
    assert r_f is None
    s_r, a_r, rm = mx.score_varlen(Q, toks, cu, want_rowmax=True)
    assert torch.equal(a_f, a_r)
    assert torch.equal(s_f, s_r)
    assert np.array_equal(s_r.cpu().numpy(), seq_sum_f64(rm.cpu().numpy()))


def test_fused_forward_launch_count():
    """One kernel per C2-shape forward (the CTA-pair kernel; no rowsum launch) when the sum is fused."""
    g = torch.Generator(device="cuda").manual_seed(1)
    Q = unit(g, (1, 1024, 128))
    D = unit(g, (64, 1024, 128))
    mx.score_dense(Q, D, want_argmax=False, validate=False)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        mx.score_dense(Q, D, want_argmax=False, validate=False)
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    kern = [n for n in names if "kernel" in n]
    assert len(kern) == 1 and "fwd_pair_kernel" in kern[0], kern


# ------------------------------------------------------------------ validation (maxsim/forward.py:173-176)
def test_dense_valid_lens_validation():
    Q = torch.zeros(1, 4, 16, device="cuda", dtype=torch.bfloat16)
    D = torch.zeros(3, 8, 16, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(EmptyDocument) as e:
        mx.score_dense(Q, D, torch.tensor([3, 0, 2], device="cuda", dtype=torch.int32))
    assert e.value.index == 1
    with pytest.raises(ShapeMismatch, match="exceeds document rows 8"):
        mx.score_dense(Q, D, torch.tensor([3, 9, 2], device="cuda", dtype=torch.int32))
    with pytest.raises(ShapeMismatch):
        mx.score_dense(Q, D, torch.tensor([3, 2], device="cuda", dtype=torch.int32))
    with pytest.raises(EmptyDocument):
        mx.maxsim(Q.float().requires_grad_(), D.float(), torch.tensor([1, -2, 1], device="cuda"))
    # validated lengths pass
    s, _, _ = mx.score_dense(Q, D, torch.tensor([8, 1, 5], device="cuda", dtype=torch.int32))
    assert s.shape == (1, 3)


def test_int8_valid_lens_validation():
    qq = torch.zeros(1, 4, 16, device="cuda", dtype=torch.int8)
    qs = torch.ones(1, 4, device="cuda")
    dq = torch.zeros(2, 8, 16, device="cuda", dtype=torch.int8)
    ds = torch.ones(2, 8, device="cuda")
    with pytest.raises(EmptyDocument):
        mx.score_int8(qq, qs, dq, ds, torch.tensor([0, 2], device="cuda"))
    with pytest.raises(ShapeMismatch):
        mx.score_int8(qq, qs, dq, ds, torch.tensor([1, 12], device="cuda"))


def test_varlen_cu_seqlens_validation():
    Q = torch.zeros(1, 4, 16, device="cuda", dtype=torch.bfloat16)
    T = torch.zeros(10, 16, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(EmptyDocument) as e:
        mx.score_varlen(Q, T, torch.tensor([0, 4, 4, 10], device="cuda"))
    assert e.value.index == 1
    with pytest.raises(EmptyDocument):
        mx.score_varlen(Q, T, torch.tensor([0, 6, 3, 10], device="cuda"))
    with pytest.raises(ShapeMismatch, match="cu\\[0\\] = 0"):
        mx.score_varlen(Q, T, torch.tensor([1, 4, 10], device="cuda"))
    with pytest.raises(ShapeMismatch, match="does not match token count 10"):
        mx.score_varlen(Q, T, torch.tensor([0, 4, 9], device="cuda"))
    with pytest.raises(EmptyDocument):
        mx.maxsim_varlen(Q, T, torch.tensor([0, 0, 10], device="cuda"))


def test_cabi_validate_entry_points():
    lib = _lib.load()
    bi, bv = ctypes.c_int64(), ctypes.c_int64()
    vl = torch.tensor([5, 7, 0, 3, -1], device="cuda", dtype=torch.int32)
    st = lib.mxs_validate_lens(_dev.ptr(vl), 5, 8, ctypes.byref(bi), ctypes.byref(bv), _dev.stream_handle())
    assert st == 3 and bi.value == 2 and bv.value == 0
    vl = torch.tensor([5, 9, 1], device="cuda", dtype=torch.int32)
    st = lib.mxs_validate_lens(_dev.ptr(vl), 3, 8, ctypes.byref(bi), ctypes.byref(bv), _dev.stream_handle())
    assert st == 2 and bi.value == 1 and bv.value == 9
    big = torch.randint(1, 1025, (1_000_003,), device="cuda", dtype=torch.int32)
    assert lib.mxs_validate_lens(_dev.ptr(big), big.numel(), 1024, None, None, _dev.stream_handle()) == 0
    big[777_777] = 1025
    st = lib.mxs_validate_lens(_dev.ptr(big), big.numel(), 1024, ctypes.byref(bi), None, _dev.stream_handle())
    assert st == 2 and bi.value == 777_777
    cu = torch.tensor([0, 3, 3, 8], device="cuda", dtype=torch.int64)
    st = lib.mxs_validate_cu_seqlens(_dev.ptr(cu), 3, 8, ctypes.byref(bi), None, _dev.stream_handle())
    assert st == 3 and bi.value == 1
