"""The C-ABI library loads on a GPU-less host and exports every symbol include/maxsim_b200.h declares."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "maxsim_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|int64_t|void|size_t|const char\*)\s+(mxs_\w+)\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_29517_b200 import _build, _lib

    _build.build()
    return _lib.load()


def test_header_declares_the_operator_surface():
    names = declared()
    for must in ("mxs_fused_score_batch", "mxs_fused_score_int8", "mxs_fused_score_varlen", "mxs_quantize_per_token",
                 "mxs_build_inverse_csr", "mxs_grad_docs_csr", "mxs_grad_query", "mxs_topk"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    from paper_2605_29517_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", _lib.lib_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (mxs_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    for n in declared():
        assert hasattr(lib, n)
    assert sorted(_lib.declared_symbols()) == declared()


def test_library_is_sm100a(lib):
    from paper_2605_29517_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_status_strings(lib):
    assert b"sm_100a" in lib.mxs_version()
    assert lib.mxs_status_string(0) == b"ok"
    assert lib.mxs_status_string(3) == b"EmptyDocument"
    assert lib.mxs_status_string(6) == b"KTooLarge"


def test_argument_validation_maps_to_reference_errors(lib):
    from paper_2605_29517_b200 import _lib, errors

    # null pointers are rejected before any CUDA call
    with pytest.raises(errors.ShapeMismatch):
        _lib.call("mxs_fused_score_batch", 2, None, 1, 4, None, 1, 4, 8, None, None, None, None, 0, None)
    with pytest.raises(errors.KTooLarge):
        _lib.call("mxs_topk", ctypes.c_void_p(8), 3, 5, 0, ctypes.c_void_p(8), ctypes.c_void_p(8), None, 0, None)
    msg = lib.mxs_last_error().decode()
    assert "top-5" in msg and "3 documents" in msg


def test_workspace_sizes(lib):
    assert lib.mxs_csr_workspace_bytes(64, 65536) == 0  # histograms live in shared memory / sort scratch
    assert lib.mxs_topk_workspace_bytes(10000, 20) == 0  # one 16384-element selection slice (k <= 128)
    assert lib.mxs_topk_workspace_bytes(20000, 20) == 2 * 20 * 16
    assert lib.mxs_topk_workspace_bytes(10000, 200) == 3 * 200 * 16  # 4096-element bitonic slices
    assert lib.mxs_topk_workspace_bytes(4096, 200) == 0
