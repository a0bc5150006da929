"""Build libmaxsim_b200.so (all sm_100a kernels + the C-ABI) in-tree with nvcc.

The shared library lands next to this file in `lib/` so it travels with the repository
snapshot to the GPU box; nothing is installed into site-packages.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG_DIR, "csrc")
LIB_DIR = os.path.join(PKG_DIR, "lib")
LIB_PATH = os.path.join(LIB_DIR, "libmaxsim_b200.so")
ROOT = os.path.dirname(PKG_DIR)

# Translation units (compiled in parallel, then linked); each includes the kernel headers it
# instantiates, and every kernel header is included by exactly one of them.
SOURCES = ["host.cu", "capi.cu", "launch_ts_bf16.cu", "launch_ts_f16.cu", "launch_ts_i8.cu", "launch_ss.cu",
           "launch_r3.cu", "launch_pair.cu", "launch_varlen.cu", "launch_exact.cu", "launch_bwd.cu", "launch_misc.cu"]
OBJ_DIR = os.path.join(LIB_DIR, "obj")
GENCODE = "-gencode=arch=compute_100a,code=sm_100a"


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libmaxsim_b200.so")
    return cand


def _inputs():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h"))]
    files.append(os.path.join(ROOT, "include", "maxsim_b200.h"))
    return files


def up_to_date() -> bool:
    if not os.path.exists(LIB_PATH):
        return False
    t = os.path.getmtime(LIB_PATH)
    return all(os.path.getmtime(f) <= t for f in _inputs())


def _obj(src: str) -> str:
    return os.path.join(OBJ_DIR, os.path.splitext(src)[0] + ".o")


def _deps(src: str):
    """Dependencies of one TU from nvcc's -MD file (falls back to every source when absent)."""
    dfile = _obj(src)[:-2] + ".d"
    if not os.path.exists(dfile):
        return None
    text = open(dfile).read().replace("\\\n", " ")
    _, _, rhs = text.partition(":")
    return [d for d in rhs.split() if d]


def _stale(src: str) -> bool:
    obj = _obj(src)
    if not os.path.exists(obj):
        return True
    deps = _deps(src)
    if deps is None:
        deps = _inputs()
    t = os.path.getmtime(obj)
    return any((not os.path.exists(d)) or os.path.getmtime(d) > t for d in deps)


def _base_flags():
    return [GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include")]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB_PATH
    os.makedirs(OBJ_DIR, exist_ok=True)
    nvcc = _nvcc()
    todo = [s for s in SOURCES if force or _stale(s)]
    procs = []
    for src in todo:
        obj = _obj(src)
        cmd = [nvcc] + _base_flags() + ["-MD", "-MF", obj[:-2] + ".d", "-c", os.path.join(CSRC, src), "-o", obj + ".tmp"]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    errs = []
    for src, obj, pr in procs:
        out, err = pr.communicate()
        if pr.returncode != 0:
            errs.append(f"nvcc failed on {src} ({pr.returncode}):\n{out}\n{err}")
        else:
            os.replace(obj + ".tmp", obj)
            if verbose and err:
                print(err, file=sys.stderr)
    if errs:
        raise RuntimeError("\n".join(errs))
    tmp = LIB_PATH + ".tmp"
    cmd = [nvcc, GENCODE, "-shared", "-Xcompiler", "-fPIC", "-Xlinker", "--no-undefined", "-o", tmp] + [_obj(s) for s in SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
