"""Build an A/B variant of libmaxsim_b200.so: one translation unit recompiled with extra -D flags,
linked with the current objects of the others.  Usage:
  python scripts/build_variant.py OUT.so launch_bwd.cu -DMXS_GRAD_GU=4 ...
(probe with MXS_LIB_PATH=OUT.so)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29517_b200 import _build  # noqa: E402

out, tu, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
_build.build()
obj = out + "." + tu + ".o"
cmd = [_build._nvcc()] + _build._base_flags() + defs + ["-c", os.path.join(_build.CSRC, tu), "-o", obj]
subprocess.run(cmd, check=True)
objs = [obj if s == tu else _build._obj(s) for s in _build.SOURCES]
subprocess.run([_build._nvcc(), _build.GENCODE, "-shared", "-Xcompiler", "-fPIC", "-o", out] + objs, check=True)
os.remove(obj)
print(out)
