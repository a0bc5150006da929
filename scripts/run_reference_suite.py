"""Run the reference's OWN test modules against the GPU kernels.

The unmodified reference package (`baseline/_ref/maxsim`) is imported, its hot-path entry points
are rebound to this package's sm_100a kernels with `paper_2605_29517_b200.dropin.install`, and the
reference's test files (copied at build time to `baseline/_ref_tests`, git-ignored, from
/root/reference/pkg/tests) run unmodified under pytest.  Writes a JSON summary (per module: passed /
failed / errors, each failure's first assertion line) to argv[1] (default
gpurun_out/reference_suite.json).
"""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.environ.get("REF_TESTS", os.path.join(ROOT, "baseline", "_ref_tests"))
MODULES = ["test_forward.py", "test_backward.py", "test_quant.py", "test_varlen.py", "test_chamfer.py",
           "test_types.py", "test_reference.py", "test_instrument.py", "test_streamio.py", "test_acceptance.py",
           "test_cli.py"]


class DropIn:
    """pytest plugin: rebinds the reference before any test module imports from it."""

    def __init__(self):
        self.results = {}

    def pytest_configure(self, config):
        import torch

        assert torch.cuda.is_available(), "the drop-in run needs the GPU"
        import maxsim

        import paper_2605_29517_b200.dropin as dropin

        assert os.path.realpath(maxsim.__file__).startswith(os.path.realpath(REF)), maxsim.__file__
        if os.environ.get("REF_ONLY") != "1":  # REF_ONLY=1: control run of the unpatched reference
            dropin.install(maxsim)

    def pytest_runtest_logreport(self, report):
        if report.when == "call" or report.outcome != "passed":
            mod = report.nodeid.split("::")[0].split("/")[-1]
            r = self.results.setdefault(mod, {"passed": 0, "failed": 0, "skipped": 0, "failures": {}})
            if report.outcome == "passed":
                r["passed"] += 1
            elif report.outcome == "skipped":
                r["skipped"] += 1
            else:
                r["failed"] += 1
                text = str(report.longrepr)
                line = next((ln.strip() for ln in text.splitlines() if ln.startswith("E ")), text.splitlines()[-1])
                r["failures"][report.nodeid.split("::", 1)[1] + f" [{report.when}]"] = line[:300]


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "reference_suite.json")
    sys.path[:0] = [REF, TESTS, ROOT]
    plugin = DropIn()
    mods = [os.path.join(TESTS, m) for m in MODULES if os.path.exists(os.path.join(TESTS, m))]
    if not mods:
        print(f"no reference tests under {TESTS}")
        return 2
    rc = pytest.main(["-q", "-p", "no:cacheprovider", "--rootdir", TESTS, "-o", "addopts=", *mods], plugins=[plugin])
    total = {k: sum(r[k] for r in plugin.results.values()) for k in ("passed", "failed", "skipped")}
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as fh:
        json.dump({"total": total, "modules": plugin.results, "pytest_rc": int(rc)}, fh, indent=1)
    print(json.dumps(total))
    return 0


if __name__ == "__main__":
    sys.exit(main())
