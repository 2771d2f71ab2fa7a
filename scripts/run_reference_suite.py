#!/usr/bin/env python
"""Run the reference's own unit tests unchanged against the GPU package.

SURVEY.md section 4: the reference's pkg/tests are the parity suite.  This
script (1) copies the in-scope test modules from /root/reference/pkg/tests
into baseline/_ref/refsuite (untracked; baseline/_ref travels to the GPU box
with the snapshot) when /root/reference is present, and (2) runs them with
the ``dacresample`` name shim (tests/refsuite_shim) on the GPU package,
writing a summary.  Out-of-scope modules (test_bench / test_weightgen /
test_acceptance need bench.py, weightgen.py and cli.py of the reference,
which this package does not re-implement) are listed, not run.

    python scripts/run_reference_suite.py [--out profiles/r2/reference_suite.txt]
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = Path("/root/reference/pkg/tests")
DST = ROOT / "baseline" / "_ref" / "refsuite"
IN_SCOPE = ["helpers.py", "test_cdf.py", "test_randkit.py", "test_samplers.py"]
OUT_OF_SCOPE = {"test_bench.py": "reference bench.py (timing harness)", "test_weightgen.py": "weightgen.py",
                "test_acceptance.py": "bench.py + weightgen.py + cli.py"}
# reference tests that observe the CPU implementation itself, not the contract
XFAIL = {
    "test_samplers.py::TestDacRecursionShape::test_first_search_targets_middle_uniform_over_full_range":
        "monkeypatches samplers.upper_bound_search to record the CPU recursion's calls; "
        "the GPU search never calls the Python bisection",
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r2" / "reference_suite.txt"))
    args = ap.parse_args()
    if SRC.exists():
        DST.mkdir(parents=True, exist_ok=True)
        for f in IN_SCOPE:
            shutil.copy2(SRC / f, DST / f)
    if not all((DST / f).exists() for f in IN_SCOPE):
        print(f"no reference tests at {DST} (run once where /root/reference exists)")
        return 1
    (DST / "conftest.py").write_text(
        "import pytest\n"
        f"XFAIL = {XFAIL!r}\n"
        "def pytest_collection_modifyitems(config, items):\n"
        "    for it in items:\n"
        "        for k, why in XFAIL.items():\n"
        "            if it.nodeid.endswith(k):\n"
        "                it.add_marker(pytest.mark.xfail(reason=why, strict=True))\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(ROOT / "tests" / "refsuite_shim"), str(ROOT)]))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-rfEx", "-p", "no:cacheprovider", str(DST)],
                       cwd=str(DST), env=env, capture_output=True, text=True)
    out = Path(args.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    text = ("reference pkg/tests run unchanged against paper_2604_01356_b200 via tests/refsuite_shim\n"
            f"in scope: {', '.join(IN_SCOPE[1:])}\n"
            "not run (out of scope): " + "; ".join(f"{k} ({v})" for k, v in OUT_OF_SCOPE.items()) + "\n"
            f"expected failures: {XFAIL}\n\n" + r.stdout[-20000:] + r.stderr[-5000:])
    out.write_text(text)
    print(r.stdout[-3000:])
    return r.returncode


if __name__ == "__main__":
    sys.exit(main())
