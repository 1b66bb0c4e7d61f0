"""The reference-suite runner (tests/run_reference_suite.py) installs the
drop-in before the reference's own test modules are collected.  Runs only
where the reference is staged under baseline/_ref (git-ignored)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")),
                                reason="reference suite not staged under baseline/_ref")


def test_collects_reference_suite_with_dropin_installed(tmp_path):
    out = tmp_path / "collect.json"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "run_reference_suite.py"), "--out", str(out),
                        "--", "--collect-only"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "180 tests collected" in r.stdout
    import json

    meta = json.loads(out.read_text())["meta"]
    assert "map_charge" in meta["installed"] and "poisson_ik" in meta["installed"]
    assert meta["pppm_file"].startswith(REF)
