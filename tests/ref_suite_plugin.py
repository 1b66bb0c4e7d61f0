"""pytest plugin: run the reference's own test suite against the B200 drop-in.

Loaded with ``-p ref_suite_plugin`` (``tests/run_reference_suite.py``).  At
configure time, before any reference test module is collected (their
``from pppm import ...`` binds names at import), it puts the staged
reference package (``baseline/_ref``, a git-ignored install of
``/root/reference/pkg`` that travels to the GPU box) on ``sys.path``, imports
``pppm`` and calls ``paper_1702_04250_b200.install(pppm)`` so the hot-path
names (map_charge, distribute_force_ik/_ad, build_plan, poisson_ik/_ad,
kspace_energy, build_table) and the driver's pair loop / compute_forces /
integrate_nve resolve to the device operators.  Every test outcome is
recorded and written as JSON at the end of the session.
"""

from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
_results = {}
_meta = {}


def pytest_addoption(parser):
    group = parser.getgroup("b200")
    group.addoption("--b200-precision", default="fp64", help="drop-in precision: fp64 (default) or mixed")
    group.addoption("--b200-ref", default=os.path.join(ROOT, "baseline", "_ref"),
                    help="directory holding the installed reference package `pppm`")
    group.addoption("--b200-report", default=None, help="write per-test outcomes here (JSON)")
    group.addoption("--b200-no-install", action="store_true",
                    help="run the reference unmodified (control run)")


def pytest_load_initial_conftests(early_config, parser, args):
    """Runs before the reference's conftest.py (which imports pppm) is loaded."""
    ns = early_config.known_args_namespace
    ref = getattr(ns, "b200_ref", None) or os.path.join(ROOT, "baseline", "_ref")
    for p in (ROOT, ref):
        if p not in sys.path:
            sys.path.insert(0, p)
    import pppm

    _meta["pppm_file"] = pppm.__file__
    _meta["precision"] = getattr(ns, "b200_precision", None) or "fp64"
    _meta["installed"] = []
    if getattr(ns, "b200_no_install", False):
        return
    import paper_1702_04250_b200 as pb

    pb.set_precision(_meta["precision"])
    names = pb.install(pppm)
    # the rebinding must be visible through every path the tests import from
    import pppm.driver
    import pppm.gridmap
    import pppm.kspace

    assert pppm.map_charge is pb.map_charge and pppm.gridmap.map_charge is pb.map_charge
    assert pppm.driver.poisson_ik is pb.poisson_ik and pppm.kspace.kspace_energy is pb.kspace_energy
    _meta["installed"] = names
    _meta["library"] = pb.library_path()


def pytest_report_header(config):
    return (f"b200 drop-in: precision={_meta.get('precision')} installed={_meta.get('installed')} "
            f"pppm={_meta.get('pppm_file')}")


def pytest_runtest_logreport(report):
    if report.when == "call" or (report.when == "setup" and report.outcome != "passed"):
        entry = {"outcome": report.outcome, "seconds": round(report.duration, 4)}
        if report.outcome == "failed":
            entry["error"] = str(report.longrepr).splitlines()[-1][:400] if report.longrepr else ""
        _results[report.nodeid] = entry


def pytest_sessionfinish(session, exitstatus):
    path = session.config.getoption("--b200-report")
    if not path:
        return
    counts = {}
    for r in _results.values():
        counts[r["outcome"]] = counts.get(r["outcome"], 0) + 1
    out = {"meta": dict(_meta, exitstatus=int(exitstatus), when=time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())),
           "counts": counts, "tests": _results}
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
