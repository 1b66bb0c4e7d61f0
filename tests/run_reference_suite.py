"""Run the reference's own pytest suite against the B200 drop-in.

    python tests/run_reference_suite.py [--precision fp64|mixed] [--ref DIR] [--out FILE] [-- pytest args]

Stage the reference first (once, in the build container; ``baseline/_ref`` is
git-ignored and travels to the GPU box with the snapshot):

    cp -r /root/reference/pkg /tmp/refpkg
    python -m pip install --no-index --no-build-isolation --no-deps \\
        --target baseline/_ref /tmp/refpkg
    mkdir -p baseline/_ref/tests && cp /root/reference/pkg/tests/*.py baseline/_ref/tests/

The runner collects ``<ref>/tests`` with ``tests/ref_suite_plugin.py`` loaded,
which installs the drop-in into the reference package before collection and
writes every outcome to ``--out`` (JSON).  ``--control`` runs the unmodified
reference (no install) for comparison.
"""

from __future__ import annotations

import argparse
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    extra = []
    if "--" in argv:
        i = argv.index("--")
        argv, extra = argv[:i], argv[i + 1:]
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", default="fp64", choices=("fp64", "mixed"))
    ap.add_argument("--ref", default=os.path.join(ROOT, "baseline", "_ref"))
    ap.add_argument("--out", default=None)
    ap.add_argument("--control", action="store_true", help="run the unmodified reference")
    args = ap.parse_args(argv)
    tests = os.path.join(args.ref, "tests")
    if not os.path.isdir(tests) or not os.path.isdir(os.path.join(args.ref, "pppm")):
        print(f"reference suite not staged under {args.ref} (see this file's docstring)", file=sys.stderr)
        return 2
    if HERE not in sys.path:
        sys.path.insert(0, HERE)
    import pytest

    opts = [tests, "-q", "-p", "ref_suite_plugin", "--rootdir", args.ref, "-p", "no:cacheprovider",
            "--b200-precision", args.precision, "--b200-ref", args.ref]
    if args.out:
        opts += ["--b200-report", args.out]
    if args.control:
        opts += ["--b200-no-install"]
    return pytest.main(opts + extra)


if __name__ == "__main__":
    sys.exit(main())
