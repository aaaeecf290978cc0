#!/usr/bin/env python3
"""Run the reference's OWN test suites against the B200 kernels.

    python scripts/run_reference_suite.py [--out profiles/r02/reference_suite.json] [pytest args...]

The unmodified reference (tomokit + tomokit_layers, installed into
baseline/_ref by scripts/install_reference.sh together with a copy of its
tests) is imported, and its kernel layer is rebound to libtkb200.so with
`paper_2511_08427_b200.tomokit_kernels.install` -- the six `_kernels`
entry points (_kernels.py:160-322) and `filters.fft_filter`
(filters.py:136-151).  Every reference code path above that layer
(projectors, filters, autodiff, tomokit_layers.ops, torch_layer) then runs on
the GPU unchanged, and pytest runs:

  pkg/tests/test_projectors.py, test_filters.py, test_autodiff.py,
  test_acceptance.py, test_geometry.py, test_grids.py, test_phantoms.py,
  test_artifacts.py; pkg/bindings/tests/test_boundary.py,
  test_torch_layer.py, test_acceptance.py

(test_cli.py is skipped: it runs the CLI in a subprocess, i.e. on the
reference's own numba kernels, so it says nothing about this library.)

Expected differences: the reference computes in float64 and some of its tests
compare to analytic values or across code paths at float64 tolerances
(1e-9..1e-12); the library computes in float32 (the north star's rel-L2 1e-4
contract).  Every outcome is written to the JSON report with the failure
message, so each failure can be classified.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"


class Recorder:
    def __init__(self):
        self.results = {}
        self.bound = []

    def pytest_configure(self, config):
        import tomokit

        from paper_2511_08427_b200 import tomokit_kernels

        self.bound = [f"{m.__name__}.{a}" for m, a, _ in tomokit_kernels.install(tomokit)]

    def pytest_runtest_logreport(self, report):
        if report.when == "call" or (report.when == "setup" and report.outcome != "passed"):
            msg = ""
            if report.outcome == "failed":
                msg = str(report.longrepr).strip().splitlines()[-1][:400] if report.longrepr else ""
            elif report.outcome == "skipped" and report.longrepr:
                msg = str(report.longrepr[-1])[:200] if isinstance(report.longrepr, tuple) else ""
            self.results[report.nodeid] = {"outcome": report.outcome, "message": msg,
                                           "seconds": round(report.duration, 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "reference_suite.json"))
    args, extra = ap.parse_known_args()
    if not (REF / "tomokit").is_dir() or not (REF / "ref_tests").is_dir():
        raise SystemExit("baseline/_ref missing: run scripts/install_reference.sh first")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tk_numba_cache")
    sys.path.insert(0, str(REF))
    sys.path.insert(0, str(ROOT))
    import pytest

    tests = REF / "ref_tests"
    # importlib mode does not put test directories on sys.path; the suites import siblings
    # (test_acceptance.py: `from test_geometry import ...`)
    sys.path.insert(0, str(tests / "pkg_tests"))
    sys.path.insert(0, str(tests / "bindings_tests"))
    files = [tests / "pkg_tests" / f for f in ("test_projectors.py", "test_filters.py", "test_autodiff.py",
                                                "test_acceptance.py", "test_geometry.py", "test_grids.py",
                                                "test_phantoms.py", "test_artifacts.py")]
    files += [tests / "bindings_tests" / f for f in ("test_boundary.py", "test_torch_layer.py",
                                                     "test_acceptance.py")]
    rec = Recorder()
    t0 = time.time()
    # importlib mode: the two suites each have a test_acceptance.py (basename clash under rootdir-relative imports)
    rc = pytest.main(["-q", "-p", "no:cacheprovider", "--import-mode=importlib", "--rootdir", str(tests),
                      *map(str, files), *extra],
                     plugins=[rec])
    counts = {}
    for r in rec.results.values():
        counts[r["outcome"]] = counts.get(r["outcome"], 0) + 1
    report = {"kernel_layer_bound_to": "paper_2511_08427_b200/libtkb200.so (tomokit_kernels.install)",
              "rebound": rec.bound, "pytest_rc": int(rc), "counts": counts,
              "seconds": round(time.time() - t0, 1),
              "failed": {k: v for k, v in rec.results.items() if v["outcome"] == "failed"},
              "results": rec.results}
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(report, indent=1))
    print(json.dumps({"counts": counts, "rebound": len(rec.bound), "out": args.out}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
