#!/usr/bin/env python
"""Run the reference's OWN test files, unmodified, against this package (drop-in check).

The reference package is installed (pip --no-deps, offline) into the git-ignored
``baseline/_ref`` together with a copy of its tests (``baseline/_ref/ref_tests``); both
travel to the GPU box with the repo snapshot.  Before the reference package is imported,
``floodstream.analytics``, ``floodstream.backends`` and ``floodstream.rasters`` are bound
to this package's modules — the hot path (fs/analytics.py, fs/backends.py,
fs/rasters.py) — so every reference module and test that uses them (streaming,
service, store, bench, the analytics / property / acceptance suites) now runs on the
B200 kernels; everything off the path (cost model, simulator, calibration, stats, CLI)
stays the reference's own code.  Prints one JSON summary line (per-file outcomes and the
failing test ids) after pytest's own report.

Usage: python tools/run_reference_tests.py [--boundary-only] [pytest args ...]
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
REF = REPO / "baseline" / "_ref"


def bind_floodstream(boundary_only: bool = False) -> dict:
    """Make ``import floodstream`` = the reference package with our hot-path modules.
    ``boundary_only``: bind just the backend registry (fs/backends.py:21-47), so the
    reference's OWN analytics.py drives our C-ABI protocol module primitive by primitive
    (INTEGRATION.md §B)."""
    sys.path.insert(0, str(REPO))
    import paper_2104_14667_b200.analytics as analytics
    import paper_2104_14667_b200.backends as backends
    import paper_2104_14667_b200.rasters as rasters

    bound = {"backends": backends} if boundary_only else {
        "analytics": analytics, "backends": backends, "rasters": rasters}

    import importlib.util

    pkg_dir = REF / "floodstream"
    # a real package spec (importlib.resources reads the bundled profiles through it)
    spec = importlib.util.spec_from_file_location(
        "floodstream", pkg_dir / "__init__.py", submodule_search_locations=[str(pkg_dir)])
    pkg = importlib.util.module_from_spec(spec)
    sys.modules["floodstream"] = pkg
    for name, mod in bound.items():
        sys.modules[f"floodstream.{name}"] = mod
        setattr(pkg, name, mod)
    spec.loader.exec_module(pkg)
    return {f"floodstream.{n}": m.__name__ for n, m in bound.items()}


class Collector:
    def __init__(self):
        self.outcomes: dict[str, dict[str, int]] = {}
        self.failed: list[str] = []

    def pytest_runtest_logreport(self, report):
        if report.when != "call" and not (report.when == "setup" and report.outcome != "passed"):
            return
        f = report.nodeid.split("::")[0].split("/")[-1]
        d = self.outcomes.setdefault(f, {"passed": 0, "failed": 0, "skipped": 0})
        d[report.outcome] = d.get(report.outcome, 0) + 1
        if report.outcome == "failed":
            self.failed.append(report.nodeid)


def main(argv: list[str]) -> int:
    if not (REF / "floodstream").exists() or not (REF / "ref_tests").exists():
        print(json.dumps({"unavailable": "baseline/_ref (reference install + ref_tests) missing"}))
        return 0
    boundary_only = "--boundary-only" in argv
    argv = [a for a in argv if a != "--boundary-only"]
    binding = bind_floodstream(boundary_only)
    import floodstream

    assert floodstream.backends.__name__ == "paper_2104_14667_b200.backends"
    assert floodstream.analytics.kernels.NAME == "cuda"
    import pytest

    col = Collector()
    args = [str(REF / "ref_tests"), "-q", "-p", "no:cacheprovider", "--rootdir",
            str(REF / "ref_tests")] + argv
    rc = pytest.main(args, plugins=[col])
    print(json.dumps({"binding": binding,
                      "files": col.outcomes,
                      "passed": sum(d.get("passed", 0) for d in col.outcomes.values()),
                      "failed": col.failed}))
    return int(rc)


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
