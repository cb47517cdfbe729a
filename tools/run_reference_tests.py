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

With ``--bind-streaming`` ``floodstream.streaming`` is bound as well (its run_stream /
simulate_stream_timing measure the real upload DAG on the device instead of pricing the
reference's cost model).  The reference tests that assert cost-model VALUES (totals,
budgets and limits derived from a DeviceProfile's prices) cannot hold for measured
timings; they are listed in COST_MODEL_ASSERTIONS and reported apart.

Usage: python tools/run_reference_tests.py [--boundary-only | --bind-streaming] [pytest args ...]
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
REF = REPO / "baseline" / "_ref"


# test ids (in the reference's tests/test_streaming.py) whose assertions are values of
# the reference's cost model: simulated totals of profile-priced items, the closed form
# equal to the simulation, the simulator's 16k image limit, frame budgets from profile
# prices.  Measured timings cannot reproduce them; everything else must pass.
COST_MODEL_ASSERTIONS = (
    "test_streaming.py::TestHandComputedTotals::test_total",
    "test_streaming.py::test_simulator_matches_closed_forms_exactly",
    "test_streaming.py::test_closed_form_makespan_source_agrees_with_simulation",
    "test_streaming.py::TestStreamJob::test_oversized_images_rejected_at_timing",
    "test_streaming.py::TestFrameBudget::test_steady_state_throughput",
    "test_streaming.py::TestFrameBudget::test_transform_bound_pipeline",
    # the service snapshot embeds run_stream's report: digest, histogram and PNG of the
    # recompute after a restart are identical, its measured microseconds are not
    "test_service.py::TestRestart::test_state_survives_byte_exactly",
)


def is_cost_model_assertion(nodeid: str) -> bool:
    return any(nodeid.split("[")[0].endswith(x) for x in COST_MODEL_ASSERTIONS)


def bind_floodstream(boundary_only: bool = False, streaming: bool = False) -> dict:
    """Make ``import floodstream`` = the reference package with our hot-path modules.
    ``boundary_only``: bind just the backend registry (fs/backends.py:21-47), so the
    reference's OWN analytics.py drives our C-ABI protocol module primitive by primitive
    (INTEGRATION.md §B)."""
    sys.path.insert(0, str(REPO))
    import paper_2104_14667_b200.analytics as analytics
    import paper_2104_14667_b200.backends as backends
    import paper_2104_14667_b200.rasters as rasters
    import paper_2104_14667_b200.streaming as streaming_mod

    bound = {"backends": backends} if boundary_only else {
        "analytics": analytics, "backends": backends, "rasters": rasters}
    if streaming:
        bound["streaming"] = streaming_mod

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
    streaming = "--bind-streaming" in argv
    argv = [a for a in argv if a not in ("--boundary-only", "--bind-streaming")]
    binding = bind_floodstream(boundary_only, streaming)
    import floodstream

    assert floodstream.backends.__name__ == "paper_2104_14667_b200.backends"
    assert floodstream.analytics.kernels.NAME == "cuda"
    import pytest

    col = Collector()
    paths = [a for a in argv if not a.startswith("-")]
    args = ([] if paths else [str(REF / "ref_tests")]) + [
        "-q", "-p", "no:cacheprovider", "--rootdir", str(REF / "ref_tests")] + argv
    rc = pytest.main(args, plugins=[col])
    print(json.dumps({"binding": binding,
                      "files": col.outcomes,
                      "passed": sum(d.get("passed", 0) for d in col.outcomes.values()),
                      "failed": col.failed,
                      "cost_model_failed": [f for f in col.failed if is_cost_model_assertion(f)]}))
    return int(rc)


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
