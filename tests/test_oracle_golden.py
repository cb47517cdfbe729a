"""Pin the oracle before trusting it: the NumPy and C restatements in oracle/ must
reproduce every golden vector the reference package produced (tests/golden/)."""

import sys
from pathlib import Path

import numpy as np
import pytest

import oracle_c
from golden_inputs import c1_cells, edge_cases, random_case, sha, stream_case
from oracle import fs_oracle as O

REPO = Path(__file__).resolve().parent.parent


def _check_record(rec, cells, ids, taus, *, use_c=False):
    assert [sha(c) for c in cells] == rec["input_sha"], "input generator drifted"
    h, w = cells[0].shape
    k = len(cells)
    counts = O.accumulate(cells, w, h)
    assert sha(counts) == rec["counts_sha"]
    assert O.grid_digest(w, h, k, counts) == rec["digest"]
    assert O.overlap_counts(counts.reshape(-1), k).tolist() == rec["bins"]
    assert sha(O.composite(counts, k)) == rec["composite_sha"]
    g = O.gram(cells)
    assert sha(g) == rec["gram_sha"]
    if rec["gram"] is not None:
        assert g.tolist() == rec["gram"]
    sim = O.similarity_from_gram(g)
    assert sha(sim) == rec["sim_sha"]
    for t in taus:
        assert O.cluster(sim, ids, t) == rec["clusters"][repr(t)]
    if k >= 2:
        scores = O.outlier_scores(sim, ids)
        assert {s: float(v).hex() for s, v in scores.items()} == rec["outliers"]
    if use_c:
        cc = oracle_c.accumulate(cells)
        assert sha(cc.reshape(h, w)) == rec["counts_sha"]
        assert oracle_c.histogram(cc, k).tolist() == rec["bins"]
        assert sha(oracle_c.composite(cc, k).reshape(h, w, 4)) == rec["composite_sha"]
        assert sha(oracle_c.gram(cells)) == rec["gram_sha"]


def test_c1_golden(golden):
    cells = c1_cells()
    rec = golden["c1"]
    _check_record(rec, cells, rec["ids"], [0.8, 0.3], use_c=True)
    flat = [c.reshape(-1) for c in cells]
    assert list(O.pair_counts(flat[0], flat[1])) == rec["pair01"] == [261767, 786289]
    assert list(oracle_c.pair_counts(flat[0], flat[1])) == rec["pair01"]


def test_c1_matches_survey_appendix(golden):
    """The survey's independently recorded goldens."""
    rec = golden["c1"]
    assert rec["counts_sha"] == "77d021e6d517dd04f97e80d1c72f066da12d8a415d8d9fc49c5980ac2529c4a8"
    assert rec["digest"] == "2b5fb38ce5f3760af1b2e0b3ac04a8c38fa20cb1b19440eeb7b9f84459f4952d"
    assert rec["composite_sha"] == "3d7336d4bd6c0e695d347eb074b44af7f0f5f1f215b6fa801cd45e9d1792cd31"
    assert rec["gram_sha"] == "0cc185412df021f9afe9a11c6b81c5ff2cda9e2543166ce7c4b4150d8a992901"
    assert rec["sim_sha"] == "0ec539d5dd36d26f6ce957f4c365252ec48b95f60a661044dce6600b31f7a8a0"
    assert float.fromhex(rec["outliers"]["s00"]) == 0.666704126486352


@pytest.mark.parametrize("case", range(40))
def test_random_golden(golden, case):
    rec = golden["random"][case]
    cells, ids, tau = random_case(case)
    assert rec["tau"] == tau
    _check_record(rec, cells, ids, [tau], use_c=(case % 4 == 0))


@pytest.mark.parametrize("name", sorted(edge_cases()))
def test_edge_golden(golden, name):
    cells, ids, taus = edge_cases()[name]
    _check_record(golden["edge"][name], cells, ids, taus, use_c=True)


@pytest.mark.parametrize("case", range(6))
def test_stream_golden(golden, case):
    rec = golden["stream"][case]
    cells, n = stream_case(case)
    h, w = cells[0].shape
    counts = O.run_stream_counts(cells, n, w, h)
    assert O.grid_digest(w, h, n, counts) == rec["digest"]
    assert O.overlap_counts(counts.reshape(-1), n).tolist() == rec["bins"]
    assert sha(O.composite(counts, n)) == rec["composite_sha"]


def test_schedule_golden(golden):
    for variant, rec in golden["schedule"].items():
        deps = O.build_schedule_deps(variant, 5)
        assert [n[0] for n in rec["nodes"]] == list(deps)
        for node_id, _, d in rec["nodes"]:
            assert tuple(d) == deps[node_id]


def test_reference_cython_accelerator_agrees(golden):
    """oracle/_ref = the reference's own _accel.pyx compiled from its sources."""
    ref_dir = REPO / "oracle" / "_ref"
    if not any(ref_dir.glob("_accel*.so")):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    sys.path.insert(0, str(ref_dir))
    import _accel

    cells = c1_cells()
    counts = np.zeros(1 << 20, dtype=np.uint32)
    for c in cells:
        _accel.accumulate_into(counts, c.reshape(-1))
    assert sha(counts.reshape(1024, 1024)) == golden["c1"]["counts_sha"]
    assert list(_accel.overlap_counts(counts, 16)) == golden["c1"]["bins"]


def test_cluster_unique_ids_matches_cluster():
    """The linkage-matrix form of the oracle clusterer (used at n = 1024) gives the same
    lists as the literal restatement of fs/analytics.py:184-226, ties included."""
    rng = np.random.default_rng(0)
    for t in range(200):
        n = int(rng.integers(1, 25))
        x = rng.random((n, n))
        if t % 3 == 0:
            x = np.round(x * 4) / 4  # many exact ties
        s = np.minimum(x, x.T)
        np.fill_diagonal(s, 1.0)
        ids = [f"s{i:03d}" for i in rng.permutation(n)]
        tau = float(rng.choice([0.1, 0.25, 0.5, 0.75, 0.8, 1.0]))
        assert O.cluster(s, ids, tau) == O.cluster_unique_ids(s, ids, tau), t


def test_blocked_c_gram_matches_pair_loop():
    """oracle/fs_oracle.c's blocked Gram (full-size configs) equals the pair loop."""
    import oracle_c

    rng = np.random.default_rng(1)
    for k, n in [(1, 5), (3, 100), (17, 1000), (40, 70001), (130, 3000)]:
        cells = [(rng.random(n) < rng.random()).astype(np.uint8) *
                 rng.integers(0, 3, n).astype(np.uint8) for _ in range(k)]
        assert np.array_equal(oracle_c.gram(cells), O.gram(cells)), (k, n)
