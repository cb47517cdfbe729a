"""GPU parity: every CUDA path against the oracle and the reference's golden vectors.

Bit-exact for counts, histograms, RGBA, Gram; float64 results (Jaccard, outliers) must
be identical to the reference's because they are computed from the same exact integers
with the same operation order.  All calls go through the product package / C ABI.
"""

import numpy as np
import pytest

from golden_inputs import c1_cells, edge_cases, random_case, sha, stream_case
from oracle import fs_oracle as O

pytestmark = pytest.mark.gpu

import paper_2104_14667_b200 as fs  # noqa: E402
from paper_2104_14667_b200 import _kernels_cuda as K  # noqa: E402
from paper_2104_14667_b200 import _native as N  # noqa: E402
from paper_2104_14667_b200.ensemble import DeviceEnsemble  # noqa: E402
from paper_2104_14667_b200.rasters import RasterSurface  # noqa: E402
from paper_2104_14667_b200.synth import synth_cells  # noqa: E402


def surfaces_of(cells, ids=None):
    return [RasterSurface(id=(ids[i] if ids else f"s{i:02d}"), name="x", width=c.shape[1],
                          height=c.shape[0], cells=c) for i, c in enumerate(cells)]


def test_backend_is_cuda():
    assert fs.analytics.kernels.NAME == "cuda"
    assert N.device_count() >= 1


# ---- protocol primitives ------------------------------------------------------------

@pytest.mark.parametrize("n", [1, 15, 16, 17, 31, 32, 33, 4095, 4096, 8191, 8192, 8193,
                               100_003, 1 << 20])
def test_primitives_match_oracle(n):
    rng = np.random.default_rng(n)
    a = (rng.integers(0, 4, n)).astype(np.uint8)
    b = (rng.random(n) < 0.3).astype(np.uint8) * 200
    counts = rng.integers(0, 5, n).astype(np.uint32)
    want = counts.copy()
    O.accumulate_into(want, a)
    K.accumulate_into(counts, a)
    assert np.array_equal(counts, want)
    assert np.array_equal(K.overlap_counts(counts, 5), O.overlap_counts(counts, 5))
    assert K.pair_counts(a, b) == O.pair_counts(a, b)
    o1 = np.zeros((n, 4), np.uint8)
    o2 = np.zeros((n, 4), np.uint8)
    K.composite_fill(counts, 5, o1)
    O.composite_fill(counts, 5, o2)
    assert np.array_equal(o1, o2)


@pytest.mark.parametrize("n_inputs", [0, 1, 2, 3, 7, 255, 256, 1000, 4095, 4096, 10_000,
                                      (1 << 20) + 5])
def test_composite_and_histogram_all_classes(n_inputs):
    c = np.arange(min(n_inputs, 300_000) + 1, dtype=np.uint32)
    c = np.concatenate([c, c[::-1], np.full(33, min(n_inputs, c[-1]), np.uint32)])
    o1 = np.zeros((c.size, 4), np.uint8)
    o2 = np.zeros((c.size, 4), np.uint8)
    K.composite_fill(c, n_inputs, o1)
    O.composite_fill(c, n_inputs, o2)
    assert np.array_equal(o1, o2)
    assert np.array_equal(K.overlap_counts(c, n_inputs), O.overlap_counts(c, n_inputs))


def test_protocol_backend_parity_reference_case():
    """test_analytics.py:261-285 inputs (seed 11, 4096 px, p = 0.4) vs the oracle."""
    rng = np.random.default_rng(11)
    cells = (rng.random(4096) < 0.4).astype(np.uint8)
    other = (rng.random(4096) < 0.4).astype(np.uint8)
    got, want = np.zeros(4096, np.uint32), np.zeros(4096, np.uint32)
    for x in (cells, other):
        K.accumulate_into(got, x)
        O.accumulate_into(want, x)
    assert np.array_equal(got, want)
    o1, o2 = np.zeros((4096, 4), np.uint8), np.zeros((4096, 4), np.uint8)
    K.composite_fill(got, 2, o1)
    O.composite_fill(want, 2, o2)
    assert np.array_equal(o1, o2)
    assert K.pair_counts(cells, other) == O.pair_counts(cells, other)
    assert np.array_equal(K.overlap_counts(got, 2), O.overlap_counts(want, 2))


# ---- analytics against golden vectors --------------------------------------------------

def _check_analytics(rec, cells, ids, taus):
    s = surfaces_of(cells, ids)
    grid = fs.accumulate(s)
    assert sha(grid.counts) == rec["counts_sha"]
    assert grid.digest() == rec["digest"]
    assert fs.overlap_histogram(grid).bins == rec["bins"]
    assert sha(fs.composite_map(grid).pixels) == rec["composite_sha"]
    sim = fs.similarity_matrix(s)
    assert sha(sim) == rec["sim_sha"]
    for t in taus:
        assert fs.cluster_surfaces(s, t) == rec["clusters"][repr(t)]
    if len(s) >= 2:
        got = {k: float(v).hex() for k, v in fs.outlier_scores(s).items()}
        assert got == rec["outliers"]


def test_c1_goldens(golden):
    rec = golden["c1"]
    _check_analytics(rec, c1_cells(), rec["ids"], [0.8, 0.3])


@pytest.mark.parametrize("case", range(40))
def test_random_goldens(golden, case):
    cells, ids, tau = random_case(case)
    _check_analytics(golden["random"][case], cells, ids, [tau])


@pytest.mark.parametrize("name", sorted(edge_cases()))
def test_edge_goldens(golden, name):
    cells, ids, taus = edge_cases()[name]
    _check_analytics(golden["edge"][name], cells, ids, taus)


def test_jaccard_pairs_match_reference(golden):
    cells, ids, _ = random_case(1)
    s = surfaces_of(cells, ids)
    g = np.array(golden["random"][1]["gram"])
    for i in range(len(s)):
        for j in range(len(s)):
            inter = int(g[i, j])
            union = int(g[i, i]) + int(g[j, j]) - inter
            assert fs.jaccard(s[i], s[j]) == O.jaccard_from_counts(inter, union)


# ---- streaming ------------------------------------------------------------------------

@pytest.mark.parametrize("case", range(6))
@pytest.mark.parametrize("variant", [v.value for v in fs.Variant])
def test_run_stream_goldens(golden, case, variant):
    rec = golden["stream"][case]
    cells, n = stream_case(case)
    h, w = cells[0].shape
    job = fs.StreamJob(variant=fs.Variant(variant), n=n, width=w, height=h,
                       surfaces=surfaces_of(cells))
    grid, report = fs.run_stream(job)
    assert grid.digest() == rec["digest"]
    assert fs.overlap_histogram(grid).bins == rec["bins"]
    assert sha(fs.composite_map(grid).pixels) == rec["composite_sha"]
    assert report.n == n and len(report.per_item_c) == n
    assert report.total_time_us >= 1 and report.makespan_source == "measured"
    assert all(x >= 0 for x in report.per_item_c + report.per_item_m + report.per_item_p)


@pytest.mark.parametrize("case", range(6))
def test_ensemble_cycled_overlap(golden, case):
    """Fused overlap with cycles/remainder == run_stream's cycled grid (streaming.py:417)."""
    rec = golden["stream"][case]
    cells, n = stream_case(case)
    h, w = cells[0].shape
    k = len(cells)
    with DeviceEnsemble(w, h, k) as ens:
        ens.upload(cells)
        cyc, rem = divmod(n, k)
        c, b, r = ens.overlap(list(range(k)), cycles=cyc, remainder=rem)
    assert O.grid_digest(w, h, n, c) == rec["digest"]
    assert b.tolist() == rec["bins"]
    assert sha(r) == rec["composite_sha"]


# ---- Gram engines ----------------------------------------------------------------------

@pytest.mark.parametrize("engine", ["popc", "tc", "tc-f4"])
@pytest.mark.parametrize("k,h,w", [(1, 3, 5), (2, 1, 1), (16, 64, 64), (31, 17, 129),
                                   (128, 32, 32), (129, 40, 33), (200, 64, 80),
                                   (256, 32, 64), (257, 16, 33), (300, 24, 40)])
def test_gram_engines_exact(engine, k, h, w):
    rng = np.random.default_rng(k * 1000 + h)
    cells = [(rng.random((h, w)) < rng.uniform(0.05, 0.95)).astype(np.uint8) for _ in range(k)]
    if k > 3:
        cells[3] = cells[0].copy()
    want = O.gram(cells)
    with DeviceEnsemble(w, h, k) as ens:
        ens.upload(cells)
        got = ens.gram(list(range(k)), engine=engine)
        # permuted / repeated slot lists
        perm = rng.permutation(k)
        got_p = ens.gram(perm.tolist(), engine=engine)
    assert np.array_equal(got, want)
    assert np.array_equal(got_p, want[np.ix_(perm, perm)])


@pytest.mark.parametrize("engine", ["popc", "tc", "tc-f4"])
def test_gram_large_pixels(engine):
    """Many K stages and K chunks: 24 flood-like masks of 1536 x 1100 px."""
    cells = [synth_cells(1100, 1536, i, members=6, eps=0.05) for i in range(24)]
    want = O.gram(cells)
    with DeviceEnsemble(1100, 1536, 24) as ens:
        ens.upload(cells)
        got = ens.gram(engine=engine)
    assert np.array_equal(got, want)


# ---- transform, synth ------------------------------------------------------------------

@pytest.mark.parametrize("pixels", [1, 31, 4095, 4096, 4097, 8191, 8192, 8193, 3 * 8192 + 17,
                                    9 * 4096 + 4095, 1 << 20, 612 * 499])
@pytest.mark.parametrize("engine", [0, 1, 2, 3, 4])
def test_pack_engines(pixels, engine):
    rng = np.random.default_rng(pixels)
    cells = [rng.integers(0, 3, pixels).astype(np.uint8).reshape(1, pixels) for _ in range(3)]
    N.call("fs_set_pack_engine", engine)
    try:
        with DeviceEnsemble(pixels, 1, 3) as ens:
            ens.upload(cells)
            c, b, r = ens.overlap([0, 1, 2])
            g = ens.gram([0, 1, 2], engine="popc")
    finally:
        N.call("fs_set_pack_engine", 4)
    want = O.accumulate(cells, pixels, 1)
    assert np.array_equal(c, want)
    assert np.array_equal(g, O.gram(cells))


def test_device_synth_equals_host_synth():
    w, h = 1000, 777
    with DeviceEnsemble(w, h, 5) as dev_ens, DeviceEnsemble(w, h, 5) as host_ens:
        dev_ens.synth(0, 5, seed=2104, members=2, eps=0.03, mask_index0=10)
        host = [synth_cells(w, h, 10 + i, seed=2104, members=2, eps=0.03) for i in range(5)]
        host_ens.upload(host)
        a = dev_ens.overlap()
        b = host_ens.overlap()
        assert np.array_equal(a[0], b[0])
        assert np.array_equal(dev_ens.gram(engine="tc"), host_ens.gram(engine="popc"))
    assert np.array_equal(a[0], O.accumulate(host, w, h))


def test_band_ensembles_tile_the_raster():
    """Row bands (the multi-GPU shard) reassemble to the full result."""
    w, h, k = 300, 97, 7
    cells = [synth_cells(w, h, i, members=3) for i in range(k)]
    full = O.accumulate(cells, w, h)
    g = np.zeros((k, k), np.int64)
    bins = np.zeros(k + 1, np.int64)
    parts = []
    for row0, rows in [(0, 30), (30, 40), (70, 27)]:
        with DeviceEnsemble(w, h, k, row0=row0, rows=rows) as ens:
            ens.upload(cells)
            c, b, _ = ens.overlap()
            parts.append(c)
            bins += b
            g += ens.gram()
    assert np.array_equal(np.concatenate(parts), full)
    assert np.array_equal(bins, O.overlap_counts(full.reshape(-1), k))
    assert np.array_equal(g, O.gram(cells))


# ---- full-size properties ------------------------------------------------------------

def test_c2_scale_properties():
    """256 masks of 8192 x 8192 (config 2), device-generated: size-independent
    invariants — histogram mass, count mass = Gram trace, composite consistency, and
    exact agreement of the two Gram engines."""
    w = h = 8192
    k = 256
    with DeviceEnsemble(w, h, k) as ens:
        ens.synth(0, k, seed=2104, members=16, eps=0.02)
        c, b, r = ens.overlap()
        g_tc = ens.gram(engine="tc")
        g_pc = ens.gram(engine="popc")
        g_f4 = ens.gram(engine="tc-f4")
    assert np.array_equal(g_tc, g_pc)
    assert np.array_equal(g_f4, g_pc)
    assert int(b.sum()) == w * h
    assert int(c.sum(dtype=np.uint64)) == int(np.trace(g_tc))
    assert np.array_equal(b, np.bincount(c.reshape(-1), minlength=k + 1))
    idx = np.random.default_rng(0).integers(0, w * h, 200_000)
    cc = c.reshape(-1)[idx]
    want = np.zeros((idx.size, 4), np.uint8)
    O.composite_fill(cc, k, want)
    assert np.array_equal(r.reshape(-1, 4)[idx], want)
    sim = fs.similarity_from_gram(g_tc)
    assert np.array_equal(sim, O.similarity_from_gram(g_tc))


# ---- sharded / pipelined recompute (single rank) ---------------------------------------

def test_sharded_recompute_and_pipelined_frames():
    """dist.ShardedEnsemble on one rank: recompute() and double-buffered run_frames()
    reproduce the oracle's maps, histogram, Gram, outliers and clusters."""
    from paper_2104_14667_b200.dist import ShardedEnsemble

    w, h, k = 700, 333, 20
    cells = [synth_cells(w, h, i, members=5, eps=0.04) for i in range(k)]
    ids = [f"s{i:04d}" for i in range(k)]
    counts = O.accumulate(cells, w, h)
    g = O.gram(cells)
    sim = O.similarity_from_gram(g)
    sh = ShardedEnsemble(w, h, k)
    try:
        sh.ens.upload(cells)
        r = sh.recompute(range(k), tau=0.8, ids=ids)
        assert np.array_equal(r["counts"], counts)
        assert np.array_equal(r["rgba"], O.composite(counts, k))
        assert r["bins"].tolist() == O.overlap_counts(counts.reshape(-1), k).tolist()
        assert np.array_equal(r["gram"], g)
        assert r["clusters"] == O.cluster(sim, ids, 0.8)
        assert r["outliers"] == O.outlier_scores(sim, ids)
        frames = sh.run_frames(range(k), 5, tau=0.8, ids=ids, maps_to_host=True)
        assert len(frames) == 5
        for f in frames[-2:]:  # map views of the last two frames are still valid
            assert np.array_equal(f["counts"], counts)
        for f in frames:
            assert np.array_equal(f["gram"], g)
            assert f["clusters"] == O.cluster(sim, ids, 0.8)
    finally:
        sh.close()


def test_gram_f4_chunk_cap_large_k_range():
    """FP4 accumulates in f32: a K chunk is capped at 2^24 px.  One 128-panel of 3 masks
    over 40 Mpx forces several capped chunks per CTA grid; all-ones masks make the
    diagonal entries as large as possible."""
    w, h = 8192, 5000
    cells = [np.ones((h, w), np.uint8), synth_cells(w, h, 1, members=2, eps=0.3),
             np.zeros((h, w), np.uint8)]
    with DeviceEnsemble(w, h, 3) as ens:
        ens.upload(cells)
        got = ens.gram(engine="tc-f4")
        ref = ens.gram(engine="popc")
    assert np.array_equal(got, ref)
    assert got[0, 0] == w * h


# ---- fused recompute: overlap products out of the Gram kernel -------------------------

@pytest.mark.parametrize("engine", ["tc-f4", "tc", "popc"])
@pytest.mark.parametrize("k,h,w", [(1, 5, 7), (3, 33, 31), (16, 64, 64), (100, 40, 70),
                                   (128, 32, 33), (129, 17, 65), (256, 24, 40),
                                   (257, 16, 33), (300, 9, 130), (64, 1500, 1100),
                                   (200, 700, 2000), (256, 613, 1999),
                                   # narrow panel (MMA N = roundup(k, 16) < 128), many K chunks
                                   (33, 1100, 1500), (127, 300, 700)])
def test_products_match_oracle(engine, k, h, w):
    rng = np.random.default_rng(7 * k + h)
    cells = [(rng.random((h, w)) < rng.uniform(0.05, 0.95)).astype(np.uint8) *
             rng.integers(1, 256, (h, w)).astype(np.uint8) for _ in range(k)]
    want = O.accumulate(cells, w, h)
    with DeviceEnsemble(w, h, k + 3) as ens:
        ens.upload(cells, first=2)
        slots = list(range(2, k + 2))
        c, b, r, g, fused = ens.products(slots, engine=engine)
        perm = [2 + int(x) for x in rng.permutation(k)]
        c2, b2, r2, g2, fused2 = ens.products(perm, engine=engine)  # gathered slots
    # k <= 256: overlap out of the diagonal CTAs; FP4 beyond one panel: partial counts
    # from the diagonal CTAs + a combine pass
    assert fused == (engine != "popc" and (k <= 256 or engine == "tc-f4"))
    assert np.array_equal(c, want)
    assert b.tolist() == O.overlap_counts(want.reshape(-1), k).tolist()
    assert np.array_equal(r, O.composite(want, k))
    gw = O.gram(cells)
    assert np.array_equal(g, gw)
    assert np.array_equal(c2, want) and np.array_equal(r2, r) and np.array_equal(b2, b)
    p = np.asarray(perm) - 2
    assert np.array_equal(g2, gw[np.ix_(p, p)])


def test_products_c1_goldens(golden):
    """The reference bench inputs through the fused path: every C1 golden."""
    cells = c1_cells()
    rec = golden["c1"]
    with DeviceEnsemble(1024, 1024, 16) as ens:
        ens.upload(cells)
        c, b, r, g, fused = ens.products(engine="tc-f4")
    assert fused
    assert O.grid_digest(1024, 1024, 16, c) == rec["digest"]
    assert b.tolist() == rec["bins"]
    assert sha(r) == rec["composite_sha"]
    assert sha(g) == rec["gram_sha"]


def test_products_c2_scale_fused_equals_unfused():
    """Config 2 (256 x 8192^2) on the device: the fused kernel's maps, histogram and
    Gram equal the separate overlap kernel + popc Gram, bit for bit."""
    w = h = 8192
    k = 256
    with DeviceEnsemble(w, h, k) as ens:
        ens.synth(0, k, seed=2104, members=16, eps=0.02)
        c, b, r, g, fused = ens.products(engine="tc-f4")
        c0, b0, r0 = ens.overlap()
        g0 = ens.gram(engine="popc")
    assert fused
    assert np.array_equal(b, b0)
    assert np.array_equal(g, g0)
    assert np.array_equal(c, c0)
    assert np.array_equal(r, r0)


# ---- measured sweep suites (config 5) -------------------------------------------------

def test_transform_sweep_and_transfer_suites():
    from paper_2104_14667_b200.sweep import (RateMap, SweepSpec, render_rate_map,
                                             run_backend_comparison, run_transfer_baseline,
                                             run_transform_sweep)

    spec = SweepSpec(64, 500, 1100)
    rm = run_transform_sweep(spec, reps=2)
    assert rm.rates.shape == (3, 3) and (rm.rates > 0).all()
    assert RateMap.from_json(rm.to_json()).rates.tolist() == rm.rates.tolist()
    assert rm.to_csv().splitlines()[0] == "width,height,rate_gbps"
    assert render_rate_map(rm).shape == (3, 3, 4)
    rep = run_transfer_baseline(points=[1 << 16, 1 << 20], repeats=2)
    assert [r["bytes"] for r in rep.rows] == [1 << 16, 1 << 20]
    assert all(r["rate_gbps"] > 0 for r in rep.rows)
    back = run_backend_comparison(pixels=1 << 16, n_surfaces=4, repeats=1)
    assert {r["backend"] for r in back.rows} == {"cuda", "cuda-batched"}


def test_dual_buffer_suite_measured():
    """The paper's four strategies measured through the real event DAG (bench.py:231-309
    schema): every (variant, N) row present, positive totals, efficiency in (0, 1.5)."""
    from paper_2104_14667_b200.sweep import VARIANTS, run_dual_buffer_suite

    rep = run_dual_buffer_suite(["96x64", (200, 30)], [3, 7], repeats=1, pool=2)
    assert len(rep.rows) == 2 * len(VARIANTS) * 2
    for r in rep.rows:
        assert r["total_us"] > 0 and 0 < r["efficiency"] < 1.5
        assert r["closed_form_us"] > 0 and len(r["samples_us"]) == 1
    assert rep.to_csv().splitlines()[0] == "variant,n,width,height,total_us,rate_gbps,efficiency"


# ---- config 3 at full size --------------------------------------------------------------

def test_c3_scale_gram_and_clusters():
    """1024 flood-like masks of 4096 x 4096 (config 3, device-generated): the tensor-core
    Gram equals the CUDA-core AND+POPC engine bit for bit, Σcounts = trace(Gram), and
    complete linkage at tau 0.8 recovers the 32 prototypes x 32 members."""
    w = h = 4096
    k, members = 1024, 32
    with DeviceEnsemble(w, h, k) as ens:
        ens.synth(0, k, seed=2104, members=members, eps=0.02)
        c, b, r, g, fused = ens.products(engine="tc-f4")
        g_pc = ens.gram(engine="popc")
    assert fused  # k > 256: per-panel partial counts from the diagonal CTAs + combine
    assert np.array_equal(g, g_pc)
    assert int(b.sum()) == w * h
    assert int(c.sum(dtype=np.uint64)) == int(np.trace(g))
    ids = [f"s{i:04d}" for i in range(k)]
    sim = fs.similarity_from_gram(g)
    clusters = fs.cluster_from_similarity(sim, ids, 0.8)
    assert clusters == [ids[p * members:(p + 1) * members] for p in range(k // members)]
    sub = list(range(0, k, 37))  # the host oracle on a subset of the exact matrix
    assert fs.cluster_from_similarity(sim[np.ix_(sub, sub)], [ids[i] for i in sub], 0.8) == \
        O.cluster(sim[np.ix_(sub, sub)], [ids[i] for i in sub], 0.8)


@pytest.mark.parametrize("k,h,w", [(520, 30, 70), (300, 1100, 1536), (1100, 9, 100),
                                   (4096, 4, 64)])
def test_gram_pair_kernel_multi_panel(k, h, w):
    """k > 256: off-diagonal 256 x 256 tiles run on CTA pairs (cta_group::2, mxf4);
    several panels and many K chunks against the CUDA-core engine and the oracle."""
    rng = np.random.default_rng(k + h)
    if h * w > 100_000:
        cells = [synth_cells(w, h, i, members=7, eps=0.05) for i in range(k)]
    else:
        cells = [(rng.random((h, w)) < rng.uniform(0.05, 0.95)).astype(np.uint8) for _ in range(k)]
    with DeviceEnsemble(w, h, k) as ens:
        ens.upload(cells)
        got = ens.gram(engine="tc-f4")
        ref = ens.gram(engine="popc")
        c, b, r, g2, fused = ens.products(engine="tc-f4")  # multi-panel fused recompute
    assert fused
    assert np.array_equal(got, ref) and np.array_equal(g2, ref)
    counts = O.accumulate(cells, w, h)
    assert np.array_equal(c, counts)
    assert b.tolist() == O.overlap_counts(counts.reshape(-1), k).tolist()
    assert np.array_equal(r, O.composite(counts, k))
    if h * w <= 100_000 and k <= 1100:
        assert np.array_equal(got, O.gram(cells))


@pytest.mark.parametrize("k", [1, 2, 3, 64, 300])
def test_device_similarity_and_outliers_bitwise(k):
    """fs_similarity_outliers_device (the frame pipeline's Jaccard + outliers) equals the
    reference formulas bit for bit, empty unions included."""
    import torch

    rng = np.random.default_rng(k)
    cells = [(rng.random(500) < rng.uniform(0.05, 0.95)).astype(np.uint8) for _ in range(k)]
    if k > 2:
        cells[1] = np.zeros(500, np.uint8)
        cells[2] = np.zeros(500, np.uint8)
    g = O.gram(cells)
    d_g = torch.from_numpy(g).cuda()
    d_s = torch.empty(k * k, dtype=torch.float64, device="cuda")
    d_o = torch.empty(max(k, 1), dtype=torch.float64, device="cuda")
    N.call("fs_similarity_outliers_device", d_g.data_ptr(), k, d_s.data_ptr(),
           d_o.data_ptr() if k >= 2 else None, None)
    N.call("fs_synchronize")
    sim = O.similarity_from_gram(g)
    assert d_s.cpu().numpy().reshape(k, k).tobytes() == sim.tobytes()
    if k >= 2:
        ids = [f"s{i}" for i in range(k)]
        want = O.outlier_scores(sim, ids)
        got = d_o.cpu().numpy()
        assert [float(x).hex() for x in got] == [float(want[i]).hex() for i in ids]


def test_error_mapping_on_device():
    """C-ABI status codes surface as the reference's error kinds: bad arguments ->
    ValueError, device allocation failure -> MemoryError; the handle stays usable."""
    cells = [synth_cells(64, 32, i, members=2) for i in range(3)]
    with DeviceEnsemble(64, 32, 3) as ens:
        ens.upload(cells)
        with pytest.raises(ValueError, match="slot"):
            ens.overlap([0, 3])
        with pytest.raises(ValueError):
            ens.stream(cells + cells, first=1)
        with pytest.raises(ValueError):
            ens.products([])
        c, _, _ = ens.overlap()
        assert np.array_equal(c, O.accumulate(cells, 64, 32))
    with pytest.raises(MemoryError):
        DeviceEnsemble(1 << 20, 1 << 16, 4096)  # 2^36 px x 4096 masks: far beyond 180 GB


def test_concurrent_callers():
    """The reference calls the primitives from its recompute worker, the request
    threadpool and job threads at once (service.py:92-95,198,289-324): protocol calls
    from 6 threads plus shared-ensemble recomputes stay exact."""
    from concurrent.futures import ThreadPoolExecutor

    w, h, k = 300, 97, 12
    cells = [synth_cells(w, h, i, members=3, eps=0.05) for i in range(k)]
    want_counts = O.accumulate(cells, w, h)
    want_gram = O.gram(cells)
    surfaces = surfaces_of(cells)
    with DeviceEnsemble(w, h, k) as ens:
        ens.upload(cells)

        def job(t):
            if t % 3 == 0:
                g = fs.accumulate(surfaces)
                return np.array_equal(g.counts, want_counts)
            if t % 3 == 1:
                c, b, r, g, _ = ens.products(engine="tc-f4")
                return np.array_equal(c, want_counts) and np.array_equal(g, want_gram)
            a, b = cells[t % k].reshape(-1), cells[(t + 1) % k].reshape(-1)
            return K.pair_counts(a, b) == O.pair_counts(a, b)

        with ThreadPoolExecutor(max_workers=6) as pool:
            assert all(pool.map(job, range(36)))


def test_bench_cli_suites(tmp_path):
    """The measured `bench` suites through the module CLI (fs/cli.py:72-150 shape)."""
    import json as _json
    import subprocess
    import sys

    for argv, out in ([["backends", "--pixels", "65536", "--surfaces", "3", "--repeats", "1"],
                       "b.json"],
                      [["dual", "--dims", "96x64", "--n", "3", "--repeats", "1"], "d.csv"],
                      [["transfer", "--min-bytes", "65536", "--max-bytes", "131072",
                        "--step-bytes", "65536", "--repeats", "1"], "t.json"],
                      [["sweep", "--start", "64", "--step", "500", "--stop", "1100", "--reps",
                        "1"], "s.json"]):
        p = tmp_path / out
        r = subprocess.run([sys.executable, "-m", "paper_2104_14667_b200", "bench", *argv,
                            "--out", str(p)], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        assert p.exists() and p.stat().st_size > 0
        if out.endswith(".json"):
            _json.loads(p.read_text())


@pytest.mark.parametrize("seed", range(12))
def test_randomized_overlap_and_products(seed):
    """Randomised shapes against the oracle: k in 1..320, odd raster sizes, masks in
    permuted / gathered slots of a larger ensemble, cycled inputs (weights w1 = c + 1
    for the first `remainder` surfaces, c for the rest, streaming.py:417-425), and the
    fused recompute on the same slots."""
    rng = np.random.default_rng(900 + seed)
    k = int(rng.integers(1, 321))
    h, w = int(rng.integers(1, 40)), int(rng.integers(1, 300))
    cap = k + int(rng.integers(0, 5))
    cells = [(rng.random((h, w)) < rng.uniform(0.0, 1.0)).astype(np.uint8) *
             rng.integers(1, 256, (h, w)).astype(np.uint8) for _ in range(k)]
    slots = rng.permutation(cap)[:k].tolist()
    cyc, rem = int(rng.integers(1, 4)), int(rng.integers(0, k + 1))
    with DeviceEnsemble(w, h, cap) as ens:
        for s, c in zip(slots, cells):
            ens.upload([c], first=s)
        c1, b1, r1 = ens.overlap(slots, cycles=cyc, remainder=rem)
        c2, b2, r2, g2, _ = ens.products(slots, engine="tc-f4")
    n = cyc * k + rem
    seq = [cells[i % k] for i in range(n)]  # run_stream's cycling order
    want = O.accumulate(seq, w, h)
    assert np.array_equal(c1, want)
    assert b1.tolist() == O.overlap_counts(want.reshape(-1), n).tolist()
    assert np.array_equal(r1, O.composite(want, n))
    once = O.accumulate(cells, w, h)
    assert np.array_equal(c2, once)
    assert b2.tolist() == O.overlap_counts(once.reshape(-1), k).tolist()
    assert np.array_equal(r2, O.composite(once, k))
    assert np.array_equal(g2, O.gram(cells))


@pytest.mark.parametrize("k,h,w", [(20, 97, 300), (300, 33, 64)])
def test_native_pipeline(k, h, w):
    """fs_pipeline_*: the native frame loop gives the oracle's histogram, Gram,
    similarity, outliers and clusters (last frame of several in flight)."""
    cells = [synth_cells(w, h, i, members=5, eps=0.04) for i in range(k)]
    ids = [f"m{i:04d}" for i in range(k)]
    g = O.gram(cells)
    sim = O.similarity_from_gram(g)
    counts = O.accumulate(cells, w, h)
    with DeviceEnsemble(w, h, k) as ens:
        ens.upload(cells)
        with ens.pipeline(list(range(k)), ids=ids, depth=3) as pipe:
            r1 = pipe.run(1)
            r = pipe.run(9)
    for res in (r1, r):
        assert res["bins"].tolist() == O.overlap_counts(counts.reshape(-1), k).tolist()
        assert np.array_equal(res["gram"], g)
        assert res["similarity"].tobytes() == sim.tobytes()
        assert res["clusters"] == O.cluster(sim, ids, 0.8)
        assert res["outliers"] == O.outlier_scores(sim, ids)
    assert r["device_ms"] > 0
