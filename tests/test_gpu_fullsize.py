"""Oracle parity at the BASELINE configs' full sizes (C2 256 x 8192^2,
C3 1024 x 4096^2, C4 64 x 32768^2).

The inputs are uint8 HOST rasters (depths 0..255) and every product goes through the
public path a user calls — pinned host rasters -> streamed upload (H2D + binarize/pack
transform on the device) -> recompute -> D2H — so the transform, the packed layout, the
chunk planner and the kernels are all inside what is checked.  The checker is the
oracle's C restatement (oracle/fs_oracle.c, OpenMP: fs/_kernels_np.py + the pair loop
of fs/analytics.py:174-181) and its NumPy restatement of fs/analytics.py:165-240 for
the float64 products, run on the same host bytes: counts, histogram, RGBA and the int64
Gram bit-exact; Jaccard matrix and outlier scores bitwise; cluster lists identical.

Three masks of each ensemble are replaced by inputs from outside the product's
generator (all dry, all wet at depth 255, and NumPy Bernoulli masks with random depths),
so the extremes of every count class are exercised.
"""

import hashlib

import numpy as np
import pytest

import oracle_c
from oracle import fs_oracle as O

pytestmark = pytest.mark.gpu

import paper_2104_14667_b200 as fs  # noqa: E402
from paper_2104_14667_b200 import _native as N  # noqa: E402
from paper_2104_14667_b200.ensemble import DeviceEnsemble  # noqa: E402
from paper_2104_14667_b200.synth import synth_cells_gpu  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def host_ensemble(w, h, k, members, eps, seed=2104, band_rows=None):
    """k pinned (h, w) uint8 rasters: the flood-like generator's bytes, except masks
    0, 1, 2 = all dry / all wet (255) / NumPy Bernoulli(0.5) x random depth."""
    bufs = [N.PinnedBuffer((h, w)) for _ in range(k)]
    for i in range(k):
        synth_cells_gpu(w, h, i, seed=seed, members=members, eps=eps, out=bufs[i].array)
    bufs[0].array[:] = 0
    bufs[1].array[:] = 255
    rng = np.random.default_rng(seed)
    for r0 in range(0, h, 1024):  # row blocks: bounded temporaries
        n = min(1024, h - r0)
        wet = rng.random((n, w)) < 0.5
        bufs[2].array[r0:r0 + n] = wet * rng.integers(1, 256, (n, w), dtype=np.uint8)
    return bufs


def oracle_products(arrays, k):
    flat = [a.reshape(-1) for a in arrays]
    counts = oracle_c.accumulate(flat)
    bins = oracle_c.histogram(counts, k)
    rgba = oracle_c.composite(counts, k)
    gram = oracle_c.gram(flat)
    return counts, bins, rgba, gram


def check_analytics(gram, sim, outliers, clusters, ids, tau, *, fast_cluster=False):
    want_sim = O.similarity_from_gram(gram)
    assert sim.tobytes() == want_sim.tobytes()
    want_out = O.outlier_scores(want_sim, ids)
    assert {s: float(v).hex() for s, v in outliers.items()} == \
        {s: float(v).hex() for s, v in want_out.items()}
    want_cl = (O.cluster_unique_ids if fast_cluster else O.cluster)(want_sim, ids, tau)
    assert clusters == want_cl
    return want_cl


@pytest.fixture(scope="module")
def c2_host():
    w = h = 8192
    k = 256
    bufs = host_ensemble(w, h, k, members=16, eps=0.02)
    arrays = [b.array for b in bufs]
    want = oracle_products(arrays, k)
    yield w, h, k, arrays, want
    for b in bufs:
        b.free()


def test_c2_full_size_products_vs_oracle(c2_host):
    """C2 through DeviceEnsemble: 2b-final stream from pinned rasters, ONE fused
    recompute (tensor-core Gram + counter warps), host outputs."""
    w, h, k, arrays, (counts, bins, rgba, gram) = c2_host
    with DeviceEnsemble(w, h, k) as ens:
        ens.stream(arrays, variant="2b-final")
        c, b, r, g, fused = ens.products(engine="tc-f4")
    assert fused
    assert sha(c) == sha(counts)
    assert b.tolist() == bins.tolist()
    assert sha(r) == sha(rgba)
    assert np.array_equal(g, gram)
    assert int(g[1, 1]) == w * h and int(g[0, 0]) == 0 and int(b[0]) == 0


def test_c2_full_size_e2e_frames_vs_oracle(c2_host):
    """C2 end to end exactly as bench.py's e2e leg runs it: every frame re-streams all
    256 rasters (2b-final) before the recompute, maps D2H on a side stream, device
    Jaccard/outliers, host linkage — two frames, the last one checked in full."""
    from paper_2104_14667_b200.dist import ShardedEnsemble

    w, h, k, arrays, (counts, bins, rgba, gram) = c2_host
    ids = [f"s{i:04d}" for i in range(k)]
    sh = ShardedEnsemble(w, h, k)
    try:
        def upload(_f):
            sh.ens.stream(arrays, variant="2b-final", already_banded=True)

        r = sh.run_frames(range(k), 2, tau=0.8, engine="tc-f4", ids=ids, maps_to_host=True,
                          keep=False, before_frame=upload)[-1]
        assert sha(r["counts"]) == sha(counts)
        assert sha(r["rgba"]) == sha(rgba)
        assert r["bins"].tolist() == bins.tolist()
        assert np.array_equal(r["gram"], gram)
        cl = check_analytics(gram, r["similarity"], r["outliers"], r["clusters"], ids, 0.8)
        # the native frame loop on the same resident ensemble
        with sh.ens.pipeline(range(k), tau=0.8, engine="tc-f4", ids=ids, depth=3) as pipe:
            rn = pipe.run(3)
        assert np.array_equal(rn["gram"], gram) and rn["bins"].tolist() == bins.tolist()
        assert rn["similarity"].tobytes() == O.similarity_from_gram(gram).tobytes()
        assert rn["clusters"] == cl
    finally:
        sh.close()


def test_c3_full_size_vs_oracle():
    """C3 (1024 x 4096^2): multi-panel plan — diagonal FP4 tiles with per-panel partial
    counts, CTA-pair off-diagonal tiles, combine pass — against the oracle, plus the
    32 x 32 cluster structure and outliers through the analytics."""
    w = h = 4096
    k, members = 1024, 32
    bufs = host_ensemble(w, h, k, members=members, eps=0.02)
    try:
        arrays = [b.array for b in bufs]
        counts, bins, rgba, gram = oracle_products(arrays, k)
        with DeviceEnsemble(w, h, k) as ens:
            ens.stream(arrays, variant="2b-final")
            c, b, r, g, fused = ens.products(engine="tc-f4")
        assert fused
        assert sha(c) == sha(counts)
        assert b.tolist() == bins.tolist()
        assert sha(r) == sha(rgba)
        assert np.array_equal(g, gram)
        ids = [f"s{i:04d}" for i in range(k)]
        sim = fs.similarity_from_gram(g)
        out = fs.outliers_from_similarity(sim, ids)
        cl = fs.cluster_from_similarity(sim, ids, 0.8)
        want_cl = check_analytics(gram, sim, out, cl, ids, 0.8, fast_cluster=True)
        # prototypes 0..31 of 32 members; masks 0-2 were replaced, so they leave
        # prototype 0 (singletons), the rest of it clusters together
        assert len(want_cl) == 31 + 1 + 3
    finally:
        for b in bufs:
            b.free()


def test_c4_full_size_banded_vs_oracle():
    """C4 (64 x 32768^2 = 68.7 GB of uint8 rasters): BandedStream from pinned host
    rasters, band by band (H2D + transform + fused recompute + D2H of the maps); the
    oracle checks every band's counts/RGBA rows and the summed histogram and Gram."""
    from paper_2104_14667_b200.banded import BandedStream

    w = h = 32768
    k, members = 64, 8
    bufs = host_ensemble(w, h, k, members=members, eps=0.02)
    try:
        arrays = [b.array for b in bufs]
        counts_out = N.PinnedBuffer((h, w), np.uint32)
        rgba_out = N.PinnedBuffer((h, w, 4), np.uint8)
        try:
            ids = [f"s{i:04d}" for i in range(k)]
            with BandedStream(w, h, k, band_rows=4096) as bs:
                r = bs.run(arrays, tau=0.8, ids=ids, counts_out=counts_out.array,
                           rgba_out=rgba_out.array, engine="tc-f4")
            bins = np.zeros(k + 1, np.int64)
            gram = np.zeros((k, k), np.int64)
            step = 4096
            for r0 in range(0, h, step):
                part = [a[r0:r0 + step] for a in arrays]
                c, b, rg, g = oracle_products(part, k)
                assert sha(counts_out.array[r0:r0 + step]) == sha(c), r0
                assert sha(rgba_out.array[r0:r0 + step]) == sha(rg), r0
                bins += b
                gram += g
            assert r["bins"].tolist() == bins.tolist()
            assert np.array_equal(r["gram"], gram)
            check_analytics(gram, r["similarity"], r["outliers"], r["clusters"], ids, 0.8)
        finally:
            counts_out.free()
            rgba_out.free()
    finally:
        for b in bufs:
            b.free()
