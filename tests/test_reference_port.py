"""The reference's own hot-path tests, restated against this package on the B200.

Each test names the reference test it follows (paths under /root/reference/pkg/tests/):
test_analytics.py (known answers, validation, composite, Jaccard, clustering,
outliers, backend parity), test_properties.py:106-139 (hypothesis invariants on 4x6
masks) and test_acceptance.py:208-308 (100 random instances, seed 55, exact, with an
independent Lance-Williams clusterer).  Every call goes through the public API, i.e.
the CUDA backend behind the C ABI; expected values are brute-force numpy on the test
side, exactly as in the reference.

Deviation: the reference compares outlier scores with Python's built-in
``sum`` over floats, which Python 3.12 compensates; ``outlier_scores`` itself (and this
package) sums np.float64 left to right, so the restated check uses that order.
"""

from __future__ import annotations

import io
import math

import numpy as np
import numpy.testing as npt
import pytest

pytestmark = pytest.mark.gpu

hyp = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    from paper_2104_14667_b200 import _native as N

    if N.device_count() == 0:
        pytest.skip("needs a CUDA device")
    N.set_device(0)


def fs():
    import paper_2104_14667_b200 as m

    return m


def wet_sum(surfaces):
    return sum((s.cells > 0).astype(np.uint32) for s in surfaces)


# -- test_analytics.py:24-59 -------------------------------------------------------
def test_depths_count_once(make_surface):
    grid = fs().accumulate([make_surface(np.array([[0, 1], [9, 255]], dtype=np.uint8))])
    npt.assert_array_equal(grid.counts, [[0, 1], [1, 1]])


def test_accumulate_brute_force(make_surface):
    rng = np.random.default_rng(3)
    for _ in range(20):
        w, h = int(rng.integers(1, 65)), int(rng.integers(1, 65))
        k = int(rng.integers(1, 51))
        stack = [make_surface((w, h), seed=int(rng.integers(1 << 30))) for _ in range(k)]
        grid = fs().accumulate(stack)
        npt.assert_array_equal(grid.counts, wet_sum(stack))
        assert grid.n_inputs == k


def test_accumulate_order_free(make_surface):
    stack = [make_surface((40, 30), seed=i) for i in range(10)]
    a, b = fs().accumulate(stack), fs().accumulate(stack[::-1])
    npt.assert_array_equal(a.counts, b.counts)
    assert a.digest() == b.digest()


def test_accumulate_validation(make_surface):
    AE = fs().AnalyticsError
    with pytest.raises(AE, match="at least one"):
        fs().accumulate([])
    with pytest.raises(AE, match="odd-one"):
        fs().accumulate([make_surface((8, 8), seed=0), make_surface((9, 8), seed=1, id="odd-one")])
    with pytest.raises(AE, match="unknown kernel variant"):
        fs().accumulate([make_surface((4, 4), seed=0)], variant="image9")


# -- test_analytics.py:62-96 -------------------------------------------------------
def test_grid_validation_and_digest():
    m = fs()
    with pytest.raises(m.AnalyticsError, match="exceeds"):
        m.AccumulationGrid(width=2, height=2, n_inputs=2, counts=np.full((2, 2), 3, np.uint32))
    with pytest.raises(m.AnalyticsError, match="uint32"):
        m.AccumulationGrid(width=2, height=2, n_inputs=1, counts=np.zeros((2, 2)))
    with pytest.raises(m.AnalyticsError, match="shape"):
        m.AccumulationGrid(width=2, height=3, n_inputs=1, counts=np.zeros((2, 2), np.uint32))
    z = np.zeros((2, 2), np.uint32)
    assert (m.AccumulationGrid(width=2, height=2, n_inputs=0, counts=z).digest()
            != m.AccumulationGrid(width=2, height=2, n_inputs=5, counts=z.copy()).digest())


def test_histogram_bincount_and_empty(make_surface):
    m = fs()
    grid = m.accumulate([make_surface((32, 24), seed=i) for i in range(7)])
    hist = m.overlap_histogram(grid)
    npt.assert_array_equal(hist.bins, np.bincount(grid.counts.ravel(), minlength=8))
    assert len(hist.bins) == 8 and sum(hist.bins) == 32 * 24 and hist.n_inputs == 7
    assert m.overlap_histogram(m.AccumulationGrid.empty(5, 4)).bins == [20]


# -- test_analytics.py:99-147 ------------------------------------------------------
def test_composite_formula(make_surface):
    m = fs()
    grid = m.accumulate([make_surface((16, 16), seed=i) for i in range(5)])
    px = m.composite_map(grid).pixels
    c = grid.counts
    cov = c > 0
    assert (px[~cov] == 0).all()
    grey = np.floor(255.0 * (1.0 - c[cov] / 5) + 0.5).astype(np.uint8)
    npt.assert_array_equal(px[cov][:, 0], grey)
    npt.assert_array_equal(px[cov][:, 1], grey)
    assert (px[cov][:, 2] == 255).all() and (px[cov][:, 3] == 255).all()


def test_composite_saturated_basemap_and_png(make_surface):
    m = fs()
    ones = np.ones((4, 4), np.uint8)
    g = m.accumulate([make_surface(ones, id="a"), make_surface(ones, id="b")])
    npt.assert_array_equal(m.composite_map(g).pixels[0, 0], [0, 0, 255, 255])
    cells = np.zeros((2, 2), np.uint8)
    cells[0, 0] = 1
    base = m.CompositeImage(width=2, height=2, pixels=np.full((2, 2, 4), 7, np.uint8))
    merged = m.composite_map(m.accumulate([make_surface(cells)]), basemap=base)
    npt.assert_array_equal(merged.pixels[0, 0], [0, 0, 255, 255])
    npt.assert_array_equal(merged.pixels[1, 1], [7, 7, 7, 7])
    with pytest.raises(m.AnalyticsError, match="basemap"):
        m.composite_map(m.AccumulationGrid.empty(4, 4),
                        basemap=m.CompositeImage(width=2, height=2,
                                                 pixels=np.zeros((2, 2, 4), np.uint8)))
    from PIL import Image

    img = m.composite_map(m.accumulate([make_surface((8, 6), seed=1)]))
    npt.assert_array_equal(np.asarray(Image.open(io.BytesIO(img.png_bytes()))), img.pixels)


# -- test_analytics.py:150-179 -----------------------------------------------------
def test_jaccard_known_answers(make_surface):
    m = fs()
    a, b = np.zeros((1, 40), np.uint8), np.zeros((1, 40), np.uint8)
    a[0, :25] = 1
    b[0, 15:40] = 1
    assert m.jaccard(make_surface(a), make_surface(b)) == 0.25
    s = make_surface((10, 10), seed=1)
    assert m.jaccard(s, s) == 1.0
    left, right = np.zeros((1, 4), np.uint8), np.zeros((1, 4), np.uint8)
    left[0, 0] = right[0, 3] = 1
    assert m.jaccard(make_surface(left), make_surface(right)) == 0.0
    e = np.zeros((3, 3), np.uint8)
    assert m.jaccard(make_surface(e, id="a"), make_surface(e, id="b")) == 1.0
    with pytest.raises(m.AnalyticsError):
        m.jaccard(make_surface((3, 3), seed=0), make_surface((4, 3), seed=1))
    sim = m.similarity_matrix([make_surface((12, 12), seed=i) for i in range(6)])
    npt.assert_array_equal(sim, sim.T)
    npt.assert_array_equal(np.diag(sim), np.ones(6))


def _trio(make_surface):
    base = np.zeros((8, 8), np.uint8)
    s1, s2, s3 = base.copy(), base.copy(), base.copy()
    s1.flat[0:10] = 1
    s2.flat[0:9] = 1
    s3.flat[[0, 1, 2, 20, 21, 22, 23, 24, 25, 26]] = 1
    return [make_surface(x, id=n) for x, n in ((s1, "s1"), (s2, "s2"), (s3, "s3"))]


# -- test_analytics.py:194-258 -----------------------------------------------------
def test_clustering_known_answers(make_surface):
    m = fs()
    trio = _trio(make_surface)
    assert m.cluster_surfaces(trio, tau=0.8) == [["s1", "s2"], ["s3"]]
    assert m.cluster_surfaces(trio, tau=0.01) == [["s1", "s2", "s3"]]
    assert m.cluster_surfaces(trio[::-1], tau=0.8) == [["s1", "s2"], ["s3"]]
    base = np.zeros((10, 10), np.uint8)
    chain = []
    for n, lo in (("a", 0), ("b", 1), ("c", 2)):
        x = base.copy()
        x.flat[lo:lo + 10] = 1
        chain.append(make_surface(x, id=n))
    cl = m.cluster_surfaces(chain, tau=0.8)
    assert len(cl) == 2 and (["c"] in cl or ["a"] in cl)
    one = [make_surface((4, 4), seed=0)]
    for bad in (0.0, 1.5):
        with pytest.raises(m.AnalyticsError, match="tau"):
            m.cluster_surfaces(one, tau=bad)
    assert m.cluster_surfaces([make_surface((4, 4), seed=0, id="only")]) == [["only"]]


def test_outliers_known_answers(make_surface):
    m = fs()
    trio = _trio(make_surface)
    sim = m.similarity_matrix(trio)
    sc = m.outlier_scores(trio)
    assert sc["s1"] == 1.0 - (np.float64(0.0) + sim[0, 1] + sim[0, 2]) / 2
    assert sc["s3"] == 1.0 - (np.float64(0.0) + sim[2, 0] + sim[2, 1]) / 2
    assert sc["s3"] == max(sc.values())
    with pytest.raises(m.AnalyticsError, match="at least two"):
        m.outlier_scores([make_surface((4, 4), seed=0)])


# -- test_analytics.py:261-285, all backends against the NumPy formulas -------------
def test_backend_protocol_parity():
    from paper_2104_14667_b200.backends import available_backends

    rng = np.random.default_rng(11)
    cells = (rng.random(4096) < 0.4).astype(np.uint8)
    other = (rng.random(4096) < 0.4).astype(np.uint8)
    want_counts = (cells > 0).astype(np.uint32) + (other > 0)
    want_bins = np.bincount(want_counts, minlength=3)
    want_pair = (int(((cells > 0) & (other > 0)).sum()), int(((cells > 0) | (other > 0)).sum()))
    g = np.floor(255.0 * (1.0 - want_counts / 2) + 0.5).astype(np.uint8)
    want_rgba = np.where((want_counts > 0)[:, None],
                         np.stack([g, g, np.full_like(g, 255), np.full_like(g, 255)], 1), 0)
    backends = available_backends()
    assert "cuda" in backends
    for name, mod in backends.items():
        counts = np.zeros(4096, np.uint32)
        mod.accumulate_into(counts, cells)
        mod.accumulate_into(counts, other)
        out = np.zeros((4096, 4), np.uint8)
        mod.composite_fill(counts, 2, out)
        npt.assert_array_equal(counts, want_counts)
        npt.assert_array_equal(np.asarray(mod.overlap_counts(counts, 2)), want_bins)
        assert mod.pair_counts(cells, other) == want_pair
        assert all(type(x) is int for x in mod.pair_counts(cells, other))
        npt.assert_array_equal(out, want_rgba)


# -- test_properties.py:106-139 ----------------------------------------------------
_masks = st.integers(min_value=0, max_value=2**24 - 1)


def _bits(sid, bits):
    from paper_2104_14667_b200.rasters import RasterSurface

    flat = np.array([(bits >> i) & 1 for i in range(24)], dtype=np.uint8)
    return RasterSurface(id=sid, name=sid, width=6, height=4, cells=flat.reshape(4, 6))


@settings(max_examples=80, deadline=None)
@given(_masks, _masks)
def test_property_jaccard_is_a_similarity(a_bits, b_bits):
    m = fs()
    a, b = _bits("a", a_bits), _bits("b", b_bits)
    ab = m.jaccard(a, b)
    assert 0.0 <= ab <= 1.0 and ab == m.jaccard(b, a) and m.jaccard(a, a) == 1.0
    inter, union = bin(a_bits & b_bits).count("1"), bin(a_bits | b_bits).count("1")
    assert ab == (1.0 if union == 0 else inter / union)


@settings(max_examples=40, deadline=None)
@given(st.lists(_masks, min_size=1, max_size=8))
def test_property_counts_bounded_histogram_complete(bit_list):
    m = fs()
    stack = [_bits(f"s{i}", b) for i, b in enumerate(bit_list)]
    grid = m.accumulate(stack)
    n = len(stack)
    assert grid.n_inputs == n and grid.counts.max() <= n
    bins = m.overlap_histogram(grid).bins
    assert len(bins) == n + 1 and sum(bins) == 24
    npt.assert_array_equal(grid.counts, wet_sum(stack))


@settings(max_examples=40, deadline=None)
@given(st.lists(_masks, min_size=1, max_size=8), st.randoms())
def test_property_accumulation_order_free(bit_list, rnd):
    m = fs()
    stack = [_bits(f"s{i}", b) for i, b in enumerate(bit_list)]
    shuffled = list(stack)
    rnd.shuffle(shuffled)
    assert m.accumulate(stack).digest() == m.accumulate(shuffled).digest()


# -- test_acceptance.py:208-308 ----------------------------------------------------
def _lance_williams(ids, pair_sim, tau):
    """Independent complete-linkage clusterer (the acceptance test's own oracle)."""
    members = {i: [ids[i]] for i in range(len(ids))}
    link = {(i, j): pair_sim[(ids[i], ids[j])] for i in members for j in members if i < j}
    while len(members) > 1:
        best = None
        for (i, j), score in link.items():
            lo, hi = sorted((min(members[i]), min(members[j])))
            key = (-score, lo, hi)
            if best is None or key < best[0]:
                best = (key, (i, j))
        if best is None or -best[0][0] < tau:
            break
        i, j = best[1]
        members[i] = members[i] + members[j]
        del members[j]
        del link[(i, j)]
        for q in list(members):
            if q != i:
                a, b = (min(i, q), max(i, q)), (min(j, q), max(j, q))
                link[a] = min(link[a], link.pop(b))
    return sorted((sorted(c) for c in members.values()), key=lambda c: c[0])


def test_acceptance_analytics_brute_force():
    from paper_2104_14667_b200.rasters import RasterSurface

    m = fs()
    rng = np.random.default_rng(55)
    for case in range(100):
        h, w = int(rng.integers(1, 65)), int(rng.integers(1, 65))
        count = int(rng.integers(2, 51))
        tau = float(rng.uniform(0.05, 0.95))
        stack = [RasterSurface(id=f"s{i:02d}", name=f"s{i:02d}", width=w, height=h,
                               cells=rng.integers(0, 4, size=(h, w)).astype(np.uint8))
                 for i in range(count)]
        wet = {s.id: s.cells > 0 for s in stack}
        grid = m.accumulate(stack)
        want = sum(wet[s.id].astype(np.int64) for s in stack)
        assert np.array_equal(grid.counts, want), case
        bins = m.overlap_histogram(grid).bins
        assert bins == [int((want == q).sum()) for q in range(count + 1)], case
        pair_sim = {}
        for a in stack:
            for b in stack:
                if a.id < b.id:
                    union = int((wet[a.id] | wet[b.id]).sum())
                    inter = int((wet[a.id] & wet[b.id]).sum())
                    pair_sim[(a.id, b.id)] = 1.0 if union == 0 else inter / union
                    assert m.jaccard(a, b) == pair_sim[(a.id, b.id)], (case, a.id, b.id)
        ids = [s.id for s in stack]
        expected = _lance_williams(ids, pair_sim, tau)
        assert m.cluster_surfaces(stack, tau) == expected, case
        scores = m.outlier_scores(stack)
        for sid in ids:
            acc = np.float64(0.0)  # outlier_scores' np.float64 left-to-right order
            for o in ids:
                if o != sid:
                    acc = acc + pair_sim[(min(sid, o), max(sid, o))]
            assert scores[sid] == 1.0 - acc / (count - 1), (case, sid)
        order = rng.permutation(count)
        shuffled = [stack[i] for i in order]
        g2 = m.accumulate(shuffled)
        assert g2.digest() == grid.digest() and m.overlap_histogram(g2).bins == bins, case
        assert m.cluster_surfaces(shuffled, tau) == expected, case
        s2 = m.outlier_scores(shuffled)
        assert all(math.isclose(s2[q], scores[q], rel_tol=1e-12, abs_tol=1e-12) for q in scores)
