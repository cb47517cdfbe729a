"""The batched drop-in calls' device cache (fs_accumulate_many / fs_gram_many keep the
stack bit-packed in HBM keyed by a fingerprint of each raster's bytes): hits, partial
misses after in-place edits, duplicate contents, growth, size changes and release —
every result against the oracle."""

import numpy as np
import pytest

from oracle import fs_oracle as O

pytestmark = pytest.mark.gpu

import paper_2104_14667_b200 as fs  # noqa: E402
from paper_2104_14667_b200 import _kernels_cuda as K  # noqa: E402


def rand_cells(rng, k, h, w):
    return [((rng.random((h, w)) < rng.uniform(0.1, 0.9)) *
             rng.integers(1, 256, (h, w))).astype(np.uint8) for _ in range(k)]


def surfaces(cells):
    return [fs.RasterSurface(id=f"s{i:03d}", name="", width=c.shape[1], height=c.shape[0],
                             cells=c) for i, c in enumerate(cells)]


def test_drop_in_sequence_uploads_once_and_tracks_edits():
    K.release_stack_cache()
    rng = np.random.default_rng(5)
    h, w, k = 300, 517, 40
    cells = rand_cells(rng, k, h, w)
    s = surfaces(cells)
    grid = fs.accumulate(s)
    assert np.array_equal(grid.counts, O.accumulate(cells, w, h))
    info = K.stack_cache_info()
    assert info["resident"] == k and info["pixels"] == h * w
    g = O.gram(cells)
    sim = O.similarity_from_gram(g)
    ids = [x.id for x in s]
    for _ in range(2):  # hits: same content, nothing new resident
        assert np.array_equal(fs.similarity_matrix(s), sim)
        assert fs.outlier_scores(s) == O.outlier_scores(sim, ids)
        assert fs.cluster_surfaces(s, 0.5) == O.cluster(sim, ids, 0.5)
        assert K.stack_cache_info()["resident"] == k
    # in-place edit of two masks: only they change, results follow the new bytes
    cells[3][:10] = 0
    cells[17][:, :5] = 200
    g = O.gram(cells)
    assert np.array_equal(K.gram_many(cells), g)
    assert np.array_equal(fs.accumulate(s).counts, O.accumulate(cells, w, h))
    # depth-only edit (same wet mask, new bytes): still correct
    cells[5][cells[5] > 0] = 1
    assert np.array_equal(K.gram_many(cells), g)
    # reordered subset with duplicate contents
    sub = [cells[9], cells[2], cells[9], cells[30], cells[2]]
    assert np.array_equal(K.gram_many(sub), O.gram(sub))
    counts = np.arange(h * w, dtype=np.uint32) % 7
    want = counts.copy()
    for c in sub:
        O.accumulate_into(want, c.reshape(-1))
    K.accumulate_many(counts, sub)
    assert np.array_equal(counts, want)


def test_cache_grows_and_switches_raster_size():
    K.release_stack_cache()
    rng = np.random.default_rng(6)
    a = rand_cells(rng, 20, 64, 96)
    assert np.array_equal(K.gram_many(a), O.gram(a))
    b = rand_cells(rng, 70, 64, 96)  # more distinct masks than the capacity
    both = a + b
    assert np.array_equal(K.gram_many(both), O.gram(both))
    assert K.stack_cache_info()["capacity"] >= 90
    c = rand_cells(rng, 5, 33, 17)  # other raster size: the cache is rebuilt
    assert np.array_equal(K.gram_many(c), O.gram(c))
    assert K.stack_cache_info()["pixels"] == 33 * 17
    K.release_stack_cache()
    assert K.stack_cache_info() == {"resident": 0, "capacity": 0, "pixels": 0}
    assert np.array_equal(K.gram_many(c), O.gram(c))


def test_cache_with_concurrent_callers():
    from concurrent.futures import ThreadPoolExecutor

    rng = np.random.default_rng(7)
    sets = [rand_cells(rng, int(rng.integers(1, 30)), 50, 70) for _ in range(8)]
    want = [O.gram(x) for x in sets]
    with ThreadPoolExecutor(6) as pool:
        got = list(pool.map(K.gram_many, sets * 3))
    for i, gg in enumerate(got):
        assert np.array_equal(gg, want[i % len(sets)])
