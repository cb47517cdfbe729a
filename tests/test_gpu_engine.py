"""GPU tests of the resident working-set engine (the service recompute path,
fs/service.py:143-175 and :289-307) against the oracle: only new surfaces are
loaded/uploaded on a working-set change, and every snapshot field — counts, histogram,
grid digest, composite PNG bytes, outliers, clusters — equals the reference formulas
on the same working set."""

import threading

import numpy as np
import pytest

from oracle import fs_oracle as O

pytestmark = pytest.mark.gpu

from paper_2104_14667_b200.engine import AnalyticsEngine, ResidentEngine  # noqa: E402
from paper_2104_14667_b200.rasters import RasterSurface, rgba_to_png_bytes  # noqa: E402
from paper_2104_14667_b200.synth import synth_cells  # noqa: E402


class FakeStore:
    """In-memory stand-in for SurfaceStore (fs/store.py:196-221): versioned working set,
    surface(sid) decodes on demand (counted)."""

    def __init__(self, w, h, n):
        self.w, self.h = w, h
        self.cells = {f"id{i:03d}": synth_cells(w, h, i, members=4, eps=0.05) for i in range(n)}
        self.version = 0
        self.ws: list[str] = []
        self.loads = 0
        self.lock = threading.Lock()

    def snapshot_state(self):
        with self.lock:
            return self.version, list(self.ws)

    def set_working_set(self, ids):
        with self.lock:
            self.ws = list(dict.fromkeys(ids))
            self.version += 1
            return self.version

    def dims(self):
        return (self.w, self.h)

    def surface(self, sid):
        self.loads += 1
        return RasterSurface(id=sid, name=sid, width=self.w, height=self.h, cells=self.cells[sid])


def _check(snap, store, ids, tau=0.8):
    cells = [store.cells[s] for s in ids]
    w, h = store.w, store.h
    counts = O.accumulate(cells, w, h)
    assert snap.n_inputs == len(ids)
    assert np.array_equal(snap.counts, counts)
    assert snap.histogram == O.overlap_counts(counts.reshape(-1), len(ids)).tolist()
    assert snap.grid_digest == O.grid_digest(w, h, len(ids), counts)
    assert snap.composite_png == rgba_to_png_bytes(O.composite(counts, len(ids)))
    sim = O.similarity_from_gram(O.gram(cells))
    assert np.array_equal(snap.similarity, sim)
    assert snap.clusters == O.cluster(sim, ids, tau)
    assert snap.outliers == O.outlier_scores(sim, ids)


def test_resident_engine_uploads_only_new_surfaces():
    store = FakeStore(300, 200, 12)
    ids_all = sorted(store.cells)
    with ResidentEngine(300, 200, 8) as eng:
        ws1 = ids_all[:6]
        s1 = eng.compute(1, ws1, store.surface)
        assert store.loads == 6 and s1.report["uploaded"] == 6
        _check(s1, store, ws1)
        ws2 = [ids_all[5], ids_all[2], ids_all[7], ids_all[0]]  # reorder + one new
        s2 = eng.compute(2, ws2, store.surface)
        assert store.loads == 7 and s2.report["uploaded"] == 1
        _check(s2, store, ws2)
        ws3 = ids_all[4:12]  # needs evictions (capacity 8)
        s3 = eng.compute(3, ws3, store.surface)
        _check(s3, store, ws3)
        assert s3.report["evicted"] >= 1
        s4 = eng.compute(4, ws3, store.surface)  # no change: nothing moves
        assert s4.report["uploaded"] == 0 and s4.grid_digest == s3.grid_digest
        e = eng.compute(5, [], store.surface)
        assert e.histogram == [300 * 200] and e.n_inputs == 0
        assert e.grid_digest == O.grid_digest(300, 200, 0, np.zeros((200, 300), np.uint32))


def test_analytics_engine_worker_follows_the_store():
    store = FakeStore(128, 96, 10)
    ids = sorted(store.cells)
    store.set_working_set(ids[:4])
    eng = AnalyticsEngine(store, capacity=16)
    try:
        snap = eng.snapshot()
        assert snap.version == 1
        _check(snap, store, ids[:4])
        v = store.set_working_set(ids[3:9])
        eng.schedule()
        snap = eng.wait_snapshot(v - 1, timeout_s=30)
        assert snap is not None and snap.version == v
        _check(snap, store, ids[3:9])
        assert eng.wait_snapshot(v, timeout_s=0.2) is None  # nothing newer
        j = snap.to_json()
        assert j["version"] == v and j["n_inputs"] == 6 and j["histogram"] == snap.histogram
    finally:
        eng.stop()


def test_ingest_files_stream_into_ensemble(tmp_path):
    """PGM (read straight into pinned staging) and PNG files decoded one batch ahead of
    the 2b-final upload reproduce the oracle's maps and Gram."""
    import io as _io

    from PIL import Image

    from paper_2104_14667_b200.ensemble import DeviceEnsemble
    from paper_2104_14667_b200.ingest import stream_files
    from paper_2104_14667_b200.rasters import write_pgm

    w, h, k = 333, 129, 11
    cells = [synth_cells(w, h, i, members=3, eps=0.05) for i in range(k)]
    sources = []
    for i, c in enumerate(cells):
        if i % 3 == 2:
            b = _io.BytesIO()
            Image.fromarray(c, "L").save(b, format="PNG")
            sources.append(b.getvalue())
        else:
            p = tmp_path / f"s{i}.pgm"
            p.write_bytes(write_pgm(c))
            sources.append(str(p))
    with DeviceEnsemble(w, h, k + 2) as ens:
        rep = stream_files(ens, sources, first=2, batch=4)
        c, b, r = ens.overlap(list(range(2, k + 2)))
        g = ens.gram(list(range(2, k + 2)), engine="tc-f4")
    assert rep["files"] == k
    want = O.accumulate(cells, w, h)
    assert np.array_equal(c, want)
    assert np.array_equal(g, O.gram(cells))


def test_resident_engine_beyond_one_panel():
    """A working set of 300 surfaces (> one 256-mask panel: unfused overlap + CTA-pair
    Gram tiles) in shuffled order, then a partial swap."""
    store = FakeStore(96, 40, 320)
    ids_all = sorted(store.cells)
    rng = np.random.default_rng(3)
    with ResidentEngine(96, 40, 310) as eng:
        ws = [ids_all[i] for i in rng.permutation(300)]
        _check(eng.compute(1, ws, store.surface), store, ws)
        ws2 = ws[20:] + ids_all[300:310]
        s2 = eng.compute(2, ws2, store.surface)
        assert s2.report["uploaded"] == 10
        _check(s2, store, ws2)


@pytest.mark.parametrize("seed", range(4))
def test_resident_engine_random_working_sets(seed):
    """A sequence of random working sets (growing, shrinking, reordered, evicting) on a
    small-capacity engine: every snapshot equals the reference formulas."""
    rng = np.random.default_rng(77 + seed)
    store = FakeStore(64, 48, 40)
    ids_all = sorted(store.cells)
    with ResidentEngine(64, 48, 24) as eng:
        for v in range(6):
            n = int(rng.integers(1, 25))
            ws = [ids_all[i] for i in rng.choice(40, n, replace=False)]
            snap = eng.compute(v, ws, store.surface)
            if n >= 2:
                _check(snap, store, ws)
            else:
                assert snap.histogram == O.overlap_counts(
                    O.accumulate([store.cells[ws[0]]], 64, 48).reshape(-1), 1).tolist()
