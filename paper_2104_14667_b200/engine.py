"""Interactive recompute over a device-resident working set.

The reference service recomputes its snapshot on every working-set change
(``AnalyticsEngine._compute``, fs/service.py:143-175): it re-reads and re-decodes
EVERY selected surface from disk (fs/store.py:156-170), streams them through
``run_stream``, then builds the histogram, the composite PNG and the grid digest;
``/clusters`` and ``/outliers`` (fs/service.py:289-307) decode everything again and
run the pairwise path.  Here the bit-packed masks stay in HBM, keyed by surface id
(ids are content-addressed: ``_surface_id(name, payload)``, fs/store.py:107-123), so a
working-set change uploads only the surfaces that are not resident yet and every
recompute reads HBM only:

* ``SlotMap``          — which surface occupies which ensemble slot (pure host logic);
* ``ResidentEngine``   — the device cache + one recompute: counts, histogram,
                         composite, Gram -> similarity / outliers / clusters;
* ``AnalyticsEngine``  — a drop-in for the reference's recompute worker (same
                         ``snapshot`` / ``wait_snapshot`` / ``schedule`` / ``stop``)
                         over any store exposing ``snapshot_state``, ``surface`` and
                         ``dims``.

The snapshot's grid digest (sha256 over the uint32 counts, analytics.py:57-59) and
PNG (Pillow, rasters.py:120-125) are inherently sequential host work; they are
computed lazily, on first access, from the exact device results.
"""

from __future__ import annotations

import hashlib
import threading
import time

import numpy as np

from .analytics import (
    AccumulationGrid,
    CompositeImage,
    cluster_from_similarity,
    outliers_from_similarity,
    similarity_from_gram,
)
from .rasters import rgba_to_png_bytes


class SlotMap:
    """Surface id -> slot of a fixed-capacity ensemble.

    ``plan(ids)`` keeps resident ids in place, evicts ids that are not wanted when
    room is needed (least recently used first), and returns the placements for the
    missing ones, grouped in runs of consecutive slots (one streamed upload each).
    """

    def __init__(self, capacity: int):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self.capacity = int(capacity)
        self.slot_of: dict[str, int] = {}
        self._last_use: dict[str, int] = {}
        self._tick = 0

    def resident(self) -> list[str]:
        return sorted(self.slot_of, key=self.slot_of.get)

    def plan(self, ids: list[str]) -> tuple[list[tuple[int, list[str]]], list[str]]:
        """(runs of (first_slot, [ids...]) to upload, evicted ids) for working set ids."""
        want = list(dict.fromkeys(ids))
        if len(want) > self.capacity:
            raise ValueError(f"working set of {len(want)} exceeds capacity {self.capacity}")
        self._tick += 1
        wanted = set(want)
        missing = [s for s in want if s not in self.slot_of]
        used = set(self.slot_of.values())
        free = [q for q in range(self.capacity) if q not in used]
        evicted: list[str] = []
        if len(free) < len(missing):
            victims = sorted((s for s in self.slot_of if s not in wanted),
                             key=lambda s: self._last_use.get(s, 0))
            for s in victims[:len(missing) - len(free)]:
                free.append(self.slot_of.pop(s))
                self._last_use.pop(s, None)
                evicted.append(s)
            free.sort()
        placed = dict(zip(missing, free))
        self.slot_of.update(placed)
        for s in want:
            self._last_use[s] = self._tick
        runs: list[tuple[int, list[str]]] = []
        for sid, q in sorted(placed.items(), key=lambda kv: kv[1]):
            if runs and runs[-1][0] + len(runs[-1][1]) == q:
                runs[-1][1].append(sid)
            else:
                runs.append((q, [sid]))
        return runs, evicted

    def slots(self, ids: list[str]) -> list[int]:
        return [self.slot_of[s] for s in ids]

    def drop(self, sid: str) -> None:
        self.slot_of.pop(sid, None)
        self._last_use.pop(sid, None)


class EngineSnapshot:
    """One recompute of the working set (fields of the reference's service Snapshot,
    fs/service.py:53-73, plus the pairwise products).  The per-pixel maps stay in
    device memory until first read (``counts``, ``rgba``); the grid digest and the PNG
    are computed on first access."""

    def __init__(self, version: int, ids: list[str], width: int, height: int, n_inputs: int,
                 histogram: list[int], *, d_counts=None, d_rgba=None, gram=None,
                 report: dict | None = None):
        self.version, self.ids = version, ids
        self.width, self.height, self.n_inputs = width, height, n_inputs
        self.histogram = histogram
        self.gram = gram
        self.similarity = None
        self.outliers = None
        self.clusters = None
        self.report = report
        self._d_counts, self._d_rgba = d_counts, d_rgba
        self._counts = self._rgba = None
        self._digest = self._png = None
        self._lock = threading.Lock()

    @property
    def counts(self) -> np.ndarray | None:
        with self._lock:
            if self._counts is None and self._d_counts is not None:
                self._counts = self._d_counts.cpu().numpy().view(np.uint32).reshape(
                    self.height, self.width)
                self._d_counts = None
            return self._counts

    @property
    def rgba(self) -> np.ndarray | None:
        with self._lock:
            if self._rgba is None and self._d_rgba is not None:
                self._rgba = self._d_rgba.cpu().numpy().reshape(self.height, self.width, 4)
                self._d_rgba = None
            return self._rgba

    @property
    def grid(self) -> AccumulationGrid:
        c = self.counts
        if c is None:
            return AccumulationGrid.empty(self.width, self.height)
        return AccumulationGrid._from_device(self.width, self.height, self.n_inputs, c)

    @property
    def grid_digest(self) -> str:
        if self._digest is None:
            c = self.counts
            if c is None:
                self._digest = AccumulationGrid.empty(self.width, self.height).digest()
            else:
                head = f"{self.width}x{self.height}:{self.n_inputs}:".encode()
                h = hashlib.sha256(head)
                h.update(memoryview(np.ascontiguousarray(c)).cast("B"))
                self._digest = h.hexdigest()
        return self._digest

    @property
    def composite(self) -> CompositeImage | None:
        r = self.rgba
        if r is None:
            return None
        return CompositeImage(width=self.width, height=self.height, pixels=r)

    @property
    def composite_png(self) -> bytes:
        if self._png is None:
            r = self.rgba
            if not (self.width and self.height):  # no dims yet: the 1x1 placeholder
                self._png = rgba_to_png_bytes(np.zeros((1, 1, 4), np.uint8))
            elif r is None:  # empty working set: transparent composite
                self._png = rgba_to_png_bytes(np.zeros((self.height, self.width, 4), np.uint8))
            else:
                self._png = rgba_to_png_bytes(r)
        return self._png

    def to_json(self) -> dict:
        return {
            "version": self.version,
            "n_inputs": self.n_inputs,
            "grid_digest": self.grid_digest,
            "histogram": self.histogram,
            "composite_url": f"/composite.png?version={self.version}",
            "report": self.report,
        }


class ResidentEngine:
    """Bit-packed working set resident in HBM, keyed by surface id."""

    def __init__(self, width: int, height: int, capacity: int, *, device: int | None = None,
                 engine: str = "auto", tau: float = 0.8):
        from .ensemble import DeviceEnsemble

        import torch

        self.width, self.height = int(width), int(height)
        self.ens = DeviceEnsemble(width, height, capacity, device=device)
        self.dev = torch.device("cuda", self.ens.device)
        # the ensemble computes on torch's current stream of its device, so the
        # caching allocator orders the reuse of snapshot buffers after the kernels
        self.ens.use_stream(torch.cuda.current_stream(self.dev).cuda_stream)
        self.slots = SlotMap(capacity)
        self.engine = engine
        self.tau = float(tau)
        self._lock = threading.RLock()

    def close(self) -> None:
        self.ens.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def update(self, ids: list[str], load) -> dict:
        """Make ``ids`` resident; ``load(sid) -> RasterSurface`` is called only for
        ids that are not resident yet.  Returns what moved and the measured upload."""
        with self._lock:
            runs, evicted = self.slots.plan(ids)
            uploaded, upload_us = [], 0.0
            try:
                for first, run in runs:
                    surfaces = [load(s) for s in run]
                    for s in surfaces:
                        if (s.width, s.height) != (self.width, self.height):
                            raise ValueError(f"surface {s.id!r} is {s.width}x{s.height}, "
                                             f"expected {self.width}x{self.height}")
                    st = self.ens.upload(surfaces, first=first)
                    upload_us += st.total_us
                    uploaded += run
            except Exception:
                for _, run in runs:  # failed placements must not look resident
                    for s in run:
                        if s not in uploaded:
                            self.slots.drop(s)
                raise
            return {"uploaded": uploaded, "evicted": evicted,
                    "reused": len(set(ids)) - len(uploaded), "upload_us": upload_us}

    def compute(self, version: int, ids: list[str], load=None, *, pairwise: bool = True,
                tau: float | None = None) -> EngineSnapshot:
        """One recompute of working set ``ids`` (in order): counts, histogram,
        composite and (``pairwise``) the Gram, similarity, outliers and clusters."""
        import torch

        tau = self.tau if tau is None else tau
        with self._lock:
            t0 = time.perf_counter()
            moved = self.update(ids, load) if load is not None else None
            ids = list(dict.fromkeys(ids))
            missing = [s for s in ids if s not in self.slots.slot_of]
            if missing:
                raise KeyError(f"surfaces not resident (pass a loader): {missing[:5]}")
            if not ids:
                return EngineSnapshot(version, [], self.width, self.height, 0,
                                      [self.width * self.height], report={"uploaded": 0})
            # the kernels read slots in ascending order (a contiguous run needs no
            # gather); the Gram is permuted back to working-set order on the host
            sl = np.asarray(self.slots.slots(ids), dtype=np.int64)
            order = np.argsort(sl, kind="stable")
            k = len(ids)
            nb = k + 1
            d_counts = torch.empty(self.width * self.height, dtype=torch.int32, device=self.dev)
            d_rgba = torch.empty(self.width * self.height * 4, dtype=torch.uint8, device=self.dev)
            d_part = torch.empty(nb + (k * k if pairwise else 0), dtype=torch.int64,
                                 device=self.dev)
            _, _, _, _, fused = self.ens.products(
                sl[order], engine=self.engine, gram=pairwise, out_counts=d_counts.data_ptr(),
                out_rgba=d_rgba.data_ptr(), out_bins=d_part.data_ptr(),
                out_gram=d_part.data_ptr() + nb * 8 if pairwise else None, device_outputs=True)
            kernel_ms = self.ens.kernel_ms("recompute")  # waits for the recompute
            part = d_part.cpu().numpy()
        g = None
        if pairwise:
            inv = np.argsort(order)
            g = part[nb:].reshape(k, k)[np.ix_(inv, inv)]
        snap = EngineSnapshot(version, ids, self.width, self.height, k,
                              [int(x) for x in part[:nb]], d_counts=d_counts, d_rgba=d_rgba,
                              gram=g)
        if pairwise:
            snap.similarity = similarity_from_gram(g)
            snap.outliers = outliers_from_similarity(snap.similarity, ids) if k >= 2 else None
            snap.clusters = cluster_from_similarity(snap.similarity, ids, tau)
        snap.report = {
            "uploaded": 0 if moved is None else len(moved["uploaded"]),
            "evicted": 0 if moved is None else len(moved["evicted"]),
            "upload_us": 0.0 if moved is None else moved["upload_us"],
            "recompute_ms": kernel_ms, "fused": fused,
            "wall_ms": (time.perf_counter() - t0) * 1e3,
            "makespan_source": "measured",
        }
        return snap


class AnalyticsEngine:
    """Drop-in for the reference's recompute worker (fs/service.py:76-175) over a
    device-resident working set: ``schedule()`` after a working-set mutation, one
    daemon thread recomputes, ``snapshot()`` / ``wait_snapshot()`` read results."""

    def __init__(self, store, *, capacity: int | None = None, device: int | None = None,
                 engine: str = "auto", tau: float = 0.8, pairwise: bool = True):
        self.store = store
        self.capacity = capacity
        self.device = device
        self.engine_kind = engine
        self.tau = tau
        self.pairwise = pairwise
        self._resident: ResidentEngine | None = None
        self._cond = threading.Condition()
        self._dirty = False
        self._stopped = False
        self._snapshot = self._compute()
        self._thread = threading.Thread(target=self._worker, name="floodstream-recompute",
                                        daemon=True)
        self._thread.start()

    def stop(self) -> None:
        with self._cond:
            self._stopped = True
            self._cond.notify_all()
        self._thread.join(timeout=5)
        if self._resident is not None:
            self._resident.close()
            self._resident = None

    def schedule(self) -> None:
        with self._cond:
            self._dirty = True
            self._cond.notify_all()

    def _worker(self) -> None:
        while True:
            with self._cond:
                self._cond.wait_for(lambda: self._dirty or self._stopped)
                if self._stopped:
                    return
                self._dirty = False
            snap = self._compute()
            with self._cond:
                if snap.version >= self._snapshot.version:
                    self._snapshot = snap
                    self._cond.notify_all()

    def snapshot(self) -> EngineSnapshot:
        with self._cond:
            return self._snapshot

    def wait_snapshot(self, min_version: int, timeout_s: float) -> EngineSnapshot | None:
        with self._cond:
            ok = self._cond.wait_for(lambda: self._snapshot.version > min_version or self._stopped,
                                     timeout=timeout_s)
            if not ok or self._snapshot.version <= min_version:
                return None
            return self._snapshot

    def _compute(self) -> EngineSnapshot:
        version, ids = self.store.snapshot_state()
        dims = self.store.dims()
        if dims is None:
            return EngineSnapshot(version, [], 0, 0, 0, [0])
        w, h = dims
        n = len(set(ids))
        if (self._resident is None or (self._resident.width, self._resident.height) != (w, h)
                or n > self._resident.slots.capacity):
            if self._resident is not None:
                self._resident.close()
            cap = max(self.capacity or 0, 64, 2 * n)
            self._resident = ResidentEngine(w, h, cap, device=self.device,
                                            engine=self.engine_kind, tau=self.tau)
        return self._resident.compute(version, ids, self.store.surface, pairwise=self.pairwise)
