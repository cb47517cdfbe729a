"""Measured benchmark suites of the transform / transfer path.

API-compatible with the sweep half of ``floodstream.bench``
(/root/reference/pkg/src/floodstream/bench.py:55-126 ``SweepSpec``/``RateMap``,
:129-163 ``BenchReport``, :193-228 ``run_transfer_baseline``, :312-339
``run_transform_sweep``, :342-364 ``render_rate_map``, :456-499
``run_backend_comparison``).  The reference prices the transform and the bus with a
fitted cost model (``transform_time`` / ``transfer_time``, device.py:376-390); here
every number is MEASURED on the B200 with CUDA events: the binarize + bit-pack
transform kernel on a raster already in HBM (``fs_time_transform``) and pinned /
pageable host->device copies (``fs_time_h2d``).  That is the paper's dimension study
(§6, Fig. 9-10) redone on the real kernel.
"""

from __future__ import annotations

import csv
import ctypes as C
import io
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

KIB = 1024
MIB = 1024 * 1024


class BenchError(ValueError):
    pass


@dataclass(frozen=True)
class SweepSpec:
    """The dimension grid of a transform sweep: widths and heights from ``start`` up to
    ``max`` every ``step`` pixels (fs/bench.py:55-76 schema)."""

    start: int
    step: int
    max: int
    repeats: int = 1

    def __post_init__(self) -> None:
        if self.start < 1 or self.step < 1:
            raise BenchError("sweep start and step must be >= 1")
        if self.max < self.start:
            raise BenchError("sweep max must be >= start")
        if self.repeats < 1:
            raise BenchError("sweep repeats must be >= 1")

    @property
    def points(self) -> list[int]:
        return list(range(self.start, self.max + 1, self.step))

    @property
    def cells(self) -> int:
        return len(self.points) ** 2


@dataclass
class RateMap:
    """Measured transform throughput on the sweep grid, in GB/s of uint8 raster; row r is
    height ``start + r*step`` and column c width ``start + c*step``."""

    spec: SweepSpec
    rates: np.ndarray = field(repr=False)

    def __post_init__(self) -> None:
        n = len(self.spec.points)
        if self.rates.shape != (n, n):
            raise BenchError(f"rate grid shape {self.rates.shape} does not match spec ({n}x{n})")

    def to_json(self) -> dict:
        s = self.spec
        return {"spec": {"start": s.start, "step": s.step, "max": s.max, "repeats": s.repeats},
                "rates": [[float(v) for v in row] for row in self.rates]}

    @staticmethod
    def from_json(doc: dict) -> "RateMap":
        return RateMap(spec=SweepSpec(**doc["spec"]),
                       rates=np.asarray(doc["rates"], dtype=np.float64))

    def to_csv(self) -> str:
        """One ``width,height,rate_gbps`` line per grid cell (the reference's calibration CSV
        layout)."""
        buf = io.StringIO()
        wr = csv.writer(buf)
        wr.writerow(["width", "height", "rate_gbps"])
        pts = self.spec.points
        for r, h in enumerate(pts):
            for c, w in enumerate(pts):
                wr.writerow([w, h, repr(float(self.rates[r, c]))])
        return buf.getvalue()


@dataclass
class BenchReport:
    suite: str
    rows: list[dict]
    environment: dict = field(default_factory=dict)
    summary: dict = field(default_factory=dict)
    csv_columns: list[str] = field(default_factory=list)

    def to_json(self) -> dict:
        return {"suite": self.suite, "rows": self.rows, "environment": self.environment,
                "summary": self.summary, "csv_columns": self.csv_columns}

    def to_csv(self) -> str:
        buf = io.StringIO()
        wr = csv.writer(buf)
        wr.writerow(self.csv_columns)
        for row in self.rows:
            wr.writerow([row.get(col, "") for col in self.csv_columns])
        return buf.getvalue()


def transform_time_us(width: int, height: int, *, reps: int = 5, engine: int = -1) -> tuple[float, float]:
    """(mean, min) µs of the device transform of one width x height raster."""
    mean, mn = C.c_double(), C.c_double()
    N.call("fs_time_transform", int(width), int(height), int(reps), int(engine), C.byref(mean),
           C.byref(mn))
    return mean.value, mn.value


def h2d_time_us(nbytes: int, *, reps: int = 5, pinned: bool = True) -> tuple[float, float]:
    mean, mn = C.c_double(), C.c_double()
    N.call("fs_time_h2d", int(nbytes), int(reps), int(bool(pinned)), C.byref(mean), C.byref(mn))
    return mean.value, mn.value


def run_transform_sweep(spec: SweepSpec, *, cell_cap: int = 40_000, reps: int | None = None,
                        engine: int = -1, max_dim: int = 32768) -> RateMap:
    """Measured transform rate at every (width, height) of the sweep (bench.py:312-339):
    rate = w*h / t_us / 1000 GB/s of uint8 raster, t = mean of ``reps`` launches."""
    if spec.cells > cell_cap:
        raise BenchError(f"sweep would cover {spec.cells} cells (cap {cell_cap}); reduce max or "
                         "enlarge step, or raise cell_cap")
    pts = spec.points
    if pts and pts[-1] > max_dim:
        raise BenchError(f"sweep max {pts[-1]} exceeds the supported dimension {max_dim}")
    reps = spec.repeats if reps is None else reps
    n = len(pts)
    rates = np.zeros((n, n), dtype=np.float64)
    for r, h in enumerate(pts):
        for c, w in enumerate(pts):
            t_us, _ = transform_time_us(w, h, reps=reps, engine=engine)
            rates[r, c] = w * h / max(t_us, 1e-3) / 1000.0
    return RateMap(spec=spec, rates=rates)


def render_rate_map(rmap: RateMap, *, scale_gbps: float = 32.0) -> np.ndarray:
    """RGBA pixels of a rate map, bottom-left = (start, start): a 32-step grey ramp over
    [0, scale) and pure blue above (bench.py:342-364 uses scale 32 GB/s — every B200
    cell would be blue, so the scale is a parameter here)."""
    n = len(rmap.spec.points)
    out = np.zeros((n, n, 4), dtype=np.uint8)
    for r in range(n):
        for c in range(n):
            v = float(rmap.rates[r, c]) * 32.0 / scale_gbps
            row = n - 1 - r
            if v > 32.0:
                out[row, c] = (0, 0, 255, 255)
            else:
                k = min(int(v), 31)
                g = round(255.0 * (1.0 - k / 31.0))
                out[row, c] = (g, g, g, 255)
    return out


def run_transfer_baseline(min_bytes: int = 64 * KIB, max_bytes: int = 64 * MIB,
                          step_bytes: int = 64 * KIB, repeats: int = 5, *,
                          pinned: bool = True, points: list[int] | None = None) -> BenchReport:
    """Measured host->device copy rate per size (bench.py:193-228).  ``points`` overrides
    the arithmetic size ladder (a full 64 KiB-step ladder is 1024 copies)."""
    if min_bytes < 1 or step_bytes < 1:
        raise BenchError("sizes and step must be >= 1")
    if min_bytes > max_bytes:
        raise BenchError("min size must not exceed max size")
    if repeats < 1:
        raise BenchError("repeats must be >= 1")
    sizes = points if points is not None else list(range(min_bytes, max_bytes + 1, step_bytes))
    rows = []
    for size in sizes:
        t_us, t_min = h2d_time_us(size, reps=repeats, pinned=pinned)
        rows.append({"bytes": size, "time_us": t_us, "min_us": t_min,
                     "rate_gbps": size / t_us / 1000.0, "repeats": repeats})
    return BenchReport(suite="transfer", rows=rows,
                       environment={"device": "B200", "pinned": pinned, "measured": True},
                       csv_columns=["bytes", "time_us", "rate_gbps"])


def run_backend_comparison(pixels: int = 1 << 20, n_surfaces: int = 16, repeats: int = 3,
                           seed: int = 0) -> BenchReport:
    """bench.py:456-499 on this framework's backends: best-of-repeats wall clock of the
    per-surface ``accumulate_into`` loop (the protocol path, host buffers) and of the
    batched ``accumulate_many`` extension, same seeded inputs (p = 0.5)."""
    from .backends import available_backends

    if pixels < 1 or n_surfaces < 1 or repeats < 1:
        raise BenchError("pixels, surfaces and repeats must all be >= 1")
    rng = np.random.default_rng(seed)
    cells = [(rng.random(pixels) < 0.5).astype(np.uint8) for _ in range(n_surfaces)]
    rows = []
    for name, module in available_backends().items():
        variants = [(name, lambda counts: [module.accumulate_into(counts, c) for c in cells])]
        if hasattr(module, "accumulate_many"):
            variants.append((f"{name}-batched", lambda counts: module.accumulate_many(counts, cells)))
        for label, fn in variants:
            best = float("inf")
            for _ in range(repeats):
                counts = np.zeros(pixels, dtype=np.uint32)
                t0 = time.perf_counter()
                fn(counts)
                best = min(best, time.perf_counter() - t0)
            rows.append({"backend": label, "pixels": pixels, "surfaces": n_surfaces,
                         "best_s": best, "mpix_per_s": pixels * n_surfaces / best / 1e6})
    return BenchReport(suite="backends", rows=rows,
                       environment={"pixels": pixels, "surfaces": n_surfaces, "repeats": repeats},
                       csv_columns=["backend", "pixels", "surfaces", "best_s", "mpix_per_s"])


# the paper's image sizes (bench.py:41-46 of the reference)
DIMS = {"2k": (1856, 2208), "4k": (3712, 4416), "8k": (7424, 8832), "16k": (14848, 17664)}
VARIANTS = ("1b-initial", "2b-initial", "1b-final", "2b-final")


def resolve_dims(entry) -> tuple[str, int, int]:
    """Normalise an image-size argument — a named size ('2k', '4k', '8k'), a 'WxH'
    string or a (w, h) pair — to (label, width, height) (fs/bench.py:167-181)."""
    if isinstance(entry, str):
        if entry in DIMS:
            return (entry,) + DIMS[entry]
        if "x" in entry:
            try:
                w_s, h_s = entry.lower().split("x", 1)
                return entry, int(w_s), int(h_s)
            except ValueError:
                pass
        raise BenchError(f"unknown image size {entry!r}")
    w, h = entry
    return f"{w}x{h}", int(w), int(h)


def run_dual_buffer_suite(dims_list, n_list, repeats: int = 3, *, pool: int = 8,
                          with_kernel: bool = True) -> BenchReport:
    """The four upload strategies MEASURED on the device (the reference simulates them,
    bench.py:231-309; the paper's Figs. 5-8): for each size, strategy and N, N rasters
    (cycled from a pool of ``pool`` pinned host rasters) stream through the variant's
    event DAG — H2D, bit-pack transform, per-item accumulate — and the device clock
    gives the total.  efficiency = N x (isolated pinned copy time) / total, the paper's
    definition; ``closed_form_us`` is the §7.1 model evaluated on the
    measured per-item c/m/p (streaming.closed_form_times)."""
    from .ensemble import DeviceEnsemble
    from .streaming import closed_form_times
    from .synth import synth_cells_gpu

    if not dims_list or not n_list:
        raise BenchError("dims and n lists must be nonempty")
    if repeats < 1:
        raise BenchError("repeats must be >= 1")
    rows = []
    for entry in dims_list:
        label, w, h = resolve_dims(entry)
        P = w * h
        bufs = [N.PinnedBuffer((h, w)) for _ in range(pool)]
        try:
            for i, b in enumerate(bufs):
                synth_cells_gpu(w, h, i, seed=2104, members=4, eps=0.05, out=b.array)
            c_iso = h2d_time_us(P, reps=5, pinned=True)[1]
            with DeviceEnsemble(w, h, 2) as ens:
                for variant in VARIANTS:
                    for n in n_list:
                        if n < 1:
                            raise BenchError("N values must be >= 1")
                        rasters = [bufs[i % pool].array for i in range(n)]
                        ens.stream(rasters[:min(n, 4)], variant=variant, with_kernel=with_kernel,
                                   slot_wrap=2)  # warm-up
                        samples, last = [], None
                        for _ in range(repeats):
                            last = ens.stream(rasters, variant=variant, with_kernel=with_kernel,
                                              slot_wrap=2)
                            samples.append(last.total_us)
                        total = float(np.median(samples))
                        t_dual, t_single = closed_form_times(last.copy_us, last.xform_us,
                                                             last.kernel_us)
                        rows.append({"dims": label, "width": w, "height": h, "variant": variant,
                                     "n": n, "total_us": total,
                                     "rate_gbps": n * P / total / 1000.0,
                                     "efficiency": n * c_iso / total,
                                     "isolated_copy_us": c_iso,
                                     "mean_copy_us": float(np.mean(last.copy_us)),
                                     "mean_xform_us": float(np.mean(last.xform_us)),
                                     "mean_kernel_us": float(np.mean(last.kernel_us)),
                                     "mean_host_us": float(np.mean(last.host_us)),
                                     "closed_form_us": t_dual if variant.startswith("2b") else t_single,
                                     "samples_us": samples})
        finally:
            for b in bufs:
                b.free()
    return BenchReport(suite="dual", rows=rows,
                       environment={"device": "B200", "measured": True, "repeats": repeats,
                                    "pool": pool, "with_kernel": with_kernel},
                       csv_columns=["variant", "n", "width", "height", "total_us", "rate_gbps",
                                    "efficiency"])
