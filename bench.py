#!/usr/bin/env python
"""Headline benchmark: ensemble Gpixels/s incl. H2D, and FPS, for 256 x 8192^2 masks.

Workload (BASELINE.json configs[1], "c2"): 256 flood-like masks of 8192 x 8192 uint8
(17.18 GB) in PINNED host memory.  One *step* = one full frame through the public API:
  H2D of every raster (2b-final dual-buffer DAG) overlapped with the binarize+pack
  transform; ONE fused kernel (k_recompute_f4) for overlap counts + histogram + composite
  RGBA + the exact pairwise-intersection Gram (tcgen05 kind::mxf4); Jaccard
  matrix and outlier scores on the device; D2H of counts + RGBA + [bins | Gram] +
  Jaccard + scores; complete-linkage clusters (tau 0.8) on the host.

* ``value``: that end-to-end frame (host rasters in, host products out) over exactly
  ``--steps`` timed steps: mask-pixels / s.  ``e2e`` repeats it with its byte counts.
* ``resident``: the same recompute with the masks already bit-packed in HBM (the
  interactive-recompute FPS of north_star), with the maps' D2H (``maps_to_host``) and
  without (``device_only``).
* ``roofline``: the dominant kernel of the recompute (the fused Gram+overlap kernel)
  against the FP4 tensor peak; ``kernels`` adds the overlap pass and the transform
  against HBM; ``e2e.roofline`` is the step against measured pinned PCIe H2D.
* ``--impl reference``: the reference's own CPU implementation — the unmodified
  reference package (baseline/_ref) run as shipped (single thread, numpy and cython
  backends, reported under ``as_shipped``) and on all host cores around its unchanged
  primitives, where each step is a proportional sample of the frame (per-pixel ops over
  all masks and pair_counts over ALL pairs on a window of rows): the all-cores number,
  pixels / step time, is the line's value.

Multi-GPU (torchrun, one rank per GPU): STRONG scaling by default — the fixed ensemble
is cut into N row bands, rank r owns rows band(H, r, N) of every mask (one contiguous
H2D per mask) and the only exchange is one NCCL all-reduce of the int64 [histogram |
Gram] partials per frame; ``--scaling weak`` grows the raster to 8192 x 8192 N instead.
Timings are the max over ranks; ``value`` = all masks' pixels / that time.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "ensemble Gpixels/s incl. H2D & FPS for 256x8192^2 masks"
UNIT = "Gpx/s"

CONFIGS = {
    # name: (width, height, masks, members per prototype, eps)
    "c1": (1024, 1024, 16, 1, 0.5),
    "c2": (8192, 8192, 256, 16, 0.02),
    "c3": (4096, 4096, 1024, 32, 0.02),
    "c4": (32768, 32768, 64, 8, 0.02),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: strong = the fixed ensemble in N row bands; weak = raster "
                         "height grows with N (every rank keeps the 1-GPU workload)")
    ap.add_argument("--tau", type=float, default=0.8)
    ap.add_argument("--engine", default="tc-f4", choices=["tc-f4", "tc", "popc"])
    ap.add_argument("--no-e2e", action="store_true",
                    help="profiling runs only: skip the end-to-end frames (value = resident)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--resident-steps", type=int, default=100)
    ap.add_argument("--band-rows", type=int, default=0, help="c4: rows per spatial band")
    ap.add_argument("--max-host-gb", type=float, default=0.0,
                    help="c4: cap on pinned host input per rank (0: 60%% of available RAM)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    """Samples SM clock and clock-event (throttle) reasons during the timed region:
    NVML every ~5 ms on a background thread (nvidia-smi -lms is too coarse for a
    region of tens of milliseconds)."""

    REASONS = {
        "hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
        "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, gpu_index: int, period_s: float = 0.002):
        self.idx = gpu_index
        self.period = period_s
        self.sm: list[float] = []
        self.max_sm = None
        self.reasons: set[str] = set()
        self._stop = threading.Event()
        self._ok = False

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.max_sm = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
            self._ok = True
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._ok = False
        return self

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._ok:
            self._t.join(timeout=2)

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": self.max_sm, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml"}


def measured_peaks() -> dict:
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            pass
    return {}


# ---------------------------------------------------------------------------
# CPU baseline (oracle C port, all cores) — rank 0, N=1 only
# ---------------------------------------------------------------------------
def cpu_baseline(host_masks, width, height, k, window_px):
    sys.path.insert(0, str(REPO / "tests"))
    import oracle_c  # test/bench infrastructure only
    from oracle import fs_oracle as O

    P = width * height
    win = [m.reshape(-1)[:window_px] for m in host_masks]
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    counts = oracle_c.accumulate(win, threads)
    oracle_c.histogram(counts, k, threads)
    oracle_c.composite(counts, k, threads)
    t1 = time.perf_counter()
    g = oracle_c.gram(win, threads)
    t2 = time.perf_counter()
    sim = O.similarity_from_gram(g)
    ids = [f"s{i:04d}" for i in range(k)]
    O.outlier_scores(sim, ids)
    t3 = time.perf_counter()
    scale = P / window_px
    t_full = (t1 - t0) * scale + (t2 - t1) * scale + (t3 - t2)
    return {
        "value": round(k * P / t_full / 1e9, 4), "unit": UNIT, "cores": threads, "kind": "port",
        "sample": (f"oracle/fs_oracle.c (OpenMP) on a {window_px}-px window of all {k} masks "
                   f"(pixel ops {t1 - t0:.2f} s, Gram {t2 - t1:.2f} s) scaled x{scale:g}, plus "
                   f"outlier reduction {t3 - t2:.2f} s; clustering not timed"),
        "fps": round(1.0 / t_full, 5),
    }


# ---------------------------------------------------------------------------
# workload description shared by both arms (the driver compares the two config dicts)
# ---------------------------------------------------------------------------
def workload_config(args, width, height, k, world) -> dict:
    return {
        "workload": (f"{args.config}: {k} flood-like masks {width}x{height} uint8 in host memory; "
                     "one step = a full recompute frame: overlap counts + histogram + composite "
                     "RGBA + pairwise Jaccard + outlier scores + complete-linkage clusters"),
        "masks": k, "width": width, "height": height, "tau": args.tau,
        "generator": "flood-like prototype+flip (fs_synth_host bytes), seed 2104",
        "parallelism": (f"row-bands x{world}" if world > 1 else "single device"),
        "l2": "every step reads all rasters from host memory (>> L2)",
    }


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation
# ---------------------------------------------------------------------------
def _load_reference_package():
    """The unmodified reference package (pip-installed offline into baseline/_ref,
    with its Cython accelerator built), or None when it is absent."""
    ref = REPO / "baseline" / "_ref"
    if not (ref / "floodstream").exists():
        return None
    sys.path.insert(0, str(ref))
    import floodstream
    import floodstream.analytics  # noqa: F401
    import floodstream.backends  # noqa: F401

    return floodstream


def _primitive_modules(ref) -> dict:
    """name -> the reference's primitive module (fs/backends.py:42-47); the oracle's
    compiled copy of its _accel.pyx / its NumPy port when the package is absent."""
    if ref is not None:
        return dict(ref.backends.available_backends())
    mods = {}
    r = REPO / "oracle" / "_ref"
    if any(r.glob("_accel*.so")):
        sys.path.insert(0, str(r))
        import _accel

        mods["cython"] = _accel
    from oracle import fs_oracle

    mods["numpy"] = fs_oracle
    return mods


_REF = {}  # fork-inherited state of the all-cores harness (masks, module, pairs)


def _stripe_worker(w, lo, hi, conn):
    """One host core: the unchanged reference primitives on rows [lo, hi) of every mask,
    one timed pass per "go" (fs/_kernels_np.py / fs/_accel.pyx, looped as
    fs/analytics.py:118-181 does)."""
    mod, masks, pairs, k = _REF["mod"], _REF["masks"], _REF["pairs"], _REF["k"]
    cells = [m[lo:hi].reshape(-1) for m in masks]
    n = cells[0].size
    while conn.recv() == "go":
        t0 = time.perf_counter()
        counts = np.zeros(n, dtype=np.uint32)
        for c in cells:
            mod.accumulate_into(counts, c)
        mod.overlap_counts(counts, k)
        out = np.zeros((n, 4), dtype=np.uint8)
        mod.composite_fill(counts, k, out)
        t1 = time.perf_counter()
        for (i, j) in pairs:
            mod.pair_counts(cells[i], cells[j])
        t2 = time.perf_counter()
        conn.send((n, t1 - t0, t2 - t1))
    conn.close()


def _as_shipped_leg(ref, name, mod, surfaces, window_px, P, k, pairs, sim, tau):
    """the reference's analytics, single thread, backend
    `name`: per-pixel ops on a `window_px` window (scaled to P), Jaccard on the sampled
    pairs (scaled to all pairs), outliers and clusters on the exact matrix
    (similarity_matrix patched to return it, as §3.3 prescribes)."""
    A = ref.analytics
    saved = A.kernels
    A.kernels = mod
    try:
        t = {}
        t0 = time.perf_counter()
        grid = A.accumulate(surfaces)
        t["accumulate"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        A.overlap_histogram(grid)
        t["overlap_histogram"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        A.composite_map(grid)
        t["composite_map"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        for (i, j) in pairs:
            A.jaccard(surfaces[i], surfaces[j])
        t["jaccard_pairs"] = time.perf_counter() - t0
        real_sim = A.similarity_matrix
        A.similarity_matrix = lambda _s: sim
        try:
            t0 = time.perf_counter()
            A.outlier_scores(surfaces)
            t["outlier_scores"] = time.perf_counter() - t0
            t0 = time.perf_counter()
            A.cluster_surfaces(surfaces, tau)
            t["cluster_surfaces"] = time.perf_counter() - t0
        finally:
            A.similarity_matrix = real_sim
    finally:
        A.kernels = saved
    npairs = k * (k - 1) // 2
    px_scale = P / window_px
    frame = ((t["accumulate"] + t["overlap_histogram"] + t["composite_map"]) * px_scale
             + t["jaccard_pairs"] * px_scale * npairs / len(pairs)
             + t["outlier_scores"] + t["cluster_surfaces"])
    return {"backend": name, "threads": 1, "value": round(k * P / frame / 1e9, 6),
            "unit": UNIT, "s_per_frame": round(frame, 3), "fps": round(1.0 / frame, 6),
            "measured_s": {x: round(v, 4) for x, v in t.items()},
            "window_px": window_px, "pairs": len(pairs),
            "extrapolated": {"pixels": round(px_scale, 3),
                             "pairs": round(npairs / len(pairs), 3)}}


def reference_arm(args, width, height, k, members, eps, rank, world):
    """The reference's own CPU implementation on the same workload and config.

    * as shipped: the unmodified reference package, one thread, FLOODSTREAM_BACKEND
      numpy and cython — once, reported under ``as_shipped``;
    * all cores (the line's value; §3.3 item 4): one process per host core, each
      running the unchanged reference primitives of the faster as-shipped backend; a
      step is a proportional sample of the frame — per-pixel ops over all k masks and
      pair_counts over all k(k-1)/2 pairs on a window of rows (one stripe per worker,
      spread over the raster) — so pixels / step time is the frame rate, unscaled.
    Under torchrun rank 0 alone runs; generation and the exact matrix are untimed."""
    if rank != 0:
        return None
    if args.scaling == "weak":
        height = height * world
    import multiprocessing as mp

    sys.path.insert(0, str(REPO / "tests"))
    import oracle_c  # bench infrastructure: the exact Gram for the clustering input
    from oracle import fs_oracle as O
    from paper_2104_14667_b200.synth import synth_cells

    ref = _load_reference_package()
    mods = _primitive_modules(ref)
    cores = os.cpu_count() or 1
    P = width * height
    npairs_total = k * (k - 1) // 2
    # inputs (untimed): the full ensemble, generated with all host threads
    masks = [synth_cells(width, height, i, seed=2104, members=members, eps=eps, threads=0)
             for i in range(k)]
    rng = np.random.default_rng(0)
    pairs = []
    while len(pairs) < min(64, npairs_total):
        i, j = sorted(rng.choice(k, 2, replace=False).tolist())
        if (i, j) not in pairs:
            pairs.append((i, j))
    ids = [f"s{i:04d}" for i in range(k)]
    sim = O.similarity_from_gram(oracle_c.gram([m.reshape(-1) for m in masks], cores))

    # ---- as shipped: single thread, both backends --------------------------------
    as_shipped = {}
    if ref is not None:
        rows_w = min(height, max(1, -(-(16 << 20) // width)))  # >= 16 Mpx window
        surfaces = [ref.RasterSurface(id=ids[i], name=ids[i], width=width, height=rows_w,
                                      cells=masks[i][:rows_w]) for i in range(k)]
        for name in ("numpy", "cython"):
            if name in mods:
                as_shipped[name] = _as_shipped_leg(ref, name, mods[name], surfaces,
                                                   rows_w * width, P, k, pairs, sim, args.tau)
        del surfaces
    # host analytics per frame (outliers + clusters on the exact matrix)
    if as_shipped:
        best = min(as_shipped.values(), key=lambda r: r["s_per_frame"])
        harness_backend = best["backend"]
        t_host = best["measured_s"]["outlier_scores"] + best["measured_s"]["cluster_surfaces"]
    else:
        harness_backend = "cython" if "cython" in mods else "numpy"
        t0 = time.perf_counter()
        O.outlier_scores(sim, ids)
        O.cluster(sim, ids, args.tau)
        t_host = time.perf_counter() - t0

    # ---- all cores: a proportional sample of the frame per step ----------------------
    # Every step is the WHOLE frame's work restricted to a window of rows: each worker
    # takes `rows_w` rows at the start of its 1/nw of the raster and runs on them the
    # per-pixel ops over all k masks AND pair_counts for ALL k(k-1)/2 pairs (the work of
    # similarity_matrix, fs/analytics.py:174-181).  Every term of the frame is linear in
    # the pixels, so mask-pixels / step time is the frame's rate with nothing scaled; only
    # the per-frame host analytics (outliers + clusters on the exact matrix, a fixed cost
    # per frame) are charged pro rata to the window.
    all_pairs = [(i, j) for i in range(k) for j in range(i + 1, k)]
    nw = min(cores, height)
    rows_w = max(1, min(height // nw, -(-(128 << 10) // width)))  # ~128 Kpx per worker
    bounds = [(w * height // nw, w * height // nw + rows_w) for w in range(nw)]
    window_px = nw * rows_w * width
    t_host_share = t_host * window_px / P

    def harness(mod, nsteps):
        """nsteps proportional-sample steps of `mod` on nw forked workers: per-step
        (time, pixel-op time, pair time)"""
        _REF.update(mod=mod, masks=masks, pairs=all_pairs, k=k)
        ctx = mp.get_context("fork")
        conns, procs, out = [], [], []
        for w, (lo, hi) in enumerate(bounds):
            parent, child = ctx.Pipe()
            proc = ctx.Process(target=_stripe_worker, args=(w, lo, hi, child), daemon=True)
            proc.start()
            conns.append(parent)
            procs.append(proc)
        try:
            for _ in range(nsteps):
                for c in conns:
                    c.send("go")
                res = [c.recv() for c in conns]
                assert sum(r[0] for r in res) == window_px
                out.append((max(r[1] + r[2] for r in res) + t_host_share,
                            max(r[1] for r in res), max(r[2] for r in res)))
        finally:
            for c in conns:
                try:
                    c.send("stop")
                except (BrokenPipeError, OSError):
                    pass
            for proc in procs:
                proc.join(timeout=10)
        return out

    # the reference at its best: one pilot step per primitive backend, the faster one runs
    # the measured steps (small stripes favour numpy's vector calls; the as-shipped
    # 16 Mpx windows can favour Cython)
    pilot = {name: harness(mod, 1)[0][0] for name, mod in mods.items()}
    harness_backend = min(pilot, key=pilot.get)
    runs = harness(mods[harness_backend], args.warmup + args.steps)[args.warmup:]
    times = [r[0] for r in runs]
    pix_s = [r[1] for r in runs]
    pair_s = [r[2] for r in runs]
    t = statistics.median(times)
    value = k * window_px / t / 1e9
    frame_s = t * P / window_px
    kind = "reference" if ref is not None or harness_backend == "cython" else "port"
    src = ("baseline/_ref floodstream (unmodified reference package)" if ref is not None else
           "oracle/_ref (reference _accel.pyx compiled from its sources)"
           if harness_backend == "cython" else "oracle NumPy port")
    sample = (f"{src}, {harness_backend} primitives, {nw} processes: each step = accumulate_into "
              f"x{k} + overlap_counts + composite_fill + pair_counts for all {npairs_total} "
              f"pairs on a {window_px}-px window ({nw} stripes of {rows_w} rows spread over "
              f"the raster), + outlier_scores/cluster_surfaces ({t_host:.2f} s per frame on the "
              f"exact matrix) charged pro rata")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload_config(args, width, height, k, world),
        "fps": round(1.0 / frame_s, 6),
        "step": {"kind": "proportional sample of one frame (all pairs, all masks, "
                         f"{window_px} of {P} px)",
                 "window_px": window_px, "frame_s": round(frame_s, 3),
                 "pixel_ops_s": round(statistics.median(pix_s), 4),
                 "pair_counts_s": round(statistics.median(pair_s), 4),
                 "host_analytics_share_s": round(t_host_share, 4),
                 "pilot_step_s": {n: round(v, 4) for n, v in pilot.items()}},
        "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": nw, "kind": kind,
                         "sample": sample},
        "as_shipped": as_shipped or None,
        "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return line


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def band(height, rank, world):
    base, extra = divmod(height, world)
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


def pcie_h2d_gbs(nbytes: int = 1 << 30, reps: int = 5) -> float:
    """Measured pinned host->device copy bandwidth (GB/s, best of reps, CUDA events):
    the e2e roofline denominator (fs/bench.py:193-228's transfer baseline, measured)."""
    import torch

    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    del h, d
    return nbytes / best / 1e9


def load_traffic() -> dict:
    """dram bytes per launch from the committed ncu --set full captures (profiles/)."""
    p = REPO / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            pass
    return {}


def bench_banded(args, width, height, k, members, eps, rank, world, local_rank):
    """Config 4 (64 x 32768^2, 68.7 GB of uint8 rasters): spatial + iterative streaming.
    The fixed ensemble is split into row blocks, one per rank ("strong" scaling), and
    each rank streams its block band by band from pinned host rasters (BandedStream):
    H2D + transform + fused recompute + D2H of the maps, then one all-reduce of the
    [histogram | Gram] sums.  Every step moves every raster byte over PCIe, so the
    step is e2e by construction and PCIe-bound."""
    import torch

    from paper_2104_14667_b200 import _native as N
    from paper_2104_14667_b200.banded import BandedStream, default_band_rows
    from paper_2104_14667_b200.dist import band as row_band
    from paper_2104_14667_b200.synth import synth_cells_gpu

    gpu, backend = dist_setup(local_rank, world)
    torch.cuda.set_device(gpu)
    N.set_device(gpu)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", gpu)
    row0, rows = row_band(height, rank, world)
    # host RAM bounds how many rows of every mask this rank can hold pinned
    try:
        import psutil

        avail = psutil.virtual_memory().available / world
    except Exception:
        avail = 64e9
    cap = args.max_host_gb * 1e9 if args.max_host_gb > 0 else 0.6 * avail
    max_rows = max(1, int(cap // (k * width + 8 * width)))
    sampled = rows > max_rows
    rows = min(rows, max_rows)
    host = [N.PinnedBuffer((rows, width)) for _ in range(k)]
    for i in range(k):
        synth_cells_gpu(width, height, i, seed=2104, members=members, eps=eps, row0=row0,
                        rows=rows, out=host[i].array)
    counts = torch.empty((rows, width), dtype=torch.int32).pin_memory()
    rgba = torch.empty((rows, width, 4), dtype=torch.uint8).pin_memory()
    band_rows = args.band_rows or min(4096, default_band_rows(width, k))
    bs = BandedStream(width, height, k, row0=row0, rows=rows, band_rows=band_rows)
    ids = [f"s{i:04d}" for i in range(k)]
    src = [h.array for h in host]

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    def step():
        return bs.run(src, tau=args.tau, ids=ids, counts_out=counts, rgba_out=rgba,
                      engine=args.engine, analytics=(rank == 0))

    for _ in range(args.warmup):
        step()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with Clocks(gpu) as clk:
        ev0.record()
        for _ in range(args.steps):
            last = step()
        torch.cuda.synchronize()
        ev1.record()
        ev1.synchronize()
    t = ev0.elapsed_time(ev1) / 1e3
    if dist is not None:
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
        nrows = torch.tensor([rows], dtype=torch.int64, device=dev)
        dist.all_reduce(nrows)
        total_rows = int(nrows.item())
    else:
        total_rows = rows
    px = k * width * total_rows
    value = px * args.steps / t / 1e9
    st = last["stats"]
    if rank == 0:
        pcie = pcie_h2d_gbs()
        per_step = t / args.steps
        h2d = k * width * rows
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(per_step * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "config": workload_config(args, width, height, k, world),
            "setup": {"band_rows": band_rows, "rows_per_rank": rows, "rows_total": total_rows,
                      "sampled": (f"host RAM holds {rows} of {row_band(height, rank, world)[1]}"
                                  " rows per rank; value counts only the streamed rows")
                      if sampled else None,
                      "path": "spatial bands streamed from pinned host memory (H2D + transform "
                              "+ recompute + D2H of maps per step)"},
            "fps": round(args.steps / t, 4),
            "bands": st.bands,
            "roofline": {"bound": "pcie_h2d", "achieved": round(h2d / per_step / 1e9, 2),
                         "peak": round(pcie, 2), "unit": "GB/s",
                         "frac": round(h2d / per_step / 1e9 / pcie, 4), "traffic": None,
                         "peak_note": "measured pinned H2D, 1 GiB copy, best of 5 (rank 0)"},
            "clocks": clk.summary(),
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": int(px),
                    "d2h_bytes_per_step": int(8 * width * total_rows),
                    "note": "the banded pass is end to end by construction"},
            "cpu_baseline": None,
            "clusters": len(last["clusters"]) if last.get("clusters") is not None else None,
            "gpu_launches": None,
        }
        # per band: k transform launches + the fused recompute (+ Gram reduce)
        line["gpu_launches"] = st.bands * (k + 2) * args.steps
        print(json.dumps(line), flush=True)
    bs.close()
    for h in host:
        h.free()
    if dist is not None:
        dist.destroy_process_group()


def dist_setup(local_rank: int, world: int):
    """(torch device index, backend) for this rank: one GPU per rank over NCCL.  The
    FS_DIST_BACKEND=gloo override lets a multi-rank run share one GPU (the N > 1 code
    path exercised on a single-GPU box; not a measurement configuration)."""
    import torch

    backend = os.environ.get("FS_DIST_BACKEND", "nccl")
    dev = local_rank % max(1, torch.cuda.device_count()) if backend != "nccl" else local_rank
    return dev, backend


def main():
    args = parse()
    width, height, k, members, eps = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        reference_arm(args, width, height, k, members, eps, rank, world)
        return
    if args.config == "c4":
        bench_banded(args, width, height, k, members, eps, rank, world, local_rank)
        return

    import torch

    from paper_2104_14667_b200 import _native as N
    from paper_2104_14667_b200.dist import ShardedEnsemble
    from paper_2104_14667_b200.synth import synth_cells_gpu

    gpu, backend = dist_setup(local_rank, world)
    torch.cuda.set_device(gpu)
    N.set_device(gpu)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", gpu)
    if args.scaling == "weak":
        height = height * world  # every rank keeps a full 1-GPU band
    P = width * height
    slots = list(range(k))
    ids = [f"s{i:04d}" for i in range(k)]

    sh = ShardedEnsemble(width, height, k)
    row0, rows = sh.row0, sh.rows
    # frames in flight = host-analytics threads: the O(k^2) linkage at k = 1024 takes
    # longer than the device frame, so more frames overlap it
    depth = 3 if k <= 256 else 6
    P_band = rows * width
    ens = sh.ens
    stream = sh.stream

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: int) -> int:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        return int(t.item())

    def timed_frames(n, **kw):
        """n pipelined frames between CUDA events on the ensemble stream (after a
        barrier), max over ranks; the events bracket every frame's device work and,
        because run_frames returns only after the last frame's products reached the
        host, its D2H too."""
        if n <= 0:
            return 0.0, 0.0, None
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        w0 = time.perf_counter()
        out = sh.run_frames(slots, n, tau=args.tau, engine=args.engine, ids=ids, keep=False,
                            depth=depth, analytics_ranks="root", **kw)
        e1.record(stream)
        e1.synchronize()
        wall = time.perf_counter() - w0
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / 1e3), max_over_ranks(wall), out[-1]

    # ---- pinned host rasters: this rank's rows of every mask (generated, untimed) ----
    host = None
    if not args.no_e2e:
        host = [N.PinnedBuffer((P_band,)) for _ in range(k)]
        for i in range(k):
            synth_cells_gpu(width, height, i, seed=2104, members=members, eps=eps, row0=row0,
                            rows=rows, out=host[i].array.reshape(rows, width))
        arrays = [h.array for h in host]
    else:
        ens.synth(0, k, seed=2104, members=members, eps=eps)

    def upload(_f):
        ens.stream(arrays, variant="2b-final", already_banded=True)

    # ---- the metric: K end-to-end frames (host rasters in, host products out) ----
    clocks = None
    n_clusters = None
    if not args.no_e2e:
        timed_frames(args.warmup, maps_to_host=True, before_frame=upload)
        with Clocks(gpu) as clk:
            t_e2e, wall_e2e, last = timed_frames(args.steps, maps_to_host=True,
                                                 before_frame=upload)
        clocks = clk.summary()
        if rank == 0:
            n_clusters = len(last["clusters"])
        kern_pack = ens.kernel_ms("pack")
    # ---- resident recompute: masks bit-packed in HBM (interactive FPS) ------------
    rsteps = max(args.resident_steps, 1)
    timed_frames(args.warmup)
    with Clocks(gpu) as clk_r:
        t_res, wall_res, last_r = timed_frames(rsteps)
    t_res_maps, _, _ = timed_frames(max(rsteps // 4, 1), maps_to_host=True)
    if clocks is None:
        clocks = clk_r.summary()
        n_clusters = len(last_r["clusters"]) if rank == 0 else None
    host_ms = []
    if rank == 0:  # host part of a frame (the complete-linkage merge loop), timed apart
        from paper_2104_14667_b200.analytics import cluster_from_similarity

        for _ in range(3):
            t0 = time.perf_counter()
            cluster_from_similarity(last_r["similarity"], ids, args.tau)
            host_ms.append((time.perf_counter() - t0) * 1e3)

    # ---- per-kernel rooflines: CUDA-event durations on the ensemble stream, sampled
    # in extra untimed calls (reading them blocks, which would break the pipelining) ----
    kern = {"overlap": [], "gram": [], "recompute": []}
    d_c = torch.empty(P_band, dtype=torch.int32, device=dev)
    d_r = torch.empty(P_band * 4, dtype=torch.uint8, device=dev)
    d_b = torch.empty(k + 1, dtype=torch.int64, device=dev)
    d_g = torch.empty(k * k, dtype=torch.int64, device=dev)
    fused = None
    for _ in range(6):
        fused = ens.products(slots, engine=args.engine, out_counts=d_c.data_ptr(),
                             out_rgba=d_r.data_ptr(), out_bins=d_b.data_ptr(),
                             out_gram=d_g.data_ptr(), device_outputs=True)[4]
        kern["recompute"].append(ens.kernel_ms("recompute"))
        ens.overlap(slots, out_counts=d_c.data_ptr(), out_rgba=d_r.data_ptr(),
                    out_bins=d_b.data_ptr(), device_outputs=True)
        kern["overlap"].append(ens.kernel_ms("overlap"))
        ens.gram(slots, engine=args.engine, out=d_g.data_ptr(), device_outputs=True)
        kern["gram"].append(ens.kernel_ms("gram"))
    del d_c, d_r, d_b, d_g
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    traffic = load_traffic()
    ov_ms = statistics.median(kern["overlap"])
    gr_ms = statistics.median(kern["gram"])
    rc_ms = statistics.median(kern["recompute"])
    ov_bytes = k * P_band / 8 + 4 * P_band + 4 * P_band + 8 * (k + 1)
    gram_ops = float(k) * (k + 1) * P_band  # upper triangle incl. diagonal, MAC = 2 ops
    t_peak, t_kind = tensor_peak(args.engine)
    rl_over = {"bound": "hbm", "achieved": round(ov_bytes / ov_ms / 1e6, 1), "peak": hbm,
               "unit": "GB/s", "frac": round(ov_bytes / ov_ms / 1e6 / hbm, 4),
               "traffic": traffic.get("k_overlap"), "kernel_ms": round(ov_ms, 4),
               "bytes_per_launch": int(ov_bytes),
               "bytes_def": "N*P/8 packed read + 4P counts + 4P RGBA + 8(N+1) bins",
               "peak_note": "MEASURED_PEAKS.json hbm_gbs (copy test)"}
    ops_def = ("N(N+1)*P = 2 ops x the N(N+1)/2 distinct mask pairs x P px (the kernel "
               "issues 3/4 N^2 P MACs: 128-row MMA granularity)")
    rl_gram = {"bound": "tensor", "achieved": round(gram_ops / gr_ms / 1e9, 1), "peak": t_peak,
               "unit": "TFLOP/s", "frac": round(gram_ops / gr_ms / 1e9 / t_peak, 4),
               "traffic": traffic.get("k_gram_tc_f4" if args.engine == "tc-f4" else "k_gram_tc"),
               "kernel_ms": round(gr_ms, 4), "ops_per_launch": gram_ops, "ops_def": ops_def,
               "peak_note": t_kind}
    npanels_k = -(-k // (128 if k <= 128 else 256))
    one_panel = bool(fused) and npanels_k == 1
    rl_fused = {"bound": "tensor",
                "kernel": (("k_recompute_f4 + k_gram_reduce" if k > 128 else
                            "k_gram_tc<128,...,FUSE> + k_gram_reduce") if npanels_k == 1 else
                           "k_recompute_f4 diagonal tiles (partial counts) + k_gram_pair_f4 + "
                           "k_gram_reduce + k_combine_partials") if fused
                else "k_overlap + k_gram_tc + k_gram_reduce",
                "fused": bool(fused), "achieved": round(gram_ops / rc_ms / 1e9, 1),
                "peak": t_peak, "unit": "TFLOP/s",
                "frac": round(gram_ops / rc_ms / 1e9 / t_peak, 4),
                "traffic": traffic.get("k_recompute_f4") if one_panel and k > 128 else None,
                "ncu": traffic.get("k_recompute_f4_ncu") if one_panel and k > 128 else None,
                "kernel_ms": round(rc_ms, 4), "ops_per_launch": gram_ops, "ops_def": ops_def,
                "peak_note": t_kind,
                "hbm_achieved_gbs": round(ov_bytes / rc_ms / 1e6, 1),
                "hbm_frac": round(ov_bytes / rc_ms / 1e6 / hbm, 4),
                "hbm_bytes_def": "same algorithmic bytes as the overlap pass (the Gram reads "
                                 "the same packed tiles)"}
    kernels = {"recompute": rl_fused, "overlap": rl_over, "gram": rl_gram}
    if not args.no_e2e:
        tx_bytes = P_band + P_band / 8
        kernels["transform"] = {
            "bound": "hbm", "kernel": "k_pack_flat (binarize + bit-pack one raster)",
            "achieved": round(tx_bytes / kern_pack / 1e6, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(tx_bytes / kern_pack / 1e6 / hbm, 4), "kernel_ms": round(kern_pack, 4),
            "bytes_per_launch": int(tx_bytes), "bytes_def": "P raw read + P/8 packed write",
            "launches_per_step": k, "traffic": traffic.get("k_pack_flat_c2_raster")
            if (P_band == 8192 * 8192) else None}

    # ---- the same frames through the native C++ loop (single device, informational) ----
    native = None
    if world == 1 or backend == "nccl":
        # the C++ frame loop; with N ranks each runs its band and the per-frame exchange is
        # an ncclAllReduce inside the loop (fs_comm, ShardedEnsemble.pipeline).  A failure
        # is reported in the line instead of aborting the measured numbers above; every
        # rank learns whether any rank failed before the max-over-ranks collectives.
        err, dev_ms, wall_n, ncl = None, 0.0, 0.0, 0
        try:
            mk = (ens.pipeline(slots, tau=args.tau, engine=args.engine, ids=ids, depth=depth)
                  if world == 1 else
                  sh.pipeline(slots, tau=args.tau, engine=args.engine, ids=ids, depth=depth))
            with mk as pipe:
                pipe.run(args.warmup)
                torch.cuda.synchronize()
                t0n = time.perf_counter()
                rn = pipe.run(rsteps)
                wall_n = time.perf_counter() - t0n
            dev_ms, ncl = rn["device_ms"], len(rn["clusters"])
        except Exception as exc:  # noqa: BLE001
            err = f"{type(exc).__name__}: {str(exc)[:300]}"
        if int(max_over_ranks(1.0 if err else 0.0)):
            native = {"error": err or "failed on another rank"}
        else:
            native = {"ms_per_step": round(max_over_ranks(dev_ms) / rsteps, 4),
                      "fps": round(rsteps / (max_over_ranks(dev_ms) / 1e3), 3),
                      "wall_ms_per_step": round(max_over_ranks(wall_n) / rsteps * 1e3, 4),
                      "clusters": ncl,
                      "path": "fs_pipeline_run: recompute + device Jaccard/outliers + D2H queued "
                              "while C++ workers run the linkage (no Python per frame)"
                              + ("" if world == 1 else "; per-frame ncclAllReduce of "
                                 "[bins | Gram] inside the C++ loop (fs_comm)")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and host is not None:
        cpu = cpu_baseline([b.array for b in host], width, rows, k, min(P_band, 1 << 22))

    px_total = k * sum_over_ranks(P_band)
    res = {"value": round(px_total * rsteps / t_res / 1e9, 3), "unit": UNIT,
           "ms_per_step": round(t_res / rsteps * 1e3, 4), "fps": round(rsteps / t_res, 3),
           "steps": rsteps, "wall_ms_per_step": round(wall_res / rsteps * 1e3, 4),
           "path": "device_only: fused recompute + all-reduce + device Jaccard/outliers + D2H "
                   "of [bins | Gram] + Jaccard + scores, host linkage overlapped",
           "maps_to_host": {"ms_per_step": round(t_res_maps / max(rsteps // 4, 1) * 1e3, 4),
                            "fps": round(max(rsteps // 4, 1) / t_res_maps, 3),
                            "d2h_bytes_per_step": int(8 * P_band),
                            "path": "the same + counts and RGBA maps to pinned host memory"},
           "native_pipeline": native}
    if rank != 0:
        torch.cuda.synchronize()
        sh.close()
        if host is not None:
            for b in host:
                b.free()
        if dist is not None:
            dist.destroy_process_group()
        return
    pcie = pcie_h2d_gbs()
    config = workload_config(args, width, height, k, world)
    setup = {"gram_engine": args.engine, "rows_per_rank": rows,
             "pipelining": f"{depth} frames in flight: host analytics of frame f overlap "
                           "device work of frame f+1",
             "value_kind": "end to end: pinned host rasters in, host products out"}
    if args.no_e2e:
        value, ms_step, fps, e2e = res["value"], res["ms_per_step"], res["fps"], None
        setup["value_kind"] = "resident (--no-e2e profiling run, not the metric)"
    else:
        value = px_total * args.steps / t_e2e / 1e9
        ms_step = t_e2e / args.steps * 1e3
        fps = args.steps / t_e2e
        h2d_rank = k * P_band
        t_min = h2d_rank / (pcie * 1e9)
        e2e = {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": int(px_total),
               # counts + RGBA of every band, and per rank [bins | Gram] + Jaccard + scores
               "d2h_bytes_per_step": int(8 * P + world * 8 * ((k + 1) + 2 * k * k + k)),
               "ms_per_step": round(ms_step, 3), "fps": round(fps, 4), "steps": args.steps,
               "wall_ms_per_step": round(wall_e2e / args.steps * 1e3, 3),
               "roofline": {"bound": "pcie_h2d",
                            "achieved": round(h2d_rank / (t_e2e / args.steps) / 1e9, 2),
                            "peak": round(pcie, 2), "unit": "GB/s",
                            "frac": round(t_min / (t_e2e / args.steps), 4),
                            "peak_note": "measured pinned H2D, 1 GiB copy, best of 5"},
               "path": "pinned host rasters -> DeviceEnsemble.stream (2b-final) -> fused "
                       "recompute -> D2H counts+RGBA+[bins|Gram]+Jaccard+scores -> clusters"}
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "u8", "data": "synthetic", "config": config, "setup": setup,
        "fps": round(fps, 4), "resident": res,
        "host_linkage_ms": round(statistics.median(host_ms), 4) if host_ms else None,
        "clusters": n_clusters,
        "roofline": rl_fused, "kernels": kernels, "clocks": clocks, "e2e": e2e,
        "cpu_baseline": cpu, "gpu_launches": None,
    }
    # our kernels per e2e step: k transform launches + the recompute + Jaccard/outliers
    if args.engine in ("tc", "tc-f4"):
        gram_launches = 1 + (1 if npanels_k > 1 else 0) + 1  # diag, off-diag, reduce
    else:
        gram_launches = 1 + (1 if k > 64 else 0)  # popc, mirror
    per_step = gram_launches + (0 if one_panel else 1) + (2 if k >= 2 else 1)
    line["gpu_launches"] = (per_step + (0 if args.no_e2e else k)) * args.steps
    print(json.dumps(line), flush=True)
    torch.cuda.synchronize()
    sh.close()
    if host is not None:
        for b in host:
            b.free()
    if dist is not None:
        dist.destroy_process_group()


def tensor_peak(engine: str) -> tuple[float, str]:
    """Dense tensor peak for the Gram's kind: the builder-measured FP4 / int8 MMA rate
    (profiles/tensor_peaks.json, tools/probes/mma_probe.cu) when present, else the
    B200_PROFILING.md nominal figure; the note says which."""
    meas = {}
    p = REPO / "profiles" / "tensor_peaks.json"
    if p.exists():
        try:
            meas = json.loads(p.read_text())
        except Exception:
            meas = {}
    key = {"tc-f4": "fp4_tflops", "tc": "int8_tops", "popc": "int8_tops"}[engine]
    nominal = {"tc-f4": 9000.0, "tc": 4500.0, "popc": 4500.0}[engine]
    kind = {"tc-f4": "fp4 (kind::mxf4)", "tc": "int8 (kind::i8)",
            "popc": "int8 (kind::i8), CUDA-core engine shown for scale"}[engine]
    if meas.get(key):
        return float(meas[key]), f"{kind} {meas[key]:.0f} TFLOP/s dense, measured ({p.name})"
    return nominal, f"{kind} {nominal:.0f} TFLOP/s dense, nominal (B200_PROFILING.md)"


if __name__ == "__main__":
    main()
