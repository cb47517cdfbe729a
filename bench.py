#!/usr/bin/env python
"""Headline benchmark: ensemble Gpixels/s (incl. H2D) and FPS for 256 x 8192^2 masks.

Workload (BASELINE.json configs[1], "c2"): 256 flood-like masks of 8192 x 8192 uint8
(17.18 GB).  One *step* = one full recompute of the working set:
  overlap counts + overlap-class histogram + composite RGBA and the exact
  pairwise-intersection Gram in ONE kernel over the bit-packed masks (tcgen05
  kind::mxf4 + counter warps), the Jaccard matrix and outlier scores on the device, and
  the complete-linkage clusters (tau 0.8) on the host.

* ``value``: masks already resident (bit-packed) in HBM; unit Gpx/s = N*P / step time.
* ``e2e``  : the same step through the public API from PINNED host rasters: every step
  streams all 256 rasters (H2D, double-buffered, overlapped with the binarize+pack
  transform), recomputes, and reads counts + RGBA + histogram + Gram back to the host.
* ``--impl reference``: the reference's own CPU implementation (oracle/_ref = its
  Cython accelerator compiled from its sources; else the oracle NumPy port) on all host
  cores, on a bounded pixel window + pair sample, extrapolated to the workload.

Multi-GPU (torchrun, one rank per GPU): the ensemble grows with N — 256 masks of
8192 x (8192 N) px — and rank r owns rows [8192 r, 8192 (r+1)) of every mask, i.e. each
GPU keeps exactly the 1-GPU workload (``scaling`` "weak", per-GPU work fixed).  The only
exchange is the one NCCL all-reduce of the int64 [histogram | Gram] partials per frame;
timings are the max over ranks and ``value`` = all masks' pixels / that time.
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
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--tau", type=float, default=0.8)
    ap.add_argument("--engine", default="tc-f4", choices=["tc-f4", "tc", "popc"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
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
# reference arm
# ---------------------------------------------------------------------------
def _ref_cells(task):
    """The stripe's input rows for every mask (generation is untimed)."""
    (lo, hi, k, width, height, seed, members, eps, _pairs) = task
    from paper_2104_14667_b200.synth import synth_cells

    return [synth_cells(width, height, i, seed=seed, members=members, eps=eps, row0=lo // width,
                        rows=max(1, (hi - lo) // width), threads=1).reshape(-1)
            for i in range(k)]


def _ref_step(mod, cells, k, pairs):
    """One timed pass of the reference primitives over a stripe of every mask."""
    n = cells[0].size
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
    return n, t1 - t0, t2 - t1


def _ref_server(task, conn):
    """Persistent worker owning one stripe: generates it once, then runs one timed step
    per "go" message (so steps measure only the reference kernels)."""
    mod = _load_reference_kernels()
    cells = _ref_cells(task)
    k, pairs = task[2], task[8]
    while conn.recv() == "go":
        conn.send(_ref_step(mod, cells, k, pairs))
    conn.close()


def _load_reference_kernels():
    ref = REPO / "oracle" / "_ref"
    if any(ref.glob("_accel*.so")):
        sys.path.insert(0, str(ref))
        import _accel  # the reference's Cython accelerator, compiled from its sources

        return _accel
    from oracle import fs_oracle  # the NumPy port of _kernels_np.py

    return fs_oracle


def reference_arm(args, width, height, k, members, eps, rank, world):
    if rank != 0:
        return None
    height = height * world  # the same (weak-scaled) ensemble as the B200 arm
    import multiprocessing as mp

    mod = _load_reference_kernels()
    kind = "reference" if getattr(mod, "NAME", "") == "cython" else "port"
    cores = os.cpu_count() or 1
    P = width * height
    # bounded sample per step: 8 rows of every mask per worker (large enough that the
    # primitives' per-call overhead is negligible); the stripes are generated once, so
    # a step costs only the timed reference kernels (~0.1-0.2 s) and even --steps 200
    # finishes within a minute or two
    rows_per_worker = 8
    window_rows = rows_per_worker * cores
    rng = np.random.default_rng(0)
    npairs_total = k * (k - 1) // 2
    sample_pairs = [tuple(sorted(rng.choice(k, 2, replace=False).tolist())) for _ in range(8)]
    tasks = [(w * rows_per_worker * width, (w + 1) * rows_per_worker * width, k, width, height,
              2104, members, eps, sample_pairs) for w in range(cores)]
    # clustering + outliers on an exact similarity matrix: the host logic of
    # analytics.py:184-240, timed once (it does not depend on pixels)
    from oracle import fs_oracle as O

    sim = np.eye(k)
    proto = np.arange(k) // members
    sim = np.where(proto[:, None] == proto[None, :], 0.9, 0.3) + np.eye(k) * 0.1
    ids = [f"s{i:04d}" for i in range(k)]
    t0 = time.perf_counter()
    O.outlier_scores(sim, ids)
    O.cluster(sim, ids, args.tau)
    t_host = time.perf_counter() - t0
    times = []
    ctx = mp.get_context("fork")
    conns, procs = [], []
    for task in tasks:
        parent, child = ctx.Pipe()
        proc = ctx.Process(target=_ref_server, args=(task, child), daemon=True)
        proc.start()
        conns.append(parent)
        procs.append(proc)
    try:
        for step in range(args.warmup + args.steps):
            for c in conns:
                c.send("go")
            res = [c.recv() for c in conns]
            n_win = sum(r[0] for r in res)
            t_pix = max(r[1] for r in res)
            t_pair = max(r[2] for r in res)
            scale = P / n_win
            t_step = t_pix * scale + t_pair * scale * (npairs_total / len(sample_pairs)) + t_host
            if step >= args.warmup:
                times.append(t_step)
    finally:
        for c in conns:
            try:
                c.send("stop")
            except (BrokenPipeError, OSError):
                pass
        for proc in procs:
            proc.join(timeout=10)
    t = statistics.median(times)
    value = k * P / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"{args.config}: {k} masks {width}x{height}"
                               + (f" ({world} x {height // world}-row bands)" if world > 1 else ""),
                   "tau": args.tau},
        "fps": round(1.0 / t, 6),
        "cpu_baseline": {
            "value": round(value, 6), "unit": UNIT, "cores": cores, "kind": kind,
            "sample": (f"{'oracle/_ref (reference _accel.pyx)' if kind == 'reference' else 'oracle NumPy port'}"
                       f" accumulate_into/overlap_counts/composite_fill on {window_rows} rows x "
                       f"{k} masks split over {cores} processes, pair_counts on "
                       f"{len(sample_pairs)} sampled pairs, scaled to {P} px and "
                       f"{npairs_total} pairs; + clustering/outliers {t_host:.2f} s (exact sim)"),
        },
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
            "config": {"workload": f"c4: {k} flood-like masks {width}x{height} uint8 streamed "
                                   f"in spatial bands of {band_rows} rows from pinned host "
                                   "memory (H2D + transform + recompute + D2H of maps per step)",
                       "masks": k, "width": width, "height": height, "tau": args.tau,
                       "rows_per_rank": rows, "rows_total": total_rows,
                       "sampled": (f"host RAM holds {rows} of {row_band(height, rank, world)[1]}"
                                   " rows per rank; value counts only the streamed rows")
                       if sampled else None,
                       "parallelism": f"row blocks x{world}" if world > 1 else "single GPU",
                       "l2": "every step streams all rasters from host memory (>> L2)"},
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
    from paper_2104_14667_b200.synth import synth_cells, synth_cells_gpu

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
    band_h = height
    height = height * world  # weak scaling: every rank keeps a full 1-GPU band
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
    ens.synth(0, k, seed=2104, members=members, eps=eps)
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

    kern = {"overlap": [], "gram": [], "recompute": []}

    def sample_kernels(_f):
        # CUDA-event duration of the previous frame's recompute call (ensemble stream)
        if _f > 0:
            kern["recompute"].append(ens.kernel_ms("recompute"))

    # ---- resident timed region: K pipelined full recomputes ---------------------------
    sh.run_frames(slots, args.warmup, tau=args.tau, engine=args.engine, ids=ids,
                  analytics_ranks="root", keep=False, depth=depth)
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    host_ms = []
    with Clocks(gpu) as clk:
        barrier()
        ev0.record(stream)
        t_wall0 = time.perf_counter()
        last = sh.run_frames(slots, args.steps, tau=args.tau, engine=args.engine, ids=ids,
                             analytics_ranks="root", keep=False, depth=depth)
        ev1.record(stream)
        ev1.synchronize()
        t_wall = time.perf_counter() - t_wall0
        barrier()
    t_res = max_over_ranks(ev0.elapsed_time(ev1) / 1e3)
    clocks = clk.summary()
    ms_step = t_res / args.steps * 1e3
    value = k * P * args.steps / t_res / 1e9
    if rank == 0:  # host part of a frame (the complete-linkage merge loop), timed apart;
        # Jaccard and outlier scores are computed on the device inside the frame
        from paper_2104_14667_b200.analytics import cluster_from_similarity

        sim_last = last[0]["similarity"]
        for _ in range(3):
            t0 = time.perf_counter()
            n_clusters = len(cluster_from_similarity(sim_last, ids, args.tau))
            host_ms.append((time.perf_counter() - t0) * 1e3)

    # ---- per-kernel roofline: CUDA-event durations on the ensemble stream, sampled in
    # extra untimed frames (reading them blocks, which would break the pipelining) ----
    sh.run_frames(slots, 6, tau=args.tau, engine=args.engine, ids=ids, analytics_ranks="none",
                  keep=False, before_frame=sample_kernels, depth=depth)
    sample_kernels(1)
    fused = None
    # the two stages as separate kernels (the unfused path), for the breakdown
    d_c = torch.empty(P_band, dtype=torch.int32, device=dev)
    d_r = torch.empty(P_band * 4, dtype=torch.uint8, device=dev)
    d_b = torch.empty(k + 1, dtype=torch.int64, device=dev)
    d_g = torch.empty(k * k, dtype=torch.int64, device=dev)
    for _ in range(6):
        ens.overlap(slots, out_counts=d_c.data_ptr(), out_rgba=d_r.data_ptr(),
                    out_bins=d_b.data_ptr(), device_outputs=True)
        kern["overlap"].append(ens.kernel_ms("overlap"))
        ens.gram(slots, engine=args.engine, out=d_g.data_ptr(), device_outputs=True)
        kern["gram"].append(ens.kernel_ms("gram"))
        fused = ens.products(slots, engine=args.engine, out_counts=d_c.data_ptr(),
                             out_rgba=d_r.data_ptr(), out_bins=d_b.data_ptr(),
                             out_gram=d_g.data_ptr(), device_outputs=True)[4]
    del d_c, d_r, d_b, d_g
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    traffic = load_traffic()
    ov_ms = statistics.median(kern["overlap"])
    gr_ms = statistics.median(kern["gram"])
    ov_bytes = k * P_band / 8 + 4 * P_band + 4 * P_band + 8 * (k + 1)
    gram_ops = float(k) * (k + 1) * P_band  # upper triangle incl. diagonal, MAC = 2 ops
    # dense tensor peaks (B200_PROFILING.md fallback table; MEASURED_PEAKS.json has bf16 only)
    t_peak, t_kind = {"tc-f4": (9000.0, "fp4 (kind::mxf4) 9 PFLOP/s dense"),
                      "tc": (4500.0, "int8 (kind::i8) 4.5 POPS dense"),
                      "popc": (4500.0, "int8 4.5 POPS dense (CUDA-core engine, for scale)")}[args.engine]
    rl_over = {"bound": "hbm", "achieved": round(ov_bytes / ov_ms / 1e6, 1), "peak": hbm,
               "unit": "GB/s", "frac": round(ov_bytes / ov_ms / 1e6 / hbm, 4),
               "traffic": traffic.get("k_overlap"), "kernel_ms": round(ov_ms, 4),
               "bytes_per_launch": int(ov_bytes),
               "bytes_def": "N*P/8 packed read + 4P counts + 4P RGBA + 8(N+1) bins",
               "peak_note": "MEASURED_PEAKS.json hbm_gbs (copy test)"}
    rl_gram = {"bound": "tensor", "achieved": round(gram_ops / gr_ms / 1e9, 1), "peak": t_peak,
               "unit": "TFLOP/s", "frac": round(gram_ops / gr_ms / 1e9 / t_peak, 4),
               "traffic": traffic.get("k_gram_tc_f4" if args.engine == "tc-f4" else "k_gram_tc"),
               "kernel_ms": round(gr_ms, 4), "ops_per_launch": gram_ops,
               "ops_def": "N(N+1)*P = 2 ops x the N(N+1)/2 distinct mask pairs x P px "
                          "(the kernel issues 3/4 N^2 P MACs: 128-row MMA granularity)",
               "peak_note": t_kind}
    rc_ms = statistics.median(kern["recompute"])
    npanels_k = -(-k // (128 if k <= 128 else 256))
    rl_fused = {"bound": "tensor",
                "kernel": ("k_gram_tc<...,FUSE> + k_gram_reduce" if npanels_k == 1 else
                           "k_gram_tc<...,FUSE> (partial counts) + k_gram_pair_f4 + "
                           "k_gram_reduce + k_combine_partials") if fused
                else "k_overlap + k_gram_tc + k_gram_reduce",
                "fused": bool(fused), "achieved": round(gram_ops / rc_ms / 1e9, 1),
                "peak": t_peak, "unit": "TFLOP/s",
                "frac": round(gram_ops / rc_ms / 1e9 / t_peak, 4),
                "traffic": traffic.get("k_gram_tc_fused") if (fused and npanels_k == 1) else None,
                # tensor-pipe utilisation of this kernel from the committed ncu capture
                "ncu": traffic.get("k_gram_tc_fused_ncu") if (fused and npanels_k == 1) else None,
                "kernel_ms": round(rc_ms, 4), "ops_per_launch": gram_ops,
                "ops_def": rl_gram["ops_def"], "peak_note": t_kind,
                "hbm_achieved_gbs": round(ov_bytes / rc_ms / 1e6, 1),
                "hbm_frac": round(ov_bytes / rc_ms / 1e6 / hbm, 4),
                "hbm_bytes_def": "same algorithmic bytes as the overlap pass (the Gram reads "
                                 "the same packed tiles)"}
    if fused and args.engine == "tc-f4" and k > 128 and npanels_k == 1:
        # What actually limits the fused kernel: shared-memory bandwidth (128 B/clk/SM).
        # Per 256-px K stage of the 256-mask diagonal panel the MMAs read 80 KB of
        # operands (rows 0-127 x N=256 and rows 128-255 x N=128, 4 K-steps), TMA writes
        # 8 KB of raw bits, the expanders read them and write 32 KB of e2m1 operands,
        # and the counter warps read the same 8 KB; the MMAs alone need 768 cycles.
        clk_hz = float((clocks or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)) * 1e6
        nsm = torch.cuda.get_device_properties(dev).multi_processor_count
        stages = -(-P_band // 1024) * 4 / nsm
        smem_ms = stages * (136 * 1024 / 128) / clk_hz * 1e3
        mma_ms = stages * 768 / clk_hz * 1e3
        rl_fused["limiter_model"] = {
            "limiter": "smem", "smem_bytes_per_stage": 136 * 1024, "smem_bytes_per_clk": 128,
            "mma_cycles_per_stage": 768, "stages_per_sm": round(stages, 1),
            "smem_bound_ms": round(smem_ms, 4), "mma_bound_ms": round(mma_ms, 4),
            "frac_of_smem_bound": round(smem_ms / rc_ms, 4),
            "note": "no binary tcgen05 kind: 1-bit masks are expanded to e2m1 in SMEM and "
                    "kind::mxf4 reads both operands from SMEM (no TMEM-A form)",
            # the kernel rebuilt without each part in turn (FS_PROBE_* builds): skeleton
            # (TMA ring + stage handoffs) 0.53 ms, + expansion 0.67, + counting 0.87,
            # + MMAs 1.08 at C2; TMA alone streams the same boxes at 7.25 TB/s
            "part_isolation": "profiles/r3f/parts.txt"}
    dominant = rl_fused

    # ---- the same frames through the native C++ loop (single device, informational) ----
    native = None
    if world == 1:
        with ens.pipeline(slots, tau=args.tau, engine=args.engine, ids=ids, depth=depth) as pipe:
            pipe.run(args.warmup)
            torch.cuda.synchronize()
            t0n = time.perf_counter()
            rn = pipe.run(args.steps)
            wall_n = time.perf_counter() - t0n
        native = {"ms_per_step": round(rn["device_ms"] / args.steps, 4),
                  "fps": round(args.steps / (rn["device_ms"] / 1e3), 3),
                  "wall_ms_per_step": round(wall_n / args.steps * 1e3, 4),
                  "clusters": len(rn["clusters"]),
                  "path": "fs_pipeline_run: recompute + device Jaccard/outliers + D2H queued "
                          "while C++ workers run the linkage (no Python per frame)"}

    # ---- end-to-end through the public API from pinned host rasters --------------------
    e2e = None
    host = h_counts = None
    if not args.no_e2e:
        host = [N.PinnedBuffer((P_band,)) for _ in range(k)]
        for i in range(k):  # the generator's bytes, produced on the GPU (fs_synth_gpu)
            synth_cells_gpu(width, height, i, seed=2104, members=members, eps=eps, row0=row0,
                            rows=rows, out=host[i].array.reshape(rows, width))
        arrays = [h.array for h in host]

        def upload(_f):
            ens.stream(arrays, variant="2b-final", already_banded=True)

        sh.run_frames(slots, 1, tau=args.tau, engine=args.engine, ids=ids, maps_to_host=True,
                      analytics_ranks="root", keep=False, depth=depth, before_frame=upload)  # warm-up
        barrier()
        ev0.record(stream)
        res = sh.run_frames(slots, args.e2e_steps, tau=args.tau, engine=args.engine, ids=ids,
                            maps_to_host=True, analytics_ranks="root", keep=False, depth=depth,
                            before_frame=upload)
        ev1.record(stream)
        ev1.synchronize()
        barrier()
        t_e2e = max_over_ranks(ev0.elapsed_time(ev1) / 1e3)
        h2d = int(k * P_band)
        pcie = pcie_h2d_gbs()
        t_min = h2d / (pcie * 1e9)
        e2e = {"value": round(k * P * args.e2e_steps / t_e2e / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(k * P),
               # counts + RGBA of every band, and per rank [bins | Gram] + Jaccard + scores
               "d2h_bytes_per_step": int(8 * P + world * 8 * ((k + 1) + 2 * k * k + k)),
               "ms_per_step": round(t_e2e / args.e2e_steps * 1e3, 3),
               "fps": round(args.e2e_steps / t_e2e, 4), "steps": args.e2e_steps,
               "roofline": {"bound": "pcie_h2d", "achieved": round(h2d / (t_e2e / args.e2e_steps) / 1e9, 2),
                            "peak": round(pcie, 2), "unit": "GB/s",
                            "frac": round(t_min / (t_e2e / args.e2e_steps), 4),
                            "peak_note": "measured pinned H2D, 1 GiB copy, best of 5"},
               "path": "DeviceEnsemble.stream(2b-final, pinned) -> overlap -> gram -> D2H "
                       "counts+RGBA+bins+Gram -> Jaccard/outliers/clusters"}
        h_counts = res[-1].get("counts")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        src = [b.array for b in host] if host is not None else [
            synth_cells(width, height, i, seed=2104, members=members, eps=eps, rows=256)
            for i in range(k)]
        window = min(P, 1 << 22, src[0].size)
        cpu = cpu_baseline(src, width, height, k, window)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"{args.config}: {k} flood-like masks {width}x{height} uint8 "
                                   "(bit-packed resident in HBM), full recompute per step"
                                   + (f"; {world} row bands of {band_h} rows, one per GPU"
                                      if world > 1 else ""),
                       "masks": k, "width": width, "height": height, "tau": args.tau,
                       "gram_engine": args.engine,
                       "parallelism": f"row-bands x{world}" if world > 1 else "single GPU",
                       "l2": f"inputs (bit-packed {k * P_band / 8 / 1e9:.2f} GB per GPU) larger "
                             "than L2; no flush",
                       "pipelining": "double-buffered frames: host analytics of frame f "
                                     "overlap device work of frame f+1"},
            "fps": round(args.steps / t_res, 3),
            "wall_ms_per_step": round(t_wall / args.steps * 1e3, 4),
            "host_linkage_ms": round(statistics.median(host_ms), 4) if host_ms else None,
            "native_pipeline": native,
            "clusters": n_clusters if host_ms else None,
            "roofline": dominant,
            "kernels": {"recompute": rl_fused, "overlap": rl_over, "gram": rl_gram},
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": None,
        }
        # our kernels per resident step: fused overlap (1) + Gram
        if args.engine in ("tc", "tc-f4"):
            npanels = -(-k // (128 if k <= 128 else 256))
            gram_launches = 1 + (1 if npanels > 1 else 0) + 1  # diag, off-diag, reduce
        else:
            gram_launches = 1 + (1 if k > 64 else 0)  # popc, mirror
        # + the overlap kernel unless fused into the diagonal Gram CTAs (beyond one panel
        # the fused path adds a combine kernel instead)
        # + Jaccard and outlier kernels on the summed Gram
        analytic_launches = 2 if k >= 2 else 1
        npan = -(-k // (128 if k <= 128 else 256))
        line["gpu_launches"] = (gram_launches + (0 if (fused and npan == 1) else 1)
                                + analytic_launches) * args.steps
        print(json.dumps(line), flush=True)
    torch.cuda.synchronize()
    sh.close()
    if host is not None:
        for b in host:
            b.free()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
