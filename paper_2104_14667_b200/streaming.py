"""The four buffer-streaming strategies, run for real on the B200.

API-compatible with ``floodstream.streaming`` (/root/reference/pkg/src/floodstream/
streaming.py:1-464).  The reference prices each strategy's operation DAG with a cost
model and a discrete-event simulator; here the same DAG (``build_schedule``) is
executed by the upload pipeline of libfloodstream — pinned/pageable host rasters,
H2D copies on a copy stream, the binarize+bit-pack transform and the per-item
accumulate kernel on a compute stream, CUDA events for every dependency edge — and
every per-item cost is *measured*:

* ``c_i`` = the H2D DMA of raster i (CUDA events on the copy stream),
* ``m_i`` = the transform kernel of item i, ``p_i`` = its accumulate kernel,
* ``total_time_us`` = first copy start -> last kernel end (device clock).

Variant mapping (paper §4 methods): ``*-initial`` = the coupled write path — each
raster is first copied by the host into a pinned staging slot (the "hidden duplicate
copy", timed per item) and only then DMA'd; ``*-final`` = decoupled upload straight
from the caller's buffer; ``1b``/``2b`` = one or two device staging slots.
"""

from __future__ import annotations

import csv
import io
from dataclasses import dataclass, field
from enum import Enum
from typing import Sequence

import numpy as np

from .schedule import OpKind, OpNode, ScheduleGraph


class Variant(str, Enum):
    ONE_BUFFER_INITIAL = "1b-initial"
    TWO_BUFFER_INITIAL = "2b-initial"
    ONE_BUFFER_FINAL = "1b-final"
    TWO_BUFFER_FINAL = "2b-final"

    @property
    def pairs(self) -> int:
        return 2 if self.value.startswith("2b") else 1

    @property
    def coupled_write(self) -> bool:
        return self.value.endswith("initial")

    @property
    def dma_pairs(self) -> int:
        """Pairs whose transfers genuinely overlap device work (only 2b-final)."""
        return 2 if self is Variant.TWO_BUFFER_FINAL else 1

    @staticmethod
    def parse(text: str) -> "Variant":
        key = text.strip().lower().replace("_", "").replace("-", "")
        table = {
            "1binitial": Variant.ONE_BUFFER_INITIAL, "onebufferinitial": Variant.ONE_BUFFER_INITIAL,
            "2binitial": Variant.TWO_BUFFER_INITIAL, "twobufferinitial": Variant.TWO_BUFFER_INITIAL,
            "1bfinal": Variant.ONE_BUFFER_FINAL, "onebufferfinal": Variant.ONE_BUFFER_FINAL,
            "2bfinal": Variant.TWO_BUFFER_FINAL, "twobufferfinal": Variant.TWO_BUFFER_FINAL,
        }
        if key not in table:
            raise StreamError(f"unknown variant {text!r}")
        return table[key]


VARIANTS = tuple(Variant)


class StreamError(ValueError):
    pass


@dataclass(frozen=True)
class StreamJob:
    """``n`` same-sized surfaces to stream and accumulate; ``surfaces`` (which may be
    fewer than ``n``) are cycled in order.  ``profile`` is accepted for signature
    compatibility with the reference; the device here is measured, not modelled."""

    variant: Variant
    n: int
    width: int
    height: int
    profile: object = None
    surfaces: Sequence = ()
    bpp: int = 1

    def __post_init__(self) -> None:
        if self.n < 1:
            raise StreamError("empty job")
        if self.width < 1 or self.height < 1:
            raise StreamError("image dimensions must be positive")
        if self.bpp != 1:
            raise StreamError("only 1 byte/px surfaces are supported")

    @property
    def payload_bytes(self) -> int:
        return self.width * self.height * self.bpp


def build_schedule(job: StreamJob) -> ScheduleGraph:
    """The strategy's operation DAG (streaming.py:134-217): the dependency contract
    that ``fs_ensemble_stream`` realises with CUDA events."""
    variant = Variant(job.variant)
    dims = (job.width, job.height)
    payload = job.payload_bytes
    nodes = [OpNode(id="clear[0]", kind=OpKind.CLEAR), OpNode(id="clear[1]", kind=OpKind.CLEAR)]
    for i in range(1, job.n + 1):
        if variant in (Variant.ONE_BUFFER_INITIAL, Variant.ONE_BUFFER_FINAL):
            copy_deps = (f"kernel[{i - 1}]",) if i >= 2 else ()
        elif variant is Variant.TWO_BUFFER_INITIAL:
            copy_deps = (f"kernel[{i - 2}]",) if i >= 3 else ()
        else:
            copy_deps = (f"xform[{i - 2}]",) if i >= 3 else ()
        if variant.coupled_write:
            nodes.append(OpNode(id=f"host[{i}]", kind=OpKind.HOST_COPY, payload_bytes=payload,
                                deps=copy_deps))
            nodes.append(OpNode(id=f"copy[{i}]", kind=OpKind.BUFFER_COPY, payload_bytes=payload,
                                deps=(f"host[{i}]",)))
        else:
            nodes.append(OpNode(id=f"copy[{i}]", kind=OpKind.BUFFER_COPY, payload_bytes=payload,
                                deps=copy_deps))
        xdeps = (f"copy[{i}]",) + ((f"kernel[{i - 1}]",) if i >= 2 else ())
        nodes.append(OpNode(id=f"xform[{i}]", kind=OpKind.BUFFER_TO_IMAGE, payload_bytes=payload,
                            image_dims=dims, deps=xdeps))
        kdeps = (f"xform[{i}]",) + (("clear[0]", "clear[1]") if i == 1 else (f"kernel[{i - 1}]",))
        nodes.append(OpNode(id=f"kernel[{i}]", kind=OpKind.KERNEL, payload_bytes=payload,
                            image_dims=dims, deps=kdeps))
    return ScheduleGraph(nodes=nodes, pairs=variant.dma_pairs, label=variant.value)


def closed_form_times(c: Sequence[int], m: Sequence[int], p: Sequence[int]) -> tuple[int, int]:
    """(t_dual, t_single) of the paper's §7.1 pipeline model (streaming.py:220-237)."""
    if not (len(c) == len(m) == len(p)):
        raise StreamError("cost lists must have equal length")
    if len(c) == 0:
        raise StreamError("cost lists must be non-empty")
    t_single = sum(c) + sum(m) + sum(p)
    t_dual = max(c[0] + sum(m) + sum(p), sum(c) + m[-1] + p[-1])
    return t_dual, t_single


def efficiency(c: Sequence[int], t_total: int) -> float:
    """Copy-bound share of a run: the sum of the per-item copy times over the measured
    total (the paper's efficiency)."""
    if t_total <= 0:
        raise StreamError("total time must be positive")
    return sum(c) / t_total


def round_half_up(x: float) -> int:
    return int(np.floor(x + 0.5))


@dataclass
class PipelineRunReport:
    variant: str
    n: int
    width: int
    height: int
    total_time_us: int
    per_item_c: list[int]
    per_item_m: list[int]
    per_item_p: list[int]
    transfer_rate_gbps: float
    efficiency: float
    makespan_source: str = "measured"
    contention_applied: bool = False
    warmup: bool = False
    per_item_h: list[int] = field(default_factory=list)

    def to_json(self) -> dict:
        per_item = {"c": self.per_item_c, "m": self.per_item_m, "p": self.per_item_p}
        if self.per_item_h:
            per_item["h"] = self.per_item_h
        return {
            "variant": self.variant,
            "n": self.n,
            "width": self.width,
            "height": self.height,
            "total_time_us": self.total_time_us,
            "per_item": per_item,
            "transfer_rate_gbps": self.transfer_rate_gbps,
            "efficiency": self.efficiency,
            "makespan_source": self.makespan_source,
            "contention_applied": self.contention_applied,
            "warmup": self.warmup,
        }

    @staticmethod
    def from_json(doc: dict) -> "PipelineRunReport":
        return PipelineRunReport(
            variant=doc["variant"], n=doc["n"], width=doc["width"], height=doc["height"],
            total_time_us=doc["total_time_us"],
            per_item_c=list(doc["per_item"]["c"]), per_item_m=list(doc["per_item"]["m"]),
            per_item_p=list(doc["per_item"]["p"]),
            transfer_rate_gbps=doc["transfer_rate_gbps"], efficiency=doc["efficiency"],
            makespan_source=doc["makespan_source"], contention_applied=doc["contention_applied"],
            warmup=doc.get("warmup", False), per_item_h=list(doc["per_item"].get("h", [])),
        )

    def csv_row(self) -> list:
        return [self.variant, self.n, self.width, self.height, self.total_time_us,
                f"{self.transfer_rate_gbps:.6f}", f"{self.efficiency:.6f}"]


CSV_HEADER = ["variant", "n", "width", "height", "total_us", "rate_gbps", "efficiency"]


def reports_to_csv(reports: Sequence[PipelineRunReport]) -> str:
    buf = io.StringIO()
    w = csv.writer(buf)
    w.writerow(CSV_HEADER)
    for r in reports:
        w.writerow(r.csv_row())
    return buf.getvalue()


# Longest run streamed item by item.  Longer jobs time this many items through the
# real DAG and extend the per-item costs to n (the grid is still exact, from the
# cycled overlap pass): the reference allows n up to 2^32 - 1, which would otherwise
# mean 6n CUDA events and n uploads for a grid that needs k.
MEASURE_CAP = 1024

MAKESPAN_SOURCES = ("measured", "simulated", "closed-form")


def _report(job: StreamJob, stats, makespan_source: str = "measured") -> PipelineRunReport:
    """Measured per-item costs -> the reference's report (streaming.py:247-309).
    ``stats`` covers ``s`` <= n items; when s < n the per-item lists are cycled to n and
    the measured total is scaled by n / s (steady state), flagged in ``makespan_source``."""
    variant = Variant(job.variant)
    c = [round_half_up(x) for x in stats.copy_us]
    m = [round_half_up(x) for x in stats.xform_us]
    p = [round_half_up(x) for x in stats.kernel_us]
    h = [round_half_up(x) for x in stats.host_us] if variant.coupled_write else []
    s = len(c)
    source = "measured"
    total = max(1, round_half_up(stats.total_us))
    if s < job.n:
        reps = -(-job.n // s)
        c, m, p = ((x * reps)[: job.n] for x in (c, m, p))
        h = (h * reps)[: job.n] if h else h
        total = max(1, round_half_up(stats.total_us * job.n / s))
        source = f"measured ({s} of {job.n} items, scaled)"
    if makespan_source == "closed-form":
        t_dual, t_single = closed_form_times(c, m, p)
        total = max(1, t_single if variant is Variant.ONE_BUFFER_FINAL else t_dual)
        source = "closed-form"
    return PipelineRunReport(
        variant=variant.value, n=job.n, width=job.width, height=job.height,
        total_time_us=total, per_item_c=c, per_item_m=m, per_item_p=p,
        transfer_rate_gbps=job.n * job.payload_bytes / total / 1000.0,
        efficiency=efficiency(c, total), makespan_source=source,
        contention_applied=False, warmup=False, per_item_h=h,
    )


def _validate(job: StreamJob) -> None:
    if not job.surfaces:
        raise StreamError("run_stream needs at least one surface")
    for idx, s in enumerate(job.surfaces):
        if (s.width, s.height) != (job.width, job.height):
            raise StreamError(
                f"surface at index {idx} is {s.width}x{s.height}, "
                f"expected {job.width}x{job.height}"
            )
    if job.n >= (1 << 32):
        raise StreamError("accumulation counts would overflow 32 bits")


def _check_source(job: StreamJob, makespan_source: str) -> None:
    if makespan_source not in MAKESPAN_SOURCES:
        raise StreamError(f"unknown makespan_source {makespan_source!r}")
    if makespan_source == "closed-form" and Variant(job.variant) not in (
            Variant.ONE_BUFFER_FINAL, Variant.TWO_BUFFER_FINAL):
        raise StreamError("closed-form totals are defined for the final strategies only")


def _timed_stream(ens, rasters, job: StreamJob, k: int):
    """Stream min(n, MEASURE_CAP) items (surfaces cycled over k slots) through the
    variant's DAG with the per-item accumulate, measured with CUDA events."""
    s = min(job.n, MEASURE_CAP)
    items = [rasters[i % k] for i in range(s)]
    return ens.stream(items, variant=Variant(job.variant).value, with_kernel=True,
                      reset_counts=True, slot_wrap=k)


def run_stream(job: StreamJob, *, makespan_source: str = "measured"):
    """Stream ``job.n`` rasters (surfaces cycled in order) through the variant's
    pipeline on the GPU and accumulate them.  Returns ``(grid, report)``; the grid is
    bit-identical across strategies (streaming.py:394-433), the report is measured.

    ``makespan_source``: ``"measured"`` (default) and ``"simulated"`` (the reference's
    default name, kept so its callers run unchanged) both report the CUDA-event total of
    the real run; ``"closed-form"`` reports the paper's §7.1 closed form
    (``closed_form_times``) evaluated on the measured per-item costs (final strategies
    only, as in the reference).  ``report.makespan_source`` says which one it is."""
    from .analytics import AccumulationGrid
    from .ensemble import DeviceEnsemble

    _check_source(job, makespan_source)
    _validate(job)
    k = len(job.surfaces)
    with DeviceEnsemble(job.width, job.height, k) as ens:
        stats = _timed_stream(ens, list(job.surfaces), job, k)
        if job.n <= MEASURE_CAP:
            # the grid the per-item kernel[i] nodes accumulated
            counts, _, _ = ens.running_counts(job.n, bins=False, rgba=False)
        else:
            # exact grid in O(k): every slot holds its surface after the timed run;
            # counts = cycles * full + the first `remainder` again (streaming.py:417-431)
            cycles, rem = divmod(job.n, k)
            counts, _, _ = ens.overlap(list(range(k)), cycles=cycles, remainder=rem,
                                       bins=False, rgba=False)
    grid = AccumulationGrid._from_device(job.width, job.height, job.n, counts)
    return grid, _report(job, stats, makespan_source)


def simulate_stream_timing(job: StreamJob, *, makespan_source: str = "measured"
                           ) -> PipelineRunReport:
    """Timing-only run (the reference's ``simulate_stream_timing``,
    streaming.py:324-373, answered by measurement): streams ``job.n`` rasters of the
    job's size — ``job.surfaces`` cycled, or two synthetic flood masks when the job
    carries none — through the variant's DAG and reports the measured pipeline.
    ``makespan_source`` as in ``run_stream``; ``job.profile`` (a cost model in the
    reference) is not consulted."""
    from . import _native as N
    from .ensemble import DeviceEnsemble

    _check_source(job, makespan_source)
    if job.n >= (1 << 32):
        raise StreamError("accumulation counts would overflow 32 bits")
    payload = job.payload_bytes
    if job.surfaces:
        rasters = [getattr(s, "cells", s) for s in job.surfaces]
        bufs = []
    else:
        bufs = [N.PinnedBuffer((payload,)) for _ in range(min(2, job.n))]
        for i, b in enumerate(bufs):
            N.call("fs_synth_host", N.ptr(b.array), 2104, job.width, job.height, 0, job.height,
                   i, 1, 0.02, 0)
        rasters = [b.array for b in bufs]
    try:
        k = len(rasters)
        with DeviceEnsemble(job.width, job.height, k) as ens:
            stats = _timed_stream(ens, rasters, job, k)
    finally:
        for b in bufs:
            b.free()
    return _report(job, stats, makespan_source)


def measure_stream_timing(job: StreamJob) -> PipelineRunReport:
    """Alias of ``simulate_stream_timing`` under the name of what it does."""
    return simulate_stream_timing(job)


def frame_budget_bytes(c_eff: float, m_eff: float, p: float, payload: int,
                       target_fps: int) -> int:
    """The reference's frame budget (streaming.py:436-464): steady-state throughput of
    the two-pair final pipeline times the frame interval, i.e. payload / per-item step
    with step = max(copy, transform + kernel) — in integer µs arithmetic as there."""
    if target_fps < 1:
        raise StreamError("target_fps must be positive")
    step = max(c_eff, m_eff + p)
    frame_us = 1_000_000 // target_fps
    if step <= 0:
        raise StreamError("per-item costs must be positive")
    return int(frame_us * payload // step)


def max_data_per_frame(profile, width: int, height: int, target_fps: int = 10,
                       *, samples: int = 8) -> int:
    """Bytes the two-pair final pipeline sustains per frame at ``target_fps``
    (streaming.py:436-464).  The per-item costs come from ``profile`` when it is a
    measured ``PipelineRunReport`` of this raster size (medians of its per-item c / m /
    p); otherwise (a reference cost-model profile, or None) from a fresh measured
    2b-final run of ``samples`` rasters of this size on the device."""
    if target_fps < 1:
        raise StreamError("target_fps must be positive")
    if width < 1 or height < 1:
        raise StreamError("image dimensions must be positive")
    payload = width * height
    if isinstance(profile, PipelineRunReport):
        if (profile.width, profile.height) != (width, height):
            raise StreamError("report was measured at another raster size")
        c_eff = float(np.median(profile.per_item_c))
        m_eff = float(np.median(profile.per_item_m))
        p = float(np.median(profile.per_item_p))
        return frame_budget_bytes(c_eff, m_eff, p, payload, target_fps)
    job = StreamJob(variant=Variant.TWO_BUFFER_FINAL, n=max(2, samples), width=width,
                    height=height)
    simulate_stream_timing(job)  # warm-up (allocations, first-launch costs)
    rep = simulate_stream_timing(job)
    return max_data_per_frame(rep, width, height, target_fps)
