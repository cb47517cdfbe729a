"""paper_2104_14667_b200 — B200-native flood-ensemble overlap path (arXiv 2104.14667).

Drop-in for the hot path of the reference package ``floodstream``
(/root/reference/pkg/src/floodstream/__init__.py:74-133): the raster type, the
ensemble analytics (overlap counts, histogram, composite, Jaccard, similarity,
clusters, outliers), the streaming strategies and their reports — computed by
hand-written sm_100a kernels in ``_lib/libfloodstream.so`` through a C ABI
(``include/floodstream.h``).  There is no CPU fallback.
"""

from .analytics import (
    AccumulationGrid,
    AnalyticsError,
    CompositeImage,
    KERNEL_VARIANTS,
    OverlapHistogram,
    accumulate,
    cluster_from_similarity,
    cluster_surfaces,
    composite_map,
    jaccard,
    outlier_scores,
    outliers_from_similarity,
    overlap_histogram,
    similarity_from_gram,
    similarity_matrix,
)
from .backends import available_backends, select_backend
from .banded import BandedStream
from .engine import AnalyticsEngine, EngineSnapshot, ResidentEngine, SlotMap
from .ensemble import DeviceEnsemble, Snapshot, StreamStats
from .ingest import stream_files
from .rasters import RasterError, RasterSurface, load_surface
from .schedule import Channel, OpKind, OpNode, ScheduleError, ScheduleGraph
from .streaming import (
    PipelineRunReport,
    StreamError,
    StreamJob,
    Variant,
    build_schedule,
    closed_form_times,
    efficiency,
    frame_budget_bytes,
    max_data_per_frame,
    measure_stream_timing,
    reports_to_csv,
    run_stream,
    simulate_stream_timing,
)

__version__ = "0.1.0"

__all__ = [
    "AccumulationGrid",
    "AnalyticsEngine",
    "AnalyticsError",
    "BandedStream",
    "Channel",
    "CompositeImage",
    "DeviceEnsemble",
    "EngineSnapshot",
    "KERNEL_VARIANTS",
    "OpKind",
    "OpNode",
    "OverlapHistogram",
    "PipelineRunReport",
    "RasterError",
    "RasterSurface",
    "ResidentEngine",
    "ScheduleError",
    "ScheduleGraph",
    "SlotMap",
    "Snapshot",
    "StreamError",
    "StreamJob",
    "StreamStats",
    "Variant",
    "accumulate",
    "available_backends",
    "build_schedule",
    "closed_form_times",
    "cluster_from_similarity",
    "cluster_surfaces",
    "composite_map",
    "efficiency",
    "frame_budget_bytes",
    "jaccard",
    "load_surface",
    "max_data_per_frame",
    "measure_stream_timing",
    "outlier_scores",
    "outliers_from_similarity",
    "overlap_histogram",
    "reports_to_csv",
    "run_stream",
    "select_backend",
    "similarity_from_gram",
    "similarity_matrix",
    "simulate_stream_timing",
    "stream_files",
]
