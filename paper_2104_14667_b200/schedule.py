"""Operation DAG of the streaming strategies (types only).

Same node/graph types as ``floodstream.schedule`` (/root/reference/pkg/src/floodstream/
schedule.py:32-112).  In the reference these graphs are *simulated* against a cost
model; here they are the contract the real upload pipeline implements with CUDA
events (csrc/fs_capi.cu, fs_ensemble_stream), and the timings are measured, so the
discrete-event simulator itself is not part of this package.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum
from typing import Mapping


class Channel(str, Enum):
    TRANSFER = "transfer"
    TRANSFORM = "transform"
    COMPUTE = "compute"


class OpKind(str, Enum):
    HOST_COPY = "host_copy"
    BUFFER_COPY = "buffer_copy"
    BUFFER_TO_IMAGE = "buffer_to_image"
    KERNEL = "kernel"
    CLEAR = "clear"


_CHANNEL_OF = {
    OpKind.HOST_COPY: Channel.TRANSFER,
    OpKind.BUFFER_COPY: Channel.TRANSFER,
    OpKind.BUFFER_TO_IMAGE: Channel.TRANSFORM,
    OpKind.KERNEL: Channel.COMPUTE,
    OpKind.CLEAR: Channel.COMPUTE,
}


class ScheduleError(ValueError):
    """Malformed graph."""


@dataclass(frozen=True)
class OpNode:
    id: str
    kind: OpKind
    payload_bytes: int = 0
    image_dims: tuple[int, int] | None = None
    deps: tuple[str, ...] = ()
    kernel_variant: str = "image1"
    channel: Channel = None  # type: ignore[assignment]

    def __post_init__(self) -> None:
        if self.channel is None:
            object.__setattr__(self, "channel", _CHANNEL_OF[self.kind])
        if self.kind in (OpKind.BUFFER_TO_IMAGE, OpKind.KERNEL) and self.image_dims is None:
            raise ScheduleError(f"node {self.id!r}: {self.kind.value} nodes carry image_dims")
        if self.payload_bytes < 0:
            raise ScheduleError(f"node {self.id!r}: negative payload")


@dataclass
class ScheduleGraph:
    """The DAG of one pipeline run as a node list; listing order doubles as the order in
    which each channel (copy / compute) receives its work."""

    nodes: list[OpNode] = field(default_factory=list)
    pairs: int = 1
    label: str = ""

    def __post_init__(self) -> None:
        self.validate()

    def validate(self) -> None:
        seen: set[str] = set()
        for node in self.nodes:
            if node.id in seen:
                raise ScheduleError(f"duplicate node id {node.id!r}")
            for dep in node.deps:
                if dep not in seen:
                    raise ScheduleError(
                        f"node {node.id!r} depends on {dep!r} which does not precede it"
                    )
            seen.add(node.id)

    def by_id(self) -> Mapping[str, OpNode]:
        return {n.id: n for n in self.nodes}
