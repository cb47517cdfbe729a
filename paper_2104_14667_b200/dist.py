"""Multi-GPU sharding of the overlap path: one process per GPU, row bands of every mask.

SURVEY §8(e): the per-pixel products (counts, histogram, composite) have no stencil
and no halo, and the Gram is a sum over pixels, so the ensemble shards by spatial ROW
BANDS — rank r owns rows [row0_r, row0_r + rows_r) of every mask (one contiguous H2D
per mask, one contiguous slice of every output).  The only exchange is one bucketed
``all_reduce(sum)`` of the int64 partials [histogram | Gram] (8 (n+1) + 8 k^2 bytes;
8 MiB at 1024 masks); counts/RGBA bands stay on their rank or are gathered to rank 0
(``gather_rows``).  Jaccard, outliers and clusters then run on the exact summed Gram,
so every rank (or rank 0 alone) produces results bit-identical to one GPU.

Reference: the partitioning ``north_star`` prescribes ("spatial tiles sharded across
GPUs ... partial Gram matrices summed with NCCL allreduce"); the single-device
semantics are fs/analytics.py:106-240 and fs/service.py:143-175.

The collective helpers take torch tensors and a process group, so the same code runs
over NCCL on B200s and over gloo on CPU in the tests.
"""

from __future__ import annotations

import numpy as np

from . import _native as N


def band(height: int, rank: int, world: int) -> tuple[int, int]:
    """(row0, rows) of rank's band: rows split as evenly as possible, lower ranks first."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(int(height), int(world))
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


def partial_layout(k: int, n_inputs: int | None = None) -> tuple[int, int]:
    """Offsets of the bucketed int64 partial buffer: bins at [0, n+1), Gram after."""
    nb = (k if n_inputs is None else n_inputs) + 1
    return nb, nb + k * k


def allreduce_partials(buf, group=None) -> None:
    """Sum the bucketed int64 [bins | Gram] partial buffer over all ranks, in place.
    One collective per recompute (launch latency, not link count, dominates at 8 MiB)."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)


def gather_rows(local, height: int, group=None, dst: int = 0):
    """Assemble per-rank row bands (first dim = rows of the band) into the full raster on
    ``dst`` (other ranks get None).  Bands are padded to the largest band for the
    collective and trimmed on arrival."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    rmax = band(height, 0, world)[1]
    pad = torch.zeros((rmax,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, parts, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([parts[r][: band(height, r, world)[1]] for r in range(world)], dim=0)


class NativeComm:
    """An NCCL communicator inside libfloodstream (fs_comm_*) for this rank's device, so
    the native frame loop (fs_pipeline_run) can sum the bands' [bins | Gram] partials
    itself.  Rank 0 draws the NCCL unique id; it reaches the other ranks through the
    torch.distributed group (any backend) — torch stays plumbing, the per-frame exchange
    runs in C++ on the ensemble stream."""

    def __init__(self, group=None, device: int | None = None):
        import ctypes as C

        import torch
        import torch.distributed as dist

        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = (C.c_uint8 * 128)()
        err = None
        if self.rank == 0:
            try:
                N.call("fs_comm_unique_id", uid)
            except (RuntimeError, ValueError) as exc:
                err = str(exc)
        if self.world > 1:
            # every rank learns rank 0's outcome, so a failure cannot leave the others
            # waiting inside the collective init
            obj = [None if err else bytes(uid)]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0)
                                       if group is not None else 0, group=group)
            if obj[0] is None:
                raise RuntimeError(f"fs_comm_unique_id failed on rank 0: {err or '?'}")
            uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        elif err:
            raise RuntimeError(err)
        dev = torch.cuda.current_device() if device is None else int(device)
        N.set_device(dev)
        h = C.c_void_p()
        N.call("fs_comm_create", uid, self.world, self.rank, C.byref(h))
        self._h = h

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            N.load().fs_comm_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class ShardedEnsemble:
    """This rank's row band of a bit-packed ensemble plus the exchange step.

    ``recompute()`` runs the fused overlap pass and the Gram on this rank's band with
    device outputs written straight into one bucketed buffer, sums the partials with a
    single all-reduce on the ensemble's stream, and returns host (numpy) results:
    this band's counts and RGBA, and the GLOBAL histogram and Gram.
    """

    def __init__(self, width: int, height: int, capacity: int, *, group=None,
                 device: int | None = None):
        import torch
        import torch.distributed as dist

        from .ensemble import DeviceEnsemble

        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.width, self.height = int(width), int(height)
        self.row0, self.rows = band(height, self.rank, self.world)
        dev = torch.cuda.current_device() if device is None else int(device)
        self.device = torch.device("cuda", dev)
        self.ens = DeviceEnsemble(width, height, capacity, row0=self.row0, rows=self.rows,
                                  device=dev)
        self.stream = torch.cuda.Stream(device=self.device)
        self.ens.use_stream(self.stream.cuda_stream)
        self.capacity = int(capacity)
        self._bufs: dict = {}

    def close(self) -> None:
        if getattr(self, "_pool", None) is not None:
            self._pool.shutdown(wait=True)
            self._pool = None
        if getattr(self, "_comm", None) is not None:
            self._comm.close()
            self._comm = None
        self.ens.close()

    def pipeline(self, slots=None, *, tau: float = 0.8, engine: str = "auto", depth: int = 3,
                 ids=None):
        """The native frame loop (fs_pipeline_*) on this rank's band with the per-frame
        all-reduce of the [bins | Gram] partials inside it (fs_comm, NCCL): every rank
        ends each frame with the GLOBAL histogram, Gram, Jaccard, outliers and clusters."""
        if getattr(self, "_comm", None) is None:
            self._comm = NativeComm(self.group, device=self.device.index)
        return self.ens.pipeline(slots, tau=tau, engine=engine, depth=depth, ids=ids,
                                 comm=self._comm)

    def _make_buffers(self, k: int, n_inputs: int, maps: bool):
        import torch

        nb, total = partial_layout(k, n_inputs)
        px = self.rows * self.width
        b = dict(nb=nb, k=k,
                 part=torch.empty(total, dtype=torch.int64, device=self.device),
                 counts=torch.empty(px, dtype=torch.int32, device=self.device),
                 rgba=torch.empty(px * 4, dtype=torch.uint8, device=self.device),
                 h_part=torch.empty(total, dtype=torch.int64).pin_memory(),
                 # Jaccard matrix + outlier scores, computed on the device from the
                 # summed Gram (fs_similarity_outliers_device)
                 sim=torch.empty(k * k, dtype=torch.float64, device=self.device),
                 scores=torch.empty(max(k, 1), dtype=torch.float64, device=self.device),
                 h_sim=torch.empty(k * k, dtype=torch.float64).pin_memory(),
                 h_scores=torch.empty(max(k, 1), dtype=torch.float64).pin_memory(),
                 event=torch.cuda.Event())
        if maps:
            b["h_counts"] = torch.empty(px, dtype=torch.int32).pin_memory()
            b["h_rgba"] = torch.empty(px * 4, dtype=torch.uint8).pin_memory()
            b["event_maps"] = torch.cuda.Event()
        return b

    def _enqueue(self, sl: np.ndarray, b, *, engine: str, cycles: int = 1, remainder: int = 0,
                 maps_to_host: bool = False):
        """Overlap + Gram into the bucketed buffer, one all-reduce, D2H of the partials
        (and of this band's maps when asked), then an event — all on the ensemble
        stream, nothing synchronised."""
        import torch

        part = b["part"]
        if cycles == 1 and remainder == 0:
            # one call: fused overlap + Gram when the engine and k allow it
            self.ens.products(sl, engine=engine, out_counts=b["counts"].data_ptr(),
                              out_rgba=b["rgba"].data_ptr(), out_bins=part.data_ptr(),
                              out_gram=part.data_ptr() + b["nb"] * 8, device_outputs=True)
        else:
            self.ens.overlap(sl, cycles=cycles, remainder=remainder,
                             out_counts=b["counts"].data_ptr(), out_rgba=b["rgba"].data_ptr(),
                             out_bins=part.data_ptr(), device_outputs=True)
            self.ens.gram(sl, engine=engine, out=part.data_ptr() + b["nb"] * 8,
                          device_outputs=True)
        if maps_to_host:
            # the maps' D2H (8 B/px) runs on a side stream: PCIe is full duplex, so it
            # overlaps the next frame's H2D upload instead of delaying it
            if getattr(self, "d2h_stream", None) is None:
                self.d2h_stream = torch.cuda.Stream(device=self.device)
            ready = torch.cuda.Event()
            ready.record(self.stream)
            self.d2h_stream.wait_event(ready)
            with torch.cuda.stream(self.d2h_stream):
                b["h_counts"].copy_(b["counts"], non_blocking=True)
                b["h_rgba"].copy_(b["rgba"], non_blocking=True)
                b["event_maps"].record(self.d2h_stream)
        # the exchange and the small D2H of the partials run on a side stream, so the
        # next frame's recompute starts right behind this one's kernels (a slot's
        # buffers are reused only after _finish saw its event)
        if getattr(self, "x_stream", None) is None:
            self.x_stream = torch.cuda.Stream(device=self.device)
        done = torch.cuda.Event()
        done.record(self.stream)
        self.x_stream.wait_event(done)
        with torch.cuda.stream(self.x_stream):
            allreduce_partials(part, self.group)
            k = b["k"]
            N.call("fs_similarity_outliers_device", part.data_ptr() + b["nb"] * 8, k,
                   b["sim"].data_ptr(), b["scores"].data_ptr() if k >= 2 else None,
                   self.x_stream.cuda_stream)
            b["h_part"].copy_(part, non_blocking=True)
            b["h_sim"].copy_(b["sim"], non_blocking=True)
            b["h_scores"].copy_(b["scores"], non_blocking=True)
            b["event"].record(self.x_stream)

    def _finish(self, b, ids, tau: float, analytics: bool, maps_to_host: bool, free=None):
        """Wait for a frame's D2H, copy out its histogram and Gram, run the host
        analytics; then hand the buffer slot back (``free``).  Runs on a pool thread:
        the C analytics release the GIL, so frames' host work overlaps each other and
        the main thread's enqueueing."""
        from .analytics import cluster_from_similarity

        try:
            b["event"].synchronize()
            part = b["h_part"].numpy()
            k = b["k"]
            out = {"bins": part[: b["nb"]].copy(), "gram": part[b["nb"]:].reshape(k, k).copy()}
            # copy the frame's analytics out of the pinned slot BEFORE the slot can be
            # handed back: the main thread reuses it for frame f + depth, whose D2H
            # would otherwise land under these reads
            sim = b["h_sim"].numpy().reshape(k, k).copy() if analytics else None
            scores = b["h_scores"].numpy()[:k].copy() if (analytics and k >= 2) else None
            if maps_to_host:
                b["event_maps"].synchronize()
                # views of the pinned slot: valid until the slot is reused (``depth``
                # frames later) — copy them to keep them longer
                out["counts"] = b["h_counts"].numpy().view(np.uint32).reshape(self.rows, self.width)
                out["rgba"] = b["h_rgba"].numpy().reshape(self.rows, self.width, 4)
            elif free is not None:
                free.set()
                free = None
            if analytics:
                out["similarity"] = sim
                out["outliers"] = ({sid: scores[i] for i, sid in enumerate(ids)}
                                   if k >= 2 else None)
                out["clusters"] = cluster_from_similarity(sim, ids, tau)
            return out
        finally:
            if free is not None:
                free.set()

    def _executor(self, workers: int):
        from concurrent.futures import ThreadPoolExecutor

        if getattr(self, "_pool", None) is None or self._pool_workers != workers:
            if getattr(self, "_pool", None) is not None:
                self._pool.shutdown(wait=True)
            self._pool = ThreadPoolExecutor(max_workers=workers, thread_name_prefix="fs-frames")
            self._pool_workers = workers
        return self._pool

    def run_frames(self, slots, n_frames: int, *, tau: float = 0.8, engine: str = "auto",
                   ids=None, maps_to_host: bool = False, analytics_ranks: str = "all",
                   before_frame=None, keep: bool = True, depth: int = 3):
        """``n_frames`` full recomputes of the working set, pipelined over a ring of
        ``depth`` frame buffers: the main thread keeps enqueueing device work
        (overlap + Gram, all-reduce, D2H) while pool threads wait for earlier frames and
        run their host analytics (Jaccard, outliers, clusters) — the interactive
        recompute loop of service.py:143-175 at GPU rate.  ``before_frame(f)`` runs first
        in each frame (e.g. streaming new rasters in).  Results come back in frame
        order (only the last one unless ``keep``)."""
        import threading
        from collections import deque

        sl = np.ascontiguousarray(np.asarray(list(slots), dtype=np.uint32))
        k = int(sl.size)
        ids = list(ids) if ids is not None else [f"s{i:04d}" for i in sl.tolist()]
        depth = max(2, int(depth))
        # one ring of frame buffers per (k, maps, depth), kept across calls: pinned
        # host slots cost milliseconds per MiB to allocate, so switching between map and
        # map-less frames must not reallocate them (at most two rings are kept)
        key = (k, maps_to_host, depth)
        if key not in self._bufs:
            if len(self._bufs) >= 2:
                self._bufs.pop(next(iter(self._bufs)))
            ring = {"b": [self._make_buffers(k, k, maps_to_host) for _ in range(depth)],
                    "free": [threading.Event() for _ in range(depth)]}
            for e in ring["free"]:
                e.set()
            self._bufs[key] = ring
        bufs, free = self._bufs[key]["b"], self._bufs[key]["free"]
        pool = self._executor(depth)
        # "all": every rank runs the host analytics; "root": rank 0 only; "none": skip
        analytics = analytics_ranks == "all" or (analytics_ranks == "root" and self.rank == 0)
        results, futs = [], deque()
        for f in range(n_frames):
            if before_frame is not None:
                before_frame(f)
            i = f % depth
            free[i].wait()
            free[i].clear()
            self._enqueue(sl, bufs[i], engine=engine, maps_to_host=maps_to_host)
            futs.append(pool.submit(self._finish, bufs[i], ids, tau, analytics, maps_to_host,
                                    free[i]))
            while futs and futs[0].done():
                r = futs.popleft().result()
                if keep:
                    results.append(r)
        while futs:
            r = futs.popleft().result()
            if keep or not futs:
                results.append(r)
        return results if keep else results[-1:]

    def recompute(self, slots, *, tau: float = 0.8, engine: str = "auto", ids=None):
        """One full recompute: this band's counts/RGBA + the global histogram, Gram,
        similarity, outliers and clusters (identical on every rank)."""
        r = self.run_frames(slots, 1, tau=tau, engine=engine, ids=ids, maps_to_host=True)[0]
        r["counts"], r["rgba"] = r["counts"].copy(), r["rgba"].copy()
        return r
