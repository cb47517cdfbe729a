"""Multi-process (world_size 2, gloo on CPU) tests of the row-band sharding.

Each rank computes its band's partial histogram / Gram / counts with the oracle (the
device kernels are covered by the GPU parity tests; here the point is the sharding
arithmetic and the exchange step of paper_2104_14667_b200.dist), then the SAME
collective helpers the NCCL path uses sum and gather them.  Rank 0 must reproduce the
single-process oracle exactly.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2104_14667_b200.dist import allreduce_partials, band, gather_rows, partial_layout


def test_band_partitions_rows():
    for h in (1, 2, 3, 7, 8, 1000, 8192, 8193):
        for world in (1, 2, 3, 4, 8):
            spans = [band(h, r, world) for r in range(world)]
            assert spans[0][0] == 0
            for (a0, an), (b0, _) in zip(spans, spans[1:]):
                assert a0 + an == b0
            assert spans[-1][0] + spans[-1][1] == h
            sizes = [s[1] for s in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        band(10, 2, 2)


def test_partial_layout():
    assert partial_layout(4) == (5, 21)
    assert partial_layout(4, n_inputs=9) == (10, 26)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, width, height, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import fs_oracle as O

        rng = np.random.default_rng(42)
        cells = [(rng.random((height, width)) < rng.uniform(0.1, 0.9)) *
                 rng.integers(1, 256, (height, width)) for _ in range(k)]
        cells = [c.astype(np.uint8) for c in cells]
        row0, rows = band(height, rank, world)
        mine = [c[row0:row0 + rows] for c in cells]
        counts = O.accumulate(mine, width, rows)
        nb, total = partial_layout(k)
        part = torch.zeros(total, dtype=torch.int64)
        part[:nb] = torch.from_numpy(O.overlap_counts(counts.reshape(-1), k))
        part[nb:] = torch.from_numpy(O.gram(mine).reshape(-1))
        allreduce_partials(part)
        full_counts = gather_rows(torch.from_numpy(counts.view(np.int32)), height)
        rgba = gather_rows(torch.from_numpy(O.composite(counts, k)), height)
        if rank == 0:
            want_counts = O.accumulate(cells, width, height)
            ok = {
                "bins": part[:nb].tolist() == O.overlap_counts(want_counts.reshape(-1), k).tolist(),
                "gram": np.array_equal(part[nb:].numpy().reshape(k, k), O.gram(cells)),
                "counts": np.array_equal(full_counts.numpy().view(np.uint32), want_counts),
                "rgba": np.array_equal(rgba.numpy(), O.composite(want_counts, k)),
            }
            q.put(ok)
        else:
            q.put(None if full_counts is None else "non-dst got data")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("width,height,k", [(37, 29, 6), (64, 3, 3), (16, 1, 2)])
def test_two_rank_bands_reproduce_single_process(width, height, k):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, width, height, k, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    oks = [r for r in results if isinstance(r, dict)]
    assert len(oks) == 1 and all(oks[0].values()), oks
    assert all(r is None for r in results if not isinstance(r, dict))


# ---- banded (spatial + iterative) streaming: rank rows, bands, the exchange -----------

def test_split_bands():
    from paper_2104_14667_b200.banded import split_bands

    assert split_bands(10, 4) == [(0, 4), (4, 4), (8, 2)]
    assert split_bands(8, 8) == [(0, 8)]
    assert split_bands(0, 3) == []
    with pytest.raises(ValueError):
        split_bands(5, 0)


def _banded_worker(rank, world, port, width, height, k, band_rows, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import fs_oracle as O
        from paper_2104_14667_b200.banded import _allreduce_cpu_or_device, rank_rows, split_bands

        rng = np.random.default_rng(7)
        cells = [(rng.random((height, width)) < 0.4).astype(np.uint8) for _ in range(k)]
        row0, rows = rank_rows(height)
        nb, total = partial_layout(k)
        part = torch.zeros(total, dtype=torch.int64)
        counts = np.zeros((rows, width), np.uint32)
        for r0, n in split_bands(rows, band_rows):  # the per-band partials of run()
            mine = [c[row0 + r0:row0 + r0 + n] for c in cells]
            bc = O.accumulate(mine, width, n)
            counts[r0:r0 + n] = bc
            part[:nb] += torch.from_numpy(O.overlap_counts(bc.reshape(-1), k))
            part[nb:] += torch.from_numpy(O.gram(mine).reshape(-1))
        _allreduce_cpu_or_device(part, None, None)
        full = gather_rows(torch.from_numpy(counts.view(np.int32)), height)
        if rank == 0:
            want = O.accumulate(cells, width, height)
            q.put({"bins": part[:nb].tolist() == O.overlap_counts(want.reshape(-1), k).tolist(),
                   "gram": np.array_equal(part[nb:].numpy().reshape(k, k), O.gram(cells)),
                   "counts": np.array_equal(full.numpy().view(np.uint32), want)})
        else:
            q.put(None)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("width,height,k,band_rows", [(33, 41, 5, 6), (16, 3, 2, 1)])
def test_two_rank_banded_partials_reproduce_single_process(width, height, k, band_rows):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_banded_worker,
                         args=(r, world, port, width, height, k, band_rows, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    oks = [r for r in results if isinstance(r, dict)]
    assert len(oks) == 1 and all(oks[0].values()), oks
