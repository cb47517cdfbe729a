"""The native frame loop's exchange (fs_comm_*, NCCL loaded at run time) on one GPU:
a world-1 communicator attached to fs_pipeline makes every frame run the ncclAllReduce of
the [bins | Gram] partials inside the C++ loop; results must equal the loop without it
and the oracle.  (N > 1 needs one GPU per rank: tests/_dist2_worker.py records it.)"""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_world1_comm_pipeline_matches_oracle():
    from oracle import fs_oracle as O
    from paper_2104_14667_b200 import _native as N
    from paper_2104_14667_b200.dist import NativeComm
    from paper_2104_14667_b200.ensemble import DeviceEnsemble

    N.set_device(0)
    rng = np.random.default_rng(7)
    w, h, k = 333, 211, 150
    cells = [((rng.random((h, w)) < rng.uniform(0.1, 0.9)) * 3).astype(np.uint8) for _ in range(k)]
    ids = [f"s{i:03d}" for i in range(k)]
    g = O.gram(cells)
    sim = O.similarity_from_gram(g)
    counts = O.accumulate(cells, w, h)
    comm = NativeComm()
    assert (comm.world, comm.rank) == (1, 0)
    try:
        with DeviceEnsemble(w, h, k) as ens:
            ens.upload(cells)
            with ens.pipeline(range(k), tau=0.7, ids=ids) as p0:
                ref = p0.run(4)
            with ens.pipeline(range(k), tau=0.7, ids=ids, comm=comm) as p1:
                got = p1.run(4)
        for key in ("bins", "gram", "similarity"):
            assert np.array_equal(got[key], ref[key]), key
        assert got["bins"].tolist() == O.overlap_counts(counts.reshape(-1), k).tolist()
        assert np.array_equal(got["gram"], g)
        assert got["similarity"].tobytes() == sim.tobytes()
        assert got["outliers"] == O.outlier_scores(sim, ids)
        assert got["clusters"] == O.cluster(sim, ids, 0.7) == ref["clusters"]
    finally:
        comm.close()


def test_comm_allreduce_world1_is_identity():
    import torch

    from paper_2104_14667_b200 import _native as N
    from paper_2104_14667_b200.dist import NativeComm

    N.set_device(0)
    comm = NativeComm()
    try:
        x = torch.arange(1 << 20, dtype=torch.int64, device="cuda") * 3 - 7
        y = x.clone()
        s = torch.cuda.current_stream()
        N.call("fs_comm_allreduce_i64", comm.handle, C.c_void_p(y.data_ptr()), y.numel(),
               C.c_void_p(s.cuda_stream))
        torch.cuda.synchronize()
        assert torch.equal(x, y)
    finally:
        comm.close()
