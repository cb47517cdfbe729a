"""Worker for tests/test_gpu_dist2.py: one rank of a world-2 run on ONE GPU (gloo
process group, FS_DIST_BACKEND=gloo): ShardedEnsemble.run_frames and BandedStream.run
end to end (upload -> recompute -> exchange -> analytics) on this rank's row band,
checked against the oracle on the full rasters.  Writes one JSON verdict per rank to
$FS_DIST2_OUT/rank<r>.json (the oracle is the checker only)."""

import json
import os
import sys
import traceback
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def ensemble(seed, k, h, w):
    rng = np.random.default_rng(seed)
    return [((rng.random((h, w)) < rng.uniform(0.05, 0.95)) *
             rng.integers(1, 256, (h, w))).astype(np.uint8) for _ in range(k)]


def main():
    from oracle import fs_oracle as O
    from paper_2104_14667_b200 import _native as N
    from paper_2104_14667_b200.banded import BandedStream, rank_rows
    from paper_2104_14667_b200.dist import ShardedEnsemble, band

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    N.set_device(0)
    checks = {}
    w, h, k = 301, 67, 37
    sets = [ensemble(s, k, h, w) for s in (11, 12, 13)]
    ids = [f"s{i:04d}" for i in range(k)]
    want = []
    for cells in sets:
        c = O.accumulate(cells, w, h)
        g = O.gram(cells)
        sim = O.similarity_from_gram(g)
        want.append(dict(counts=c, rgba=O.composite(c, k), bins=O.overlap_counts(c.reshape(-1), k),
                         gram=g, sim=sim, out=O.outlier_scores(sim, ids),
                         cl=O.cluster(sim, ids, 0.6)))
    row0, rows = band(h, rank, world)

    # ---- ShardedEnsemble: each frame streams a different ensemble before recomputing
    sh = ShardedEnsemble(w, h, k)
    try:
        assert (sh.row0, sh.rows) == (row0, rows)
        order = [0, 1, 2, 1, 0, 2, 2]

        def upload(f):
            sh.ens.upload(sets[order[f]])

        frames = sh.run_frames(range(k), len(order), tau=0.6, engine="tc-f4", ids=ids,
                               maps_to_host=False, before_frame=upload, depth=3)
        for f, r in enumerate(frames):
            x = want[order[f]]
            assert r["bins"].tolist() == x["bins"].tolist(), f
            assert np.array_equal(r["gram"], x["gram"]), f
            assert r["similarity"].tobytes() == x["sim"].tobytes(), f
            assert r["outliers"] == x["out"], f
            assert r["clusters"] == x["cl"], f
        # maps stay per band: this rank's rows of counts / RGBA
        r = sh.recompute(range(k), tau=0.6, ids=ids)
        x = want[order[-1]]
        assert np.array_equal(r["counts"], x["counts"][row0:row0 + rows])
        assert np.array_equal(r["rgba"], x["rgba"][row0:row0 + rows])
        assert np.array_equal(r["gram"], x["gram"])
        checks["sharded_frames"] = len(frames)
        # the native frame loop with the exchange inside it (fs_comm = NCCL).  NCCL refuses
        # two ranks of one communicator on the same GPU ("Duplicate GPU"); these boxes have
        # one GPU, so that refusal is recorded instead of a result.
        try:
            with sh.pipeline(range(k), tau=0.6, ids=ids) as pipe:
                r = pipe.run(3)
            x = want[order[-1]]
            assert r["bins"].tolist() == x["bins"].tolist()
            assert np.array_equal(r["gram"], x["gram"])
            assert r["similarity"].tobytes() == x["sim"].tobytes()
            assert r["outliers"] == x["out"]
            assert r["clusters"] == x["cl"]
            checks["native_pipeline_nccl"] = "ok"
        except N.NativeError as e:
            if "duplicate" not in str(e).lower() and "invalid usage" not in str(e).lower():
                raise
            checks["native_pipeline_nccl"] = "nccl refused two ranks on one GPU: " + str(e)[:200]
    finally:
        sh.close()

    # ---- BandedStream: this rank's row block, in bands, exchange at the end
    r0, nr = rank_rows(h)
    assert (r0, nr) == (row0, rows)
    cells = sets[1]
    with BandedStream(w, h, k, row0=r0, rows=nr, band_rows=5) as bs:
        out = bs.run([c[r0:r0 + nr] for c in cells], tau=0.6, ids=ids, engine="tc-f4")
    x = want[1]
    assert np.array_equal(out["counts"], x["counts"][r0:r0 + nr])
    assert np.array_equal(out["rgba"], x["rgba"][r0:r0 + nr])
    assert out["bins"].tolist() == x["bins"].tolist()
    assert np.array_equal(out["gram"], x["gram"])
    assert out["clusters"] == x["cl"]
    checks["banded_bands"] = out["stats"].bands
    dist.barrier()
    dist.destroy_process_group()
    return {"rank": rank, "world": world, "rows": [row0, rows], "ok": True, "checks": checks}


if __name__ == "__main__":
    outdir = Path(os.environ["FS_DIST2_OUT"])
    rank = int(os.environ.get("RANK", "0"))
    try:
        res = main()
    except Exception:
        res = {"rank": rank, "ok": False, "error": traceback.format_exc()}
    (outdir / f"rank{rank}.json").write_text(json.dumps(res))
    sys.exit(0 if res["ok"] else 1)
