"""The N > 1 path on one GPU: torchrun with two ranks over a gloo process group
(FS_DIST_BACKEND=gloo), both ranks on cuda:0, each owning a row band.  Drives
ShardedEnsemble.run_frames (a different ensemble streamed in before each frame, the
exchange, device Jaccard/outliers, host linkage) and BandedStream.run (row block in
bands, exchange at the end) end to end, every product checked against the oracle on the
full rasters (tests/_dist2_worker.py); and bench.py's strong-scaling N = 2 line."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parent.parent


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(args, env_extra, timeout=900):
    env = dict(os.environ, FS_DIST_BACKEND="gloo", **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port())] + args
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=REPO, env=env)


def test_two_ranks_sharded_frames_and_banded_stream(tmp_path):
    r = _torchrun([str(REPO / "tests" / "_dist2_worker.py")], {"FS_DIST2_OUT": str(tmp_path)})
    res = [json.loads((tmp_path / f"rank{i}.json").read_text()) for i in range(2)
           if (tmp_path / f"rank{i}.json").exists()]
    assert len(res) == 2, (r.stdout[-2000:], r.stderr[-4000:])
    for x in res:
        assert x["ok"], x.get("error")
    assert res[0]["rows"][0] == 0 and res[0]["rows"][1] + res[1]["rows"][1] == 67
    assert r.returncode == 0, r.stderr[-2000:]


def test_bench_two_ranks_strong_scaling():
    """bench.py under torchrun (N = 2 ranks on one GPU via gloo): the fixed C1 ensemble
    in two row bands, one JSON line from rank 0 with n_gpus 2 and strong scaling."""
    r = _torchrun([str(REPO / "bench.py"), "--gpus", "2", "--config", "c1", "--steps", "3",
                   "--warmup", "3", "--resident-steps", "8"], {})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.strip().splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["parallelism"] == "row-bands x2"
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 16 * 1024 * 1024
    assert line["clusters"] is not None
