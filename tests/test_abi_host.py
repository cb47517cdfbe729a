"""CPU tests of the C-ABI boundary (no GPU needed).

* libfloodstream loads and exports every entry point include/floodstream.h declares,
  and the ctypes table binds each of them;
* device entry points fail loudly (RuntimeError, never a silent host fallback) when no
  CUDA device is visible;
* the exact host-side analytics behind the boundary (Jaccard from the Gram, outlier
  reduction, complete-linkage clustering; analytics.py:165-240 of the reference) agree
  with the oracle on seeded inputs, including tie-heavy similarity matrices.
"""

import re
from pathlib import Path

import numpy as np
import pytest

from oracle import fs_oracle as O

REPO = Path(__file__).resolve().parent.parent
HEADER = REPO / "include" / "floodstream.h"


def header_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fs_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = header_functions()
    for required in ("fs_accumulate_into", "fs_overlap_counts", "fs_pair_counts",
                     "fs_composite_fill", "fs_ensemble_overlap", "fs_ensemble_gram"):
        assert required in names


def test_library_exports_every_header_symbol():
    from paper_2104_14667_b200 import _native as N

    lib = N.load()
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, f"declared but not exported: {missing}"


def test_ctypes_table_covers_header():
    from paper_2104_14667_b200 import _native as N

    assert set(header_functions()) == set(N.EXPORTED_SYMBOLS)


def test_library_is_built_for_sm100a():
    """The fatbin carries sm_100a SASS (cuobjdump is part of the toolkit here)."""
    import shutil
    import subprocess

    from paper_2104_14667_b200 import _native as N

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(tool).exists():
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", str(N.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_version():
    from paper_2104_14667_b200 import _native as N

    assert N.load().fs_abi_version() == 1


def test_device_calls_fail_loudly_without_gpu():
    from paper_2104_14667_b200 import _kernels_cuda as K
    from paper_2104_14667_b200 import _native as N

    if N.device_count() > 0:
        pytest.skip("a GPU is visible")
    counts = np.zeros(64, np.uint32)
    with pytest.raises(RuntimeError):
        K.accumulate_into(counts, np.ones(64, np.uint8))
    with pytest.raises(RuntimeError):
        K.pair_counts(np.ones(64, np.uint8), np.ones(64, np.uint8))


def test_cpu_backends_are_refused():
    from paper_2104_14667_b200.backends import select_backend

    with pytest.raises(RuntimeError):
        select_backend("numpy")
    with pytest.raises(ValueError):
        select_backend("nope")
    assert select_backend("cuda").NAME == "cuda"


# ---- exact host analytics behind the boundary ----------------------------------------

def random_gram(rng, k, pixels):
    cells = [(rng.random(pixels) < rng.uniform(0.05, 0.95)).astype(np.uint8) for _ in range(k)]
    if k > 2:
        cells[1] = np.zeros(pixels, np.uint8)  # empty surface: union 0 with another empty
        cells[2] = np.zeros(pixels, np.uint8)
    return O.gram(cells)


@pytest.mark.parametrize("seed", range(6))
def test_similarity_from_gram_matches_oracle(seed):
    from paper_2104_14667_b200.analytics import similarity_from_gram

    rng = np.random.default_rng(seed)
    g = random_gram(rng, int(rng.integers(1, 40)), 777)
    got = similarity_from_gram(g)
    want = O.similarity_from_gram(g)
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("seed", range(6))
def test_outliers_match_oracle_bitwise(seed):
    from paper_2104_14667_b200.analytics import outliers_from_similarity

    rng = np.random.default_rng(100 + seed)
    k = int(rng.integers(2, 60))
    sim = O.similarity_from_gram(random_gram(rng, k, 513))
    ids = [f"m{i:03d}" for i in range(k)]
    got = outliers_from_similarity(sim, ids)
    want = O.outlier_scores(sim, ids)
    assert {s: float(v).hex() for s, v in got.items()} == {s: float(v).hex() for s, v in want.items()}


def test_outliers_need_two():
    from paper_2104_14667_b200.analytics import AnalyticsError, outliers_from_similarity

    with pytest.raises(AnalyticsError, match="at least two"):
        outliers_from_similarity(np.ones((1, 1)), ["a"])


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("tau", [0.05, 0.3, 0.5, 0.8, 1.0])
def test_clustering_matches_oracle(seed, tau):
    from paper_2104_14667_b200.analytics import cluster_from_similarity

    rng = np.random.default_rng(1000 + seed)
    k = int(rng.integers(1, 24))
    if seed % 3 == 0:
        # tie-heavy: similarities on a coarse grid, shuffled ids (lexical tie-break)
        sim = rng.integers(0, 5, (k, k)) / 4.0
        sim = np.triu(sim, 1)
        sim = sim + sim.T + np.eye(k)
    else:
        sim = O.similarity_from_gram(random_gram(rng, k, 257))
    ids = [f"s{v:03d}" for v in rng.permutation(k)]
    assert cluster_from_similarity(sim, ids, tau) == O.cluster(sim, ids, tau)


def test_clustering_duplicate_ids():
    from paper_2104_14667_b200.analytics import cluster_from_similarity

    sim = np.array([[1.0, 0.9, 0.9], [0.9, 1.0, 0.9], [0.9, 0.9, 1.0]])
    ids = ["b", "a", "a"]
    assert cluster_from_similarity(sim, ids, 0.95) == O.cluster(sim, ids, 0.95)
    assert cluster_from_similarity(sim, ids, 0.5) == O.cluster(sim, ids, 0.5)


def test_clustering_reference_known_answers():
    """test_analytics.py:182-239 of the reference: s1/s2 at J = 0.9, s3 far away; the
    a-b-c chain where complete linkage refuses the second merge."""
    from paper_2104_14667_b200.analytics import cluster_from_similarity

    base = np.zeros(64, np.uint8)
    s1, s2, s3 = base.copy(), base.copy(), base.copy()
    s1[0:10] = 1
    s2[0:9] = 1
    s3[[0, 1, 2, 20, 21, 22, 23, 24, 25, 26]] = 1
    sim = O.similarity_from_gram(O.gram([s1, s2, s3]))
    assert cluster_from_similarity(sim, ["s1", "s2", "s3"], 0.8) == [["s1", "s2"], ["s3"]]
    assert cluster_from_similarity(sim, ["s1", "s2", "s3"], 0.01) == [["s1", "s2", "s3"]]
    rev = sim[::-1, ::-1].copy()
    assert cluster_from_similarity(rev, ["s3", "s2", "s1"], 0.8) == [["s1", "s2"], ["s3"]]
    b100 = np.zeros(100, np.uint8)
    a, b, c = b100.copy(), b100.copy(), b100.copy()
    a[0:10] = 1
    b[1:11] = 1
    c[2:12] = 1
    sim = O.similarity_from_gram(O.gram([a, b, c]))
    cl = cluster_from_similarity(sim, ["a", "b", "c"], 0.8)
    assert len(cl) == 2 and (["c"] in cl or ["a"] in cl)
    assert cl == O.cluster(sim, ["a", "b", "c"], 0.8)


def test_tau_validation():
    from paper_2104_14667_b200.analytics import AnalyticsError, cluster_from_similarity

    for tau in (0.0, 1.5, -1.0):
        with pytest.raises(AnalyticsError, match="tau"):
            cluster_from_similarity(np.ones((1, 1)), ["x"], tau)
    assert cluster_from_similarity(np.ones((1, 1)), ["only"], 0.8) == [["only"]]


def test_clustering_c3_shape_blocks():
    """32 prototypes x 32 members block structure (config c3's expected answer)."""
    from paper_2104_14667_b200.analytics import cluster_from_similarity

    k, m = 1024, 32
    proto = np.arange(k) // m
    rng = np.random.default_rng(7)
    noise = rng.integers(0, 1000, (k, k)) / 1e5
    noise = np.triu(noise, 1)
    noise = noise + noise.T
    sim = np.where(proto[:, None] == proto[None, :], 0.9, 0.3) + noise
    np.fill_diagonal(sim, 1.0)
    ids = [f"s{i:04d}" for i in range(k)]
    cl = cluster_from_similarity(sim, ids, 0.8)
    assert len(cl) == 32 and all(len(c) == 32 for c in cl)
    assert cl[0] == ids[:32]


@pytest.mark.parametrize("seed", range(6))
def test_clustering_components_with_cross_block_ties(seed):
    """Complete linkage runs per connected component of {sim >= tau}; blocks whose
    internal similarities tie exactly with other blocks' (and duplicated ids across
    blocks) must still give the reference's lists."""
    from paper_2104_14667_b200.analytics import cluster_from_similarity

    rng = np.random.default_rng(77 + seed)
    nb, m = int(rng.integers(2, 7)), int(rng.integers(1, 6))
    k = nb * m
    levels = np.array([0.8, 0.85, 0.9, 1.0])
    sim = np.full((k, k), 0.1)
    for b in range(nb):
        blk = rng.choice(levels, (m, m))
        blk = np.triu(blk, 1)
        sim[b * m:(b + 1) * m, b * m:(b + 1) * m] = blk + blk.T
    # a few bridges above tau join blocks into larger components
    for _ in range(int(rng.integers(0, 3))):
        i, j = rng.integers(0, k, 2)
        if i != j:
            sim[i, j] = sim[j, i] = 0.85
    np.fill_diagonal(sim, 1.0)
    perm = rng.permutation(k)
    sim = sim[np.ix_(perm, perm)]
    ids = [f"s{v % (k - 1 if seed % 2 else k):03d}" for v in rng.permutation(k)]
    for tau in (0.8, 0.85, 0.9, 1.0):
        assert cluster_from_similarity(sim, ids, tau) == O.cluster(sim, ids, tau)


def test_bench_cli_fails_cleanly_without_gpu():
    """python -m paper_2104_14667_b200 bench <suite> (the reference's `bench` suites,
    fs/cli.py:72-150): exit code 2 and a message when no device is visible."""
    import subprocess
    import sys

    from paper_2104_14667_b200 import _native as N

    if N.device_count() > 0:
        pytest.skip("a GPU is visible")
    r = subprocess.run([sys.executable, "-m", "paper_2104_14667_b200", "bench", "backends",
                        "--pixels", "4096", "--surfaces", "2", "--repeats", "1"],
                       capture_output=True, text=True, cwd=REPO, timeout=120)
    assert r.returncode == 2 and r.stderr.startswith("error:")


@pytest.mark.parametrize("seed", range(30))
def test_clustering_duplicate_ids_list_order(seed):
    """Duplicate ids: clusters with the same first id keep the reference's list order
    (smallest member index first, fs/analytics.py:220-226) — e.g. ids a b x x y with
    sim(0,1)=.9, sim(1,3)=.85, sim(3,4)=.95 gives [[a, b], [x], [x, y]]."""
    from paper_2104_14667_b200.analytics import cluster_from_similarity

    ids = ["a", "b", "x", "x", "y"]
    s = np.eye(5)
    for i, j, v in [(0, 1, .9), (1, 3, .85), (3, 4, .95)]:
        s[i, j] = s[j, i] = v
    assert cluster_from_similarity(s, ids, 0.8) == [["a", "b"], ["x"], ["x", "y"]]
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 30))
    x = np.round(rng.random((n, n)) * 5) / 5
    s = np.minimum(x, x.T)
    np.fill_diagonal(s, 1.0)
    ids = [str(v) for v in rng.integers(0, max(2, n // 3), n)]
    tau = float(rng.choice([0.2, 0.4, 0.6, 0.8]))
    assert cluster_from_similarity(s, ids, tau) == O.cluster(s, ids, tau)


def test_comm_unique_id_without_gpu_and_create_needs_a_device():
    """fs_comm_unique_id only asks libnccl for a bootstrap id (works on CPU); creating a
    communicator needs a CUDA device and fails loudly without one."""
    import ctypes as C

    from paper_2104_14667_b200 import _native as N

    uid = (C.c_uint8 * 128)()
    N.call("fs_comm_unique_id", uid)
    assert any(bytes(uid))
    h = C.c_void_p()
    with pytest.raises((RuntimeError, ValueError)):
        N.call("fs_comm_create", uid, 1, 0, C.byref(h))
    with pytest.raises(ValueError):
        N.call("fs_comm_create", uid, 2, 5, C.byref(h))
