"""GPU parity of the spatial + iterative (banded) streaming path and the device
synthesiser, against the oracle (bit-exact maps, histogram and Gram; identical
outliers and clusters)."""

import numpy as np
import pytest

from oracle import fs_oracle as O

pytestmark = pytest.mark.gpu

from paper_2104_14667_b200 import _native as N  # noqa: E402
from paper_2104_14667_b200.banded import BandedStream, default_band_rows  # noqa: E402
from paper_2104_14667_b200.synth import synth_cells, synth_cells_gpu  # noqa: E402


def _expect(cells, w, h, k, ids, tau=0.8):
    counts = O.accumulate(cells, w, h)
    g = O.gram(cells)
    sim = O.similarity_from_gram(g)
    return (counts, g, sim, O.cluster(sim, ids, tau),
            O.outlier_scores(sim, ids) if k >= 2 else None)


@pytest.mark.parametrize("w,h,k,band_rows", [(1000, 333, 24, 50), (96, 64, 3, 64),
                                             (257, 129, 40, 1), (4096, 40, 70, 17),
                                             (160, 37, 300, 8), (33, 9, 1, 4)])
def test_banded_matches_oracle(w, h, k, band_rows):
    cells = [synth_cells(w, h, i, members=6, eps=0.04) for i in range(k)]
    ids = [f"s{i:04d}" for i in range(k)]
    counts, g, sim, clusters, outl = _expect(cells, w, h, k, ids)
    with BandedStream(w, h, k, band_rows=band_rows) as bs:
        assert sum(n for _, n in bs.bands()) == h
        r = bs.run(cells, ids=ids)
    assert np.array_equal(r["counts"], counts)
    assert np.array_equal(r["rgba"], O.composite(counts, k))
    assert r["bins"].tolist() == O.overlap_counts(counts.reshape(-1), k).tolist()
    assert np.array_equal(r["gram"], g)
    assert r["clusters"] == clusters
    assert r["outliers"] == outl
    assert r["stats"].bands == -(-h // band_rows)


def test_banded_pinned_callable_and_partial_rows():
    """Pinned sources take the overlapped 2b-final path; a callable source and a
    row block (one rank's share) reproduce the same rows of the full result."""
    w, h, k = 640, 300, 16
    cells = [synth_cells(w, h, i, members=4, eps=0.05) for i in range(k)]
    counts = O.accumulate(cells, w, h)
    row0, rows = 77, 150
    pinned = [N.PinnedBuffer((rows, w)) for _ in range(k)]
    try:
        for i in range(k):
            pinned[i].array[:] = cells[i][row0:row0 + rows]
        with BandedStream(w, h, k, row0=row0, rows=rows, band_rows=40) as bs:
            a = bs.run([p.array for p in pinned], analytics=False)
            b = bs.run(lambda i, r0, n: cells[i][row0 + r0:row0 + r0 + n], analytics=False)
            out = np.empty((rows, w), np.uint32)
            c = bs.run(lambda i, r0, n: cells[i][row0 + r0:row0 + r0 + n], analytics=False,
                       counts_out=out, variant="1b-final")
    finally:
        for p in pinned:
            p.free()
    want = counts[row0:row0 + rows]
    g = O.gram([x[row0:row0 + rows] for x in cells])
    for r in (a, b, c):
        assert np.array_equal(r["counts"], want)
        assert np.array_equal(r["gram"], g)
    assert np.array_equal(out, want)


def test_default_band_rows_fits_budget():
    w, k = 32768, 64
    rows = default_band_rows(w, k, 8 << 30)
    assert rows >= 1 and 2 * rows * w * (k / 8 + 10) <= 8 << 30


def test_synth_gpu_equals_host():
    """fs_synth_gpu writes the bytes of fs_synth_host (host pinned, host pageable and
    device destinations; a row band not starting at 0; a width that is not a multiple
    of 8)."""
    import torch

    w, h = 1003, 517
    for (row0, rows) in [(0, h), (101, 250)]:
        want = synth_cells(w, h, 7, seed=99, members=3, eps=0.07, row0=row0, rows=rows)
        got = synth_cells_gpu(w, h, 7, seed=99, members=3, eps=0.07, row0=row0, rows=rows)
        assert np.array_equal(got, want)
        pin = N.PinnedBuffer((rows, w))
        try:
            synth_cells_gpu(w, h, 7, seed=99, members=3, eps=0.07, row0=row0, rows=rows,
                            out=pin.array)
            assert np.array_equal(pin.array, want)
        finally:
            pin.free()
        d = torch.empty(rows * w, dtype=torch.uint8, device="cuda")
        synth_cells_gpu(w, h, 7, seed=99, members=3, eps=0.07, row0=row0, rows=rows,
                        device_ptr=d.data_ptr())
        assert np.array_equal(d.cpu().numpy().reshape(rows, w), want)


def test_c4_full_size_banded_equals_resident():
    """Config 4 at full size (64 flood-like masks of 32768 x 32768): band-by-band
    streaming from host memory (bands generated on demand, 512 rows each) gives the
    same histogram and Gram as the whole ensemble bit-packed resident in HBM
    (8.6 GB), and the histogram covers every pixel."""
    from paper_2104_14667_b200.ensemble import DeviceEnsemble

    w = h = 32768
    k, members, eps = 64, 8, 0.02
    with DeviceEnsemble(w, h, k) as ens:
        ens.synth(0, k, seed=2104, members=members, eps=eps)
        _, bins_res, _, gram_res, _ = ens.products(engine="tc-f4", counts=False, rgba=False)
    def source(i, r0, n):  # band rows of mask i, generated on demand
        return synth_cells_gpu(w, h, i, seed=2104, members=members, eps=eps, row0=r0, rows=n)

    with BandedStream(w, h, k, band_rows=512) as bs:
        r = bs.run(source, maps=False, analytics=True)
    assert int(r["bins"].sum()) == w * h
    assert np.array_equal(r["bins"], bins_res)
    assert np.array_equal(r["gram"], gram_res)
    assert len(r["clusters"]) == k // members


@pytest.mark.parametrize("seed", range(6))
def test_banded_randomized(seed):
    """Random geometry / band height / row block / k (incl. > 256) / source kind."""
    rng = np.random.default_rng(4242 + seed)
    k = int(rng.integers(1, 300))
    w, h = int(rng.integers(1, 400)), int(rng.integers(1, 90))
    row0 = int(rng.integers(0, h))
    rows = int(rng.integers(1, h - row0 + 1))
    band_rows = int(rng.integers(1, rows + 3))
    cells = [(rng.random((h, w)) < rng.uniform(0, 1)).astype(np.uint8) *
             rng.integers(1, 256, (h, w)).astype(np.uint8) for _ in range(k)]
    with BandedStream(w, h, k, row0=row0, rows=rows, band_rows=band_rows) as bs:
        if seed % 2:
            r = bs.run(lambda i, r0, n: cells[i][row0 + r0:row0 + r0 + n], analytics=False)
        else:
            r = bs.run([c[row0:row0 + rows] for c in cells], analytics=False)
    part = [c[row0:row0 + rows] for c in cells]
    want = O.accumulate(part, w, rows)
    assert np.array_equal(r["counts"], want)
    assert np.array_equal(r["rgba"], O.composite(want, k))
    assert r["bins"].tolist() == O.overlap_counts(want.reshape(-1), k).tolist()
    assert np.array_equal(r["gram"], O.gram(part))
