"""PGM/PNG codecs (host side): the header scanner accepts exactly what the reference's
parser accepts (fs/rasters.py:54-76), with the same errors; ingest reads headers longer
than its first read (long comment blocks)."""

import importlib.util
import random
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2104_14667_b200 import ingest
from paper_2104_14667_b200 import rasters as R

REF_RASTERS = Path("/root/reference/pkg/src/floodstream/rasters.py")


def _parse(mod, data):
    try:
        w, h, c = mod.parse_pgm(data)
        return ("ok", w, h, c.tobytes())
    except ValueError as e:
        return ("err", str(e))


@pytest.mark.parametrize("data,want", [
    (b"P5 3 2 255\n\x00\x01\x02\x03\x04\x05", ("ok", 3, 2)),
    (b"P5\n#c\n3\n#d\n 2\n255\n\x00\x01\x02\x03\x04\x05", ("ok", 3, 2)),
    (b"P5 3 2 255 \x00\x01\x02\x03\x04\x05", ("ok", 3, 2)),
    (b"P5#c\n3 2 255\n\x00" * 2, ("err", "not a binary PGM (P5) file")),
    (b"P5 3#c\n 2 255\n\x00\x01\x02\x03\x04\x05", ("err", "not a binary PGM (P5) file")),
    (b"P5 3 2 256\n" + bytes(12), ("err", "16-bit PGM is not supported; maxval must be <= 255")),
    (b"P5 0 2 255\n", ("err", "PGM dimensions must be positive")),
    (b"P5 3 2 255\n\x00", ("err", "PGM truncated: expected 6 pixel bytes, got 1")),
    (b"P5 3 2 255", ("err", "not a binary PGM (P5) file")),
])
def test_pgm_known_answers(data, want):
    got = _parse(R, data)
    assert got[: len(want)] == want


def test_pgm_header_matches_reference_parser():
    """300k random token strings: identical accept/reject, error text and pixels."""
    if not REF_RASTERS.exists():
        pytest.skip("reference sources not present")
    spec = importlib.util.spec_from_file_location("_ref_rasters", REF_RASTERS)
    ref = importlib.util.module_from_spec(spec)
    sys.modules["_ref_rasters"] = ref
    spec.loader.exec_module(ref)
    rng = random.Random(0)
    toks = [b"P5", b"P6", b" ", b"\n", b"\t", b"\r", b"\x0b", b"\x0c", b"#c\n", b"# x y\n",
            b"#", b"3", b"2", b"12", b"255", b"256", b"0", b"x", b"\x00\x01\x02\x03\x04\x05"]
    for _ in range(300_000):
        d = b"".join(rng.choice(toks) for _ in range(rng.randint(0, 12)))
        if rng.random() < 0.7:
            d = b"P5" + d
        assert _parse(ref, d) == _parse(R, d), d
    c = np.arange(6, dtype=np.uint8).reshape(2, 3)
    assert R.write_pgm(c) == ref.write_pgm(c)


def test_ingest_reads_long_pgm_headers(tmp_path):
    """A valid P5 file whose comments push the header past the first 512-byte read."""
    cells = (np.arange(40 * 30) % 7).astype(np.uint8).reshape(30, 40)
    body = R.write_pgm(cells)
    data = b"P5\n" + b"".join(b"# comment line %04d padding padding\n" % i for i in range(300)) \
        + body[3:]
    path = tmp_path / "long.pgm"
    path.write_bytes(data)
    assert ingest.probe(path) == (40, 30)
    out = np.empty(40 * 30, np.uint8)
    assert ingest.decode_into(path, out) == (40, 30)
    assert np.array_equal(out.reshape(30, 40), cells)
    assert np.array_equal(R.parse_pgm(data)[2], cells)
    bad = tmp_path / "bad.pgm"
    bad.write_bytes(b"P5\n" + b"# unterminated" * 100)
    with pytest.raises(R.RasterError, match="not a binary PGM"):
        ingest.probe(bad)
