"""Host side of the ingest path (no GPU): header probing and decoding straight into a
caller buffer agree with the reference-compatible decoder (rasters.decode_surface_bytes,
fs/rasters.py:60-117), for PGM (path and bytes, comments in the header) and PNG."""

import io

import numpy as np
import pytest

from paper_2104_14667_b200.ingest import decode_into, probe
from paper_2104_14667_b200.rasters import RasterError, decode_surface_bytes, write_pgm


def _png(cells):
    from PIL import Image

    b = io.BytesIO()
    Image.fromarray(cells, "L").save(b, format="PNG")
    return b.getvalue()


@pytest.mark.parametrize("w,h", [(1, 1), (37, 5), (300, 211)])
def test_pgm_and_png_decode_into_buffer(tmp_path, w, h):
    rng = np.random.default_rng(w * h)
    cells = rng.integers(0, 256, (h, w)).astype(np.uint8)
    pgm = write_pgm(cells)
    commented = b"P5\n# a comment\n%d %d\n# another\n255\n" % (w, h) + cells.tobytes()
    path = tmp_path / "s.pgm"
    path.write_bytes(commented)
    for src in (pgm, commented, str(path), _png(cells)):
        assert probe(src) == (w, h)
        out = np.zeros(w * h, np.uint8)
        assert decode_into(src, out) == (w, h)
        assert np.array_equal(out.reshape(h, w), cells)
        assert np.array_equal(out.reshape(h, w), decode_surface_bytes(
            src if isinstance(src, bytes) else path.read_bytes())[2])


def test_decode_errors(tmp_path):
    cells = np.ones((4, 5), np.uint8)
    with pytest.raises(RasterError, match="buffer"):
        decode_into(write_pgm(cells), np.zeros(21, np.uint8))
    with pytest.raises(RasterError, match="truncated"):
        decode_into(write_pgm(cells)[:-3], np.zeros(20, np.uint8))
    p = tmp_path / "t.pgm"
    p.write_bytes(write_pgm(cells)[:-1])
    with pytest.raises(RasterError, match="truncated"):
        decode_into(str(p), np.zeros(20, np.uint8))
    with pytest.raises(RasterError, match="unrecognised"):
        probe(b"GIF89a....")
    with pytest.raises(RasterError, match="16-bit"):
        decode_into(b"P5 2 2 65535\n" + bytes(8), np.zeros(4, np.uint8))
