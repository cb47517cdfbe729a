"""CPU tests of the sweep-suite host logic (fs/bench.py:55-126,342-364 schemas)."""

import numpy as np
import pytest

from paper_2104_14667_b200.sweep import BenchError, RateMap, SweepSpec, render_rate_map


def test_sweep_spec_points_and_validation():
    s = SweepSpec(512, 500, 16012)
    assert s.points[0] == 512 and s.points[-1] == 16012 and len(s.points) == 32
    assert s.cells == 1024
    for bad in ((0, 1, 5), (1, 0, 5), (10, 1, 5)):
        with pytest.raises(BenchError):
            SweepSpec(*bad)
    with pytest.raises(BenchError):
        SweepSpec(1, 1, 5, repeats=0)


def test_ratemap_round_trips_and_shape_check():
    s = SweepSpec(100, 50, 200)
    r = np.arange(9, dtype=np.float64).reshape(3, 3) * 10.5
    rm = RateMap(spec=s, rates=r)
    assert RateMap.from_json(rm.to_json()).rates.tolist() == r.tolist()
    lines = rm.to_csv().splitlines()
    assert lines[0] == "width,height,rate_gbps" and len(lines) == 10
    assert lines[1].startswith("100,100,")
    assert lines[2].startswith("150,100,")  # width varies fastest within a height row
    with pytest.raises(BenchError):
        RateMap(spec=s, rates=np.zeros((2, 3)))


def test_render_rate_map_ramp_and_blue():
    s = SweepSpec(1, 1, 2)
    rm = RateMap(spec=s, rates=np.array([[0.0, 16.0], [31.5, 40.0]]))
    img = render_rate_map(rm)
    # bottom-left origin: rates[0, 0] is the bottom-left pixel
    assert img[1, 0].tolist() == [255, 255, 255, 255]     # 0 GB/s -> white
    assert img[0, 1].tolist() == [0, 0, 255, 255]         # > 32 GB/s -> blue
    assert img[0, 0].tolist() == [0, 0, 0, 255]           # step 31 -> black
    g = round(255.0 * (1.0 - 16 / 31.0))
    assert img[1, 1].tolist() == [g, g, g, 255]
    # configurable scale for B200-sized rates
    assert render_rate_map(rm, scale_gbps=64.0)[0, 1].tolist() != [0, 0, 255, 255]
