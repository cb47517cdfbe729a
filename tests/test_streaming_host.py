"""Host-side streaming logic on injected per-item costs (no GPU): the report builder,
the closed-form makespan source and the frame budget, against the reference's own
known answers (tests/test_streaming.py:111-130, :176-190, :318-336 of the reference;
fs/streaming.py:220-244, :324-373, :436-464)."""

from types import SimpleNamespace

import pytest

from paper_2104_14667_b200.streaming import (
    MEASURE_CAP,
    PipelineRunReport,
    StreamError,
    StreamJob,
    Variant,
    _check_source,
    _report,
    frame_budget_bytes,
    max_data_per_frame,
)

DIMS = (100, 60)
PAYLOAD = DIMS[0] * DIMS[1]


def stats(c, m, p, h=None, total=None):
    n = len(c)
    return SimpleNamespace(copy_us=list(c), xform_us=list(m), kernel_us=list(p),
                           host_us=list(h or [0.0] * n), total_us=total or 1.0)


def job(variant, n):
    return StreamJob(variant=variant, n=n, width=DIMS[0], height=DIMS[1])


@pytest.mark.parametrize("variant,total", [(Variant.ONE_BUFFER_FINAL, 18),
                                           (Variant.TWO_BUFFER_FINAL, 12)])
def test_closed_form_source_on_injected_costs(variant, total):
    """(c, m, p) = (3, 2, 1) per item, n = 3: the reference's hand-computed totals for
    the two final strategies (its TestHandComputedTotals)."""
    rep = _report(job(variant, 3), stats([3] * 3, [2] * 3, [1] * 3, total=99.0), "closed-form")
    assert rep.total_time_us == total
    assert rep.makespan_source == "closed-form"
    assert rep.per_item_c == [3, 3, 3] and rep.per_item_m == [2, 2, 2]
    assert rep.efficiency == 9 / total


def test_measured_source_keeps_measured_total():
    rep = _report(job(Variant.TWO_BUFFER_FINAL, 3), stats([3.4] * 3, [2] * 3, [1] * 3, total=12.5))
    assert rep.total_time_us == 13 and rep.makespan_source == "measured"
    assert rep.per_item_c == [3, 3, 3]
    assert rep.transfer_rate_gbps == 3 * PAYLOAD / 13 / 1000.0
    assert PipelineRunReport.from_json(rep.to_json()) == rep


def test_sampled_report_scales_to_n():
    """Jobs longer than MEASURE_CAP are timed on a sample: lists cycle to n, the total
    scales by n / sample, and the source says so."""
    s = stats([3, 4], [2, 2], [1, 1], total=10.0)
    rep = _report(job(Variant.TWO_BUFFER_FINAL, 5), s)
    assert rep.per_item_c == [3, 4, 3, 4, 3] and len(rep.per_item_p) == 5
    assert rep.total_time_us == 25
    assert rep.makespan_source.startswith("measured (2 of 5")
    assert MEASURE_CAP >= 64


def test_initial_strategies_carry_host_copies():
    rep = _report(job(Variant.TWO_BUFFER_INITIAL, 2), stats([3, 3], [2, 2], [1, 1], h=[4, 4.6]))
    assert rep.per_item_h == [4, 5]
    assert "h" in rep.to_json()["per_item"]


def test_makespan_source_validation():
    """As the reference (streaming.py:343-347): closed form for final strategies only."""
    with pytest.raises(StreamError, match="final strategies only"):
        _check_source(job(Variant.ONE_BUFFER_INITIAL, 5), "closed-form")
    with pytest.raises(StreamError, match="unknown makespan_source"):
        _check_source(job(Variant.ONE_BUFFER_FINAL, 5), "modelled")
    for src in ("measured", "simulated", "closed-form"):
        _check_source(job(Variant.TWO_BUFFER_FINAL, 5), src)


@pytest.mark.parametrize("c,m,p,div", [(3, 2, 1, 3), (1, 5, 2, 7)])
def test_frame_budget_reference_answers(c, m, p, div):
    """The reference's TestFrameBudget: 100 ms frame, step = max(c, m + p)."""
    assert frame_budget_bytes(c, m, p, PAYLOAD, 10) == 100_000 * PAYLOAD // div


@pytest.mark.parametrize("c,m,p,div", [(3, 2, 1, 3), (1, 5, 2, 7)])
def test_max_data_per_frame_from_measured_report(c, m, p, div):
    """max_data_per_frame takes a measured PipelineRunReport as its profile."""
    rep = _report(job(Variant.TWO_BUFFER_FINAL, 4), stats([c] * 4, [m] * 4, [p] * 4))
    assert max_data_per_frame(rep, *DIMS, target_fps=10) == 100_000 * PAYLOAD // div
    assert max_data_per_frame(rep, *DIMS, target_fps=1) == 1_000_000 * PAYLOAD // div
    with pytest.raises(StreamError, match="another raster size"):
        max_data_per_frame(rep, 10, 10)


def test_frame_budget_validation():
    with pytest.raises(StreamError):
        frame_budget_bytes(3, 2, 1, PAYLOAD, 0)
    with pytest.raises(StreamError):
        max_data_per_frame(None, 100, 100, target_fps=0)
    with pytest.raises(StreamError):
        frame_budget_bytes(0, 0, 0, PAYLOAD, 10)
