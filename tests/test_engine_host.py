"""Host logic of the resident working-set engine (no GPU): slot placement, eviction
order and upload runs of engine.SlotMap."""

import pytest

from paper_2104_14667_b200.engine import SlotMap


def test_slotmap_places_runs_and_keeps_residents():
    m = SlotMap(6)
    runs, ev = m.plan(["a", "b", "c"])
    assert runs == [(0, ["a", "b", "c"])] and ev == []
    runs, ev = m.plan(["c", "a", "d"])  # a, c stay; d goes to the first free slot
    assert runs == [(3, ["d"])] and ev == []
    assert m.slots(["c", "a", "d"]) == [2, 0, 3]
    assert m.resident() == ["a", "b", "c", "d"]


def test_slotmap_evicts_least_recently_used_unwanted():
    m = SlotMap(3)
    m.plan(["a", "b", "c"])
    m.plan(["a", "c"])          # b not used this round
    runs, ev = m.plan(["a", "x"])  # c used more recently than b
    assert ev == ["b"] and runs == [(1, ["x"])]
    runs, ev = m.plan(["y", "z", "x"])  # a@0 and c@2 both go; x stays at 1
    assert ev == ["c", "a"]
    assert runs == [(0, ["y"]), (2, ["z"])]
    assert m.slots(["y", "z", "x"]) == [0, 2, 1]


def test_slotmap_dedupes_and_rejects_overflow():
    m = SlotMap(2)
    runs, _ = m.plan(["a", "a", "b"])
    assert runs == [(0, ["a", "b"])]
    with pytest.raises(ValueError):
        m.plan(["a", "b", "c"])
    m.drop("a")
    assert m.resident() == ["b"]
