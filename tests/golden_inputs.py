"""Seeded input recipes shared by the golden-fixture generator and the tests.

Every fixture in tests/golden/golden.json was produced by running the reference
package on exactly these inputs; tests regenerate them and check the recorded sha256
before comparing outputs.
"""

from __future__ import annotations

import hashlib

import numpy as np


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def c1_cells() -> list[np.ndarray]:
    """Config 1 = the reference bench inputs (bench.py:472-475): 16 masks of 2^20 px,
    default_rng(0), p = 0.5, reshaped to 1024 x 1024."""
    rng = np.random.default_rng(0)
    return [(rng.random(1 << 20) < 0.5).astype(np.uint8).reshape(1024, 1024) for _ in range(16)]


def random_case(case: int):
    """Acceptance-style instance (test_acceptance.py:241-256): depths 0..3."""
    rng = np.random.default_rng((55, case))
    h = int(rng.integers(1, 65))
    w = int(rng.integers(1, 65))
    count = int(rng.integers(2, 51))
    tau = float(rng.uniform(0.05, 0.95))
    cells = [rng.integers(0, 4, size=(h, w)).astype(np.uint8) for _ in range(count)]
    # occasionally duplicate a mask so exact-similarity ties exercise the tie-break
    if case % 3 == 0 and count >= 4:
        cells[count - 1] = cells[1].copy()
        cells[count - 2] = cells[1].copy()
    ids = [f"s{i:02d}" for i in range(count)]
    if case % 5 == 0:  # non-monotone ids
        ids = [f"m{(7 * i) % count:03d}" for i in range(count)]
    return cells, ids, tau


def stream_case(case: int):
    rng = np.random.default_rng((7, case))
    h = int(rng.integers(1, 40))
    w = int(rng.integers(1, 70))
    k = int(rng.integers(1, 6))
    n = int(rng.integers(1, 25))
    cells = [(rng.random((h, w)) < 0.4).astype(np.uint8) * rng.integers(1, 256, size=(h, w)).astype(np.uint8)
             for _ in range(k)]
    return cells, n


def edge_cases():
    """name -> (cells list, ids, taus)."""
    z = np.zeros((3, 5), dtype=np.uint8)
    o = np.full((3, 5), 7, dtype=np.uint8)
    one = np.zeros((3, 5), dtype=np.uint8)
    one[1, 2] = 255
    rng = np.random.default_rng(99)
    ties = [(rng.random((9, 33)) < 0.5).astype(np.uint8) for _ in range(3)]
    return {
        "all_empty": ([z, z.copy(), z.copy()], ["a", "b", "c"], [0.8, 1.0]),
        "all_full": ([o, o.copy()], ["x", "y"], [1.0]),
        "empty_vs_point": ([z, one, one.copy()], ["e", "p", "q"], [0.5, 1.0]),
        "single_pixel": ([np.array([[3]], dtype=np.uint8), np.array([[0]], dtype=np.uint8)],
                         ["u", "v"], [0.5]),
        "duplicate_ids": ([ties[0], ties[1], ties[0].copy(), ties[2]], ["d", "d", "a", "d"],
                          [0.3, 0.9]),
        "exact_ties": ([ties[0], ties[0].copy(), ties[0].copy(), ties[1], ties[1].copy()],
                       ["t4", "t0", "t3", "t1", "t2"], [0.2, 0.99]),
        "single_surface": ([ties[2]], ["only"], [0.8]),
        "depths_255": ([np.arange(256, dtype=np.uint8).reshape(16, 16),
                        np.arange(256, dtype=np.uint8)[::-1].reshape(16, 16).copy()],
                       ["r", "s"], [0.5]),
        "odd_width_tail": ([(np.random.default_rng(5 + i).random((7, 1031)) < 0.3).astype(np.uint8)
                            for i in range(5)], [f"w{i}" for i in range(5)], [0.2]),
    }
