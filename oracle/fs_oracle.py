"""NumPy restatement of the reference overlap path — TEST INFRASTRUCTURE ONLY.

Follows /root/reference/pkg/src/floodstream/ (abbrev. ``fs/``) function by function.
Used by tests/ and bench.py (cpu_baseline, --impl reference) as the checker; never by
the product package.
"""

from __future__ import annotations

import hashlib

import numpy as np


# ---- the four backend primitives: fs/_kernels_np.py:16-47 -------------------------

def accumulate_into(counts: np.ndarray, cells: np.ndarray) -> None:
    """fs/_kernels_np.py:16-18 — counts[p] += cells[p] > 0."""
    np.add(counts, cells > 0, out=counts, casting="unsafe")


def overlap_counts(counts: np.ndarray, n_inputs: int) -> np.ndarray:
    """fs/_kernels_np.py:21-23 — bincount with n_inputs + 1 classes, int64."""
    return np.bincount(counts, minlength=n_inputs + 1).astype(np.int64)


def pair_counts(a: np.ndarray, b: np.ndarray) -> tuple[int, int]:
    """fs/_kernels_np.py:26-32 — (|A & B|, |A | B|) of the wet masks."""
    wa, wb = a > 0, b > 0
    return int(np.count_nonzero(wa & wb)), int(np.count_nonzero(wa | wb))


def grey_levels(counts: np.ndarray, n_inputs: int) -> np.ndarray:
    """fs/_kernels_np.py:41-42 — floor(255 * (1 - c / max(n, 1)) + 0.5) in float64."""
    sat = counts.astype(np.float64) / float(max(n_inputs, 1))
    return np.floor(255.0 * (1.0 - sat) + 0.5).astype(np.uint8)


def composite_fill(counts: np.ndarray, n_inputs: int, out: np.ndarray) -> None:
    """fs/_kernels_np.py:35-47 — RGBA (g, g, 255, 255) where covered, else 0."""
    grey = grey_levels(counts, n_inputs)
    covered = counts > 0
    out[:, 0] = np.where(covered, grey, 0)
    out[:, 1] = np.where(covered, grey, 0)
    out[:, 2] = np.where(covered, 255, 0)
    out[:, 3] = np.where(covered, 255, 0)


# ---- analytics: fs/analytics.py ------------------------------------------------------

def accumulate(cells_list, width: int, height: int) -> np.ndarray:
    """fs/analytics.py:118-120 — per-surface loop of accumulate_into; uint32 (H, W)."""
    counts = np.zeros(width * height, dtype=np.uint32)
    for cells in cells_list:
        accumulate_into(counts, np.asarray(cells).reshape(-1))
    return counts.reshape(height, width)


def grid_digest(width: int, height: int, n_inputs: int, counts: np.ndarray) -> str:
    """fs/analytics.py:57-59 — sha256 of 'WxH:n:' + counts bytes."""
    head = f"{width}x{height}:{n_inputs}:".encode()
    return hashlib.sha256(head + np.ascontiguousarray(counts, dtype=np.uint32).tobytes()).hexdigest()


def composite(counts: np.ndarray, n_inputs: int) -> np.ndarray:
    """fs/analytics.py:154-156 — (H, W, 4) uint8 via composite_fill."""
    h, w = counts.shape
    out = np.zeros((h * w, 4), dtype=np.uint8)
    composite_fill(counts.reshape(-1), n_inputs, out)
    return out.reshape(h, w, 4)


def jaccard_from_counts(inter: int, union: int) -> float:
    """fs/analytics.py:165-171 — 1.0 when union == 0 else exact int/int division."""
    if union == 0:
        return 1.0
    return inter / union


def gram(cells_list) -> np.ndarray:
    """Exact int64 intersection matrix |A_i & A_j| (diag = |A_i|): the quantity every
    pair_counts call of fs/analytics.py:178-180 reduces.  Computed as a bit-popcount
    product so the oracle stays usable at thousands of pairs."""
    wet = [np.packbits(np.asarray(c).reshape(-1) > 0) for c in cells_list]
    k = len(wet)
    g = np.zeros((k, k), dtype=np.int64)
    if k == 0:
        return g
    M = np.stack(wet)
    for i in range(k):
        inter = np.bitwise_and(M[i:i + 1], M[i:])
        g[i, i:] = np.unpackbits(inter, axis=1).sum(axis=1, dtype=np.int64)
        g[i:, i] = g[i, i:]
    return g


def similarity_from_gram(g: np.ndarray) -> np.ndarray:
    """fs/analytics.py:174-181 — float64 (n, n), diag 1.0, J = inter/union."""
    n = g.shape[0]
    sim = np.ones((n, n), dtype=np.float64)
    for i in range(n):
        for j in range(i + 1, n):
            inter = int(g[i, j])
            union = int(g[i, i]) + int(g[j, j]) - inter
            sim[i, j] = sim[j, i] = jaccard_from_counts(inter, union)
    return sim


def similarity_matrix(cells_list) -> np.ndarray:
    """fs/analytics.py:174-181 by direct pair_counts (small inputs)."""
    n = len(cells_list)
    sim = np.ones((n, n), dtype=np.float64)
    for i in range(n):
        for j in range(i + 1, n):
            inter, union = pair_counts(np.asarray(cells_list[i]).reshape(-1),
                                       np.asarray(cells_list[j]).reshape(-1))
            sim[i, j] = sim[j, i] = jaccard_from_counts(inter, union)
    return sim


def outlier_scores(sim: np.ndarray, ids) -> dict:
    """fs/analytics.py:229-240 — 1 - sum(others)/len(others), where ``others`` is a list
    of np.float64 summed by builtin sum() left to right (no compensation: np.float64 is
    not an exact float for CPython 3.12's compensated sum)."""
    n = len(ids)
    scores = {}
    for i, sid in enumerate(ids):
        others = [sim[i, j] for j in range(n) if j != i]
        scores[sid] = 1.0 - sum(others) / len(others)
    return scores


def cluster(sim: np.ndarray, ids, tau: float) -> list[list[str]]:
    """fs/analytics.py:184-226 — complete linkage, candidate key (-score, lo, hi, a, b)."""
    clusters = [[i] for i in range(len(ids))]

    def linkage(ca, cb):
        return min(sim[i, j] for i in ca for j in cb)

    while len(clusters) > 1:
        best = None
        for a in range(len(clusters)):
            for b in range(a + 1, len(clusters)):
                score = linkage(clusters[a], clusters[b])
                if score < tau:
                    continue
                ka = min(ids[i] for i in clusters[a])
                kb = min(ids[i] for i in clusters[b])
                lo, hi = sorted((ka, kb))
                cand = (-score, lo, hi, a, b)
                if best is None or cand < best:
                    best = cand
        if best is None:
            break
        _, _, _, a, b = best
        clusters[a] = clusters[a] + clusters[b]
        del clusters[b]
    named = [sorted(ids[i] for i in members) for members in clusters]
    named.sort(key=lambda c: c[0])
    return named


def cluster_unique_ids(sim: np.ndarray, ids, tau: float) -> list[list[str]]:
    """``cluster`` for UNIQUE ids at n ~ 1000 (config 3): the same merge sequence as
    fs/analytics.py:200-226, with the complete-linkage matrix kept up to date instead of
    rescanning member pairs (linkage(A u B, C) = min(linkage(A, C), linkage(B, C)) —
    min of floats, exact).  With unique ids the candidate key (-score, lo, hi, a, b) is
    decided by (-score, lo, hi), so list positions never matter.  Pinned to ``cluster``
    by tests/test_oracle_golden.py."""
    n = len(ids)
    if len(set(ids)) != n:
        raise ValueError("cluster_unique_ids needs unique ids")
    rank = np.empty(n, dtype=np.int64)
    rank[np.argsort(np.array(ids, dtype=object), kind="stable")] = np.arange(n)
    link = np.array(sim, dtype=np.float64, copy=True)
    np.fill_diagonal(link, -np.inf)
    lo_id = rank.copy()  # min id rank of the cluster rooted at i
    members = {i: [i] for i in range(n)}
    iu = np.triu(np.ones((n, n), dtype=bool), 1)
    while len(members) > 1:
        best = link[iu].max() if n > 1 else -np.inf
        if not (best >= tau):
            break
        ii, jj = np.nonzero((link == best) & iu)
        lo = np.minimum(lo_id[ii], lo_id[jj])
        hi = np.maximum(lo_id[ii], lo_id[jj])
        pick = np.lexsort((hi, lo))[0]
        a, b = int(ii[pick]), int(jj[pick])
        merged = np.minimum(link[a], link[b])
        link[a, :] = merged
        link[:, a] = merged
        link[b, :] = -np.inf
        link[:, b] = -np.inf
        link[a, a] = -np.inf
        lo_id[a] = min(lo_id[a], lo_id[b])
        members[a] = members[a] + members.pop(b)
    named = [sorted(ids[i] for i in m) for m in members.values()]
    named.sort(key=lambda c: c[0])
    return named


def run_stream_counts(cells_list, n: int, width: int, height: int) -> np.ndarray:
    """fs/streaming.py:417-431 — surfaces cycled to n: cycles*full + partial, uint32."""
    k = len(cells_list)
    cycles, rem = divmod(n, k)
    counts = np.zeros(width * height, dtype=np.uint64)
    if cycles:
        counts += accumulate(cells_list, width, height).astype(np.uint64).ravel() * cycles
    if rem:
        counts += accumulate(cells_list[:rem], width, height).astype(np.uint64).ravel()
    return counts.astype(np.uint32).reshape(height, width)


def build_schedule_deps(variant: str, n: int) -> dict:
    """fs/streaming.py:150-215 — node id -> deps for the four strategies."""
    deps = {"clear[0]": (), "clear[1]": ()}
    for i in range(1, n + 1):
        if variant in ("1b-initial", "1b-final"):
            cd = (f"kernel[{i - 1}]",) if i >= 2 else ()
        elif variant == "2b-initial":
            cd = (f"kernel[{i - 2}]",) if i >= 3 else ()
        else:
            cd = (f"xform[{i - 2}]",) if i >= 3 else ()
        if variant.endswith("initial"):
            deps[f"host[{i}]"] = cd
            deps[f"copy[{i}]"] = (f"host[{i}]",)
        else:
            deps[f"copy[{i}]"] = cd
        deps[f"xform[{i}]"] = (f"copy[{i}]",) + ((f"kernel[{i - 1}]",) if i >= 2 else ())
        deps[f"kernel[{i}]"] = (f"xform[{i}]",) + (("clear[0]", "clear[1]") if i == 1
                                                   else (f"kernel[{i - 1}]",))
    return deps
