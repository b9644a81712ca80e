"""Element-block partitioner (orodg/partition.py:29-99), vectorised.

Leaves are Morton sorted, so a partition is a list of contiguous ranges
chosen to minimise the largest per-rank weight: bisection on the capacity,
greedy packing per capacity.  The packing here walks chunk starts and takes
each chunk's length from a sequential ``np.cumsum`` of the weights after
the start -- the same left-to-right float accumulation as the reference's
scalar loop (partition.py:29-43), so boundaries are bitwise identical, but
O(n) numpy work per bisection step instead of a Python loop
(3-4 s at 220 k leaves and ~45 s at 2.5 M in the reference).
"""

from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError


@dataclass
class Partition:
    n_workers: int
    owner: np.ndarray
    ranges: list
    ghosts: list

    def imbalance(self, weights):
        tot = np.array([weights[a:b].sum() for a, b in self.ranges])
        mean = tot.mean()
        return float(tot.max() / mean) if mean > 0 else 1.0


def _pack(w, cap, limit):
    """Greedy contiguous chunks of weight <= cap; None if a single weight
    exceeds cap; stops early once more than ``limit`` chunks are needed."""
    n = len(w)
    if n and w.max() > cap:
        return None
    bounds = [0]
    s = 0
    pref = np.cumsum(w)
    while s < n:
        # window guess from the global prefix, then exact local accumulation
        base = pref[s - 1] if s else 0.0
        guess = int(np.searchsorted(pref, base + cap, side="right")) - s
        win = max(16, 2 * guess + 16)
        while True:
            c = np.cumsum(w[s:s + win])
            over = np.nonzero(c > cap)[0]
            if len(over) or s + win >= n:
                break
            win *= 2
        k = int(over[0]) if len(over) else n - s
        s += k
        bounds.append(s)
        if len(bounds) - 1 > limit:
            return bounds
    if bounds[-1] != n:
        bounds.append(n)
    return bounds


def split_contiguous(weights, n_chunks):
    w = np.asarray(weights, dtype=float)
    n = len(w)
    if n_chunks >= n:
        return list(range(n + 1)) + [n] * (n_chunks - n)
    lo, hi = float(w.max()), float(w.sum())
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        b = _pack(w, mid, n_chunks)
        if b is not None and len(b) - 1 <= n_chunks:
            hi = mid
        else:
            lo = mid
        if hi - lo <= 1e-12 * max(hi, 1.0):
            break
    b = _pack(w, hi * (1 + 1e-12), n)
    while len(b) - 1 < n_chunks:
        b.append(n)
    return b


def neighbor_pairs(mesh):
    topo = mesh.topology
    parts = [np.stack([b.left, b.right], 1) for b in topo.conforming]
    parts += [np.stack([b.coarse, b.fine], 1) for b in topo.hanging]
    return np.concatenate(parts) if parts else np.empty((0, 2), np.int64)


def partition_leaves(mesh, n_workers, weights=None):
    if n_workers < 1:
        raise ConfigurationError(f"need >= 1 worker, got {n_workers}")
    n = mesh.n_leaves
    w = np.ones(n) if weights is None else np.asarray(weights, dtype=float)
    b = split_contiguous(w, n_workers)
    ranges = [(b[p], b[p + 1]) for p in range(n_workers)]
    owner = np.empty(n, dtype=np.int64)
    for p, (a, e) in enumerate(ranges):
        owner[a:e] = p
    pairs = neighbor_pairs(mesh)
    if len(pairs) == 0:
        ghosts = [np.empty(0, dtype=np.int64) for _ in range(n_workers)]
    else:
        ol, orr = owner[pairs[:, 0]], owner[pairs[:, 1]]
        ghosts = []
        for p in range(n_workers):
            ml, mr = ol == p, orr == p
            ghosts.append(np.unique(np.concatenate([pairs[ml & ~mr, 1],
                                                    pairs[mr & ~ml, 0]])))
    return Partition(n_workers=n_workers, owner=owner, ranges=ranges, ghosts=ghosts)
