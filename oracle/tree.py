"""Cluster tree by recursive PCA-median bisection (oracle side).

P:72 ("clustering algorithms are employed to find groups of points") and
P:180 (hierarchical 2x2 partitioning); the concrete rule is reading T1-T4 /
AMB-13 in DESIGN.md:
  T1  L = max(0, ceil(log2(n/m))); every node is split exactly L times.
  T2  per node: c = mean, C = (F_P - c)^T (F_P - c), v0 from R1-R3 (seed_tree,
      i = level-major BFS id, j = feature), 20 steps v <- Cv/||Cv|| (keep v if Cv = 0).
  T3  p_i = (f_i - c).v; stable sort by (p_i, original index); left = first floor(|P|/2).
  T4  perm = leaves concatenated left to right.
Node ids are level-major BFS: node (l, i) has id 2^l - 1 + i.
"""
from __future__ import annotations

import numpy as np

from .rng import tree_start_vector

POWER_ITERS = 20


def num_levels(n: int, m: int) -> int:
    """T1 in integer arithmetic: smallest L >= 0 with m * 2^L >= n."""
    L = 0
    while m * (1 << L) < n:
        L += 1
    return L


def node_ranges(n: int, L: int):
    """ranges[l] = list of (lo, hi) for the 2^l nodes of level l (floor splits, T3)."""
    ranges = [[(0, n)]]
    for _ in range(L):
        nxt = []
        for lo, hi in ranges[-1]:
            half = (hi - lo) // 2
            nxt.append((lo, lo + half))
            nxt.append((lo + half, hi))
        ranges.append(nxt)
    return ranges


def principal_direction(X: np.ndarray, v0: np.ndarray, iters: int = POWER_ITERS) -> np.ndarray:
    """T2: `iters` normalized power steps on C = X^T X starting from v0."""
    Cm = X.T @ X
    v = v0.copy()
    for _ in range(iters):
        w = Cm @ v
        nw = np.linalg.norm(w)
        if nw == 0.0:
            break
        v = w / nw
    return v


def build_tree(F: np.ndarray, m: int, seed_tree: int):
    """Return (perm, ranges): perm[t] = original index of the point at tree position t."""
    n, r = F.shape
    L = num_levels(n, m)
    ranges = node_ranges(n, L)
    perm = np.arange(n, dtype=np.int64)
    for lvl in range(L):
        for i, (lo, hi) in enumerate(ranges[lvl]):
            idx = perm[lo:hi].copy()
            X = F[idx] - F[idx].mean(axis=0)
            v = principal_direction(X, tree_start_vector(seed_tree, (1 << lvl) - 1 + i, r))
            p = X @ v
            order = np.lexsort((idx, p))  # primary key p, ties by original index
            perm[lo:hi] = idx[order]
    return perm, ranges
