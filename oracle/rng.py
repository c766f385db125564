"""Counter-based Gaussian generator for the random test matrix Omega (oracle side).

P:184 (randomized sampling needs seeded random probe blocks); the generator
itself is reading R1-R3: splitmix64 keyed by (seed, ORIGINAL point
index i, column j), Box-Muller.  The CUDA side implements the same generator
independently; the integer stream is bitwise portable.
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(z):
    """splitmix64 finalizer on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def gaussian(seed: int, i, j) -> np.ndarray:
    """Omega[i, j] for original indices i (array) and columns j (array), broadcast.

    R1: ctr = (i << 20) | j, key = splitmix64(seed)
    R2: a = splitmix64(key + 2 ctr), b = splitmix64(key + 2 ctr + 1),
        U1 = ((a >> 11) + 0.5) 2^-53,  U2 = (b >> 11) 2^-53
    R3: sqrt(-2 ln U1) cos(2 pi U2)
    """
    i = np.asarray(i, dtype=np.uint64)
    j = np.asarray(j, dtype=np.uint64)
    key = splitmix64(np.uint64(seed))
    with np.errstate(over="ignore"):
        ctr = (i << np.uint64(20)) | j
        base = key + np.uint64(2) * ctr
        a = splitmix64(base)
        b = splitmix64(base + np.uint64(1))
    u1 = ((a >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53
    u2 = (b >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def omega(seed: int, orig_index: np.ndarray, s: int) -> np.ndarray:
    """Rows of Omega for the given ORIGINAL point indices: shape (len(orig_index), s)."""
    idx = np.asarray(orig_index, dtype=np.int64)
    return gaussian(seed, idx[:, None], np.arange(s, dtype=np.int64)[None, :])


def tree_start_vector(seed_tree: int, node_id: int, r: int) -> np.ndarray:
    """T2: v0 from R1-R3 with i = level-major BFS node id, j = feature index; normalized."""
    v = gaussian(seed_tree, np.full(r, node_id, dtype=np.int64), np.arange(r, dtype=np.int64))
    return v / np.linalg.norm(v)
