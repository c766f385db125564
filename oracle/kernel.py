"""Gaussian kernel blocks (oracle side).

P:49 / P:286: K_ij = exp(-||f_i - f_j||^2 / (2 h^2)); the printed `f_i - f_i`
is the typo AMB-4, read as f_i - f_j.  Squared distances are computed by DIRECT
differences (scipy cdist 'sqeuclidean'), the plain definition; the GPU uses the
GEMM form nu_i + nu_j - 2 f_i.f_j (clamped >= 0), a different route.
"""
from __future__ import annotations

import numpy as np
from scipy.spatial.distance import cdist


def gaussian_block(Fa: np.ndarray, Fb: np.ndarray, h: float) -> np.ndarray:
    """K(Fa, Fb): (len(Fa) x len(Fb)) block of Gaussian kernel entries."""
    Fa = np.atleast_2d(np.asarray(Fa, dtype=np.float64))
    Fb = np.atleast_2d(np.asarray(Fb, dtype=np.float64))
    if Fa.shape[0] == 0 or Fb.shape[0] == 0:
        return np.zeros((Fa.shape[0], Fb.shape[0]))
    d2 = cdist(Fa, Fb, "sqeuclidean")
    return np.exp(-d2 / (2.0 * h * h))


def dense_kernel(F: np.ndarray, h: float, cap: int = 32768) -> np.ndarray:
    """Full K (guarded: refuses n > cap; dense K is O(n^2) memory)."""
    if F.shape[0] > cap:
        raise ValueError(f"dense_kernel refuses n={F.shape[0]} > cap={cap}")
    return gaussian_block(F, F, h)


def sketch(Fp: np.ndarray, h: float, Omega_p: np.ndarray, chunk: int | None = None,
           threads: int | None = None) -> np.ndarray:
    """H1: S = K_p Omega_p as a dense product, computed in row chunks.

    Row chunks are independent and may run on a thread pool (cdist, exp and dgemm release
    the GIL); the chunk boundaries, hence the result, do not depend on the thread count."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    n = Fp.shape[0]
    S = np.empty((n, Omega_p.shape[1]))
    if chunk is None:  # bound the per-thread temporaries (chunk x n doubles) to ~1 GB
        chunk = int(max(64, min(1024, (1 << 27) // max(1, n))))

    def one(lo):
        S[lo:lo + chunk] = gaussian_block(Fp[lo:lo + chunk], Fp, h) @ Omega_p

    los = list(range(0, n, chunk))
    nt = threads if threads is not None else min(len(os.sched_getaffinity(0)), 16)
    if nt <= 1 or len(los) <= 1 or n < 8192:
        for lo in los:
            one(lo)
    else:
        with ThreadPoolExecutor(nt) as ex:
            list(ex.map(one, los))
    return S


def sketch_rows(Fp: np.ndarray, h: float, Omega_p: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """Selected rows of S (for sampled checks at sizes where the full S is too slow)."""
    return gaussian_block(Fp[rows], Fp, h) @ Omega_p
