"""Seeded synthetic workloads shaped like BASELINE.json's configs.

Draw order inside one `numpy.random.default_rng(seed_data)` stream (documented in
DESIGN.md "Input recipe"):
  cfg 0/4: (1) balanced labels (train then test, each shuffled), (2) features;
  cfg 1:   (1) features, (3) labels from a closed-form teacher, (4) flips;
  cfg 2:   (1) features, (2) teacher weights W1, W2, (3) labels, (4) flips;
  cfg 3:   (1) features, (2) teacher centres + amplitudes, (3) labels, (4) flips.
sign(0) = +1 everywhere (AMB-15).  All arrays are float64, C-contiguous, features
row-major n x r.  Labels are exactly +-1.0.
"""
from __future__ import annotations

import numpy as np

from .configs import get_config


def _sign(v: np.ndarray) -> np.ndarray:
    return np.where(v >= 0.0, 1.0, -1.0)


def _balanced_labels(rng, n: int) -> np.ndarray:
    y = np.ones(n)
    y[n // 2 + (n % 2):] = -1.0
    return y[rng.permutation(n)]


def _flip(rng, y: np.ndarray, p: float) -> np.ndarray:
    f = rng.random(y.shape[0]) < p
    return np.where(f, -y, y)


def _mixed_features(rng, N: int) -> np.ndarray:
    """cfg 3: 10 N(0,1) + one-hot(4, uniform) + one-hot(40, uniform) = 54 columns."""
    F = np.zeros((N, 54))
    F[:, :10] = rng.standard_normal((N, 10))
    a = rng.integers(0, 4, N)
    b = rng.integers(0, 40, N)
    F[np.arange(N), 10 + a] = 1.0
    F[np.arange(N), 14 + b] = 1.0
    return F


def generate(c: int, n: int | None = None, n_test: int | None = None, **_ignored):
    """Return (F_train, y_train, F_test, y_test) for config `c`.

    `n` / `n_test` override the sizes (scaled parity cases draw a fresh stream of
    the same distribution; they are not prefixes of the full-size draw).
    """
    cfg = get_config(c)
    n = cfg["n"] if n is None else int(n)
    nt = cfg["n_test"] if n_test is None else int(n_test)
    N = n + nt
    rng = np.random.default_rng(cfg["seed_data"])
    r = cfg["r"]
    if c in (0, 4):
        mean = 0.5 if c == 0 else 0.3
        y = np.concatenate([_balanced_labels(rng, n), _balanced_labels(rng, nt)])
        F = rng.standard_normal((N, r)) + mean * y[:, None]
    elif c == 1:
        F = rng.random((N, r))
        g = np.sin(3.0 * F[:, 0]) + np.cos(2.0 * F[:, 1]) + 0.5 * F[:, 2] - 0.2
        y = _flip(rng, _sign(g), 0.05)
    elif c == 2:
        F = (rng.random((N, r)) < 0.11).astype(np.float64)
        W1 = rng.standard_normal((r, 32))
        W2 = rng.standard_normal(32)
        g = np.tanh(F @ W1) @ W2
        y = _flip(rng, _sign(g - np.median(g[:n])), 0.08)
    elif c == 3:
        F = _mixed_features(rng, N)
        centres = _mixed_features(rng, 256)
        amp = rng.standard_normal(256)
        g = np.empty(N)
        cn = (centres * centres).sum(1)
        for lo in range(0, N, 65536):
            X = F[lo:lo + 65536]
            d2 = (X * X).sum(1)[:, None] + cn[None, :] - 2.0 * X @ centres.T
            g[lo:lo + 65536] = np.exp(-0.5 * np.maximum(d2, 0.0)) @ amp
        y = _flip(rng, _sign(g - np.median(g[:n])), 0.03)
    else:
        raise ValueError(f"unknown config {c}")
    F = np.ascontiguousarray(F, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return F[:n].copy(), y[:n].copy(), F[n:].copy(), y[n:].copy()
