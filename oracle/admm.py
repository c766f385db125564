"""Closed-form ADMM for the SVM dual (oracle side).

Alg. 2 with the precomputation of Alg. 3 lines 4-6 and
the x-update of P:145 / P:164 (reading AMB-1: Alg. 3 line 218 as printed, with
x^k and w2 = w^T x^k, is a typo; q^k = e + mu^k + beta z^k as in P:125):

  A0  v = K_b^-1 e;  w = Y v;  w1 = e^T v  (must be > 0)
  A1  x^0 = z^0 = mu^0 = 0                                          AMB-6
  A2  q = e + mu + beta z;  v = K_b^-1 (Y q);  x = Y v - (w^T q / w1) w
  A3  z = Pi_[0,C](x - mu / beta);  mu = mu - beta (x - z)
  A4  exactly MaxIt iterations; output z^MaxIt.
`solve` is any callable b -> K_b^-1 b (HSS ULV, or dense Cholesky for the dense oracle).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


class W1Error(RuntimeError):
    """w1 = e^T K_b^-1 e <= 0 (HSS_EW1)."""


def precompute(solve, y):
    e = np.ones_like(y)
    v = solve(e)
    w1 = float(e @ v)
    if not w1 > 0:
        raise W1Error(f"w1 = {w1} <= 0: shifted operator not positive definite")
    return y * v, w1


def x_update(solve, y, w, w1, q):
    """P:145 closed form: x = Y K_b^-1 Y q - (e^T K_b^-1 Y q / w1) Y K_b^-1 e, with
    e^T K_b^-1 Y q = w^T q (K_b symmetric)."""
    v = solve(y * q)
    return y * v - (w @ q / w1) * w


def run(solve, y, C, beta, max_it, *, trace_every=0, z0=None, mu0=None):
    """Returns dict(z, mu, x, trace=[(it, z, mu)], w, w1, lam) after max_it iterations."""
    y = np.asarray(y, dtype=np.float64)
    n = y.shape[0]
    w, w1 = precompute(solve, y)
    z = np.zeros(n) if z0 is None else np.array(z0, dtype=np.float64)
    mu = np.zeros(n) if mu0 is None else np.array(mu0, dtype=np.float64)
    x = np.zeros(n)
    e = np.ones(n)
    trace = []
    lam = 0.0
    for it in range(1, max_it + 1):
        q = e + mu + beta * z
        lam = -(w @ q) / w1
        x = x_update(solve, y, w, w1, q)
        z = np.clip(x - mu / beta, 0.0, C)
        mu = mu - beta * (x - z)
        if trace_every and (it % trace_every == 0 or it == max_it):
            trace.append((it, z.copy(), mu.copy()))
    return dict(z=z, mu=mu, x=x, trace=trace, w=w, w1=w1, lam=lam)


def run_multi(solve, y, Cs, beta, max_it, *, trace_every=0):
    """A1-A4 for several box bounds C_c at once (the factorization is shared across C):
    the nC problems are independent and advance together, column c of z / mu being problem c
    (solve takes an n x nC right-hand side).  Same arithmetic per column as run()."""
    y = np.asarray(y, dtype=np.float64)
    Cs = np.asarray(Cs, dtype=np.float64)
    n, nC = y.shape[0], Cs.shape[0]
    w, w1 = precompute(solve, y)
    z, mu, x = np.zeros((n, nC)), np.zeros((n, nC)), np.zeros((n, nC))
    trace = []
    for it in range(1, max_it + 1):
        q = 1.0 + mu + beta * z
        v = solve(y[:, None] * q)
        x = y[:, None] * v - np.outer(w, (w @ q) / w1)
        z = np.clip(x - mu / beta, 0.0, Cs[None, :])
        mu = mu - beta * (x - z)
        if trace_every and (it % trace_every == 0 or it == max_it):
            trace.append((it, z.copy(), mu.copy()))
    return dict(z=z, mu=mu, x=x, trace=trace, w=w, w1=w1)


def dense_solver(K, beta):
    """Dense oracle: Cholesky of K + beta I (equivalently of Y(K+beta I)Y = YKY + beta I,
    since Y^2 = I); returns b -> (K + beta I)^-1 b."""
    n = K.shape[0]
    c = sla.cho_factor(K + beta * np.eye(n), lower=True)
    return lambda b: sla.cho_solve(c, b)


def kkt_bordered(Kb, y, q):
    """Direct solve of the (d+1) bordered KKT system of P:131-142:
    [[Y K_b Y, -y], [-y^T, 0]] [x; lam] = [q; 0]."""
    n = y.shape[0]
    A = np.zeros((n + 1, n + 1))
    A[:n, :n] = (y[:, None] * Kb) * y[None, :]
    A[:n, n] = -y
    A[n, :n] = -y
    rhs = np.concatenate([q, [0.0]])
    sol = np.linalg.solve(A, rhs)
    return sol[:n], sol[n]
