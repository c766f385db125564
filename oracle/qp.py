"""Brute-force solution of the SVM dual QP, Eq. (1), for tiny d.

Active-set enumeration: every index is at the lower bound 0, at the upper bound C,
or free; for each of the 3^d patterns the equality-constrained QP over the free
set is solved exactly (its KKT system), kept if box-feasible; the minimum
objective over all candidates is the global optimum (the QP is convex; every
optimum is a stationary point of its own pattern).  Also the KKT conditions of
Eq. (1) and the objective-gap bound Eq. (9).
"""
from __future__ import annotations

import itertools

import numpy as np


def solve_qp_bruteforce(K, y, C, tol=1e-12):
    d = y.shape[0]
    if d > 10:
        raise ValueError("brute force QP refuses d > 10")
    Q = (y[:, None] * K) * y[None, :]
    best, best_x = np.inf, None
    for pat in itertools.product((0, 1, 2), repeat=d):   # 0: at 0, 1: at C, 2: free
        pat = np.array(pat)
        x = np.where(pat == 1, C, 0.0).astype(np.float64)
        F = np.flatnonzero(pat == 2)
        Bd = np.flatnonzero(pat != 2)
        if F.size:
            nF = F.size
            A = np.zeros((nF + 1, nF + 1))
            A[:nF, :nF] = Q[np.ix_(F, F)]
            A[:nF, nF] = -y[F]
            A[nF, :nF] = -y[F]
            rhs = np.concatenate([1.0 - Q[np.ix_(F, Bd)] @ x[Bd], [y[Bd] @ x[Bd]]])
            try:
                sol = np.linalg.solve(A, rhs)
            except np.linalg.LinAlgError:
                continue
            x[F] = sol[:nF]
            if (x[F] < -tol).any() or (x[F] > C + tol).any():
                continue
            x[F] = np.clip(x[F], 0.0, C)
        if abs(y @ x) > 1e-9:
            continue
        f = 0.5 * x @ Q @ x - x.sum()
        if f < best - 1e-15:
            best, best_x = f, x.copy()
    return best_x, best


def kkt_residual(K, y, C, z, lam, eps=1e-9):
    """Max violation of the KKT conditions of Eq. (1) with multiplier lam:
    g = Y K Y z - e;  free: g_j = lam y_j;  z_j = 0: g_j - lam y_j >= 0;  z_j = C: <= 0."""
    g = y * (K @ (y * z)) - 1.0
    r = g - lam * y
    viol = 0.0
    for j in range(z.shape[0]):
        if z[j] <= eps:
            viol = max(viol, -r[j])
        elif z[j] >= C - eps:
            viol = max(viol, r[j])
        else:
            viol = max(viol, abs(r[j]))
    return max(viol, abs(y @ z))


def gap_bound(K, Kt, y, C):
    """Eq. (9): returns (lhs, rhs) = (|f(x_bar) - f~(x~)|, 1/2 max(|x~|^2, |x_bar|^2) ||Kt - K||_2)."""
    xb, fb = solve_qp_bruteforce(K, y, C)
    xt, ft = solve_qp_bruteforce(Kt, y, C)
    lhs = abs(fb - ft)
    rhs = 0.5 * max(xt @ xt, xb @ xb) * np.linalg.norm(Kt - K, 2)
    return lhs, rhs
