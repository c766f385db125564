"""Bias, objective and prediction (oracle side).

Bias (Alg. 3) with reading AMB-2 (standard sign,
so that y_j f(f_j) = 1 on margin SVs; the printed Eq. (2)/(7) sign equals the KKT
multiplier lambda instead) and AMB-3 (margin band eps = 1e-8 C; empty M -> all
z_j > eps; still empty -> b = 0):
    b = (1/|M|) ( sum_{j in M} y_j - z_y^T Kt e_M ),   z_y = Y z.
Objective of the approximated QP, Eq. (8):  f~(z) = 1/2 z_y^T Kt z_y - e^T z.
Prediction (Alg. 3): dv(t) = sum_i (z_y)_i K(f_i, t) + b, label = +1
if dv >= 0 else -1 (AMB-15), with the EXACT kernel (AMB-19).
"""
from __future__ import annotations

import numpy as np

from .kernel import gaussian_block


def margin_set(z, C, eps_rel=1e-8):
    eps = eps_rel * C
    M = (z > eps) & (z < C - eps)
    if not M.any():
        M = z > eps
    return M


def bias(matvec, z, y, C, eps_rel=1e-8):
    """`matvec`: v -> Kt v (same point order as z, y)."""
    M = margin_set(z, C, eps_rel)
    cnt = int(M.sum())
    if cnt == 0:
        return 0.0
    u = matvec(M.astype(np.float64))
    return float((y[M].sum() - (y * z) @ u) / cnt)


def objective(matvec, z, y):
    zy = y * z
    return float(0.5 * zy @ matvec(zy) - z.sum())


def objective_dense(K, z, y):
    zy = y * z
    return float(0.5 * zy @ K @ zy - z.sum())


def decision_values(Ftrain, coef, h, b, Ftest, chunk=4096):
    dv = np.empty(Ftest.shape[0])
    for lo in range(0, Ftest.shape[0], chunk):
        dv[lo:lo + chunk] = gaussian_block(Ftest[lo:lo + chunk], Ftrain, h) @ coef + b
    return dv


def labels(dv):
    return np.where(dv >= 0.0, 1, -1).astype(np.int8)
