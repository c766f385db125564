"""Symmetric orthogonal ULV factorization and solve of K~ + beta I (oracle side).

P:188 (ULV form, U/V orthogonal, L lower triangular; computed once per h and
reused), P:209-210 (K~_beta = K~ + beta I, ULVfactorization), P:211 and the
x-update (solves with K_beta).  Concrete steps = readings U and S,
AMB-14 (Cholesky on eliminated blocks, no LU fallback):

  leaf:      Dcur = D + beta I,  Ucur = U
  internal:  Dcur = [[Dh_a, R_a B R_b^T], [R_b B^T R_a^T, Dh_b]],  Ucur = diag(R_a, R_b) U_t
  node t (non-root, k < rows):  Q^T Ucur = [R; 0] (Householder QR, complete Q);
      Dc = Q^T Dcur Q;  Dc_rr = L_r L_r^T (the last rows-k indices);
      L_sr = Dc_sr L_r^-T;  Dh = Dc_ss - L_sr L_sr^T
  pass-through (k == rows): Dh = Dcur, R = Ucur (no transform)
  root: Cholesky of Dcur.
Solve:
  forward:  c = Q^T b;  y_r = L_r^-1 c_r;  up = c_s - L_sr y_r
  root:     Cholesky solve
  backward: x_r = L_r^-T (y_r - L_sr^T x_s);  x = Q [x_s; x_r]; split between children.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla

from .hss import HSS


class NotSPDError(RuntimeError):
    """Cholesky breakdown of an eliminated block (HSS_ENOTSPD); carries the node id."""

    def __init__(self, node):
        super().__init__(f"K~ + beta I not SPD: Cholesky breakdown at node {node}")
        self.node = node


@dataclass
class ULV:
    hss: HSS
    beta: float
    Q: dict = field(default_factory=dict)
    Lr: dict = field(default_factory=dict)
    Lsr: dict = field(default_factory=dict)
    Lroot: np.ndarray = None


def _chol(A, node):
    try:
        return np.linalg.cholesky(A)
    except np.linalg.LinAlgError:
        raise NotSPDError(node) from None


def factor(hss: HSS, beta: float) -> ULV:
    f = ULV(hss=hss, beta=beta)
    L = hss.L
    Dh, Rm = {}, {}
    if L == 0:
        f.Lroot = _chol(hss.D[0] + beta * np.eye(hss.n), 0)
        return f
    for lvl in range(L, -1, -1):
        for t, lo, hi in hss.nodes(lvl):
            if lvl == L:
                Dcur = hss.D[t] + beta * np.eye(hi - lo)
                Ubase = None
            else:
                a, b = 2 * t + 1, 2 * t + 2
                off = Rm[a] @ hss.B[t] @ Rm[b].T
                Dcur = np.block([[Dh[a], off], [off.T, Dh[b]]])
                Ubase = sla.block_diag(Rm[a], Rm[b])
                del Dh[a], Dh[b], Rm[a], Rm[b]
            if lvl == 0:
                f.Lroot = _chol(Dcur, 0)
                continue
            rows, k = hss.rows[t], hss.k[t]
            if hss.is_passthrough(t):
                Dh[t] = Dcur
                Rm[t] = np.eye(rows) if Ubase is None else Ubase
                continue
            Ucur = hss.U[t] if Ubase is None else Ubase @ hss.U[t]
            Q, Rfull = np.linalg.qr(Ucur, mode="complete")
            Dc = Q.T @ Dcur @ Q
            Lr = _chol(Dc[k:, k:], t)
            Lsr = sla.solve_triangular(Lr, Dc[k:, :k], lower=True).T
            Dh[t] = Dc[:k, :k] - Lsr @ Lsr.T
            Rm[t] = Rfull[:k]
            f.Q[t], f.Lr[t], f.Lsr[t] = Q, Lr, Lsr
    return f


def solve(f: ULV, Bv: np.ndarray) -> np.ndarray:
    """x = (K~ + beta I)^-1 b in tree order (b: n or n x c)."""
    hss = f.hss
    Bv = np.asarray(Bv, dtype=np.float64)
    vec = Bv.ndim == 1
    if vec:
        Bv = Bv[:, None]
    L = hss.L
    if L == 0:
        x = sla.cho_solve((f.Lroot, True), Bv)
        return x[:, 0] if vec else x
    up, yr = {}, {}
    for lvl in range(L, 0, -1):                      # forward sweep
        for t, lo, hi in hss.nodes(lvl):
            bt = Bv[lo:hi] if lvl == L else np.vstack([up[2 * t + 1], up[2 * t + 2]])
            if hss.is_passthrough(t):
                up[t] = bt
                continue
            k = hss.k[t]
            c = f.Q[t].T @ bt
            y = sla.solve_triangular(f.Lr[t], c[k:], lower=True)
            yr[t] = y
            up[t] = c[:k] - f.Lsr[t] @ y
    broot = np.vstack([up[1], up[2]])                 # root
    xroot = sla.cho_solve((f.Lroot, True), broot)
    xs = {1: xroot[:hss.k[1]], 2: xroot[hss.k[1]:]}
    out = np.zeros_like(Bv)
    for lvl in range(1, L + 1):                       # backward sweep
        for t, lo, hi in hss.nodes(lvl):
            if hss.is_passthrough(t):
                xt = xs[t]
            else:
                xr = sla.solve_triangular(f.Lr[t].T, yr[t] - f.Lsr[t].T @ xs[t], lower=False)
                xt = f.Q[t] @ np.vstack([xs[t], xr])
            if lvl == L:
                out[lo:hi] = xt
            else:
                ka = hss.k[2 * t + 1]
                xs[2 * t + 1], xs[2 * t + 2] = xt[:ka], xt[ka:]
    return out[:, 0] if vec else out


def factor_bytes(f: ULV) -> int:
    """Bytes of Q, L_r, L_sr (explicit storage in this oracle)."""
    tot = sum(q.size for q in f.Q.values()) + sum(l.size for l in f.Lr.values())
    tot += sum(l.size for l in f.Lsr.values()) + f.Lroot.size
    return 8 * tot
