"""Randomized ID-based symmetric HSS compression of the permuted kernel (oracle side).

P:180-187 (HSS with a hierarchical 2x2 partition, randomized sampling that needs
only products with K and selected entries of K) and Alg. 3 line 1
(P:208).  The paper delegates the construction to STRUMPACK's HSS-ANN; this file
follows reading H1-H5, the randomized interpolative-decomposition
construction the paper cites ([MR2854612]) with V = U (K symmetric):

  H1  S = K_p Omega_p.
  H2  leaf t:  D_t = K(I_t, I_t);  Y_t = S(I_t) - D_t Omega_p(I_t);  Omega^_t = Omega_p(I_t);
      active rows = I_t.
  H3  non-root t:  CPQR of Y_t^T (LAPACK dgeqp3 via scipy; ties -> first index);
      k by the rank rule (AMB-10) or the fixed rank; k == rows -> pass-through
      (U = I, J = all active rows in order).  Else J~ = piv[:k] (pivot order),
      T = R11^-1 R12,  U[piv[:k]] = I_k,  U[piv[k:]] = T^T;  J_t = active[J~],
      Y_sk = Y_t[J~],  Omega'_t = U^T Omega^_t.
  H4  parent t of (a, b):  B_ab = K(J_a, J_b);
      Y_t = [Y_sk,a - B Omega'_b ; Y_sk,b - B^T Omega'_a];  Omega^_t = [Omega'_a; Omega'_b];
      active rows = [J_a; J_b].
  H5  root: B only.
N4 (SPD-preserving compression; our construction): with
  interp="spd" every non-pass-through node keeps the skeleton J_t that H3 picks, but its
  interpolation matrix is the kernel (Nystrom) interpolant onto the skeleton instead of the
  CPQR's R11^-1 R12:
      U_t = K(A_t, J_t) (K(J_t, J_t) + eps I)^-1       (A_t = the node's active rows)
  computed by a Cholesky factor of K(J_t, J_t) + eps I and two triangular solves.  Then
  D_t - U_t K(J_t,J_t) U_t^T >= 0 for every node (a generalized Schur complement), and K~ is a
  sum of such PSD terms pushed through the nested bases plus the root's principal submatrix of
  K, so K~ is positive semidefinite for every rank choice and K~ + beta I is SPD for every
  beta > 0.  Y_sk, Omega' = U^T Omega^, B = K(J_a, J_b) and the leaf D follow H2-H5 unchanged.
Also the HSS mat-vec (reading M) and an independent dense assembly from the
generators (used by tests).  All indices into points are TREE (permuted) positions.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla

from .kernel import gaussian_block, sketch as dense_sketch


@dataclass
class HSS:
    n: int
    L: int
    ranges: list            # ranges[l][i] = (lo, hi) in tree positions
    Fp: np.ndarray          # permuted features
    h: float
    D: dict = field(default_factory=dict)        # leaf id -> (m x m)
    U: dict = field(default_factory=dict)        # node id -> rows x k, or None (pass-through)
    k: dict = field(default_factory=dict)        # node id -> rank
    rows: dict = field(default_factory=dict)     # node id -> active row count
    Jloc: dict = field(default_factory=dict)     # node id -> local pivot indices (len k)
    J: dict = field(default_factory=dict)        # node id -> tree positions of skeleton (len k)
    B: dict = field(default_factory=dict)        # parent id -> (k_a x k_b)
    Rdiag: dict = field(default_factory=dict)    # node id -> |diag R| of the CPQR (for audit)
    cap_hit: dict = field(default_factory=dict)  # node id -> bool (tolerance unmet at cap)

    def node_id(self, lvl, i):
        return (1 << lvl) - 1 + i

    def is_passthrough(self, t):
        return self.U.get(t) is None

    def nodes(self, lvl):
        return [((1 << lvl) - 1 + i, lo, hi) for i, (lo, hi) in enumerate(self.ranges[lvl])]


def choose_rank(rdiag: np.ndarray, rows: int, s: int, *, fixed_rank=None,
                rel_tol=0.0, abs_tol=0.0, cap=None):
    """AMB-10: k = leading run of |R_jj| > max(rel_tol |R_11|, abs_tol sqrt(s)), then
    min(k, cap, rows).  Fixed-rank mode: min(fixed_rank, rows, len(rdiag)).
    Returns (k, cap_hit)."""
    ncand = len(rdiag)
    if fixed_rank is not None:
        return int(min(fixed_rank, rows, ncand)), False
    a = np.abs(rdiag)
    if ncand == 0:
        return 0, False
    thr = max(rel_tol * a[0], abs_tol * np.sqrt(s))
    above = a > thr
    k_tol = ncand if above.all() else int(np.argmin(above))
    k = k_tol
    cap_hit = False
    if cap is not None and k > cap:
        k, cap_hit = cap, True
    if k > rows:
        k = rows
    return int(k), cap_hit


def nystrom_u(Fp: np.ndarray, h: float, act: np.ndarray, J: np.ndarray, eps: float) -> np.ndarray:
    """N4: U = K(A, J) (K(J, J) + eps I)^-1 (rows x k), by the Cholesky factor of K(J,J) + eps I."""
    G = gaussian_block(Fp[J], Fp[J], h) + eps * np.eye(len(J))
    c = sla.cho_factor(G, lower=True)
    return sla.cho_solve(c, gaussian_block(Fp[J], Fp[act], h)).T


def compress(Fp: np.ndarray, h: float, ranges, Omega_p: np.ndarray, *, ranks=None,
             rel_tol=0.0, abs_tol=0.0, cap=None, S=None, skeletons=None,
             interp: str = "id", spd_eps: float = 1e-10) -> HSS:
    """H1-H5.  `ranks` (dict or array indexed by BFS node id) selects fixed-rank mode.

    `skeletons` (dict: node id -> tree positions J_t in pivot order, every non-root node)
    selects the fixed-skeleton diagnostic mode (AMB-12): in H3 the pivots are J_t's local
    indices followed by the other active rows in increasing order, the QR of Y_t^T is taken
    WITHOUT pivoting in that column order, k = len(J_t), and U, J, Y_sk, Omega' follow as usual
    (U[piv[k:]] = (R11^-1 R12)^T, the interpolation coefficients of the given skeleton).

    `interp` = "id" (H3, the paper's interpolative decomposition) or "spd" (N4: the same
    skeletons, U_t = K(A_t, J_t)(K(J_t, J_t) + spd_eps I)^-1; module docstring)."""
    if interp not in ("id", "spd"):
        raise ValueError(f"interp must be 'id' or 'spd', got {interp!r}")
    n, s = Omega_p.shape
    L = len(ranges) - 1
    hss = HSS(n=n, L=L, ranges=ranges, Fp=Fp, h=h)
    if S is None:
        S = dense_sketch(Fp, h, Omega_p)                          # H1
    Y, Om, act = {}, {}, {}
    for t, lo, hi in hss.nodes(L):                                # H2
        Dt = gaussian_block(Fp[lo:hi], Fp[lo:hi], h)
        hss.D[t] = Dt
        Y[t] = S[lo:hi] - Dt @ Omega_p[lo:hi]
        Om[t] = Omega_p[lo:hi]
        act[t] = np.arange(lo, hi)
    for lvl in range(L, 0, -1):
        for t, lo, hi in hss.nodes(lvl):
            if lvl < L:                                           # H4 (t is a parent)
                a, b = 2 * t + 1, 2 * t + 2
                Bt = gaussian_block(Fp[hss.J[a]], Fp[hss.J[b]], h)
                hss.B[t] = Bt
                Y[t] = np.vstack([Y[a] - Bt @ Om[b], Y[b] - Bt.T @ Om[a]])
                Om[t] = np.vstack([Om[a], Om[b]])
                act[t] = np.concatenate([hss.J[a], hss.J[b]])
                # children's Y entries now hold Y_sk; free them
                del Y[a], Y[b], Om[a], Om[b]
            Yt = Y[t]
            rows = Yt.shape[0]
            hss.rows[t] = rows
            if skeletons is not None:                             # H3, fixed skeleton
                Jt = np.asarray(skeletons[t], dtype=np.int64)
                where = {int(a): q for q, a in enumerate(act[t])}
                loc = [where[int(a)] for a in Jt]
                if len(set(loc)) != len(loc):
                    raise ValueError(f"skeleton of node {t} repeats an active row")
                rest = [q for q in range(rows) if q not in set(loc)]
                piv = np.array(loc + rest, dtype=np.int64)
                k = len(loc)
                R = sla.qr(Yt.T[:, piv], mode="r")[0] if rows else np.zeros((0, 0))
                rd = np.abs(np.diag(R)) if R.size else np.zeros(0)
                hss.Rdiag[t], hss.cap_hit[t], hss.k[t] = rd, False, k
                if k == rows:
                    if list(loc) != list(range(rows)):
                        raise ValueError(f"pass-through node {t}: skeleton must be its active rows in order")
                    hss.U[t], hss.Jloc[t], hss.J[t] = None, np.arange(rows), act[t]
                else:
                    if interp == "spd":
                        U = nystrom_u(Fp, h, act[t], act[t][piv[:k]], spd_eps)
                    else:
                        T = sla.solve_triangular(R[:k, :k], R[:k, k:], lower=False)
                        U = np.zeros((rows, k))
                        U[piv[:k]] = np.eye(k)
                        U[piv[k:]] = T.T
                    hss.U[t], hss.Jloc[t], hss.J[t] = U, piv[:k].copy(), act[t][piv[:k]]
                    Y[t] = Yt[piv[:k]]
                    Om[t] = U.T @ Om[t]
                continue
            if rows == 0:
                _Q, R, piv = None, np.zeros((0, 0)), np.zeros(0, dtype=np.int64)
            else:                                                 # H3
                _Q, R, piv = sla.qr(Yt.T, mode="economic", pivoting=True)
            rd = np.abs(np.diag(R)) if R.size else np.zeros(0)
            hss.Rdiag[t] = rd
            fixed = None if ranks is None else int(ranks[t])
            k, hit = choose_rank(rd, rows, s, fixed_rank=fixed, rel_tol=rel_tol,
                                 abs_tol=abs_tol, cap=cap)
            hss.cap_hit[t] = hit
            hss.k[t] = k
            if k == rows:                                         # pass-through
                hss.U[t] = None
                hss.Jloc[t] = np.arange(rows)
                hss.J[t] = act[t]
                # Y[t] (= Y_sk) and Om[t] (= Omega') unchanged
            else:
                if interp == "spd":                               # N4
                    U = nystrom_u(Fp, h, act[t], act[t][piv[:k]], spd_eps)
                else:
                    T = sla.solve_triangular(R[:k, :k], R[:k, k:], lower=False)
                    U = np.zeros((rows, k))
                    U[piv[:k]] = np.eye(k)
                    U[piv[k:]] = T.T
                hss.U[t] = U
                hss.Jloc[t] = piv[:k].copy()
                hss.J[t] = act[t][piv[:k]]
                Y[t] = Yt[piv[:k]]
                Om[t] = U.T @ Om[t]
    if L > 0:                                                     # H5
        Bt = gaussian_block(Fp[hss.J[1]], Fp[hss.J[2]], h)
        hss.B[0] = Bt
    else:
        hss.D[0] = gaussian_block(Fp, Fp, h)
    return hss


def skeletons_from_flat(flat, ranks, ranges, s):
    """The flat skeleton layout of the C-ABI (hss_info's skel_out, hss_opts.skeletons: levels
    1..L, nodes in BFS order, k_t tree positions each) -> dict node id -> J_t.  k_t follows the
    fixed-rank rule min(ranks[t], rows_t, s), rows_t = leaf size or the children's k."""
    L = len(ranges) - 1
    k = {}
    for lvl in range(L, 0, -1):
        for i, (lo, hi) in enumerate(ranges[lvl]):
            t = (1 << lvl) - 1 + i
            rows = hi - lo if lvl == L else k[2 * t + 1] + k[2 * t + 2]
            k[t] = int(max(0, min(int(ranks[t]), rows, s)))
    out, off = {}, 0
    flat = np.asarray(flat, dtype=np.int64)
    for lvl in range(1, L + 1):
        for i in range(len(ranges[lvl])):
            t = (1 << lvl) - 1 + i
            out[t] = flat[off:off + k[t]]
            off += k[t]
    if off != flat.size:
        raise ValueError(f"flat skeleton array has {flat.size} entries, the ranks need {off}")
    return out


def unconverged(hss: HSS, s: int, p: int, cap) -> list:
    """N2b: nodes whose rank ran into the sample budget: k > s - p while more rank was possible
    (k < min(cap, rows))."""
    bad = []
    for t, k in hss.k.items():
        lim = hss.rows[t] if cap is None else min(cap, hss.rows[t])
        if k > s - p and k < lim:
            bad.append(t)
    return bad


def compress_adaptive(Fp: np.ndarray, h: float, ranges, perm: np.ndarray, seed: int, *, s0: int, ds: int,
                      s_max: int, p: int, rel_tol=0.0, abs_tol=0.0, cap=None):
    """N2 (P:70 / P:184, adaptive randomized sampling; our reading):
      N2a  start with s = min(s0, s_max) columns of Omega (R1-R3: column j of Omega does not
           depend on s, so a larger s only appends columns);
      N2b  compress (H1-H5); if any node is unconverged (its rank reached s - p while
           min(cap, rows) allowed more), s = min(s + ds, s_max) and compress again from scratch;
      N2c  stop when every node converged or s = s_max.
    Returns (hss, s_final, rounds)."""
    from .rng import omega
    s = min(s0, s_max)
    rounds = 0
    while True:
        rounds += 1
        Om = omega(seed, perm, s)
        H = compress(Fp, h, ranges, Om, rel_tol=rel_tol, abs_tol=abs_tol, cap=cap)
        if s >= s_max or not unconverged(H, s, p, cap):
            return H, s, rounds
        s = min(s + ds, s_max)


def matvec(hss: HSS, V: np.ndarray) -> np.ndarray:
    """M: K~ V in tree order (upward U^T sweep, B coupling, downward U sweep, leaf D)."""
    V = np.asarray(V, dtype=np.float64)
    vec = V.ndim == 1
    if vec:
        V = V[:, None]
    L = hss.L
    out = np.zeros_like(V)
    if L == 0:
        out = hss.D[0] @ V
        return out[:, 0] if vec else out
    up = {}
    for lvl in range(L, 0, -1):
        for t, lo, hi in hss.nodes(lvl):
            x = V[lo:hi] if lvl == L else np.vstack([up[2 * t + 1], up[2 * t + 2]])
            up[t] = x if hss.is_passthrough(t) else hss.U[t].T @ x
    down = {}
    for lvl in range(0, L):
        for t, lo, hi in hss.nodes(lvl):
            a, b = 2 * t + 1, 2 * t + 2
            ga = hss.B[t] @ up[b]
            gb = hss.B[t].T @ up[a]
            if lvl > 0:
                g = down[t] if hss.is_passthrough(t) else hss.U[t] @ down[t]
                ka = hss.k[a]
                ga = ga + g[:ka]
                gb = gb + g[ka:]
            down[a], down[b] = ga, gb
    for t, lo, hi in hss.nodes(L):
        g = down[t] if hss.is_passthrough(t) else hss.U[t] @ down[t]
        out[lo:hi] = hss.D[t] @ V[lo:hi] + g
    return out[:, 0] if vec else out


def big_basis(hss: HSS):
    """U^big_t (node points x k_t): leaf U (or I), internal blockdiag(U^big_a, U^big_b) U_t."""
    Ub = {}
    for lvl in range(hss.L, 0, -1):
        for t, lo, hi in hss.nodes(lvl):
            if lvl == hss.L:
                base = np.eye(hi - lo)
            else:
                a, b = 2 * t + 1, 2 * t + 2
                base = sla.block_diag(Ub[a], Ub[b])
            Ub[t] = base if hss.is_passthrough(t) else base @ hss.U[t]
    return Ub


def assemble_dense(hss: HSS) -> np.ndarray:
    """K~ from its generators directly (independent of `matvec`): leaf D blocks plus
    U^big_a B_ab U^big_b^T on every sibling block."""
    n = hss.n
    if n > 16384:
        raise ValueError("assemble_dense refuses n > 16384")
    K = np.zeros((n, n))
    if hss.L == 0:
        return hss.D[0].copy()
    Ub = big_basis(hss)
    for t, lo, hi in hss.nodes(hss.L):
        K[lo:hi, lo:hi] = hss.D[t]
    for lvl in range(0, hss.L):
        for t, lo, hi in hss.nodes(lvl):
            a, b = 2 * t + 1, 2 * t + 2
            (alo, ahi), (blo, bhi) = hss.ranges[lvl + 1][2 * (t - ((1 << lvl) - 1))], \
                hss.ranges[lvl + 1][2 * (t - ((1 << lvl) - 1)) + 1]
            blk = Ub[a] @ hss.B[t] @ Ub[b].T
            K[alo:ahi, blo:bhi] = blk
            K[blo:bhi, alo:ahi] = blk.T
    return K


def memory_bytes(hss: HSS) -> int:
    """D6: bytes of the generators (D, U, B) in fp64."""
    tot = sum(d.size for d in hss.D.values())
    tot += sum(u.size for u in hss.U.values() if u is not None)
    tot += sum(b.size for b in hss.B.values())
    return 8 * tot
