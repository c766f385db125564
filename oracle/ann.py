"""HSS-ANN column sampling — oracle side.

P:186 says the construction's "matrix-times-vector operation is further approximated using a
column sampling based on Approximate Nearest Neighbours of the data points ... which uses the
similarity between them to identify the dominating entries of the kernel matrix", and P:187 that
this makes the construction O(r^2 d) (r = max HSS rank, d = points).  The details live in the
cited [9139856], which is not in PAPER.md, so the steps below are our reading (DESIGN.md
"Readings", N1-N3); every integer decision is made in exact arithmetic so that the CUDA path
can reproduce it bit for bit:

  N1  ANN.  `trees` random-projection trees over the ORIGINAL points.  Tree t has
      L_t = max(0, ceil(log2(n / leaf))) levels (every node split exactly L_t times, as T1);
      node (l, i) (BFS id b = 2^l - 1 + i) splits its points at the median of
      p_j = sum_f s_f F[j, f] (features in order, float64 adds; s_f = +1 if bit 63 of
      splitmix64(key_t + 2^20 b + f) is 0 else -1, key_t = splitmix64(seed + t)), by a stable sort
      on (p, original index), left = the first floor(|P|/2).  Candidates of point i: the other
      points of i's leaf, in every tree.  d(i, j) = sum_f (F[i,f] - F[j,f])^2 in feature order,
      each square rounded before it is added (no fused multiply-add).  ANN(i) = the `kappa`
      distinct candidates with the smallest (d, original index).
  N2  Sampled columns of a non-root node t with tree-position range [lo, hi) and active rows A_t
      (leaf: its points; parent: the children's skeletons): the pairs (d(i, j), pos(j)) for i in
      A_t and j in ANN(i) with pos(j) outside [lo, hi), ordered by (d, pos); keep the first s
      distinct positions.  If fewer than s exist, add random outside positions: for q = 0, 1, ...
      u = splitmix64(key + 2^20 b + q) (key = splitmix64(seed), b = BFS id), p = u mod (n - w)
      (w = hi - lo), p += w if p >= lo; skip positions already taken; stop at s (or when every
      outside position is taken; after 64 s draws the smallest untaken outside positions fill
      up).  C_t = the kept positions, sorted.
  N3  Y_t = K(A_t, C_t), the sampled off-diagonal block row, replaces the sketch rows in H3
      (CPQR of Y_t^T, rank rule AMB-10, U, J); there is no Omega and no sibling update.  D, B and
      everything after compression (ULV, ADMM) are unchanged.

Pins: tests/test_oracle_ann.py (brute-force kNN where the trees cannot miss, tree invariants,
sampling properties, and K~ = K when the sample is the whole off-diagonal block row).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .hss import HSS, choose_rank, nystrom_u
from .kernel import gaussian_block
from .rng import splitmix64
from .tree import node_ranges, num_levels

_TWO20 = np.uint64(1 << 20)


def rp_signs(seed: int, tree: int, node_id: int, r: int) -> np.ndarray:
    """N1: the +-1 direction of node `node_id` in tree `tree`."""
    with np.errstate(over="ignore"):
        key = splitmix64(np.uint64(seed) + np.uint64(tree))
        u = splitmix64(key + np.uint64(node_id) * _TWO20 + np.arange(r, dtype=np.uint64))
    return np.where((u >> np.uint64(63)) == 0, 1.0, -1.0)


def projection(X: np.ndarray, sgn: np.ndarray) -> np.ndarray:
    """p_j = sum_f s_f X[j, f], features in order (plain adds; s_f X exact)."""
    p = np.zeros(X.shape[0])
    for f in range(X.shape[1]):
        p = p + sgn[f] * X[:, f]
    return p


def rp_tree(F: np.ndarray, leaf: int, seed: int, tree: int):
    """N1: (perm, ranges) of random-projection tree `tree` (perm[pos] = original index)."""
    n, r = F.shape
    L = num_levels(n, leaf)
    ranges = node_ranges(n, L)
    perm = np.arange(n, dtype=np.int64)
    for lvl in range(L):
        for i, (lo, hi) in enumerate(ranges[lvl]):
            idx = perm[lo:hi].copy()
            p = projection(F[idx], rp_signs(seed, tree, (1 << lvl) - 1 + i, r))
            perm[lo:hi] = idx[np.lexsort((idx, p))]
    return perm, ranges


def sqdist(Fa: np.ndarray, Fb: np.ndarray) -> np.ndarray:
    """d(i, j) = sum_f (Fa[i,f] - Fb[j,f])^2, features in order, squares rounded first."""
    d = np.zeros((Fa.shape[0], Fb.shape[0]))
    for f in range(Fa.shape[1]):
        t = Fa[:, f][:, None] - Fb[:, f][None, :]
        d = d + t * t
    return d


def knn(F: np.ndarray, kappa: int, trees: int, leaf: int, seed: int):
    """N1: ANN lists.  Returns (idx, dist), n x kappa, original indices sorted by (d, index);
    -1 / inf where fewer than kappa candidates exist."""
    n = F.shape[0]
    cand = [[] for _ in range(n)]
    for t in range(trees):
        perm, ranges = rp_tree(F, leaf, seed, t)
        for lo, hi in ranges[-1]:
            pts = perm[lo:hi]
            for a in pts:
                cand[a].append(pts)
    idx = np.full((n, kappa), -1, dtype=np.int64)
    dist = np.full((n, kappa), np.inf)
    for i in range(n):
        c = np.unique(np.concatenate(cand[i]))
        c = c[c != i]
        if c.size == 0:
            continue
        d = sqdist(F[i:i + 1], F[c])[0]
        o = np.lexsort((c, d))[:kappa]
        idx[i, :o.size] = c[o]
        dist[i, :o.size] = d[o]
    return idx, dist


def sample_columns(node_id: int, lo: int, hi: int, n: int, active_pos: np.ndarray,
                   ann_pos: np.ndarray, ann_d: np.ndarray, s: int, seed: int) -> np.ndarray:
    """N2: the sampled column positions of a node (sorted tree positions)."""
    P = ann_pos[active_pos].ravel()
    D = ann_d[active_pos].ravel()
    keep = (P >= 0) & ((P < lo) | (P >= hi))
    P, D = P[keep], D[keep]
    o = np.lexsort((P, D))
    chosen, seen = [], set()
    for q in P[o]:
        if len(chosen) == s:
            break
        if q not in seen:
            seen.add(q)
            chosen.append(int(q))
    w = hi - lo
    target = min(s, n - w)
    if len(chosen) < target:
        key = splitmix64(np.uint64(seed))
        q = 0
        while len(chosen) < target and q < 64 * s:
            with np.errstate(over="ignore"):
                u = splitmix64(key + np.uint64(node_id) * _TWO20 + np.uint64(q))
            p = int(u % np.uint64(n - w))
            if p >= lo:
                p += w
            if p not in seen:
                seen.add(p)
                chosen.append(p)
            q += 1
        p = 0
        while len(chosen) < target:
            if (p < lo or p >= hi) and p not in seen:
                seen.add(p)
                chosen.append(p)
            p += 1
    return np.sort(np.array(chosen, dtype=np.int64))


def compress_ann(Fp: np.ndarray, h: float, ranges, perm: np.ndarray, ann_idx: np.ndarray,
                 ann_d: np.ndarray, s: int, seed: int, *, ranks=None, rel_tol=0.0, abs_tol=0.0,
                 cap=None, interp: str = "id", spd_eps: float = 1e-10) -> HSS:
    """H2-H5 with N2-N3 in place of the sketch.  ann_idx: n x kappa ORIGINAL indices (knn());
    rows of ann_* are indexed by ORIGINAL index.  interp="spd": N4's kernel interpolant onto the
    same skeletons (oracle/hss.py; the sampled columns do not depend on U here)."""
    if interp not in ("id", "spd"):
        raise ValueError(f"interp must be 'id' or 'spd', got {interp!r}")
    n = Fp.shape[0]
    L = len(ranges) - 1
    hss = HSS(n=n, L=L, ranges=ranges, Fp=Fp, h=h)
    iperm = np.empty(n, dtype=np.int64)
    iperm[perm] = np.arange(n)
    # ANN lists re-indexed by tree position (row p = point perm[p]), entries as tree positions
    ann_dp = ann_d[perm]
    ann_pos = np.where(ann_idx[perm] >= 0, iperm[np.maximum(ann_idx[perm], 0)], -1)
    act = {}
    for t, lo, hi in hss.nodes(L):
        hss.D[t] = gaussian_block(Fp[lo:hi], Fp[lo:hi], h)
        act[t] = np.arange(lo, hi)
    for lvl in range(L, 0, -1):
        for t, lo, hi in hss.nodes(lvl):
            if lvl < L:
                a, b = 2 * t + 1, 2 * t + 2
                hss.B[t] = gaussian_block(Fp[hss.J[a]], Fp[hss.J[b]], h)
                act[t] = np.concatenate([hss.J[a], hss.J[b]])
            A = act[t]
            rows = A.shape[0]
            hss.rows[t] = rows
            C = sample_columns(t, lo, hi, n, A, ann_pos, ann_dp, s, seed)         # N2
            Yt = gaussian_block(Fp[A], Fp[C], h)                                  # N3
            if rows == 0 or C.size == 0:
                R, piv = np.zeros((0, 0)), np.zeros(0, dtype=np.int64)
            else:
                _Q, R, piv = sla.qr(Yt.T, mode="economic", pivoting=True)
            rd = np.abs(np.diag(R)) if R.size else np.zeros(0)
            hss.Rdiag[t] = rd
            fixed = None if ranks is None else int(ranks[t])
            k, hit = choose_rank(rd, rows, s, fixed_rank=fixed, rel_tol=rel_tol, abs_tol=abs_tol, cap=cap)
            hss.cap_hit[t] = hit
            hss.k[t] = k
            if k == rows:
                hss.U[t] = None
                hss.Jloc[t] = np.arange(rows)
                hss.J[t] = A
            else:
                if interp == "spd":                                               # N4
                    U = nystrom_u(Fp, h, A, A[piv[:k]], spd_eps)
                else:
                    T = sla.solve_triangular(R[:k, :k], R[:k, k:], lower=False)
                    U = np.zeros((rows, k))
                    U[piv[:k]] = np.eye(k)
                    U[piv[k:]] = T.T
                hss.U[t] = U
                hss.Jloc[t] = piv[:k].copy()
                hss.J[t] = A[piv[:k]]
    if L > 0:
        hss.B[0] = gaussian_block(Fp[hss.J[1]], Fp[hss.J[2]], h)
    else:
        hss.D[0] = gaussian_block(Fp, Fp, h)
    return hss
