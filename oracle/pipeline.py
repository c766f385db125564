"""Alg. 3 end to end on the oracle side, for tests and the CPU baseline.

train(): tree (T) -> Omega (R) -> HSS (H) -> ULV (U) -> precompute + ADMM (A) per C
-> bias + objective (B) -> prediction (P).  Vectors returned in ORIGINAL point order.
"""
from __future__ import annotations

import time

import numpy as np

from . import admm as _admm
from . import hss as _hss
from . import rng as _rng
from . import svm as _svm
from . import tree as _tree
from . import ulv as _ulv


def build(F, cfg, h=None, ranks=None, S=None, timings=None):
    """Tree + Omega + compression. Returns (perm, ranges, Omega_p, hss)."""
    t = time.perf_counter()
    h = cfg["h"] if h is None else h
    perm, ranges = _tree.build_tree(F, cfg["leaf"], cfg["seed_tree"])
    t1 = time.perf_counter()
    Fp = F[perm]
    Om = _rng.omega(cfg["seed_omega"], perm, cfg["s"])
    kw = dict(ranks=ranks) if ranks is not None else dict(
        rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"], cap=cfg["cap"])
    H = _hss.compress(Fp, h, ranges, Om, S=S, **kw)
    if timings is not None:
        timings["tree"] = t1 - t
        timings["compress"] = time.perf_counter() - t1
    return perm, ranges, Om, H


def build_ann(F, cfg, h=None, ranks=None, timings=None, interp="id", spd_eps=1e-12):
    """Tree + ANN lists + HSS-ANN compression (N1-N3).  Returns (perm, ranges, (idx, d), hss)."""
    from . import ann as _ann
    t = time.perf_counter()
    h = cfg["h"] if h is None else h
    perm, ranges = _tree.build_tree(F, cfg["leaf"], cfg["seed_tree"])
    t1 = time.perf_counter()
    idx, d = _ann.knn(F, cfg["ann_neighbors"], cfg["ann_trees"], cfg["ann_leaf"], cfg["ann_seed"])
    t2 = time.perf_counter()
    kw = dict(ranks=ranks) if ranks is not None else dict(
        rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"], cap=cfg["cap"])
    H = _ann.compress_ann(F[perm], h, ranges, perm, idx, d, cfg["s"], cfg["ann_seed"], interp=interp,
                          spd_eps=spd_eps, **kw)
    if timings is not None:
        timings["tree"] = t1 - t
        timings["ann"] = t2 - t1
        timings["compress"] = time.perf_counter() - t2
    return perm, ranges, (idx, d), H


def train(F, y, cfg, *, h=None, C_list=None, ranks=None, max_it=None, trace_every=0,
          Ftest=None, timings=None):
    timings = {} if timings is None else timings
    h = cfg["h"] if h is None else h
    C_list = cfg["C"] if C_list is None else C_list
    max_it = cfg["max_it"] if max_it is None else max_it
    perm, ranges, Om, H = build(F, cfg, h=h, ranks=ranks, timings=timings)
    t = time.perf_counter()
    fac = _ulv.factor(H, cfg["beta"])
    timings["factor"] = time.perf_counter() - t
    yp = y[perm]
    solve = lambda b: _ulv.solve(fac, b)          # noqa: E731
    mv = lambda v: _hss.matvec(H, v)              # noqa: E731
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.shape[0])
    res = []
    for C in C_list:
        t = time.perf_counter()
        out = _admm.run(solve, yp, C, cfg["beta"], max_it, trace_every=trace_every)
        timings.setdefault("admm", 0.0)
        timings["admm"] += time.perf_counter() - t
        zp = out["z"]
        b = _svm.bias(mv, zp, yp, C)
        obj = _svm.objective(mv, zp, yp)
        r = dict(C=C, z=zp[inv], mu=out["mu"][inv], bias=b, obj=obj, w1=out["w1"],
                 trace=[(it, z[inv], mu[inv]) for it, z, mu in out["trace"]])
        if Ftest is not None:
            dv = _svm.decision_values(F, y * r["z"], h, b, Ftest)
            r["dv"], r["labels"] = dv, _svm.labels(dv)
        res.append(r)
    return dict(perm=perm, hss=H, ulv=fac, results=res, timings=timings)


def ranks_array(H, nnodes):
    """Per-node ranks in level-major BFS order (root = -1)."""
    a = np.full(nnodes, -1, dtype=np.int64)
    for t, k in H.k.items():
        a[t] = k
    return a
