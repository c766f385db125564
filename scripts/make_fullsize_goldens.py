"""Full-size oracle goldens for configs 2 and 3 (and the AMB-9 chaos gate), oracle only.

Calls ONLY `oracle/` and `datagen/` (never the CUDA path).  The GPU tests
(tests/test_gpu_fullsize_golden.py) compare the product, at BASELINE.json's full sizes
and in the launch configuration bench.py times, with what this script writes:

  tests/golden/cfg{c}_full.json   scalars, hashes, ranks, the AMB-9 chaos gate record
  tests/golden/cfg{c}_full.npz    sampled arrays (indices + values)

Contents (Alg. 3 end to end):
  - sha256 of perm (T1-T4), ranks array, skeletons (H3, per level and total);
  - 2048 seeded rows of the sketch S = K_p Omega_p (H1);
  - per level, two nodes' generators: 8 rows of U and U g (H3; U is sign-free),
    8 rows of B and B g (H4), 8 rows of two leaves' D (H2);
  - w1 and samples of v = K_b^-1 e (A0) and of x = K_b^-1 b for a seeded b (readings S);
  - z, mu after 10 / 100 / MaxIt iterations (A1-A4), bias (AMB-2/3) and f~ (Eq. 8);
  - decision values of 1024 seeded test points with the final z;
  - AMB-9 chaos gate: ADMM from z0 = 0 and from z0 = 1e-12 N(0,1) for MaxIt iterations,
    max |z1 - z2| (must stay < 1e-9).
Vectors are in ORIGINAL point order; samples are seeded index sets (stored).

The compressed HSS is cached (pickle, ~4 GB at cfg 3) under .golden_cache/ so that a
re-run with another beta reuses the 2.3 h oracle compression of cfg 3.
Usage: python scripts/make_fullsize_goldens.py --config 3 [--beta B] [--no-chaos]
"""
import argparse
import hashlib
import json
import os
import pickle
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import datagen  # noqa: E402
from oracle import admm, hss, kernel, pipeline, rng, svm, tree, ulv  # noqa: E402

CACHE = os.path.join(ROOT, ".golden_cache")
SPD_EPS = 1e-12  # N4 jitter (bench.py / tests use the same)
GOLD = os.path.join(ROOT, "tests", "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def build_cached(tag, cfg, F, interp="id"):
    path = os.path.join(CACHE, f"{tag}_hss.pkl")
    if os.path.exists(path):
        log("loading cached HSS", path)
        with open(path, "rb") as f:
            return pickle.load(f)
    tm = {}
    t0 = time.time()
    perm, ranges = tree.build_tree(F, cfg["leaf"], cfg["seed_tree"])
    tm["tree"] = time.time() - t0
    log("tree", tm["tree"])
    Fp = F[perm]
    Om = rng.omega(cfg["seed_omega"], perm, cfg["s"])
    t0 = time.time()
    S = kernel.sketch(Fp, cfg["h"], Om)
    tm["sketch"] = time.time() - t0
    log("sketch", tm["sketch"])
    t0 = time.time()
    H = hss.compress(Fp, cfg["h"], ranges, Om, rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"],
                     cap=cfg["cap"], S=S, interp=interp, spd_eps=SPD_EPS)
    tm["compress_after_sketch"] = time.time() - t0
    log("compress", tm["compress_after_sketch"])
    g = np.random.default_rng(50 + cfg["id"])
    rows = np.sort(g.choice(F.shape[0], min(2048, F.shape[0]), replace=False))
    out = dict(perm=perm, ranges=ranges, H=H, S_rows_idx=rows, S_rows=S[rows].copy(), timings=tm)
    del S
    os.makedirs(CACHE, exist_ok=True)
    with open(path + ".tmp", "wb") as f:
        pickle.dump(out, f, protocol=5)
    os.replace(path + ".tmp", path)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--beta", type=float, default=None)
    ap.add_argument("--h", type=float, default=None, help="config 4: one grid width")
    ap.add_argument("--no-chaos", action="store_true")
    ap.add_argument("--interp", default="id", choices=["id", "spd"],
                    help="spd: N4 SPD-preserving compression at the paper's beta schedule (tag cfg{c}_spd)")
    ap.add_argument("--n", type=int, default=None, help="smoke-test size (writes under --out)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    global GOLD, CACHE
    if a.out:
        GOLD = CACHE = a.out
    c = a.config
    cfg = datagen.get_config(c)
    tag = f"cfg{c}"
    if isinstance(cfg["h"], list):                      # config 4: one h of the grid
        cfg["h"] = a.h if a.h is not None else cfg["h"][0]
        cfg["beta"] = cfg["beta_per_h"][cfg["h"]]
        tag = f"cfg{c}_h{cfg['h']:g}"
    if a.interp == "spd":
        tag += "_spd"
        cfg["beta"] = datagen.configs.beta_schedule(cfg["n"] if a.n is None else a.n)
    beta = cfg["beta"] if a.beta is None else a.beta
    C = cfg["C"][0]
    max_it = cfg["max_it"]
    F, y, Ft, _ = datagen.generate(c, n=a.n, n_test=None if a.n is None else 2048)
    n = F.shape[0]
    log("config", c, "n", n, "beta", beta)
    B = build_cached(tag, cfg, F, a.interp)
    perm, H = B["perm"], B["H"]
    L = H.L
    nn = 2 ** (L + 1) - 1
    inv = np.empty_like(perm)
    inv[perm] = np.arange(n)
    g = np.random.default_rng(60 + c)
    nsamp = min(n, 65536)
    vidx = np.sort(g.choice(n, nsamp, replace=False)) if nsamp < n else np.arange(n)

    meta = dict(config=c, n=n, r=F.shape[1], h=cfg["h"], C=C, beta=beta, max_it=max_it, interp=a.interp,
                leaf=cfg["leaf"], cap=cfg["cap"], s=cfg["s"], rel_tol=cfg["rel_tol"],
                seed_omega=cfg["seed_omega"], seed_tree=cfg["seed_tree"], L=L,
                oracle_timings_s=dict(B["timings"]),
                host=dict(cpu=platform.processor() or platform.machine(),
                          cores=len(os.sched_getaffinity(0))))
    ranks = pipeline.ranks_array(H, nn)
    skel_lv = []
    for lv in range(1, L + 1):
        skel_lv.append(sha(np.concatenate([H.J[t] for t in range((1 << lv) - 1, (1 << (lv + 1)) - 1)])
                           .astype(np.int64)))
    skel = np.concatenate([H.J[t] for t in range(1, nn)]).astype(np.int64)
    meta.update(perm_sha256=sha(perm.astype(np.int64)), ranks=ranks.tolist(),
                skeleton_sha256=sha(skel), skeleton_level_sha256=skel_lv, skeleton_len=int(skel.size),
                cap_hits=int(sum(H.cap_hit.values())))
    arrs = dict(S_rows_idx=B["S_rows_idx"], S_rows=B["S_rows"], vidx=vidx)

    # generators of sampled nodes (two per level)
    gn = np.random.default_rng(70 + c)
    nodes, recs = [], []
    for lv in range(0, L + 1):
        lo = (1 << lv) - 1
        cnt = 1 << lv
        pick = sorted({lo, lo + int(gn.integers(0, cnt))})
        for t in pick:
            nodes.append(t)
            if lv > 0:
                rows_t, k_t = H.rows[t], H.k[t]
                U = H.U[t] if H.U[t] is not None else np.eye(rows_t)
                ri = np.sort(gn.choice(rows_t, min(8, rows_t), replace=False))
                gk = gn.standard_normal(k_t)
                arrs[f"U{t}_ri"], arrs[f"U{t}_rows"], arrs[f"U{t}_g"], arrs[f"U{t}_Ug"] = ri, U[ri], gk, U @ gk
            if lv < L:
                Bt = H.B[t]
                ri = np.sort(gn.choice(Bt.shape[0], min(8, Bt.shape[0]), replace=False))
                gk = gn.standard_normal(Bt.shape[1])
                arrs[f"B{t}_ri"], arrs[f"B{t}_rows"], arrs[f"B{t}_g"], arrs[f"B{t}_Bg"] = ri, Bt[ri], gk, Bt @ gk
            else:
                Dt = H.D[t]
                ri = np.sort(gn.choice(Dt.shape[0], min(8, Dt.shape[0]), replace=False))
                arrs[f"D{t}_ri"], arrs[f"D{t}_rows"] = ri, Dt[ri]
            recs.append(t)
    meta["sampled_nodes"] = nodes

    t0 = time.time()
    fac = ulv.factor(H, beta)
    meta["oracle_timings_s"]["factor"] = time.time() - t0
    log("factor", meta["oracle_timings_s"]["factor"])
    yp = y[perm]

    def solve(b):
        return ulv.solve(fac, b)

    # A0 and a seeded solve (vectors in original order)
    t0 = time.time()
    bvec = np.random.default_rng(80 + c).standard_normal(n)
    xs = np.empty(n)
    xs[perm] = solve(bvec[perm])
    meta["oracle_timings_s"]["solve"] = time.time() - t0
    w, w1 = admm.precompute(solve, yp)
    meta["w1"] = w1
    arrs["solve_b_seed"] = np.array([80 + c])
    arrs["x_solve"] = xs[vidx]
    meta["x_solve_norm"] = float(np.linalg.norm(xs))
    wo = np.empty(n)
    wo[perm] = w
    arrs["w"] = wo[vidx]
    meta["w_norm"] = float(np.linalg.norm(wo))

    # ADMM (A1-A4) with traces at 10, 100 and MaxIt
    t0 = time.time()
    o = admm.run(solve, yp, C, beta, max_it, trace_every=10)
    meta["oracle_timings_s"]["admm"] = time.time() - t0
    meta["oracle_timings_s"]["admm_per_iter"] = meta["oracle_timings_s"]["admm"] / max_it
    log("admm", meta["oracle_timings_s"]["admm"])
    keep = sorted({10, min(100, max_it), max_it})
    meta["trace_its"] = keep
    for it, z, mu in o["trace"]:
        if it in keep:
            zo, muo = z[inv], mu[inv]
            arrs[f"z{it}"], arrs[f"mu{it}"] = zo[vidx], muo[vidx]
            meta[f"z{it}_norm"], meta[f"mu{it}_norm"] = float(np.linalg.norm(zo)), float(np.linalg.norm(muo))
    mv = lambda v: hss.matvec(H, v)  # noqa: E731
    t0 = time.time()
    meta["bias"] = svm.bias(mv, o["z"], yp, C)
    meta["objective"] = svm.objective(mv, o["z"], yp)
    meta["oracle_timings_s"]["bias_objective"] = time.time() - t0
    zf = o["z"][inv]
    meta["n_sv"] = int((zf > 1e-8 * C).sum())
    ti = np.sort(np.random.default_rng(90 + c).choice(Ft.shape[0], 1024, replace=False))
    t0 = time.time()
    dv = svm.decision_values(F, y * zf, cfg["h"], meta["bias"], Ft[ti])
    meta["oracle_timings_s"]["predict_1024"] = time.time() - t0
    arrs["test_idx"], arrs["dv"] = ti, dv
    log("bias", meta["bias"], "objective", meta["objective"])

    os.makedirs(GOLD, exist_ok=True)
    np.savez_compressed(os.path.join(GOLD, f"{tag}_full.npz"), **arrs)
    with open(os.path.join(GOLD, f"{tag}_full.json"), "w") as f:
        json.dump(meta, f, indent=1)
    log("wrote goldens")

    if not a.no_chaos:                                  # AMB-9 chaos gate (E10)
        t0 = time.time()
        z0 = 1e-12 * np.random.default_rng(0).standard_normal(n)
        o2 = admm.run(solve, yp, C, beta, max_it, z0=z0)
        div = float(np.abs(o["z"] - o2["z"]).max())
        rec = dict(config=c, n=n, h=cfg["h"], beta=beta, interp=a.interp, chaos_it=max_it, chaos_div=div,
                   chaos_pass=bool(div < 1e-9), secs=time.time() - t0, source="make_fullsize_goldens")
        if not a.out:
            with open(os.path.join(ROOT, "configs", "beta_calibration.jsonl"), "a") as f:
                f.write(json.dumps(rec) + "\n")
        meta["chaos"] = rec
        with open(os.path.join(GOLD, f"{tag}_full.json"), "w") as f:
            json.dump(meta, f, indent=1)
        log("chaos", rec)


if __name__ == "__main__":
    main()
