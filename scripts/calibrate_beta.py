"""AMB-9 beta calibration with the ORACLE only (oracle/ + datagen/).

beta = schedule(n) if lambda_min(K~) >= 0, else
       max(schedule(n), 10^ceil(log10(-4 lambda_min(K~)))).
lambda_min from eigsh(LinearOperator(K~ matvec), which='SA').  Optionally the chaos
gate (E10): ADMM from z0 and from z0 + 1e-12 perturbation must stay < 1e-9 apart.
Usage: python scripts/calibrate_beta.py --config 1 [--n 4096] [--h 0.5] [--chaos-it 200]
Appends one JSON line to configs/beta_calibration.jsonl.
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
from scipy.sparse.linalg import LinearOperator, eigsh  # noqa: E402

import datagen  # noqa: E402
from oracle import admm, hss, pipeline, ulv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--h", type=float, default=None)
    ap.add_argument("--chaos-it", type=int, default=0)
    ap.add_argument("--sampling", default="sketch", choices=["sketch", "ann"])
    a = ap.parse_args()
    cfg = datagen.get_config(a.config)
    n = a.n or cfg["n"]
    h = a.h if a.h is not None else (cfg["h"] if not isinstance(cfg["h"], list) else cfg["h"][0])
    F, y, _, _ = datagen.generate(a.config, n=n, n_test=0)
    t0 = time.time()
    tm = {}
    if a.sampling == "ann":
        perm, ranges, _, H = pipeline.build_ann(F, cfg, h=h, timings=tm)
    else:
        perm, ranges, Om, H = pipeline.build(F, cfg, h=h, timings=tm)
    print("built", tm, flush=True)
    op = LinearOperator((n, n), matvec=lambda v: hss.matvec(H, v), dtype=np.float64)
    lmin = float(eigsh(op, k=1, which="SA", tol=1e-4, maxiter=20000)[0][0])
    print("lambda_min", lmin, "after", time.time() - t0, "s", flush=True)
    sched = datagen.beta_schedule(n)
    beta = sched if lmin >= 0 else max(sched, 10.0 ** math.ceil(math.log10(-4 * lmin)))
    rec = dict(config=a.config, n=n, h=h, lambda_min=lmin, schedule=sched, beta=beta,
               timings=tm, secs=time.time() - t0)
    if a.sampling != "sketch":
        rec["sampling"] = a.sampling
    if a.chaos_it:
        f = ulv.factor(H, beta)
        solve = lambda b: ulv.solve(f, b)  # noqa: E731
        yp = y[perm]
        C = cfg["C"][0]
        o1 = admm.run(solve, yp, C, beta, a.chaos_it)
        z0 = 1e-12 * np.random.default_rng(0).standard_normal(n)
        o2 = admm.run(solve, yp, C, beta, a.chaos_it, z0=z0)
        rec["chaos_div"] = float(np.abs(o1["z"] - o2["z"]).max())
    os.makedirs(os.path.join(ROOT, "configs"), exist_ok=True)
    with open(os.path.join(ROOT, "configs/beta_calibration.jsonl"), "a") as fo:
        fo.write(json.dumps(rec) + "\n")
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
