"""Debug: GPU vs oracle ranks/skeletons on a scaled config (SVMHSS_CPQR_MODE from the env).
    python scripts/debug_case.py CFG N CAP"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2108_04167_b200 as P  # noqa: E402
from oracle import pipeline  # noqa: E402

c, n, cap = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cfg = datagen.get_config(c)
cfg["cap"], cfg["s"] = cap, cap + 16
F, y, _, _ = datagen.generate(c, n=n, n_test=0)
perm, ranges, Om, H = pipeline.build(F, cfg)
Hg = P.hss_build(torch.from_numpy(F).cuda(), cfg["h"], leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"],
                 max_rank=cap, oversample=16, omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"])
info = Hg.info()
nn = 2 ** (H.L + 1) - 1
ro = pipeline.ranks_array(H, nn)
print("mode", os.environ.get("SVMHSS_CPQR_MODE"), "perm eq", np.array_equal(info["perm"], perm),
      "ranks eq", np.array_equal(info["ranks"].astype(np.int64), ro))
off = 0
for t in range(1, nn):
    k = int(info["ranks"][t])
    Jg = info["skeletons"][off:off + k]
    off += k
    if k != H.k[t] or not np.array_equal(Jg, H.J[t]):
        m = next((q for q in range(min(k, H.k[t])) if Jg[q] != H.J[t][q]), -1)
        rd = H.Rdiag[t]
        print("node", t, "k", k, H.k[t], "first diff", m, "rdiag near", rd[max(0, m - 1):m + 2])
        break
else:
    print("all skeletons equal")
from oracle import admm, ulv, hss as ohss  # noqa: E402
beta = float(sys.argv[4]) if len(sys.argv) > 4 else 1e4
for t in range(1, nn):
    if H.U.get(t) is not None:
        U = Hg.node_generators(t, H.L)["U"]
        e = np.abs(U - H.U[t]).max() / max(1.0, np.abs(H.U[t]).max())
        if e > 1e-9:
            print("U differs at node", t, e)
            break
fac = ulv.factor(H, beta)
Ug = P.hss_ulv_factor(Hg, beta)
b = np.random.default_rng(0).standard_normal(n)
ref = np.empty(n)
ref[perm] = ulv.solve(fac, b[perm])
x = Ug.solve(torch.from_numpy(b).cuda()).cpu().numpy()
print("solve relerr", np.linalg.norm(x - ref) / np.linalg.norm(ref))
r = admm.run(lambda v: ulv.solve(fac, v), y[perm], 1.0, beta, 60)
inv = np.empty_like(perm)
inv[perm] = np.arange(n)
g = P.admm_svm_train(Ug, torch.from_numpy(y).cuda(), [0.5, 1.0, 10.0], 60)
zg = g["z"].cpu().numpy()[:, 1]
print("z relerr", np.linalg.norm(zg - r["z"][inv]) / np.linalg.norm(r["z"]))
g1 = P.admm_svm_train(Ug, torch.from_numpy(y).cuda(), [1.0], 60)
print("z relerr nC=1", np.linalg.norm(g1["z"].cpu().numpy()[:, 0] - r["z"][inv]) / np.linalg.norm(r["z"]))
