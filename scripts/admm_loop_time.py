"""ADMM loop time per iteration at config 3 (build + factor once, then 3 x 300 iterations)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2108_04167_b200 as P  # noqa: E402

cfg = datagen.get_config(3)
F, y, _, _ = datagen.generate(3, n=cfg["n"], n_test=0)
kw = dict(leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"], max_rank=cfg["cap"],
          oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"])
H = P.hss_build(torch.from_numpy(F).cuda(), cfg["h"], **kw)
U = P.hss_ulv_factor(H, cfg["beta"])
yd = torch.from_numpy(y).cuda()
import hashlib  # noqa: E402
for r in range(3):
    res = P.admm_svm_train(U, yd, [1.0], 300)
    dig = hashlib.sha256(res["z"].cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"loop ms/it {res['stats']['ms_loop'] / 300:.4f} z {dig}", flush=True)
