"""Small end-to-end solve (config 3 shape, n=5000) in both samplings, for debugging the solve
path: python scripts/repro_top.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2108_04167_b200 as P  # noqa: E402

for sampling in ("sketch", "ann"):
    cfg = datagen.get_config(3)
    F, y, _, _ = datagen.generate(3, n=5000, n_test=0)
    Fd = torch.from_numpy(F).cuda()
    H = P.hss_build(Fd, cfg["h"], leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], max_rank=cfg["cap"], oversample=16,
                    omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"], sampling=sampling,
                    ann_neighbors=64, ann_trees=4, ann_leaf=256, ann_seed=4003)
    U = P.hss_ulv_factor(H, 1e3)
    b = torch.from_numpy(np.random.default_rng(0).standard_normal((5000, 2))).cuda()
    x = U.solve(b)
    r = H.matvec(x) + 1e3 * x - b
    print(sampling, "residual", float(torch.linalg.norm(r) / torch.linalg.norm(b)))
    res = P.admm_svm_train(U, torch.from_numpy(y).cuda(), [1.0], 30)
    print(sampling, "obj", res["obj"], "launches/iter", res["stats"]["kernel_launches_per_iter"])
