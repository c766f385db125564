"""Tiny solve through the cooperative top-levels kernel (n=5000 sketch mode) for compute-sanitizer."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2108_04167_b200 as P  # noqa: E402

cfg = datagen.get_config(3)
F, y, _, _ = datagen.generate(3, n=5000, n_test=0)
H = P.hss_build(torch.from_numpy(F).cuda(), cfg["h"], leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"],
                max_rank=cfg["cap"], oversample=16, omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"])
U = P.hss_ulv_factor(H, 1e3)
b = torch.from_numpy(np.random.default_rng(0).standard_normal(5000)).cuda()
x = U.solve(b)
print("ok", float(x.norm()))
