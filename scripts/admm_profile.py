"""ADMM-loop profiling target: config 3 (n = 524288) build + factor, one warm-up train call, then
a 3-iteration admm_svm_train between cudaProfilerStart/Stop.
    python scripts/admm_profile.py [sketch|ann]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2108_04167_b200 as P  # noqa: E402

sampling = sys.argv[1] if len(sys.argv) > 1 else "sketch"
cfg = datagen.get_config(3)
F, y, _, _ = datagen.generate(3, n=cfg["n"], n_test=0)
kw = dict(leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"], max_rank=cfg["cap"],
          oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"],
          sampling=sampling, ann_neighbors=cfg["ann_neighbors"], ann_trees=cfg["ann_trees"],
          ann_leaf=cfg["ann_leaf"], ann_seed=cfg["ann_seed"])
H = P.hss_build(torch.from_numpy(F).cuda(), cfg["h"], **kw)
U = P.hss_ulv_factor(H, cfg["beta_ann"] if sampling == "ann" else cfg["beta"])
yd = torch.from_numpy(y).cuda()
r = P.admm_svm_train(U, yd, [1.0], 200)
print("loop ms/it", r["stats"]["ms_loop"] / 200)
torch.cuda.synchronize()
torch.cuda.profiler.start()
P.admm_svm_train(U, yd, [1.0], 3)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
