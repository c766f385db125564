"""Factor-only profiling target: config 3 (n = 524288) HSS build, one unprofiled factorization
(grows the memory pool), then a second one between cudaProfilerStart/Stop, so
`ncu --profile-from-start off` captures just the factor's launches.
    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ... python scripts/factor_profile.py [sketch|ann]"""
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
H = P.hss_build(torch.from_numpy(F).cuda(), cfg["h"], leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"],
                abs_tol=cfg["abs_tol"], max_rank=cfg["cap"], oversample=cfg["s"] - cfg["cap"],
                omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"], sampling=sampling,
                ann_neighbors=cfg["ann_neighbors"], ann_trees=cfg["ann_trees"], ann_leaf=cfg["ann_leaf"],
                ann_seed=cfg["ann_seed"])
beta = cfg["beta_ann"] if sampling == "ann" else cfg["beta"]
U = P.hss_ulv_factor(H, beta)
U.free()
ts = []
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    if rep == 2:
        torch.cuda.profiler.start()
    U = P.hss_ulv_factor(H, beta)
    torch.cuda.synchronize()
    if rep == 2:
        torch.cuda.profiler.stop()
    ts.append(time.perf_counter() - t)
    U.free()
print(f"sampling={sampling} factor_s={['%.4f' % x for x in ts]}")
