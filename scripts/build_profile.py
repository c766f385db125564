"""Build-only profiling target: config 3 (n = 524288) hss_build twice; the second one runs
between cudaProfilerStart/Stop (`ncu --profile-from-start off`).
    python scripts/build_profile.py [sketch|ann] [id|spd]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2108_04167_b200 as P  # noqa: E402

sampling = sys.argv[1] if len(sys.argv) > 1 else "ann"
interp = sys.argv[2] if len(sys.argv) > 2 else "id"
cfg = datagen.get_config(3)
F, y, _, _ = datagen.generate(3, n=cfg["n"], n_test=0)
Fd = torch.from_numpy(F).cuda()
kw = dict(leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"], max_rank=cfg["cap"],
          oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"],
          sampling=sampling, ann_neighbors=cfg["ann_neighbors"], ann_trees=cfg["ann_trees"],
          ann_leaf=cfg["ann_leaf"], ann_seed=cfg["ann_seed"], interp=interp, spd_eps=1e-12)
P.hss_build(Fd, cfg["h"], **kw).free()
torch.cuda.synchronize()
t = time.perf_counter()
torch.cuda.profiler.start()
H = P.hss_build(Fd, cfg["h"], **kw)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"sampling={sampling} interp={interp} build_s={time.perf_counter() - t:.4f}")
