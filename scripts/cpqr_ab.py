"""A/B of build/factor variants (env knobs) on config 3 (n = 524288): builds the HSS with the
SVMHSS_CPQR_MODE mode given on the command line, prints the build time and a digest of the
compressed generators (must match across modes bit for bit).
    SVMHSS_TRACE=1 python scripts/cpqr_ab.py MODE [sketch|ann]"""
import hashlib
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402

os.environ["SVMHSS_CPQR_MODE"] = sys.argv[1]
import paper_2108_04167_b200 as P  # noqa: E402

sampling = sys.argv[2] if len(sys.argv) > 2 else "sketch"
cfg = datagen.get_config(3)
F, y, _, _ = datagen.generate(3, n=cfg["n"], n_test=0)
Fd = torch.from_numpy(F).cuda()
kw = dict(leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"], max_rank=cfg["cap"],
          oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"],
          sampling=sampling, ann_neighbors=cfg["ann_neighbors"], ann_trees=cfg["ann_trees"],
          ann_leaf=cfg["ann_leaf"], ann_seed=cfg["ann_seed"])
H = P.hss_build(Fd, cfg["h"], **kw)   # warm-up (module load, pools)
H.free()
torch.cuda.synchronize()
t = time.perf_counter()
H = P.hss_build(Fd, cfg["h"], **kw)
torch.cuda.synchronize()
dt = time.perf_counter() - t
info = H.info()
b = torch.from_numpy(np.random.default_rng(3).standard_normal((cfg["n"], 1))).cuda()
mv = H.matvec(b).cpu().numpy()
dig = hashlib.sha1(info["ranks"].tobytes() + info["skeletons"].tobytes()).hexdigest()[:16]
mvd = hashlib.sha1(mv.tobytes()).hexdigest()[:16]
st = {k: info[k] for k in ("kmax", "s_used") if k in info}
beta = cfg["beta_ann"] if sampling == "ann" else cfg["beta"]
torch.cuda.synchronize()
t = time.perf_counter()
U = P.hss_ulv_factor(H, beta)
torch.cuda.synchronize()
ft = time.perf_counter() - t
x = U.solve(b).cpu().numpy()
fd = hashlib.sha1(x.tobytes()).hexdigest()[:16]
print(f"mode={sys.argv[1]} sampling={sampling} build_s={dt:.3f} ms_compress={info['ms_compress']:.1f} skel_digest={dig} mv_digest={mvd} {st} factor_s={ft:.3f} solve_digest={fd}")
