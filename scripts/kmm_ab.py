"""Sketch-kernel A/B: config-3 hss_build (sketch sampling) three times, printing the sketch
phase per build.  The variant comes from the environment (SVMHSS_KMM, SVMHSS_KMM_NW).
    SVMHSS_KMM=1 python scripts/kmm_ab.py [config]"""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2108_04167_b200 as P  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = datagen.get_config(c)
F, y, _, _ = datagen.generate(c, n=cfg["n"], n_test=0)
Fd = torch.from_numpy(F).cuda()
kw = dict(leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"], max_rank=cfg["cap"],
          oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"])
h = cfg["h"] if "h" in cfg else cfg["hs"][0]
tag = f"KMM={os.environ.get('SVMHSS_KMM', 'default')} NW={os.environ.get('SVMHSS_KMM_NW', 'default')}"
for r in range(3):
    H = P.hss_build(Fd, h, **kw)
    torch.cuda.synchronize()
    hi = H.info()
    dig = hashlib.sha256(np.ascontiguousarray(hi["skeletons"]).tobytes()).hexdigest()[:12]
    print(f"{tag} cfg{c} build {r}: sketch {hi['ms_sketch']:.1f} ms compress {hi['ms_compress']:.1f} ms skeletons {dig}",
          flush=True)
    H.free()
