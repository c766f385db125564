"""Worker for tests/test_gpu_factor_paths.py: build + factor + solve + 20 ADMM iterations of a
config-3-shaped problem under the environment it is started with (the kernel-choice knobs are
read once per process), results to an .npz."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2108_04167_b200 as P  # noqa: E402

out, n = sys.argv[1], int(sys.argv[2])
cfg = datagen.get_config(3)
F, y, _, _ = datagen.generate(3, n=n, n_test=0)
H = P.hss_build(torch.from_numpy(F).cuda(), cfg["h"], leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"],
                max_rank=cfg["cap"], oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"],
                tree_seed=cfg["seed_tree"])
U = P.hss_ulv_factor(H, 1e4)
b = torch.from_numpy(np.random.default_rng(3).standard_normal((n, 2))).cuda()
x = U.solve(b)
res = (H.matvec(x) + 1e4 * x - b).norm() / b.norm()
r = P.admm_svm_train(U, torch.from_numpy(y).cuda(), [1.0], 20)
np.savez(out, x=x.cpu().numpy(), res=float(res), z=r["z"].cpu().numpy(), obj=np.asarray(r["obj"]),
         ranks=H.info()["ranks"])
