"""GPU pre-screen of beta for the AMB-9 chaos gate (the gate itself is the oracle's,
scripts/make_fullsize_goldens.py): config c, one build, then for each beta one factorization and
one MaxIt-iteration train with two C columns, C and C (1 + 1e-12); prints max |z_1 - z_2| / C.
A non-chaotic run keeps this near 1e-12; a chaotic one amplifies it.
    python scripts/beta_screen.py 3 1e6 3e6 1e7 3e7 1e8"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2108_04167_b200 as P  # noqa: E402

c = int(sys.argv[1])
betas = [float(b) for b in sys.argv[2:]]
cfg = datagen.get_config(c)
F, y, _, _ = datagen.generate(c, n=cfg["n"], n_test=0)
h = cfg["h"]
H = P.hss_build(torch.from_numpy(F).cuda(), h, leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"],
                max_rank=cfg["cap"], oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"],
                tree_seed=cfg["seed_tree"])
yd = torch.from_numpy(y).cuda()
C = cfg["C"][0]
for b in betas:
    U = P.hss_ulv_factor(H, b)
    for it in (cfg["max_it"], 2 * cfg["max_it"]):
        r = P.admm_svm_train(U, yd, [C, C * (1 + 1e-12)], it)
        z = r["z"]
        div = (z[:, 0] - z[:, 1]).abs().max().item() / C
        print(f"cfg{c} beta {b:.0e} it {it}: max|dz|/C = {div:.3e}  bias {r['bias'][0]:.10g}", flush=True)
    U.free()
