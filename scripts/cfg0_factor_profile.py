import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import datagen
import paper_2108_04167_b200 as P
cfg = datagen.get_config(0)
F, y, _, _ = datagen.generate(0, n=cfg["n"], n_test=0)
H = P.hss_build(torch.from_numpy(F).cuda(), cfg["h"], leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"],
                max_rank=cfg["cap"], oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"])
U = P.hss_ulv_factor(H, cfg["beta"]); U.free()
torch.cuda.synchronize(); t = time.perf_counter()
torch.cuda.profiler.start()
U = P.hss_ulv_factor(H, cfg["beta"])
torch.cuda.synchronize(); torch.cuda.profiler.stop()
print("factor s", time.perf_counter() - t, "ranks", sorted(H.info()["ranks"])[-6:])
