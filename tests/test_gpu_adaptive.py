"""Adaptive randomized sampling (readings N2a-c) on the GPU vs the oracle's
compress_adaptive: same final sample count and number of rounds, ranks and skeletons bit-exact,
mat-vec at 1e-10."""
import numpy as np
import pytest

import datagen
from oracle import hss as o_hss
from oracle import pipeline as o_pipe
from oracle import tree as o_tree

pytestmark = pytest.mark.gpu


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


@pytest.mark.parametrize("cfg_id,n,h,cap,p,tol,s0,ds", [
    (4, 3000, 2.0, 200, 16, 1e-6, 32, 32),    # smooth kernel: ranks well below the cap
    (0, 2000, 1.0, 300, 16, 1e-4, 48, 64),
    (3, 2500, 1.0, 96, 16, 1e-3, 64, 32),     # cap-bound: grows to the full budget
])
def test_adaptive_sampling_matches_oracle(gpu_lib, cfg_id, n, h, cap, p, tol, s0, ds):
    P = gpu_lib
    cfg = datagen.get_config(cfg_id)
    F, _, _, _ = datagen.generate(cfg_id, n=n, n_test=0)
    perm, ranges = o_tree.build_tree(F, cfg["leaf"], cfg["seed_tree"])
    Ho, s_o, rounds_o = o_hss.compress_adaptive(F[perm], h, ranges, perm, cfg["seed_omega"], s0=s0, ds=ds,
                                                s_max=cap + p, p=p, rel_tol=tol, cap=cap)
    Hg = P.hss_build(_t(F), h, leaf_size=cfg["leaf"], rel_tol=tol, max_rank=cap, oversample=p,
                     omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"], adaptive_s0=s0, adaptive_ds=ds)
    info = Hg.info()
    assert (info["s_used"], info["sample_rounds"]) == (s_o, rounds_o)
    assert np.array_equal(info["ranks"].astype(np.int64), o_pipe.ranks_array(Ho, 2 ** (Ho.L + 1) - 1))
    skel_o = np.concatenate([Ho.J[t] for t in range(1, 2 ** (Ho.L + 1) - 1)])
    assert np.array_equal(info["skeletons"], skel_o)
    V = np.random.default_rng(2).standard_normal((n, 2))
    ref = np.empty_like(V)
    ref[perm] = o_hss.matvec(Ho, V[perm])
    out = Hg.matvec(_t(V)).cpu().numpy()
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) <= 1e-10
