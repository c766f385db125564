"""The optional top-levels sweeps (levels 0..5 of both ULV sweeps in one launch: SVMHSS_TOP_MERGE=1
with grid barriers between levels, =2 as a dataflow queue with per-node dependency counters) must
give bitwise the same solve and ADMM iterates as the per-level kernels: they run the same item
bodies."""
import os

import numpy as np
import pytest

import datagen

pytestmark = pytest.mark.gpu


def _run(P, F, y, cfg, merge):
    import torch
    os.environ["SVMHSS_TOP_MERGE"] = str(merge)
    try:
        H = P.hss_build(torch.from_numpy(F).cuda(), cfg["h"], leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"],
                        max_rank=cfg["cap"], oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"],
                        tree_seed=cfg["seed_tree"])
        U = P.hss_ulv_factor(H, 1e3)
        b = torch.from_numpy(np.random.default_rng(5).standard_normal((F.shape[0], 3))).cuda()
        x = U.solve(b).cpu().numpy()
        r = P.admm_svm_train(U, torch.from_numpy(y).cuda(), [1.0, 5.0], 30)
        return x, r["z"].cpu().numpy(), r["mu"].cpu().numpy(), r["obj"]
    finally:
        os.environ.pop("SVMHSS_TOP_MERGE", None)


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("n", [5000, 20000])
def test_top_merge_bitwise(gpu_lib, n, mode):
    cfg = datagen.get_config(3)
    F, y, _, _ = datagen.generate(3, n=n, n_test=0)
    a = _run(gpu_lib, F, y, cfg, mode)
    b = _run(gpu_lib, F, y, cfg, 0)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
