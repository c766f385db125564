"""The ADMM iteration's fused leaf kernel (leaf level of both sweeps + the epilogue in one kernel,
DESIGN.md "Leaf level fused with the epilogue") is bitwise the unfused level-kernel sequence
(SVMHSS_LEAF_FUSE=0): z, mu, their traces, bias and objective, for leaves with their own
transform (cap < leaf size), pass-through leaves, a mix, and several right-hand sides."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import datagen, paper_2108_04167_b200 as P
c, n, cap, beta, out = %d, %d, %d, %r, %r
cfg = datagen.get_config(c)
F, y, _, _ = datagen.generate(c, n=n, n_test=0)
h = cfg["h"] if not isinstance(cfg["h"], list) else 1.0
H = P.hss_build(torch.from_numpy(F).cuda(), h, leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], max_rank=cap,
                oversample=16, omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"])
U = P.hss_ulv_factor(H, beta)
r = P.admm_svm_train(U, torch.from_numpy(y).cuda(), [0.5, 1.0, 10.0], 40, trace_every=10)
r1 = P.admm_svm_train(U, torch.from_numpy(y).cuda(), [1.0], 25)
np.savez(out, z=r["z"].cpu().numpy(), mu=r["mu"].cpu().numpy(), tz=r["trace_z"].cpu().numpy(),
         tm=r["trace_mu"].cpu().numpy(), bias=r["bias"], obj=r["obj"], z1=r1["z"].cpu().numpy(),
         pt=H.info()["passthrough"])
"""


@pytest.mark.parametrize("c,n,cap,beta", [(3, 6000, 96, 1e4), (3, 9000, 256, 1e3), (1, 9000, 128, 1e4),
                                          (4, 5000, 48, 1e3)])
def test_leaf_fusion_bitwise(tmp_path, c, n, cap, beta):
    outs = {}
    for fuse in ("1", "0"):
        out = str(tmp_path / f"f{fuse}.npz")
        env = dict(os.environ, SVMHSS_LEAF_FUSE=fuse)
        r = subprocess.run([sys.executable, "-c", CODE % (ROOT, c, n, cap, beta, out)], capture_output=True,
                           text=True, cwd=ROOT, env=env, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        outs[fuse] = dict(np.load(out))
    for k in ("z", "mu", "tz", "tm", "bias", "obj", "z1"):
        assert np.array_equal(outs["1"][k], outs["0"][k]), k


@pytest.mark.parametrize("c,n,cap,beta", [(3, 9000, 96, 1e4), (1, 9000, 128, 1e4)])
def test_columns_bitwise_independent(c, n, cap, beta):
    """The nC right-hand sides of one call (a12, the factorization cache over a grid of C) are
    independent problems: every column is bitwise the nC = 1 run with that C (z, mu, bias,
    objective), including a duplicated C value and columns beyond the first group of 8."""
    import torch
    sys.path.insert(0, ROOT)
    import datagen
    import paper_2108_04167_b200 as P
    cfg = datagen.get_config(c)
    F, y, _, _ = datagen.generate(c, n=n, n_test=0)
    h = cfg["h"] if not isinstance(cfg["h"], list) else 1.0
    H = P.hss_build(torch.from_numpy(F).cuda(), h, leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], max_rank=cap,
                    oversample=16, omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"])
    U = P.hss_ulv_factor(H, beta)
    yd = torch.from_numpy(y).cuda()
    Cs = [0.5, 1.0, 10.0, 1.0, 2.0, 3.0, 4.0, 5.0, 0.25]   # 9 columns: two groups of <= 8
    r = P.admm_svm_train(U, yd, Cs, 30)
    for j, C in enumerate(Cs):
        if j in (0, 2, 3, 8):
            r1 = P.admm_svm_train(U, yd, [C], 30)
            assert torch.equal(r["z"][:, j], r1["z"][:, 0]), j
            assert torch.equal(r["mu"][:, j], r1["mu"][:, 0]), j
            assert r["bias"][j] == r1["bias"][0] and r["obj"][j] == r1["obj"][0], j
    U.free()
    H.free()
