"""Full-size (BASELINE.json config 3, n = 524,288 / 131,072 test points, with the sketch and with
HSS-ANN sampling; config 2, n = 131,072) checks of the CUDA path in the configuration bench.py times, on outputs the oracle can compute one by one or on properties
that hold at any size (the oracle's full HSS at this n takes hours on the host):

  - tree: the permutation equals the oracle's PCA bisection (T1-T4) bit for bit;
  - ULV solve: (K~ + beta I) x = b to 1e-10 relative, K~ applied by the library's own HSS mat-vec
    (a different code path from the solve: up/down sweeps over U, B, D);
  - ADMM: z in [0, C] exactly; the x-update satisfies y^T x = 0 (x = Y K^-1 Y q - (w^T q / w1) w
    has y^T x = w^T q - (w^T q / w1) w1 = 0), x recovered from two runs one iteration apart
    (x = z + (mu_prev - mu) / beta, A3), and z = clip(x - mu_prev / beta, 0, C);
  - predict: 64 sampled test points, decision values recomputed by the oracle from the exact
    kernel — labels identical wherever |dv| > 1e-6, dv to 1e-10 relative.
"""
import numpy as np
import pytest

import datagen
from oracle import svm as o_svm
from oracle import tree as o_tree

pytestmark = pytest.mark.gpu


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


# (config, sampling): config 3 with both compressions, config 2 (n = 131072, r = 123 binary)
@pytest.fixture(scope="module", params=[(3, "sketch"), (3, "ann"), (2, "sketch")],
                ids=["cfg3-sketch", "cfg3-ann", "cfg2-sketch"])
def full(gpu_lib, request):
    P = gpu_lib
    c, sampling = request.param
    cfg = datagen.get_config(c)
    if sampling == "ann":
        cfg["beta"] = cfg["beta_ann"]
    F, y, Ft, yt = datagen.generate(c, n=cfg["n"], n_test=cfg["n_test"])
    H = P.hss_build(_t(F), cfg["h"], leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"],
                    max_rank=cfg["cap"], oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"],
                    tree_seed=cfg["seed_tree"], sampling=sampling, ann_neighbors=cfg["ann_neighbors"],
                    ann_trees=cfg["ann_trees"], ann_leaf=cfg["ann_leaf"], ann_seed=cfg["ann_seed"])
    U = P.hss_ulv_factor(H, cfg["beta"])
    yield dict(P=P, cfg=cfg, F=F, y=y, Ft=Ft, H=H, U=U)
    U.free()
    H.free()


def test_fullsize_tree_bit_exact(full):
    perm_o, _ = o_tree.build_tree(full["F"], full["cfg"]["leaf"], full["cfg"]["seed_tree"])
    assert np.array_equal(full["H"].info()["perm"], perm_o)


def test_fullsize_solve_residual(full):
    import torch
    n, beta = full["F"].shape[0], full["cfg"]["beta"]
    b = _t(np.random.default_rng(11).standard_normal((n, 2)))
    x = full["U"].solve(b)
    r = full["H"].matvec(x) + beta * x - b
    assert float(torch.linalg.norm(r) / torch.linalg.norm(b)) <= 1e-10


def test_fullsize_admm_properties_and_predict(full):
    P, cfg, y = full["P"], full["cfg"], full["y"]
    beta, C, it = cfg["beta"], cfg["C"][0], cfg["max_it"]
    yd = _t(y)
    a = P.admm_svm_train(full["U"], yd, [C], it - 1)
    b = P.admm_svm_train(full["U"], yd, [C], it)
    z, mu, mu_prev = (v.cpu().numpy()[:, 0] for v in (b["z"], b["mu"], a["mu"]))
    assert z.min() >= 0.0 and z.max() <= C
    x = z + (mu_prev - mu) / beta
    assert abs(float(y @ x)) <= 1e-9 * np.linalg.norm(x) * np.sqrt(len(x))
    assert np.allclose(np.clip(x - mu_prev / beta, 0.0, C), z, rtol=0, atol=1e-9 * max(1.0, C))
    # predict on 64 sampled test points vs the oracle's exact decision values
    Ft = full["Ft"]
    sel = np.random.default_rng(12).choice(Ft.shape[0], 64, replace=False)
    dv, lab = P.svm_predict(_t(full["F"]), yd, b["z"], cfg["h"], b["bias"], _t(Ft[sel]))
    dv, lab = dv.cpu().numpy()[:, 0], lab.cpu().numpy()[:, 0]
    dvo = o_svm.decision_values(full["F"], y * z, cfg["h"], b["bias"][0], Ft[sel])
    assert np.abs(dv - dvo).max() <= 1e-10 * max(1.0, np.abs(dvo).max())
    sure = np.abs(dvo) > 1e-6
    assert np.array_equal(lab[sure], o_svm.labels(dvo)[sure])
