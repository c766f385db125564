"""The C-ABI boundary pieces of SURVEY §8(b) beyond the main path, through the library:
  - hss_opts.perm: an imported tree (the oracle's T1-T4 output) drives the build;
  - hss_opts.skeletons (+ ranks): fixed-skeleton mode (AMB-12) — the oracle's skeletons, and an
    arbitrary non-CPQR skeleton, give the oracle's fixed-skeleton generators and solves;
  - ulv_solve with nrhs > 8 and admm_svm_train with nC > 8 (groups of 8 inside the library);
  - HSS_EW1 through the SVMHSS_FAULT_W1 test hook; argument / shape validation."""
import os
import subprocess
import sys

import numpy as np
import pytest

import datagen
from oracle import admm as o_admm
from oracle import hss as o_hss
from oracle import pipeline as o_pipe
from oracle import rng as o_rng
from oracle import tree as o_tree
from oracle import ulv as o_ulv

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def relerr(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def _kw(cfg):
    return dict(leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"], max_rank=cfg["cap"],
                oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"])


_C = {}


def _case():
    """cfg-3 knobs at n = 6000 (levels with pass-through leaves and compressed nodes), oracle
    adaptive run with its ranks and skeletons."""
    if "c" not in _C:
        cfg = datagen.get_config(3)
        F, y, _, _ = datagen.generate(3, n=6000, n_test=0)
        perm, ranges, Om, H = o_pipe.build(F, cfg)
        nn = 2 ** (H.L + 1) - 1
        ranks = o_pipe.ranks_array(H, nn).astype(np.int32)
        skel = np.concatenate([H.J[t] for t in range(1, nn)]).astype(np.int64)
        _C["c"] = dict(cfg=cfg, F=F, y=y, perm=perm, ranges=ranges, Om=Om, H=H, ranks=ranks, skel=skel, nn=nn)
    return _C["c"]


def test_perm_import_reproduces_the_built_tree(gpu_lib):
    P = gpu_lib
    c = _case()
    Fd = _t(c["F"])
    H1 = P.hss_build(Fd, c["cfg"]["h"], **_kw(c["cfg"]))
    H2 = P.hss_build(Fd, c["cfg"]["h"], perm=c["perm"], **_kw(c["cfg"]))
    i1, i2 = H1.info(), H2.info()
    assert np.array_equal(i2["perm"], c["perm"]) and np.array_equal(i1["perm"], c["perm"])
    assert np.array_equal(i1["skeletons"], i2["skeletons"])
    v = _t(np.random.default_rng(1).standard_normal(6000))
    assert np.array_equal(H1.matvec(v).cpu().numpy(), H2.matvec(v).cpu().numpy())


def test_perm_import_of_another_tree(gpu_lib):
    """A different (random) permutation: the GPU build follows it; ranks/skeletons match the
    oracle run on the same imported tree."""
    P = gpu_lib
    c = _case()
    cfg = c["cfg"]
    perm = np.random.default_rng(3).permutation(6000)
    ranges = o_tree.node_ranges(6000, o_tree.num_levels(6000, cfg["leaf"]))
    Fp = c["F"][perm]
    Om = o_rng.omega(cfg["seed_omega"], perm, cfg["s"])
    Ho = o_hss.compress(Fp, cfg["h"], ranges, Om, rel_tol=cfg["rel_tol"], cap=cfg["cap"])
    Hg = P.hss_build(_t(c["F"]), cfg["h"], perm=perm, **_kw(cfg))
    info = Hg.info()
    nn = 2 ** (Ho.L + 1) - 1
    assert np.array_equal(info["perm"], perm)
    assert np.array_equal(info["ranks"].astype(np.int64), o_pipe.ranks_array(Ho, nn))
    assert np.array_equal(info["skeletons"], np.concatenate([Ho.J[t] for t in range(1, nn)]))


def test_bad_perm_rejected(gpu_lib):
    P = gpu_lib
    c = _case()
    bad = c["perm"].copy()
    bad[5] = bad[6]
    with pytest.raises(P.HssError) as ei:
        P.hss_build(_t(c["F"]), c["cfg"]["h"], perm=bad, **_kw(c["cfg"]))
    assert ei.value.code == -1


def test_oracle_skeleton_import_matches_oracle(gpu_lib):
    """Fixed-skeleton mode with the oracle's own ranks and skeletons: the GPU keeps them and its
    generators and solves equal the oracle's (solve <= 1e-9, north-star tolerance)."""
    P = gpu_lib
    c = _case()
    cfg = c["cfg"]
    Hg = P.hss_build(_t(c["F"]), cfg["h"], ranks=c["ranks"], skeletons=c["skel"], **_kw(cfg))
    info = Hg.info()
    assert np.array_equal(info["skeletons"], c["skel"])
    H = c["H"]
    for t in (1, 2, 2 ** H.L - 2, 2 ** H.L - 1 + 3):
        if H.U.get(t) is None:
            continue
        gen = Hg.node_generators(t, H.L)
        assert np.abs(gen["U"] - H.U[t]).max() <= 1e-9 * max(1.0, np.abs(H.U[t]).max())
    beta = 1e3
    fac = o_ulv.factor(H, beta)
    U = P.hss_ulv_factor(Hg, beta)
    b = np.random.default_rng(4).standard_normal((6000, 2))
    ref = np.empty_like(b)
    ref[c["perm"]] = o_ulv.solve(fac, b[c["perm"]])
    assert relerr(U.solve(_t(b)).cpu().numpy(), ref) <= 1e-9


def test_arbitrary_skeleton_import_matches_oracle_fixed_skeleton_mode(gpu_lib):
    """A non-CPQR skeleton (each node: a seeded scramble of its active rows, first k): the GPU's
    forced-pivot CPQR gives the oracle's fixed-skeleton interpolation (U <= 1e-9, solve <= 1e-9)."""
    P = gpu_lib
    c = _case()
    cfg = c["cfg"]
    ranges, perm = c["ranges"], c["perm"]
    L = len(ranges) - 1
    g = np.random.default_rng(9)
    k = 200
    sk, ranks = {}, np.full(2 ** (L + 1) - 1, -1, dtype=np.int32)
    for lvl in range(L, 0, -1):
        for i, (lo, hi) in enumerate(ranges[lvl]):
            t = (1 << lvl) - 1 + i
            act = np.arange(lo, hi) if lvl == L else np.concatenate([sk[2 * t + 1], sk[2 * t + 2]])
            kk = min(k, len(act))
            sk[t] = act[g.permutation(len(act))[:kk]] if kk < len(act) else act
            ranks[t] = kk
    flat = np.concatenate([sk[t] for t in range(1, 2 ** (L + 1) - 1)]).astype(np.int64)
    Ho = o_hss.compress(c["F"][perm], cfg["h"], ranges, c["Om"], skeletons=sk)
    Hg = P.hss_build(_t(c["F"]), cfg["h"], ranks=ranks, skeletons=flat, **_kw(cfg))
    assert np.array_equal(Hg.info()["skeletons"], flat)
    for t in (1, 2, 5, 2 ** L - 1, 2 ** (L + 1) - 2):
        if Ho.U.get(t) is None:
            continue
        gen = Hg.node_generators(t, L)
        assert np.abs(gen["U"] - Ho.U[t]).max() <= 1e-9 * max(1.0, np.abs(Ho.U[t]).max()), t
    beta = 1e4
    fac = o_ulv.factor(Ho, beta)
    U = P.hss_ulv_factor(Hg, beta)
    b = np.random.default_rng(5).standard_normal(6000)
    ref = np.empty_like(b)
    ref[perm] = o_ulv.solve(fac, b[perm])
    assert relerr(U.solve(_t(b)).cpu().numpy(), ref) <= 1e-9


def test_bad_skeleton_rejected(gpu_lib):
    P = gpu_lib
    c = _case()
    bad = c["skel"].copy()
    bad[1] = bad[0]
    with pytest.raises(P.HssError) as ei:
        P.hss_build(_t(c["F"]), c["cfg"]["h"], ranks=c["ranks"], skeletons=bad, **_kw(c["cfg"]))
    assert ei.value.code == -1
    with pytest.raises(P.HssError):
        P.hss_build(_t(c["F"]), c["cfg"]["h"], skeletons=c["skel"], **_kw(c["cfg"]))   # no ranks


def test_solve_more_than_8_rhs_and_admm_more_than_8_C(gpu_lib):
    P = gpu_lib
    c = _case()
    cfg = c["cfg"]
    Hg = P.hss_build(_t(c["F"]), cfg["h"], **_kw(cfg))
    U = P.hss_ulv_factor(Hg, 1e3)
    fac = o_ulv.factor(c["H"], 1e3)
    B = np.random.default_rng(6).standard_normal((6000, 11))
    ref = np.empty_like(B)
    ref[c["perm"]] = o_ulv.solve(fac, B[c["perm"]])
    X = U.solve(_t(B)).cpu().numpy()
    assert relerr(X, ref) <= 1e-9
    Cs = [0.1, 0.3, 1, 3, 10, 30, 100, 300, 1000, 3000]
    yd = _t(c["y"])
    r = P.admm_svm_train(U, yd, Cs, 30, trace_every=10)
    a = P.admm_svm_train(U, yd, Cs[:8], 30, trace_every=10)
    b2 = P.admm_svm_train(U, yd, Cs[8:], 30, trace_every=10)
    z = r["z"].cpu().numpy()
    assert np.array_equal(z[:, :8], a["z"].cpu().numpy()) and np.array_equal(z[:, 8:], b2["z"].cpu().numpy())
    assert np.array_equal(r["trace_mu"].cpu().numpy()[:, :, 8:], b2["trace_mu"].cpu().numpy())
    assert np.array_equal(r["bias"], np.concatenate([a["bias"], b2["bias"]]))
    o = o_admm.run_multi(lambda v: o_ulv.solve(fac, v), c["y"][c["perm"]], Cs, 1e3, 30)
    inv = np.empty_like(c["perm"])
    inv[c["perm"]] = np.arange(6000)
    assert relerr(z, o["z"][inv]) <= 1e-7


def test_w1_error_path(gpu_lib):
    """HSS_EW1 via the SVMHSS_FAULT_W1 hook (a fresh process reads it)."""
    code = (
        "import numpy as np, torch, paper_2108_04167_b200 as P\n"
        "g = np.random.default_rng(0)\n"
        "F = torch.from_numpy(g.standard_normal((300, 3))).cuda()\n"
        "y = torch.from_numpy(np.where(g.random(300) < 0.5, 1.0, -1.0)).cuda()\n"
        "H = P.hss_build(F, 1.0, leaf_size=64, max_rank=48, oversample=16)\n"
        "U = P.hss_ulv_factor(H, 1.0)\n"
        "try:\n"
        "    P.admm_svm_train(U, y, [1.0], 5)\n"
        "except P.HssError as e:\n"
        "    print('CODE', e.code, str(e))\n"
    )
    env = dict(os.environ, SVMHSS_FAULT_W1="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, env=env, timeout=300)
    assert "CODE -6" in r.stdout and "w1" in r.stdout, r.stdout + r.stderr


def test_python_shape_checks(gpu_lib):
    P = gpu_lib
    c = _case()
    cfg = c["cfg"]
    Hg = P.hss_build(_t(c["F"]), cfg["h"], **_kw(cfg))
    U = P.hss_ulv_factor(Hg, 1e3)
    with pytest.raises(ValueError):
        U.solve(_t(np.ones(5999)))
    with pytest.raises(ValueError):
        Hg.matvec(_t(np.ones(6001)))
    with pytest.raises(ValueError):
        P.admm_svm_train(U, _t(c["y"][:100]), [1.0], 3)
    F = _t(c["F"])
    y = _t(c["y"])
    z = _t(np.zeros(6000))
    with pytest.raises(ValueError):
        P.svm_predict(F, y, z, 1.0, [0.0, 1.0], F)          # bias length != nC
    with pytest.raises(ValueError):
        P.svm_predict(F, y, z, 1.0, [0.0], _t(np.zeros((4, 3))))   # Ftest columns != r
