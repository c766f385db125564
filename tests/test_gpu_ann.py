"""HSS-ANN sampling (readings N1-N3) on the GPU vs the oracle (oracle/ann.py).

Integer work is compared bit-exactly: the ANN lists (indices AND the FMA-free squared
distances), the tree, ranks and skeletons.  Floating point at the north-star tolerances: the
mat-vec / solve vectors <= 1e-9 (1e-10 for the mat-vec), the ADMM iterates and objective <= 1e-7."""
import numpy as np
import pytest

import datagen
from oracle import admm as o_admm
from oracle import ann as o_ann
from oracle import hss as o_hss
from oracle import pipeline as o_pipe
from oracle import svm as o_svm
from oracle import ulv as o_ulv

pytestmark = pytest.mark.gpu


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def _np(t):
    return t.detach().cpu().numpy()


def relerr(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("cfg_id,n,kappa,trees,leaf", [
    (3, 5000, 64, 4, 256), (1, 3000, 64, 4, 256), (2, 2500, 32, 2, 128), (4, 3000, 64, 4, 256),
    (3, 300, 16, 2, 64), (1, 100, 64, 3, 256), (4, 257, 8, 1, 16)])
def test_ann_lists_bit_exact(gpu_lib, cfg_id, n, kappa, trees, leaf):
    F, _, _, _ = datagen.generate(cfg_id, n=n, n_test=0)
    idx_g, d_g = gpu_lib.hss_ann_lists(_t(F), kappa, trees, leaf, 4000 + cfg_id)
    idx_o, d_o = o_ann.knn(F, kappa, trees, leaf, 4000 + cfg_id)
    assert np.array_equal(_np(idx_g), idx_o)
    assert np.array_equal(_np(d_g), d_o)


CASES = {
    "cfg3a": dict(cfg=3, n=5000, max_it=100, beta=1e2),
    "cfg1a": dict(cfg=1, n=3000, max_it=100, beta=1e2),
    "cfg4a": dict(cfg=4, n=3000, max_it=100, beta=1e2, h=1.0),
    "cfg3small": dict(cfg=3, n=700, max_it=60, beta=1e2),
    "cfg3a_spd": dict(cfg=3, n=5000, max_it=100, beta=1e2, interp="spd"),   # N4 with HSS-ANN sampling
}
_CACHE = {}


def run_case(P, name):
    if name in _CACHE:
        return _CACHE[name]
    d = CASES[name]
    cfg = datagen.get_config(d["cfg"])
    if "h" in d:
        cfg["h"] = d["h"]
    cfg["beta"] = d["beta"]
    F, y, _, _ = datagen.generate(d["cfg"], n=d["n"], n_test=0)
    interp = d.get("interp", "id")
    perm, ranges, _, H = o_pipe.build_ann(F, cfg, interp=interp, spd_eps=1e-12)
    fac = o_ulv.factor(H, cfg["beta"])
    Hg = P.hss_build(_t(F), cfg["h"], leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"],
                     max_rank=cfg["cap"], oversample=cfg["s"] - cfg["cap"], tree_seed=cfg["seed_tree"],
                     sampling="ann", ann_neighbors=cfg["ann_neighbors"], ann_trees=cfg["ann_trees"],
                     ann_leaf=cfg["ann_leaf"], ann_seed=cfg["ann_seed"], interp=interp, spd_eps=1e-12)
    Ug = P.hss_ulv_factor(Hg, cfg["beta"])
    out = dict(d=d, cfg=cfg, F=F, y=y, perm=perm, H=H, fac=fac, Hg=Hg, Ug=Ug)
    _CACHE[name] = out
    return out


@pytest.mark.parametrize("name", list(CASES))
def test_ann_build_ranks_skeletons_exact(gpu_lib, name):
    c = run_case(gpu_lib, name)
    info = c["Hg"].info()
    H = c["H"]
    assert np.array_equal(info["perm"], c["perm"])
    assert np.array_equal(info["ranks"].astype(np.int64), o_pipe.ranks_array(H, 2 ** (H.L + 1) - 1))
    skel_o = np.concatenate([H.J[t] for t in range(1, 2 ** (H.L + 1) - 1)])
    assert np.array_equal(info["skeletons"], skel_o)


@pytest.mark.parametrize("name", list(CASES))
def test_ann_generators_matvec_solve(gpu_lib, name):
    c = run_case(gpu_lib, name)
    H, Hg, perm = c["H"], c["Hg"], c["perm"]
    for t in [1, 2, 2 ** H.L - 1, 2 ** (H.L + 1) - 2]:
        gen = Hg.node_generators(t, H.L)
        U = H.U[t] if H.U[t] is not None else np.eye(H.rows[t])
        assert np.abs(gen["U"] - U).max() <= 1e-9 * max(1.0, np.abs(U).max())
    g = np.random.default_rng(3)
    n = c["F"].shape[0]
    V = g.standard_normal((n, 2))
    ref = np.empty_like(V)
    ref[perm] = o_hss.matvec(H, V[perm])
    assert relerr(_np(Hg.matvec(_t(V))), ref) <= 1e-10
    ref[perm] = o_ulv.solve(c["fac"], V[perm])
    assert relerr(_np(c["Ug"].solve(_t(V))), ref) <= 1e-9


@pytest.mark.parametrize("name", list(CASES))
def test_ann_admm_trace_objective(gpu_lib, name):
    P = gpu_lib
    c = run_case(P, name)
    cfg, perm, y = c["cfg"], c["perm"], c["y"]
    it, beta, C = c["d"]["max_it"], cfg["beta"], cfg["C"][0]
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.shape[0])
    res = P.admm_svm_train(c["Ug"], _t(y), [C], it, trace_every=10)
    o = o_admm.run(lambda b: o_ulv.solve(c["fac"], b), y[perm], C, beta, it, trace_every=10)
    tz = _np(res["trace_z"])
    for ti, (_, z_o, _) in enumerate(o["trace"]):
        assert relerr(tz[ti, :, 0], z_o[inv]) <= 1e-7
    assert relerr(_np(res["z"])[:, 0], o["z"][inv]) <= 1e-7
    f_o = o_svm.objective(lambda v: o_hss.matvec(c["H"], v), o["z"], y[perm])
    assert abs(res["obj"][0] - f_o) <= 1e-7 * abs(f_o)
