"""N4 (SPD-preserving compression, interp="spd"): CUDA path through the C-ABI vs the oracle.

Same bars as tests/test_gpu_parity.py (BASELINE.json north_star): tree / ranks / skeletons
bit-exact; U at sampled nodes of every level, mat-vec and solves <= 1e-9 (mat-vec 1e-10);
ADMM z / mu traces, objective and bias <= 1e-7; labels identical where |dv| > 1e-6.  The shift
is the paper's beta schedule — the point of N4: no calibration above -lambda_min(K~).
"""
import numpy as np
import pytest

import datagen
from oracle import admm as o_admm
from oracle import hss as o_hss
from oracle import pipeline as o_pipe
from oracle import rng as o_rng
from oracle import svm as o_svm
from oracle import tree as o_tree
from oracle import ulv as o_ulv
from test_gpu_parity import _np, _t, relerr

pytestmark = pytest.mark.gpu

EPS = 1e-12
CASES = {
    "cfg1s": dict(cfg=1, n=3000, nt=700, max_it=200),
    "cfg2s": dict(cfg=2, n=2500, nt=600, max_it=100),
    "cfg3s": dict(cfg=3, n=5000, nt=900, max_it=200),
    "cfg4s": dict(cfg=4, n=3000, nt=500, max_it=100, h=1.0),
    "cfg1_full": dict(cfg=1, n=32768, nt=2048, max_it=100),
}
_CACHE = {}


def run_case(P, name):
    if name in _CACHE:
        return _CACHE[name]
    d = CASES[name]
    cfg = datagen.get_config(d["cfg"])
    h = d.get("h", cfg["h"])
    beta = datagen.configs.beta_schedule(d["n"])
    F, y, Ft, yt = datagen.generate(d["cfg"], n=d["n"], n_test=d["nt"])
    perm, ranges = o_tree.build_tree(F, cfg["leaf"], cfg["seed_tree"])
    Om = o_rng.omega(cfg["seed_omega"], perm, cfg["s"])
    H = o_hss.compress(F[perm], h, ranges, Om, rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"], cap=cfg["cap"],
                       interp="spd", spd_eps=EPS)
    fac = o_ulv.factor(H, beta)
    Hg = P.hss_build(_t(F), h, leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"],
                     max_rank=cfg["cap"], oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"],
                     tree_seed=cfg["seed_tree"], interp="spd", spd_eps=EPS)
    Ug = P.hss_ulv_factor(Hg, beta)
    Cs = cfg["C"][:1] if d["cfg"] != 4 else [1.0, 10.0]
    out = dict(d=d, cfg=cfg, F=F, y=y, Ft=Ft, perm=perm, H=H, fac=fac, Hg=Hg, Ug=Ug, Cs=Cs, h=h, beta=beta)
    _CACHE[name] = out
    return out


@pytest.mark.parametrize("name", list(CASES))
def test_spd_tree_ranks_skeletons_exact(gpu_lib, name):
    c = run_case(gpu_lib, name)
    info = c["Hg"].info()
    H = c["H"]
    assert np.array_equal(info["perm"], c["perm"])
    assert np.array_equal(info["ranks"].astype(np.int64), o_pipe.ranks_array(H, 2 ** (H.L + 1) - 1))
    assert np.array_equal(info["skeletons"], np.concatenate([H.J[t] for t in range(1, 2 ** (H.L + 1) - 1)]))
    assert sum(u is not None for u in H.U.values()) > 0     # the case compresses


@pytest.mark.parametrize("name", list(CASES))
def test_spd_generators_match(gpu_lib, name):
    c = run_case(gpu_lib, name)
    H, Hg = c["H"], c["Hg"]
    seen = 0
    for lvl in range(1, H.L + 1):
        nodes = [t for t, _, _ in H.nodes(lvl) if H.U[t] is not None]
        for t in nodes[:1] + nodes[-1:]:
            gen = Hg.node_generators(t, H.L)
            U = H.U[t]
            assert gen["U"].shape == U.shape
            assert np.abs(gen["U"] - U).max() <= 1e-9 * max(1.0, np.abs(U).max()), (lvl, t)
            seen += 1
    assert seen > 0


@pytest.mark.parametrize("name", list(CASES))
def test_spd_matvec_and_solve_match(gpu_lib, name):
    c = run_case(gpu_lib, name)
    g = np.random.default_rng(8)
    n = c["F"].shape[0]
    perm = c["perm"]
    V = g.standard_normal((n, 3))
    ref = np.empty_like(V)
    ref[perm] = o_hss.matvec(c["H"], V[perm])
    assert relerr(_np(c["Hg"].matvec(_t(V))), ref) <= 1e-10
    for B in (np.ones((n, 1)), g.standard_normal((n, 4))):
        x = _np(c["Ug"].solve(_t(B[:, 0] if B.shape[1] == 1 else B)))
        ref = np.empty_like(B)
        ref[perm] = o_ulv.solve(c["fac"], B[perm])
        assert relerr(x, ref[:, 0] if B.shape[1] == 1 else ref) <= 1e-9


@pytest.mark.parametrize("name", list(CASES))
def test_spd_admm_trace_bias_objective_labels(gpu_lib, name):
    P = gpu_lib
    c = run_case(P, name)
    perm, y, beta = c["perm"], c["y"], c["beta"]
    max_it = c["d"]["max_it"]
    yp = y[perm]
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.shape[0])
    solve = lambda b: o_ulv.solve(c["fac"], b)  # noqa: E731
    mv = lambda v: o_hss.matvec(c["H"], v)      # noqa: E731
    res = P.admm_svm_train(c["Ug"], _t(y), c["Cs"], max_it, trace_every=10)
    zg, mug, tz, tm = _np(res["z"]), _np(res["mu"]), _np(res["trace_z"]), _np(res["trace_mu"])
    for ci, C in enumerate(c["Cs"]):
        o = o_admm.run(solve, yp, C, beta, max_it, trace_every=10)
        for ti, (it, z_o, mu_o) in enumerate(o["trace"]):
            assert relerr(tz[ti, :, ci], z_o[inv]) <= 1e-7, (ci, it)
            assert relerr(tm[ti, :, ci], mu_o[inv]) <= 1e-7, (ci, it)
        assert abs(res["stats"]["w1"] - o["w1"]) <= 1e-9 * abs(o["w1"])
        b_o = o_svm.bias(mv, o["z"], yp, C)
        f_o = o_svm.objective(mv, o["z"], yp)
        assert abs(res["obj"][ci] - f_o) <= 1e-7 * abs(f_o)
        assert abs(res["bias"][ci] - b_o) <= 1e-7 * max(1.0, abs(b_o))
        dv_o = o_svm.decision_values(c["F"], y * o["z"][inv], c["h"], b_o, c["Ft"])
        dv_g, lab_g = P.svm_predict(_t(c["F"]), _t(y), _t(zg[:, ci].copy()), c["h"], [res["bias"][ci]],
                                    _t(c["Ft"]))
        sure = np.abs(dv_o) > 1e-6
        assert np.array_equal(_np(lab_g)[:, 0][sure], o_svm.labels(dv_o)[sure])
        assert np.abs(_np(dv_g)[:, 0] - dv_o).max() <= 1e-7 * max(1.0, np.abs(dv_o).max())


def test_spd_factors_where_id_breaks_down(gpu_lib):
    """The case tests/test_gpu_parity.py::test_not_spd_reports_node uses: the ID form's K~ has
    lambda_min = -1.30 (HSS_ENOTSPD at every small beta); the N4 form (lambda_min = +0.011) factors
    at beta = 1e-6 and solves as the oracle does."""
    P = gpu_lib
    g = np.random.default_rng(4)
    F = g.standard_normal((1024, 4))
    kw = dict(leaf_size=32, rel_tol=0.0, max_rank=8, oversample=16)
    Hid = P.hss_build(_t(F), 0.4, **kw)
    with pytest.raises(P.HssError) as ei:
        P.hss_ulv_factor(Hid, 1e-3)
    assert ei.value.code == -5
    H = P.hss_build(_t(F), 0.4, interp="spd", spd_eps=EPS, **kw)
    info = H.info()
    perm = info["perm"]
    Ho = o_hss.compress(F[perm], 0.4, o_tree.build_tree(F, 32, 0)[1], o_rng.omega(0, perm, 24), rel_tol=0.0,
                        cap=8, interp="spd", spd_eps=EPS)
    for beta in (1e-6, 1e-2):
        U = P.hss_ulv_factor(H, beta)
        b = g.standard_normal(1024)
        ref = np.empty_like(b)
        ref[perm] = o_ulv.solve(o_ulv.factor(Ho, beta), b[perm])
        assert relerr(_np(U.solve(_t(b))), ref) <= 1e-9


def test_spd_invalid_eps_rejected(gpu_lib):
    P = gpu_lib
    F = _t(np.random.default_rng(0).standard_normal((300, 3)))
    with pytest.raises(P.HssError) as ei:
        P.hss_build(F, 1.0, leaf_size=32, max_rank=8, interp="spd", spd_eps=-1.0)
    assert ei.value.code == -1


def test_spd_config3_full_size_sampled_nodes_and_psd(gpu_lib):
    """Config 3 at its stated size (n = 524288), in the launch configuration bench.py's
    variants.spd times: the oracle recomputes U_t = K(A_t, J_t)(K(J_t, J_t) + eps I)^-1 of sampled
    nodes of every level from the GPU's own tree and skeletons (the N4 definition, oracle/hss.py
    nystrom_u; 1e-9), and K~ + beta I factors at beta = 1e-6 (a property of the N4 form at any
    size: K~ is PSD), then ADMM runs at the paper's beta schedule (1e3)."""
    import torch
    P = gpu_lib
    cfg = datagen.get_config(3)
    F, y, _, _ = datagen.generate(3, n_test=0)
    Fd = _t(F)
    H = P.hss_build(Fd, cfg["h"], leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"],
                    max_rank=cfg["cap"], oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"],
                    tree_seed=cfg["seed_tree"], interp="spd", spd_eps=EPS)
    info = H.info()
    perm, ks, skel = info["perm"], info["ranks"].astype(np.int64), info["skeletons"].astype(np.int64)
    L = int(info["L"])
    Fp = F[perm]
    J, off = {}, 0
    for lvl in range(1, L + 1):
        for t in range((1 << lvl) - 1, (1 << (lvl + 1)) - 1):
            J[t] = skel[off:off + ks[t]]
            off += ks[t]
    ranges = o_tree.node_ranges(F.shape[0], L)
    g = np.random.default_rng(11)
    checked = 0
    for lvl in range(1, L + 1):
        lo_id = (1 << lvl) - 1
        for t in sorted({lo_id, lo_id + int(g.integers(0, 1 << lvl))}):
            if lvl == L:
                a, b = ranges[lvl][t - lo_id]
                A = np.arange(a, b)
            else:
                A = np.concatenate([J[2 * t + 1], J[2 * t + 2]])
            if ks[t] == len(A):
                continue                                     # pass-through: U = I
            gen = H.node_generators(t, L)
            U = o_hss.nystrom_u(Fp, cfg["h"], A, J[t], EPS)
            assert np.abs(gen["U"] - U).max() <= 1e-9 * max(1.0, np.abs(U).max()), (lvl, t)
            checked += 1
    assert checked >= L - 2
    U6 = P.hss_ulv_factor(H, 1e-6)                           # PSD: factors at a tiny shift
    U6.free()
    Ug = P.hss_ulv_factor(H, datagen.configs.beta_schedule(F.shape[0]))
    res = P.admm_svm_train(Ug, _t(y), [1.0], 10)
    assert torch.isfinite(res["z"]).all() and res["stats"]["w1"] > 0
    Ug.free()
    H.free()
