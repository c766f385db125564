"""Oracle pins: x-update, z/mu updates, ADMM vs brute-force QP, KKT,
bias (AMB-2/3), prediction, Eq. (9) gap bound."""
import json
import os

import numpy as np
import pytest

from oracle import admm, hss, kernel, qp, rng, svm, tree, ulv

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CF = json.load(open(os.path.join(GOLD, "closed_forms.json")))


def _toy(n, seed, h=1.0, sep=0.7):
    g = np.random.default_rng(seed)
    y = np.where(g.random(n) < 0.5, 1.0, -1.0)
    if abs(y.sum()) == n:
        y[0] = -y[0]
    F = g.standard_normal((n, 2)) + sep * y[:, None]
    return F, y, kernel.dense_kernel(F, h)


def test_xupdate_golden_2x2():
    c = CF["xupdate_2x2"]
    Kb = np.array(c["Kbeta"])
    y, q = np.array(c["y"]), np.array(c["q"])
    solve = lambda b: np.linalg.solve(Kb, b)  # noqa: E731
    w, w1 = admm.precompute(solve, y)
    x = admm.x_update(solve, y, w, w1, q)
    assert np.allclose(x, c["x"], rtol=0, atol=1e-15)
    xk, lam = admm.kkt_bordered(Kb, y, q)
    assert np.allclose(xk, c["x"], atol=1e-15) and abs(lam - c["lam"]) < 1e-15


def test_precompute_golden():
    c = CF["precompute_2"]
    A = np.array(c["K"]) + c["beta"] * np.eye(2)
    w, w1 = admm.precompute(lambda b: np.linalg.solve(A, b), np.array(c["y"]))
    assert np.allclose(w, c["w"], atol=1e-16) and w1 == c["w1"]


@pytest.mark.parametrize("seed", range(5))
def test_xupdate_equals_bordered_kkt(seed):
    F, y, K = _toy(30, seed)
    beta = 0.5 + seed
    Kb = K + beta * np.eye(30)
    g = np.random.default_rng(seed)
    q = 1.0 + g.random(30) * 3
    solve = lambda b: np.linalg.solve(Kb, b)  # noqa: E731
    w, w1 = admm.precompute(solve, y)
    x = admm.x_update(solve, y, w, w1, q)
    xk, lam = admm.kkt_bordered(Kb, y, q)
    assert np.abs(x - xk).max() < 1e-12 * max(1, np.abs(xk).max())
    assert abs(y @ x) < 1e-13 * np.linalg.norm(x) * np.sqrt(30)
    assert abs(lam - (-(w @ q) / w1)) < 1e-11 * max(1, abs(lam))


def test_z_clamp_and_mu_fixed_point():
    c = CF["zclamp"]
    z = np.clip(np.array(c["arg"]), 0.0, c["C"])
    assert np.array_equal(z, np.array(c["z"]))
    mu = np.array([0.3, -0.2])
    x = np.array([0.1, 0.4])
    assert np.array_equal(mu - 2.0 * (x - x), mu)


@pytest.mark.parametrize("seed", range(3))
def test_admm_converges_to_bruteforce_qp(seed):
    F, y, K = _toy(8, seed)
    C = 1.0
    xb, fb = qp.solve_qp_bruteforce(K, y, C)
    out = admm.run(admm.dense_solver(K, 1.0), y, C, 1.0, 3000)
    assert np.abs(out["z"] - xb).max() < 1e-9
    assert qp.kkt_residual(K, y, C, out["z"], out["lam"]) < 1e-9
    assert abs(svm.objective_dense(K, out["z"], y) - fb) < 1e-12


def test_bias_single_margin_sv_reduces_to_eq2():
    """|M| = 1: b = y_j - sum_i y_i x_i K_ij  (Eq. (2), with the standard sign AMB-2)."""
    F, y, K = _toy(6, 9)
    C = 2.0
    z = np.array([0.0, C, 0.7, C, 0.0, 0.0])
    b = svm.bias(lambda v: K @ v, z, y, C)
    j = 2
    assert abs(b - (y[j] - (y * z) @ K[:, j])) < 1e-15


def test_bias_at_convergence_margin_svs_on_margin():
    F, y, K = _toy(10, 4)
    C = 1.0
    out = admm.run(admm.dense_solver(K, 1.0), y, C, 1.0, 4000)
    z = out["z"]
    b = svm.bias(lambda v: K @ v, z, y, C)
    M = svm.margin_set(z, C)
    assert M.sum() >= 1
    f = K @ (y * z) + b
    assert np.abs(y[M] * f[M] - 1.0).max() < 1e-9        # y_j f(f_j) = 1
    assert abs(b + out["lam"]) < 1e-9                     # b = -lambda = w^T q / w1 (E3)


def test_bias_empty_margin_fallbacks():
    K = np.eye(3)
    y = np.array([1.0, -1.0, 1.0])
    assert svm.bias(lambda v: K @ v, np.zeros(3), y, 1.0) == 0.0
    z = np.array([1.0, 1.0, 0.0])                         # all at C: fall back to z > eps
    b = svm.bias(lambda v: K @ v, z, y, 1.0)
    assert abs(b - ((1 - 1) - ((y * z) @ (K @ np.array([1.0, 1.0, 0.0])))) / 2) < 1e-15


def test_prediction_matches_loop_and_sign_zero():
    g = np.random.default_rng(8)
    Ftr, Fte = g.standard_normal((13, 3)), g.standard_normal((7, 3))
    coef = g.standard_normal(13)
    dv = svm.decision_values(Ftr, coef, 0.8, 0.25, Fte, chunk=3)
    for t in range(7):
        ref = 0.25 + sum(coef[i] * np.exp(-((Ftr[i] - Fte[t]) ** 2).sum() / (2 * 0.64))
                         for i in range(13))
        assert abs(dv[t] - ref) < 1e-14
    assert svm.labels(np.array([0.0, -0.0, 1e-300, -1e-300])).tolist() == [1, 1, 1, -1]


@pytest.mark.parametrize("seed", range(10))
def test_objective_gap_bound_eq9(seed):
    F, y, K = _toy(7, 100 + seed)
    g = np.random.default_rng(seed)
    E = g.standard_normal((7, 7)) * 0.05
    Kt = K + (E + E.T) / 2                              # may be indefinite
    lhs, rhs = qp.gap_bound(K, Kt, y, 1.0)
    assert lhs <= rhs * (1 + 1e-9) + 1e-14


def test_hss_admm_tracks_dense_admm_near_exact():
    """E13 shape: near-exact HSS ADMM stays within a few rel_tol of dense-K ADMM."""
    g = np.random.default_rng(0)
    n = 800
    y = np.where(g.random(n) < 0.5, 1.0, -1.0)
    F = g.standard_normal((n, 4)) + 0.5 * y[:, None]
    perm, ranges = tree.build_tree(F, 64, 3)
    Fp, yp = F[perm], y[perm]
    H = hss.compress(Fp, 1.0, ranges, rng.omega(4, perm, 700), rel_tol=1e-6, cap=684)
    f = ulv.factor(H, 1.0)
    K = kernel.dense_kernel(Fp, 1.0)
    o1 = admm.run(lambda b: ulv.solve(f, b), yp, 1.0, 1.0, 100)
    o2 = admm.run(admm.dense_solver(K, 1.0), yp, 1.0, 1.0, 100)
    assert np.linalg.norm(o1["z"] - o2["z"]) / np.linalg.norm(o2["z"]) < 2e-5
    ft = svm.objective(lambda v: hss.matvec(H, v), o1["z"], yp)
    fd = svm.objective_dense(K, o2["z"], yp)
    assert abs(ft - fd) / abs(fd) < 1e-6


def test_run_multi_columns_converge_to_their_own_bruteforce_qp():
    """The multi-C driver (one factorization, several C): column c converges to the
    brute-force QP optimum at box bound C_c (independent of run())."""
    F, y, K = _toy(8, 7)
    Cs = [0.3, 1.0, 5.0]
    out = admm.run_multi(admm.dense_solver(K, 1.0), y, Cs, 1.0, 3000)
    for c, C in enumerate(Cs):
        xb, fb = qp.solve_qp_bruteforce(K, y, C)
        assert np.abs(out["z"][:, c] - xb).max() < 1e-9
        assert abs(svm.objective_dense(K, out["z"][:, c], y) - fb) < 1e-12
