"""Oracle pins: HSS compression (H1-H5), mat-vec (M), ULV factor/solve (U, S)."""
import json
import os

import numpy as np
import pytest

from oracle import hss, kernel, rng, tree, ulv

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _setup(n, r, m, s, h, seed=0, spread=1.0):
    g = np.random.default_rng(seed)
    F = g.standard_normal((n, r)) * spread
    perm, ranges = tree.build_tree(F, m, 11)
    Fp = F[perm]
    Om = rng.omega(22, perm, s)
    return F, perm, ranges, Fp, Om


def test_exact_compression_limit():
    """rel_tol = 0, no cap, s >= every block rank => K~ = K (SPEC S:584 criterion)."""
    F, perm, ranges, Fp, Om = _setup(256, 3, 32, 272, 0.8)
    H = hss.compress(Fp, 0.8, ranges, Om, rel_tol=0.0)
    Kt = hss.assemble_dense(H)
    K = kernel.dense_kernel(Fp, 0.8)
    assert np.abs(Kt - K).max() / np.abs(K).max() < 1e-12


@pytest.mark.parametrize("tol", [1e-3, 1e-4, 1e-6])
def test_near_exact_error_below_tolerance(tol):
    F, perm, ranges, Fp, Om = _setup(1000, 4, 64, 700, 1.0)
    H = hss.compress(Fp, 1.0, ranges, Om, rel_tol=tol, cap=684)
    Kt = hss.assemble_dense(H)
    K = kernel.dense_kernel(Fp, 1.0)
    err = np.linalg.norm(Kt - K, 2) / np.linalg.norm(K, 2)
    assert err <= tol, err
    assert err >= 1e-3 * tol            # it is an approximation, not the identity
    assert np.abs(Kt - Kt.T).max() < 1e-15


def test_matvec_equals_independent_assembly_and_is_linear():
    F, perm, ranges, Fp, Om = _setup(600, 5, 32, 48, 1.0)
    H = hss.compress(Fp, 1.0, ranges, Om, rel_tol=1e-2, cap=32)
    assert any(H.cap_hit.values())
    Kt = hss.assemble_dense(H)
    g = np.random.default_rng(5)
    V = g.standard_normal((600, 3))
    out = hss.matvec(H, V)
    assert np.linalg.norm(out - Kt @ V) / np.linalg.norm(Kt @ V) < 1e-14
    a = 1.7
    lin = hss.matvec(H, a * V[:, 0] + V[:, 1])
    assert np.allclose(lin, a * out[:, 0] + out[:, 1], rtol=0, atol=1e-12)
    assert np.abs(hss.matvec(H, np.zeros(600))).max() == 0.0


def test_interpolative_structure():
    """U[J~] = I_k and J_t are active rows of the node; Y ~ U Y(J~) exactly on J~."""
    F, perm, ranges, Fp, Om = _setup(512, 4, 64, 80, 1.0)
    H = hss.compress(Fp, 1.0, ranges, Om, rel_tol=1e-3, cap=64)
    for t, U in H.U.items():
        if U is None:
            continue
        k = H.k[t]
        assert np.array_equal(U[H.Jloc[t]], np.eye(k))
        assert U.shape == (H.rows[t], k)


def test_fixed_rank_mode_reproduces_adaptive_generators():
    F, perm, ranges, Fp, Om = _setup(500, 4, 32, 120, 1.0)
    H1 = hss.compress(Fp, 1.0, ranges, Om, rel_tol=1e-4, cap=100)
    ranks = np.full(2 ** (H1.L + 1) - 1, -1)
    for t, k in H1.k.items():
        ranks[t] = k
    H2 = hss.compress(Fp, 1.0, ranges, Om, ranks=ranks)
    for t in H1.k:
        assert H1.k[t] == H2.k[t]
        assert np.array_equal(H1.J[t], H2.J[t])
    assert np.array_equal(hss.assemble_dense(H1), hss.assemble_dense(H2))


def test_passthrough_leaves_when_cap_equals_leaf():
    F, perm, ranges, Fp, Om = _setup(512, 4, 64, 80, 1.0)
    H = hss.compress(Fp, 1.0, ranges, Om, rel_tol=1e-12, cap=64)
    for t, lo, hi in H.nodes(H.L):
        assert H.U[t] is None and H.k[t] == hi - lo   # leaves: k = rows
    for t, lo, hi in H.nodes(H.L - 1):
        assert H.k[t] == 64 and H.rows[t] == 128


# ---------------------------------------------------------------- ULV
def _ulv_case(cap, beta, n=700):
    F, perm, ranges, Fp, Om = _setup(n, 4, 48, cap + 16, 1.0)
    H = hss.compress(Fp, 1.0, ranges, Om, rel_tol=1e-8, cap=cap)
    return H, ulv.factor(H, beta)


@pytest.mark.parametrize("cap,beta", [(200, 1.0), (48, 100.0)])
def test_ulv_solve_equals_dense_solve(cap, beta):
    H, f = _ulv_case(cap, beta)
    Kt = hss.assemble_dense(H)
    A = Kt + beta * np.eye(H.n)
    b = np.random.default_rng(1).standard_normal((H.n, 2))
    x = ulv.solve(f, b)
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) < 1e-13
    assert np.linalg.norm(x - np.linalg.solve(A, b)) / np.linalg.norm(x) < 1e-12


def test_ulv_scalar_case():
    g = json.load(open(os.path.join(GOLD, "closed_forms.json")))["solve_scalar"]
    Fp = np.zeros((1, 2))
    ranges = tree.node_ranges(1, 0)
    H = hss.compress(Fp, 1.0, ranges, rng.omega(1, np.array([0]), 1))
    f = ulv.factor(H, 1.0)
    assert abs(ulv.solve(f, np.array([g["b"]]))[0] - g["x"]) <= 4e-16


def test_ulv_huge_shift_limit():
    H, f = _ulv_case(48, 1e12, n=300)
    b = np.random.default_rng(2).standard_normal(300)
    x = ulv.solve(f, b)
    assert np.linalg.norm(x - b / 1e12) / np.linalg.norm(b / 1e12) < 1e-9


def test_ulv_breakdown_names_node():
    """Capped K~ is indefinite; a tiny shift must raise NotSPD with a node id (AMB-9/14)."""
    F, perm, ranges, Fp, Om = _setup(1024, 4, 32, 24, 0.4)
    H = hss.compress(Fp, 0.4, ranges, Om, rel_tol=0.0, cap=8)
    Kt = hss.assemble_dense(H)
    lmin = np.linalg.eigvalsh(Kt)[0]
    assert lmin < -1e-3
    with pytest.raises(ulv.NotSPDError) as ei:
        ulv.factor(H, 1e-6)
    assert isinstance(ei.value.node, int)
    ulv.factor(H, -4 * lmin)   # a shift past -lambda_min succeeds


# ------------------------------------------------------------------ N2: adaptive sampling
def test_adaptive_with_full_budget_is_the_plain_compression():
    F, perm, ranges, Fp, Om = _setup(600, 5, 40, 96, 1.0)
    H1 = hss.compress(Fp, 1.0, ranges, Om, rel_tol=1e-3, cap=80)
    H2, s, rounds = hss.compress_adaptive(Fp, 1.0, ranges, perm, 22, s0=96, ds=16, s_max=96, p=16,
                                          rel_tol=1e-3, cap=80)
    assert s == 96 and rounds == 1
    assert all(H1.k[t] == H2.k[t] for t in H1.k)
    assert np.array_equal(hss.assemble_dense(H1), hss.assemble_dense(H2))


def test_adaptive_grows_until_converged_and_meets_tolerance():
    # near-exact tolerance, small start: the loop must grow s, end with every node converged
    # (or at the budget), and the compressed K~ must meet the tolerance (E6 shape)
    F, perm, ranges, Fp, _ = _setup(700, 3, 64, 16, 1.5)
    H, s, rounds = hss.compress_adaptive(Fp, 1.5, ranges, perm, 0, s0=24, ds=24, s_max=400, p=16,
                                         rel_tol=1e-6)
    assert rounds > 1 and s > 24
    assert s == 400 or not hss.unconverged(H, s, 16, None)
    K = np.exp(-((Fp[:, None, :] - Fp[None, :, :]) ** 2).sum(-1) / (2 * 1.5 ** 2))
    assert np.linalg.norm(hss.assemble_dense(H) - K, 2) <= 1e-6 * np.linalg.norm(K, 2)


def test_unconverged_rule():
    H = hss.HSS(n=0, L=1, ranges=[], Fp=np.zeros((0, 1)), h=1.0)
    H.k = {1: 40, 2: 30, 3: 50}
    H.rows = {1: 100, 2: 100, 3: 50}
    # s = 48, p = 16: k > 32 and k < min(cap, rows) -> node 1 only (node 3 is full rank)
    assert hss.unconverged(H, 48, 16, None) == [1]
    assert hss.unconverged(H, 48, 16, 40) == []     # node 1 at the cap


def test_fixed_skeleton_replay_reproduces_adaptive_generators():
    """AMB-12 diagnostic mode: replaying the adaptive run's own skeletons (pivot order) and ranks
    gives the same K~: U (sign-free interpolation coefficients), J, B equal to rounding."""
    F, perm, ranges, Fp, Om = _setup(700, 4, 64, 48, 1.0, seed=3)
    H = hss.compress(Fp, 1.0, ranges, Om, rel_tol=1e-3, cap=32)
    nn = 2 ** (H.L + 1) - 1
    ranks = np.full(nn, -1)
    for t, k in H.k.items():
        ranks[t] = k
    flat = np.concatenate([H.J[t] for t in range(1, nn)])
    sk = hss.skeletons_from_flat(flat, ranks, ranges, 48)
    assert all(np.array_equal(sk[t], H.J[t]) for t in range(1, nn))
    H2 = hss.compress(Fp, 1.0, ranges, Om, skeletons=sk)
    for t in range(1, nn):
        assert H2.k[t] == H.k[t] and np.array_equal(H2.J[t], H.J[t])
        if H.U[t] is not None:
            assert np.abs(H2.U[t] - H.U[t]).max() <= 1e-9 * max(1.0, np.abs(H.U[t]).max())
    for t in H.B:
        assert np.abs(H2.B[t] - H.B[t]).max() <= 1e-14


def test_fixed_skeleton_interpolation_is_least_squares():
    """For an arbitrary (non-CPQR) skeleton, U's non-skeleton rows are the least-squares
    interpolation coefficients of Y_t's rows on the skeleton rows (the ID of P:184 with a given
    column set): U[rest] = (pinv(Y_J^T) Y_rest^T)^T, checked with numpy lstsq (no QR route)."""
    F, perm, ranges, Fp, Om = _setup(256, 3, 64, 40, 1.0, seed=4)
    L = len(ranges) - 1
    g = np.random.default_rng(1)
    sk = {}
    k = {}
    # leaves: 24 random points in a scrambled order; parents: 24 of the children's skeletons
    for lvl in range(L, 0, -1):
        for i, (lo, hi) in enumerate(ranges[lvl]):
            t = (1 << lvl) - 1 + i
            act = np.arange(lo, hi) if lvl == L else np.concatenate([sk[2 * t + 1], sk[2 * t + 2]])
            sk[t] = act[g.permutation(len(act))[:24]]
            k[t] = 24
    H = hss.compress(Fp, 1.0, ranges, Om, skeletons=sk)
    S = kernel.sketch(Fp, 1.0, Om)
    for i, (lo, hi) in enumerate(ranges[L]):
        t = (1 << L) - 1 + i
        D = kernel.gaussian_block(Fp[lo:hi], Fp[lo:hi], 1.0)
        Y = S[lo:hi] - D @ Om[lo:hi]
        loc = np.array([int(np.where(np.arange(lo, hi) == a)[0][0]) for a in sk[t]])
        rest = np.setdiff1d(np.arange(hi - lo), loc)
        X = np.linalg.lstsq(Y[loc].T, Y[rest].T, rcond=None)[0]
        assert np.array_equal(H.J[t], sk[t])
        assert np.abs(H.U[t][loc] - np.eye(24)).max() == 0.0
        assert np.abs(H.U[t][rest] - X.T).max() <= 1e-8 * max(1.0, np.abs(X).max())
