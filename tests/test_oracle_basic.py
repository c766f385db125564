"""Oracle pins: RNG, kernel, sketch, tree (CPU only)."""
import json
import math
import os

import numpy as np
import pytest
from scipy import stats

from oracle import kernel, rng, tree

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- RNG (R1-R3)
def test_splitmix64_reference_vectors():
    g = _gold("splitmix64.json")
    golden = 0x9E3779B97F4A7C15
    M = (1 << 64) - 1
    for k, hx in enumerate(g["seed0_first3_hex"]):
        assert int(rng.splitmix64(np.uint64((k * golden) & M))) == int(hx, 16)
    for k, dec in enumerate(g["seed1234567_first5"]):
        assert int(rng.splitmix64(np.uint64((1234567 + k * golden) & M))) == int(dec)


def test_omega_is_standard_normal():
    i = np.arange(2000)
    X = rng.omega(2003, i, 500).ravel()
    assert np.isfinite(X).all()
    assert abs(X.mean()) < 5e-3 and abs(X.var() - 1.0) < 5e-3
    assert stats.kstest(X[:200000], "norm").pvalue > 1e-4


def test_omega_keyed_by_original_index_and_column():
    a = rng.omega(7, np.array([5, 9, 5]), 4)
    assert np.array_equal(a[0], a[2])          # same (i, j) -> same value
    assert not np.array_equal(a[0], a[1])
    b = rng.omega(8, np.array([5]), 4)
    assert not np.array_equal(a[0], b[0])      # different seed
    # a subset of columns is a prefix (counter keyed by j, not by s)
    assert np.array_equal(rng.omega(7, np.array([5]), 2)[0], a[0, :2])


# ---------------------------------------------------------------- kernel (AMB-4)
def test_kernel_exp_minus_one_at_two_h_squared():
    g = _gold("closed_forms.json")["kernel_exp_minus_one"]["value"]
    h = 0.7
    fa = np.array([[0.0, 0.0]])
    fb = np.array([[math.sqrt(2.0) * h, 0.0]])
    assert abs(kernel.gaussian_block(fa, fb, h)[0, 0] - g) <= 2e-16


def test_kernel_symmetry_unit_diagonal_and_gemm_form():
    r = np.random.default_rng(1)
    F = r.standard_normal((200, 11))
    K = kernel.gaussian_block(F, F, 1.3)
    assert np.array_equal(np.diag(K), np.ones(200))
    assert np.abs(K - K.T).max() == 0.0
    nu = (F * F).sum(1)
    d2 = np.maximum(nu[:, None] + nu[None, :] - 2 * F @ F.T, 0.0)
    Kg = np.exp(-d2 / (2 * 1.3 ** 2))
    assert np.abs(K - Kg).max() < 1e-13
    assert (K > 0).all() and (K <= 1).all()


def test_sketch_equals_triple_loop():
    r = np.random.default_rng(2)
    F = r.standard_normal((23, 3))
    Om = r.standard_normal((23, 5))
    h = 0.9
    S = kernel.sketch(F, h, Om, chunk=7)
    ref = np.zeros((23, 5))
    for i in range(23):
        for j in range(23):
            d2 = sum((F[i, t] - F[j, t]) ** 2 for t in range(3))
            kij = math.exp(-d2 / (2 * h * h))
            for c in range(5):
                ref[i, c] += kij * Om[j, c]
    assert np.abs(S - ref).max() < 1e-13


# ---------------------------------------------------------------- tree (T1-T4)
@pytest.mark.parametrize("n,m", [(2000, 64), (1024, 128), (257, 64), (10, 16), (64, 64)])
def test_tree_invariants(n, m):
    r = np.random.default_rng(n)
    F = r.standard_normal((n, 5))
    perm, ranges = tree.build_tree(F, m, 99)
    L = tree.num_levels(n, m)
    assert L == max(0, math.ceil(math.log2(n / m))) if n > m else L == 0
    assert np.array_equal(np.sort(perm), np.arange(n))          # bijection
    assert len(ranges) == L + 1
    for lvl in range(L + 1):
        assert ranges[lvl][0][0] == 0 and ranges[lvl][-1][1] == n
        for (a, b), (c, d) in zip(ranges[lvl][:-1], ranges[lvl][1:]):
            assert b == c
    for lo, hi in ranges[L]:
        assert 1 <= hi - lo <= m
    # T3: every split separates projections: recompute p with the oracle's direction
    for lvl in range(L):
        for i, (lo, hi) in enumerate(ranges[lvl]):
            idx = perm[lo:hi]
            X = F[idx] - F[idx].mean(0)
            v = tree.principal_direction(X, rng.tree_start_vector(99, (1 << lvl) - 1 + i, 5))
            p = X @ v
            half = (hi - lo) // 2
            assert p[:half].max() <= p[half:].min()


def test_tree_two_blobs_split_exactly():
    r = np.random.default_rng(3)
    A = r.standard_normal((50, 2)) * 0.1 + np.array([-10.0, 3.0])
    B = r.standard_normal((50, 2)) * 0.1 + np.array([10.0, -3.0])
    F = np.vstack([A, B])
    perm, ranges = tree.build_tree(F, 64, 5)
    left = set(perm[:50].tolist())
    assert left == set(range(50)) or left == set(range(50, 100))


def test_power_iteration_is_top_eigenvector_with_gap():
    r = np.random.default_rng(4)
    # covariance eigenvalues 4, 1, 0.25 ... -> lambda2/lambda1 = 0.25 <= 0.7
    X = r.standard_normal((4000, 6)) * np.array([2.0, 1.0, 0.5, 0.4, 0.3, 0.2])
    X = X - X.mean(0)
    v = tree.principal_direction(X, rng.tree_start_vector(1, 0, 6))
    w, V = np.linalg.eigh(X.T @ X)
    assert 1 - abs(v @ V[:, -1]) < 1e-12


def test_tree_constant_points_split_by_index():
    F = np.ones((40, 3))
    perm, ranges = tree.build_tree(F, 16, 1)
    assert np.array_equal(perm, np.arange(40))
