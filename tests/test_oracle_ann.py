"""Pins of the HSS-ANN oracle (oracle/ann.py; readings N1-N3 in DESIGN.md), each against
something other than the oracle's own formulas: brute-force nearest neighbours (scipy cdist),
geometric separation where random-projection trees cannot miss, set properties of the sampled
columns checked by a direct loop, and the exact-compression limit (sampling the whole
off-diagonal block row at full rank gives K~ = K)."""
import numpy as np
import pytest
from scipy.spatial.distance import cdist

from oracle import ann, hss, tree


def test_signs_are_pm1_deterministic_and_balanced():
    a = ann.rp_signs(5, 0, 3, 4000)
    b = ann.rp_signs(5, 0, 3, 4000)
    assert set(np.unique(a)) == {-1.0, 1.0} and np.array_equal(a, b)
    assert abs(a.mean()) < 0.06
    assert not np.array_equal(a, ann.rp_signs(5, 1, 3, 4000))   # another tree
    assert not np.array_equal(a, ann.rp_signs(5, 0, 4, 4000))   # another node


def test_sqdist_matches_cdist():
    g = np.random.default_rng(1)
    A, B = g.standard_normal((30, 7)), g.standard_normal((20, 7))
    assert np.allclose(ann.sqdist(A, B), cdist(A, B, "sqeuclidean"), rtol=1e-13, atol=1e-13)


def test_rp_tree_invariants():
    g = np.random.default_rng(2)
    F = g.standard_normal((1000, 6))
    perm, ranges = ann.rp_tree(F, 64, 9, 1)
    assert np.array_equal(np.sort(perm), np.arange(1000))
    L = len(ranges) - 1
    assert L == tree.num_levels(1000, 64)
    for lvl in range(L):
        for i, (lo, hi) in enumerate(ranges[lvl]):
            mid = lo + (hi - lo) // 2
            sg = ann.rp_signs(9, 1, (1 << lvl) - 1 + i, 6)
            pl = F[perm[lo:mid]] @ sg
            pr = F[perm[mid:hi]] @ sg
            assert pl.max() <= pr.min() + 1e-12


def test_single_tree_covering_all_points_gives_exact_knn():
    g = np.random.default_rng(3)
    F = g.standard_normal((300, 5))
    idx, d = ann.knn(F, 12, 1, 1000, 4)
    D = cdist(F, F, "sqeuclidean")
    np.fill_diagonal(D, np.inf)
    ex = np.argsort(D, axis=1, kind="stable")[:, :12]
    assert np.array_equal(idx, ex)
    assert np.allclose(d, np.take_along_axis(D, ex, axis=1), rtol=1e-13)


def test_separated_clusters_are_found_exactly():
    # two clusters 200 apart along every coordinate (r odd: every +-1 direction separates them),
    # each exactly one leaf of every tree -> ANN = exact kNN
    g = np.random.default_rng(4)
    A = g.standard_normal((128, 5)) - 100.0
    B = g.standard_normal((128, 5)) + 100.0
    F = np.vstack([A, B])[g.permutation(256)]
    idx, _ = ann.knn(F, 10, 3, 128, 8)
    D = cdist(F, F, "sqeuclidean")
    np.fill_diagonal(D, np.inf)
    assert np.array_equal(idx, np.argsort(D, axis=1, kind="stable")[:, :10])


def test_fewer_candidates_than_kappa_pads():
    F = np.random.default_rng(5).standard_normal((40, 3))
    idx, d = ann.knn(F, 20, 1, 8, 1)            # leaves of 5 points: 4 candidates each
    assert (idx[:, 4:] == -1).all() and np.isinf(d[:, 4:]).all()
    assert (idx[:, :4] >= 0).all()


def _sampling_case(n=900, r=4, s=40, seed=6):
    g = np.random.default_rng(seed)
    F = g.standard_normal((n, r))
    perm, ranges = tree.build_tree(F, 50, 2)
    idx, d = ann.knn(F, 8, 2, 60, 3)
    iperm = np.empty(n, dtype=np.int64)
    iperm[perm] = np.arange(n)
    ann_pos = np.where(idx[perm] >= 0, iperm[np.maximum(idx[perm], 0)], -1)
    return F, perm, ranges, ann_pos, d[perm]


@pytest.mark.parametrize("s", [5, 40, 3000])
def test_sampled_columns_properties(s):
    F, perm, ranges, ann_pos, ann_dp = _sampling_case()
    n = F.shape[0]
    lvl = 3
    for i, (lo, hi) in enumerate(ranges[lvl]):
        t = (1 << lvl) - 1 + i
        A = np.arange(lo, hi)
        C = ann.sample_columns(t, lo, hi, n, A, ann_pos, ann_dp, s, 17)
        assert np.all(np.diff(C) > 0)                            # sorted, distinct
        assert np.all((C < lo) | (C >= hi))                      # outside the node
        assert C.size == min(s, n - (hi - lo))
        # the ANN part, by a direct loop: best (min d, pos) outside positions
        best = {}
        for a in A:
            for q, dq in zip(ann_pos[a], ann_dp[a]):
                if q >= 0 and (q < lo or q >= hi):
                    best[q] = min(best.get(q, np.inf), dq)
        ranked = sorted(best, key=lambda q: (best[q], q))[:s]
        assert set(ranked) <= set(C.tolist())
        assert np.array_equal(C, ann.sample_columns(t, lo, hi, n, A, ann_pos, ann_dp, s, 17))


def test_whole_block_row_sample_is_exact():
    # s >= n: every node samples its entire off-diagonal block row; rel_tol 0, no cap ->
    # the interpolative decompositions are exact and K~ = K
    g = np.random.default_rng(7)
    n = 300
    F = g.standard_normal((n, 3))
    perm, ranges = tree.build_tree(F, 40, 5)
    idx, d = ann.knn(F, 6, 2, 40, 3)
    H = ann.compress_ann(F[perm], 1.5, ranges, perm, idx, d, n, 11, rel_tol=0.0)
    K = np.exp(-cdist(F[perm], F[perm], "sqeuclidean") / (2 * 1.5 ** 2))
    Kt = hss.assemble_dense(H)
    assert np.linalg.norm(Kt - K, 2) <= 1e-11 * np.linalg.norm(K, 2)


def test_capped_ann_compression_is_a_valid_hss():
    g = np.random.default_rng(8)
    n = 700
    F = g.standard_normal((n, 4))
    perm, ranges = tree.build_tree(F, 64, 5)
    idx, d = ann.knn(F, 16, 2, 64, 3)
    H = ann.compress_ann(F[perm], 1.0, ranges, perm, idx, d, 48, 11, rel_tol=1e-4, cap=32)
    Kt = hss.assemble_dense(H)
    assert np.allclose(Kt, Kt.T, atol=1e-14)
    assert max(H.k.values()) <= 32
    for t, U in H.U.items():                                    # interpolative: U[J~] = I
        if U is not None:
            assert np.array_equal(U[H.Jloc[t]], np.eye(H.k[t]))
    # matvec == the assembled matrix
    v = g.standard_normal(n)
    assert np.allclose(hss.matvec(H, v), Kt @ v, rtol=1e-12, atol=1e-12)
