"""Oracle pins: N4, SPD-preserving compression (interp="spd", oracle/hss.py docstring).

The construction keeps H3's skeletons and replaces the ID interpolation by the kernel
interpolant U_t = K(A_t, J_t) (K(J_t, J_t) + eps I)^-1.  Pinned here against what the
mathematics fixes, not against its own formula:
  - K~ is positive semidefinite on inputs where the paper's ID form is indefinite (the
    property N4 exists for);
  - the assembled K~ equals, term by term, the telescoping sum of one-level Schur-complement
    terms that proves it PSD (each term built from raw kernel entries, each term PSD);
  - interpolation: skeleton rows of U are the identity for eps = 0, and K~ reproduces K exactly
    on skeleton x skeleton entries of sibling blocks;
  - with no compression (every node pass-through) both forms are K itself;
  - the ULV factorization of K~ + beta I succeeds for small beta where the ID form breaks down,
    and its solve equals a dense solve of the assembled matrix.
"""
import numpy as np
import pytest
import scipy.linalg as sla

import datagen
from oracle import hss, kernel, rng, tree, ulv


def _setup(c, n, s=None, cap=None, leaf=None, h=None):
    cfg = datagen.get_config(c)
    h = h if h is not None else (cfg["h"] if not isinstance(cfg["h"], list) else 1.0)
    F, *_ = datagen.generate(c, n=n, n_test=1)
    leaf = leaf or cfg["leaf"]
    perm, ranges = tree.build_tree(F, leaf, cfg["seed_tree"])
    Fp = F[perm]
    cap = cap or cfg["cap"]
    Om = rng.omega(cfg["seed_omega"], perm, s or cfg["s"])
    return cfg, Fp, ranges, Om, h, cap


@pytest.mark.parametrize("c,n,cap,leaf", [(1, 1024, 32, 64), (3, 1024, 64, 128), (4, 1024, 16, 32)])
def test_spd_form_is_psd_where_id_form_is_not(c, n, cap, leaf):
    cfg, Fp, ranges, Om, h, _ = _setup(c, n, s=cap + 16, cap=cap, leaf=leaf)
    K = kernel.dense_kernel(Fp, h)
    nK = np.linalg.norm(K, 2)
    Hid = hss.compress(Fp, h, ranges, Om, rel_tol=cfg["rel_tol"], cap=cap, interp="id")
    Hspd = hss.compress(Fp, h, ranges, Om, rel_tol=cfg["rel_tol"], cap=cap, interp="spd", spd_eps=0.0)
    lid = np.linalg.eigvalsh(hss.assemble_dense(Hid))[0]
    Ks = hss.assemble_dense(Hspd)
    assert np.abs(Ks - Ks.T).max() < 1e-15
    lspd = np.linalg.eigvalsh(Ks)[0]
    assert lid < -1e-3 * nK, lid                  # the capped ID form is indefinite here
    assert lspd >= -1e-12 * nK, lspd              # the N4 form is not
    assert any(u is not None for u in Hspd.U.values())   # it did compress


def _telescoping_sum(H):
    """K~ as the sum the PSD proof uses, built from raw kernel entries and the U_t only:
    level l's active set A^(l) (all points at l = L, the children's skeletons above);
    W_l = blockdiag_t(U_t) (I for pass-through) maps A^(l-1) coordinates to A^(l);
    T_l = blockdiag_t(K(A_t, A_t) - U_t K(J_t, J_t) U_t^T);  K~ = T_L + W_L (T_{L-1} + W_{L-1}(...
    (T_1 + W_1 K(A^(0), A^(0)) W_1^T) ...) W_L^T."""
    Fp, h, L = H.Fp, H.h, H.L
    act = {}
    for t, lo, hi in H.nodes(L):
        act[t] = np.arange(lo, hi)
    for lvl in range(L - 1, -1, -1):
        for t, lo, hi in H.nodes(lvl):
            act[t] = np.concatenate([H.J[2 * t + 1], H.J[2 * t + 2]])
    terms, Ws = {}, {}
    for lvl in range(L, 0, -1):
        blocks_T, blocks_W = [], []
        for t, lo, hi in H.nodes(lvl):
            A = act[t]
            U = np.eye(len(A)) if H.U[t] is None else H.U[t]
            J = H.J[t]
            blocks_T.append(kernel.gaussian_block(Fp[A], Fp[A], h) - U @ kernel.gaussian_block(Fp[J], Fp[J], h) @ U.T)
            blocks_W.append(U)
        terms[lvl] = sla.block_diag(*blocks_T)
        Ws[lvl] = sla.block_diag(*blocks_W)
    A0 = act[0]
    acc = kernel.gaussian_block(Fp[A0], Fp[A0], h)
    for lvl in range(1, L + 1):
        acc = terms[lvl] + Ws[lvl] @ acc @ Ws[lvl].T
    return acc, terms


def test_assembled_spd_form_equals_the_psd_decomposition():
    cfg, Fp, ranges, Om, h, _ = _setup(3, 512, s=24, cap=8, leaf=32)
    H = hss.compress(Fp, h, ranges, Om, rel_tol=1e-3, cap=8, interp="spd", spd_eps=0.0)
    assert H.L == 4 and sum(u is not None for u in H.U.values()) > 20
    Kt = hss.assemble_dense(H)
    Ksum, terms = _telescoping_sum(H)
    assert np.abs(Kt - Ksum).max() <= 1e-12 * np.abs(Kt).max()
    for lvl, T in terms.items():                  # every Schur-complement term is PSD
        assert np.linalg.eigvalsh((T + T.T) / 2)[0] >= -1e-12, lvl
    # the ID form does NOT satisfy the decomposition's premise (its terms are indefinite)
    Hid = hss.compress(Fp, h, ranges, Om, rel_tol=1e-3, cap=8, interp="id")
    _, tid = _telescoping_sum(Hid)
    assert min(np.linalg.eigvalsh((T + T.T) / 2)[0] for T in tid.values()) < -1e-6


def test_interpolation_property_and_exact_skeleton_entries():
    cfg, Fp, ranges, Om, h, _ = _setup(1, 512, s=32, cap=16, leaf=64)
    H = hss.compress(Fp, h, ranges, Om, rel_tol=1e-4, cap=16, interp="spd", spd_eps=0.0)
    Kt = hss.assemble_dense(H)
    K = kernel.dense_kernel(Fp, h)
    checked = 0
    for t, U in H.U.items():
        if U is None:
            continue
        assert np.abs(U[H.Jloc[t]] - np.eye(U.shape[1])).max() < 1e-8
        checked += 1
    assert checked > 4
    for t, lo, hi in H.nodes(H.L - 1):            # leaf-level siblings: skeleton x skeleton exact
        Ja, Jb = H.J[2 * t + 1], H.J[2 * t + 2]
        assert np.abs(Kt[np.ix_(Ja, Jb)] - K[np.ix_(Ja, Jb)]).max() < 1e-12
    for t, lo, hi in H.nodes(H.L):                # leaf diagonal blocks are K's
        assert np.array_equal(Kt[lo:hi, lo:hi], K[lo:hi, lo:hi])


def test_no_compression_both_forms_are_k():
    cfg, Fp, ranges, Om, h, _ = _setup(0, 256, s=272, cap=None, leaf=32)
    K = kernel.dense_kernel(Fp, h)
    for interp in ("id", "spd"):
        H = hss.compress(Fp, h, ranges, Om, rel_tol=0.0, interp=interp)
        assert np.abs(hss.assemble_dense(H) - K).max() < 1e-12 * np.abs(K).max()


def test_spd_factor_at_small_beta_and_solve_equals_dense():
    cfg, Fp, ranges, Om, h, _ = _setup(3, 1024, s=80, cap=64, leaf=128)
    Hid = hss.compress(Fp, h, ranges, Om, rel_tol=1e-3, cap=64, interp="id")
    with pytest.raises(ulv.NotSPDError):
        ulv.factor(Hid, 1e-2)
    H = hss.compress(Fp, h, ranges, Om, rel_tol=1e-3, cap=64, interp="spd")
    beta = 1e-2
    fac = ulv.factor(H, beta)
    b = np.random.default_rng(3).standard_normal((1024, 2))
    x = ulv.solve(fac, b)
    ref = np.linalg.solve(hss.assemble_dense(H) + beta * np.eye(1024), b)
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) < 1e-9


def test_spd_eps_bound_keeps_psd():
    """eps > 0 (the jittered interpolant) keeps every Schur term PSD (g/(g+eps)^2 <= 1/g)."""
    cfg, Fp, ranges, Om, h, _ = _setup(3, 512, s=24, cap=8, leaf=32)
    for eps in (1e-8, 1e-2):
        H = hss.compress(Fp, h, ranges, Om, rel_tol=1e-3, cap=8, interp="spd", spd_eps=eps)
        Kt = hss.assemble_dense(H)
        Ksum, terms = _telescoping_sum(H)
        assert np.abs(Kt - Ksum).max() <= 1e-12 * np.abs(Kt).max()
        assert np.linalg.eigvalsh(Kt)[0] >= -1e-12 * np.abs(Kt).max()


def test_spd_with_ann_sampling_is_psd_and_keeps_skeletons():
    """N4 with HSS-ANN sampling (N1-N3): the sampled columns do not depend on U, so the skeletons
    equal the ID form's; the assembled K~ is the PSD decomposition's sum, and PSD."""
    from oracle import ann
    cfg = datagen.get_config(3)
    F, *_ = datagen.generate(3, n=1024, n_test=1)
    perm, ranges = tree.build_tree(F, 128, cfg["seed_tree"])
    idx, d = ann.knn(F, cfg["ann_neighbors"], cfg["ann_trees"], cfg["ann_leaf"], cfg["ann_seed"])
    kw = dict(rel_tol=1e-3, cap=48)
    Hid = ann.compress_ann(F[perm], 1.0, ranges, perm, idx, d, 64, cfg["ann_seed"], **kw)
    Hs = ann.compress_ann(F[perm], 1.0, ranges, perm, idx, d, 64, cfg["ann_seed"], interp="spd", spd_eps=0.0, **kw)
    assert all(np.array_equal(Hid.J[t], Hs.J[t]) for t in Hid.J)
    assert sum(u is not None for u in Hs.U.values()) > 4
    Kt = hss.assemble_dense(Hs)
    Ksum, terms = _telescoping_sum(Hs)
    assert np.abs(Kt - Ksum).max() <= 1e-12 * np.abs(Kt).max()
    assert np.linalg.eigvalsh(Kt)[0] >= -1e-12 * np.abs(Kt).max()
