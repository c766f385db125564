"""C-ABI error behaviour and handle ownership (include/svmhss.h) on the GPU: invalid arguments
return HSS_EINVAL, a Cholesky breakdown returns HSS_ENOTSPD naming the node (AMB-14), labels
other than +-1 are rejected, and a ulv_t keeps its hss_t alive after hss_free."""
import numpy as np
import pytest

import datagen

pytestmark = pytest.mark.gpu


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def _small(P, **kw):
    cfg = datagen.get_config(3)
    F, y, _, _ = datagen.generate(3, n=2000, n_test=0)
    opts = dict(leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], max_rank=cfg["cap"], oversample=16,
                omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"])
    opts.update(kw)
    return F, y, P.hss_build(_t(F), cfg["h"], **opts)


@pytest.mark.parametrize("kw,h", [(dict(leaf_size=0), 1.0), (dict(max_rank=0), 1.0), ({}, 0.0), ({}, -1.0),
                                  (dict(oversample=-2), 1.0), (dict(rel_tol=-1.0), 1.0),
                                  (dict(sampling="ann", ann_leaf=512), 1.0),
                                  (dict(sampling="ann", ann_trees=8, ann_neighbors=64), 1.0)])
def test_build_rejects_invalid_arguments(gpu_lib, kw, h):
    P = gpu_lib
    F, _, _, _ = datagen.generate(3, n=500, n_test=0)
    opts = dict(leaf_size=64, max_rank=32, oversample=16)
    opts.update(kw)
    with pytest.raises(P.HssError) as e:
        P.hss_build(_t(F), h, **opts)
    assert e.value.code == -1


def test_factor_breakdown_names_the_node(gpu_lib):
    P = gpu_lib
    _, _, H = _small(P, max_rank=32)
    with pytest.raises(P.HssError) as e:
        P.hss_ulv_factor(H, 1e-6)
    assert e.value.code == -5 and "node" in str(e.value)
    with pytest.raises(P.HssError) as e:
        P.hss_ulv_factor(H, 0.0)
    assert e.value.code == -1


def test_admm_rejects_bad_labels_and_sizes(gpu_lib):
    P = gpu_lib
    F, y, H = _small(P)
    U = P.hss_ulv_factor(H, 1e3)
    yb = y.copy()
    yb[7] = 0.5
    with pytest.raises(P.HssError) as e:
        P.admm_svm_train(U, _t(yb), [1.0], 5)
    assert e.value.code == -1
    with pytest.raises(P.HssError):
        P.admm_svm_train(U, _t(y), [-1.0], 5)            # C <= 0
    with pytest.raises(P.HssError):
        P.admm_svm_train(U, _t(y), [1.0], 0)             # max_it < 1


def test_ulv_keeps_hss_alive(gpu_lib):
    P = gpu_lib
    F, y, H = _small(P)
    U = P.hss_ulv_factor(H, 1e3)
    b = _t(np.random.default_rng(1).standard_normal(F.shape[0]))
    x1 = U.solve(b).cpu().numpy()
    H.free()                       # the factorization still holds a reference
    x2 = U.solve(b).cpu().numpy()
    assert np.array_equal(x1, x2)
    r = P.admm_svm_train(U, _t(y), [1.0], 10)
    assert np.isfinite(r["obj"][0])
    U.free()
