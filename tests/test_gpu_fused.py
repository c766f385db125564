"""The fused bottom level of the ADMM iteration (one 8-CTA cluster per level-(L-1) node:
backward sweep -> epilogue -> next forward sweep) must give BITWISE the same iterates as the
unfused level-by-level sweep (the default; SVMHSS_FUSE_BOTTOM=1 fuses): both use the same device functions and
the same chunk-ordered leaf sums.  Also pinned to the oracle (tests/test_gpu_parity.py covers
the unfused order at the north-star tolerances)."""
import os

import numpy as np
import pytest

import datagen

pytestmark = pytest.mark.gpu


def _train(P, F, y, cfg, beta, Cs, it, fuse):
    import torch
    os.environ["SVMHSS_FUSE_BOTTOM"] = "1" if fuse else "0"
    try:
        dev = torch.device("cuda:0")
        Fd, yd = torch.from_numpy(F).to(dev), torch.from_numpy(y).to(dev)
        H = P.hss_build(Fd, cfg["h"], leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], max_rank=cfg["cap"],
                        oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"])
        U = P.hss_ulv_factor(H, beta)
        r = P.admm_svm_train(U, yd, Cs, it, trace_every=10)
        out = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in r.items() if k != "stats"}
        out["launches"] = r["stats"]["kernel_launches_per_iter"]
        U.free()
        H.free()
        return out
    finally:
        os.environ.pop("SVMHSS_FUSE_BOTTOM", None)


@pytest.mark.parametrize("cfg_id,n,cap,Cs", [(3, 8192, 256, [1.0]), (3, 6000, 256, [0.5, 1.0, 10.0]),
                                              (1, 5000, 128, [10.0]), (3, 5000, 96, [1.0, 2.0])])
def test_fused_bottom_is_bitwise_identical_to_unfused(gpu_lib, cfg_id, n, cap, Cs):
    cfg = datagen.get_config(cfg_id)
    cfg["cap"], cfg["s"] = cap, cap + 16
    F, y, _, _ = datagen.generate(cfg_id, n=n, n_test=0)
    a = _train(gpu_lib, F, y, cfg, 1e4, Cs, 40, fuse=True)
    b = _train(gpu_lib, F, y, cfg, 1e4, Cs, 40, fuse=False)
    for k in ("z", "mu", "bias", "obj", "trace_z", "trace_mu"):
        assert np.array_equal(a[k], b[k]), k
