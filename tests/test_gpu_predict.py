"""svm_predict (a11: dv_t = sum_i coef_i K(f_i, t) + b, label = sign with 0 -> +1) on
the GPU against the oracle's exact decision values, across the predict kernel's shapes: feature
counts that select each A-fragment register width (r = 8 -> rp 8, r = 54 -> rp 56, r = 123 ->
rp 124 with 8-warp CTAs) and the wide-feature path (r > 128), coefficient widths nC = 1, 3 (padded to 4) and 16, and ragged sizes
(test points not a multiple of the 128 / 64-row CTA tile, training points not a multiple of the
64-point step, a single test point, fewer training points than one step)."""
import numpy as np
import pytest

from oracle import svm as o_svm

pytestmark = pytest.mark.gpu


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


@pytest.mark.parametrize("n,m,r,nC,h", [
    (1000, 333, 8, 1, 1.0),
    (4099, 130, 54, 1, 1.0),
    (777, 257, 54, 3, 0.7),
    (130, 1, 54, 16, 2.0),
    (50, 70, 22, 2, 0.5),
    (2050, 65, 123, 1, 2.0),
    (513, 200, 123, 16, 3.0),
    (700, 150, 150, 1, 4.0),      # r > 128: the wide-feature path (sketch kernel tiling)
    (300, 77, 203, 3, 5.0),
])
def test_predict_matches_oracle(gpu_lib, n, m, r, nC, h):
    P = gpu_lib
    g = np.random.default_rng(n * 7 + m)
    F = g.standard_normal((n, r)) * (0.3 if r > 50 else 1.0)
    Ft = g.standard_normal((m, r)) * (0.3 if r > 50 else 1.0)
    coef = g.standard_normal((n, nC))
    bias = g.standard_normal(nC)
    y = np.where(g.random(n) < 0.5, -1.0, 1.0)
    z = y[:, None] * coef          # y o z = coef exactly (sign flips)
    dv, lab = P.svm_predict(_t(F), _t(y), _t(z if nC > 1 else z[:, 0]), h, bias, _t(Ft))
    dv, lab = dv.cpu().numpy(), lab.cpu().numpy()
    for c in range(nC):
        dvo = o_svm.decision_values(F, coef[:, c], h, bias[c], Ft)
        scale = max(1.0, np.abs(coef[:, c]).sum())
        assert np.abs(dv[:, c] - dvo).max() <= 1e-12 * scale
        sure = np.abs(dvo) > 1e-6
        assert np.array_equal(lab[sure, c], o_svm.labels(dvo)[sure])


def test_predict_exact_kernel_values(gpu_lib):
    """One training point with coefficient 1 and bias 0: dv_t = K(f, t) itself, including
    t = f (K = 1 up to the distance rounding) and far points (exp underflow to 0)."""
    P = gpu_lib
    f = np.array([[0.5, -1.0, 2.0, 0.25]])
    Ft = np.array([[0.5, -1.0, 2.0, 0.25], [1.5, -1.0, 2.0, 0.25], [100.0, 0.0, 0.0, 0.0]])
    dv, lab = P.svm_predict(_t(f), _t(np.ones(1)), _t(np.ones(1)), 1.0, [0.0], _t(Ft))
    dv = dv.cpu().numpy()[:, 0]
    assert abs(dv[0] - 1.0) <= 1e-15
    assert abs(dv[1] - np.exp(-0.5)) <= 1e-15
    assert dv[2] == 0.0
    assert lab.cpu().numpy()[2, 0] == 1   # dv = 0 -> +1
