"""The factorization's tensor-core kernels (DMMA GEMMs, QR with DMMA trailing updates, blocked
Cholesky, blocked larft, DMMA TRSM) against the generic one-CTA DFMA kernels they replace
(SVMHSS_GEMM_DFMA=1 SVMHSS_QR_TC=0 SVMHSS_POTRF_TC=0 SVMHSS_TRSM_TC=0 SVMHSS_LARFT_BLK=0): the
same K~ (ranks bit-identical), solves that agree to rounding and both satisfy
(K~ + beta I) x = b to 1e-11, and ADMM iterates / objective to the north-star 1e-7."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "_factor_paths_worker.py")
GENERIC = {"SVMHSS_GEMM_DFMA": "1", "SVMHSS_QR_TC": "0", "SVMHSS_POTRF_TC": "0", "SVMHSS_TRSM_TC": "0",
           "SVMHSS_LARFT_BLK": "0"}


def _run(tmp_path, tag, n, extra):
    out = str(tmp_path / f"{tag}.npz")
    env = dict(os.environ)
    for k in GENERIC:
        env.pop(k, None)
    env.update(extra)
    r = subprocess.run([sys.executable, WORKER, out, str(n)], env=env, capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    return dict(np.load(out))


@pytest.mark.parametrize("n", [5000, 20000])
def test_tensor_core_factor_matches_generic(tmp_path, n):
    a = _run(tmp_path, "tc", n, {})
    b = _run(tmp_path, "generic", n, GENERIC)
    assert np.array_equal(a["ranks"], b["ranks"])
    assert a["res"] <= 1e-11 and b["res"] <= 1e-11
    assert np.linalg.norm(a["x"] - b["x"]) <= 1e-11 * np.linalg.norm(b["x"])
    assert np.linalg.norm(a["z"] - b["z"]) <= 1e-7 * max(1.0, np.linalg.norm(b["z"]))
    assert abs(float(a["obj"][0]) - float(b["obj"][0])) <= 1e-7 * abs(float(b["obj"][0]))
