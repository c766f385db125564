"""Predict-only profiling target: config-3-shaped prediction (n = 524288 training points, r = 54,
m test points), between cudaProfilerStart/Stop after one warm-up call.
    python scripts/predict_profile.py [m]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_04167_b200 as P  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
n, r = 524288, 54
g = np.random.default_rng(5)
F = torch.from_numpy(g.standard_normal((n, r)) * 0.3).cuda()
Ft = torch.from_numpy(g.standard_normal((m, r)) * 0.3).cuda()
coef = torch.from_numpy(g.standard_normal(n)).cuda()
ones = torch.ones(n, dtype=torch.float64, device="cuda")
P.svm_predict(F, ones, coef, 1.0, [0.0], Ft)
torch.cuda.synchronize()
t = time.perf_counter()
torch.cuda.profiler.start()
P.svm_predict(F, ones, coef, 1.0, [0.0], Ft)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"predict m={m} n={n}: {time.perf_counter() - t:.4f} s")
