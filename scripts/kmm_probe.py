"""Sketch kernel alone at config-3 shapes (r = 54, s = 272 columns), na = nb = N (default 65536):
for an ncu --set full capture of kmm_kernel.
    python scripts/kmm_probe.py [N]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_04167_b200 as P  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
g = np.random.default_rng(0)
F = torch.from_numpy(g.standard_normal((N, 54)) / np.sqrt(54)).cuda()
W = torch.from_numpy(g.standard_normal((N, 272))).cuda()
for _ in range(2):
    S = P.hss_kernel_matmul(F, F, 1.0, W, same_set=True)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
S = P.hss_kernel_matmul(F, F, 1.0, W, same_set=True)
ev1.record()
torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1)
print(f"N {N}: {ms:.2f} ms, {2 * N * N * (56 + 272) / ms / 1e9:.2f} TF/s")
