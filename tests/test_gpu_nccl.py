"""The library's NCCL communicator on the GPU box: Comm.nccl() over a torch.distributed NCCL group
(one rank per GPU available here, two when there are two), a build/factor/train through it equals
the run without a comm, and the ADMM loop is still captured as a CUDA graph (NCCL is
graph-capturable).  The in-kernel exchange through the NCCL device API (N3) runs on hardware:
with one GPU on a one-rank LSA team (self stores + LSA barrier), with more on NVLink peers."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_nccl_comm_single_rank(tmp_path):
    import torch
    n = max(1, torch.cuda.device_count())
    world = 1 if n < 2 else 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "_nccl_worker.py"), str(tmp_path)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    ref = None
    for k in range(world):
        d = np.load(os.path.join(tmp_path, f"nccl_r{k}.npz"))
        assert np.array_equal(d["z_comm"], d["z_none"]) and np.array_equal(d["obj_comm"], d["obj_none"])
        assert int(d["graph"]) == 1
        expect = np.concatenate([np.arange(7) + 100.0 * q for q in range(world)])
        assert np.array_equal(d["ex_ag"], expect) and int(d["device_api_off"]) == 0
        # NCCL 2.28 device API: in use on this NCCL, and the in-kernel exchange
        # gives the allgather's result
        assert int(d["device_api"]) == 1
        assert np.array_equal(d["ex_dev"], expect)
        if ref is None:
            ref = d["z_comm"]
        assert np.array_equal(d["z_comm"], ref)
