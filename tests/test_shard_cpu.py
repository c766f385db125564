"""Host-side logic of subtree sharding on CPU (world_size 2, gloo): the allgather callback the
library calls for its host backend gathers rank-major byte slots exactly, and the
communicator constructor validates its arguments.  The device side runs in
tests/test_gpu_shard.py."""
import ctypes as ct
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2108_04167_b200 as P
    fn = P._host_allgather(None)
    res = []
    for nbytes in (1, 24, 1 << 16, 0):
        send = (np.arange(nbytes, dtype=np.int64) * 7 + 31 * (rank + 1)).astype(np.uint8)
        recv = np.full(nbytes * world, 255, dtype=np.uint8)
        rc = fn(None, send.ctypes.data if nbytes else None, recv.ctypes.data if nbytes else None, nbytes)
        res.append((rc, recv.copy()))
    # a comm built on this backend (no device needed to create it)
    c = P.Comm.host()
    ok = c.handle is not None and c.rank == rank and c.world == world
    c.free()
    q.put((rank, res, ok))
    dist.barrier()
    dist.destroy_process_group()


def test_host_allgather_callback_is_rank_major_exact():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=180) for _ in range(world)]
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    for rank, res, ok in out:
        assert ok
        for (rc, recv), nbytes in zip(res, (1, 24, 1 << 16, 0)):
            assert rc == 0
            exp = np.concatenate([(np.arange(nbytes, dtype=np.int64) * 7 + 31 * (r + 1)).astype(np.uint8)
                                  for r in range(world)]) if nbytes else np.zeros(0, np.uint8)
            assert np.array_equal(recv, exp)


def test_comm_init_validates_arguments():
    import paper_2108_04167_b200 as P
    from paper_2108_04167_b200 import _lib
    L = _lib.load()
    fn = _lib.ALLGATHER_FN(lambda *a: 0)
    h = ct.c_void_p()
    assert L.hss_comm_init_host(2, 2, fn, None, ct.byref(h)) == -1      # rank out of range
    assert L.hss_comm_init_host(0, 0, fn, None, ct.byref(h)) == -1      # no ranks
    assert L.hss_comm_init_host(2, 1, fn, None, ct.byref(h)) == 0
    L.hss_comm_free(h)
    assert P.Comm is not None
