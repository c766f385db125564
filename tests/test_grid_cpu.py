"""Multi-process (world_size 2, gloo, CPU) test of the h-sharded grid driver: every h is
trained exactly once across ranks, with the cached factorization reused for all C (one
train call per h), and rank 0 gathers every (h, C) record.  The GPU training step is replaced
by a stub so the host logic runs here."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stub_train(F, y, Ft, yt, h, C_list, beta, max_it, opts):
    return [dict(h=h, C=C, beta=beta, accuracy=50.0, calls=1, pid=os.getpid()) for C in C_list]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import datagen
    from paper_2108_04167_b200.grid import run_grid, shard_h
    cfg = datagen.get_config(4)
    out = run_grid(None, None, None, None, cfg, rank=rank, world=world, train_fn=_stub_train)
    q.put((rank, shard_h(cfg["h"], rank, world), out))
    dist.barrier()
    dist.destroy_process_group()


def test_grid_sharded_over_two_ranks_gathers_everything():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (mine, out)) for r, mine, out in [q.get(timeout=120) for _ in range(2)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import datagen
    cfg = datagen.get_config(4)
    assert sorted(res[0][0] + res[1][0]) == sorted(cfg["h"])       # disjoint cover of h
    assert not set(res[0][0]) & set(res[1][0])
    out = res[0][1]
    assert res[1][1] is None
    assert len(out) == len(cfg["h"]) * len(cfg["C"])
    assert {(r["h"], r["C"]) for r in out} == {(h, C) for h in cfg["h"] for C in cfg["C"]}
    for r in out:
        assert r["beta"] == cfg["beta_per_h"][r["h"]]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_h_partition(world):
    from paper_2108_04167_b200.grid import shard_h
    hs = [0.25, 0.5, 1.0, 2.0, 4.0]
    parts = [shard_h(hs, r, world) for r in range(world)]
    assert sorted(sum(parts, [])) == sorted(hs)
