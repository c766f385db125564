"""Hyper-parameter grid with the factorization cache (Alg. 3 P:205-233,
P:194 "computed just once for fixed h ... reused for all the values C in the grid search").

For each kernel width h: ONE hss_build + ONE hss_ulv_factor, then all C values advance
together as the nC right-hand sides of one ULV solve per ADMM iteration (admm_svm_train with
nC > 1), then one prediction per C.  Multi-GPU: the h values are independent problems, so they
are sharded across ranks (round robin) with no data-path collective; only the small result
records are gathered to rank 0 (torch.distributed object gather, NCCL or gloo).
"""
from __future__ import annotations

import time


def shard_h(h_list, rank: int, world: int):
    """Round-robin assignment of the h values to ranks (deterministic)."""
    return [h for i, h in enumerate(h_list) if i % world == rank]


def train_h(F, y, Ft, yt, h, C_list, beta, max_it, opts, device="cuda"):
    """One h: build + factor once, ADMM for every C (batched), predict per C.  Returns a list
    of records (one per C) with accuracy and phase times (CUDA events inside the library)."""
    import numpy as np
    import torch

    from . import admm_svm_train, hss_build, hss_ulv_factor, svm_predict
    Fd = torch.from_numpy(np.ascontiguousarray(F)).to(device)
    yd = torch.from_numpy(np.ascontiguousarray(y)).to(device)
    Ftd = torch.from_numpy(np.ascontiguousarray(Ft)).to(device)
    t0 = time.perf_counter()
    H = hss_build(Fd, h, **opts)
    U = hss_ulv_factor(H, beta)
    res = admm_svm_train(U, yd, C_list, max_it, want_mu=False)
    dv, lab = svm_predict(Fd, yd, res["z"], h, res["bias"], Ftd)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    hi, ui = H.info(), U.info()
    lab = lab.cpu().numpy()
    out = []
    for c, C in enumerate(C_list):
        acc = float((lab[:, c] == yt.astype(np.int8)).mean() * 100.0)
        out.append(dict(h=h, C=C, beta=beta, accuracy=acc, bias=float(res["bias"][c]),
                        objective=float(res["obj"][c]),
                        compress_ms=hi["ms_tree"] + hi["ms_omega"] + hi["ms_sketch"] + hi["ms_compress"],
                        factor_ms=ui["ms_factor"], admm_ms=res["stats"]["ms_loop"] / len(C_list),
                        memory_mb=hi["generator_bytes"] / 2 ** 20, max_rank=hi["max_rank_used"],
                        wall_s=wall))
    U.free()
    H.free()
    return out


def run_grid(F, y, Ft, yt, cfg, rank=0, world=1, train_fn=None, group=None):
    """Run the config-4 grid on this rank's share of h; gather all records on rank 0 (others
    get None).  `train_fn` defaults to train_h (tests inject a CPU stub)."""
    import torch.distributed as dist
    train_fn = train_fn or train_h
    h_list = cfg["h"] if isinstance(cfg["h"], list) else [cfg["h"]]
    betas = cfg.get("beta_per_h", {})
    opts = dict(leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"], max_rank=cfg["cap"],
                oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"])
    mine = []
    for h in shard_h(h_list, rank, world):
        mine.extend(train_fn(F, y, Ft, yt, h, list(cfg["C"]), betas.get(h, cfg["beta"]), cfg["max_it"], opts))
    if world == 1:
        return sorted(mine, key=lambda r: (r["h"], r["C"]))
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(mine, gathered, dst=0, group=group)
    if rank != 0:
        return None
    flat = [r for part in gathered for r in part]
    return sorted(flat, key=lambda r: (r["h"], r["C"]))
