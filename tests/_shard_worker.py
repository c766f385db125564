"""Worker for the subtree-sharding tests (tests/test_gpu_shard.py): one rank of P, launched by
torchrun, exchanging through a gloo group with the library's host-callback backend
(Comm.host) — P ranks may share one GPU because no kernel ever waits on another rank.
Runs build + factor + solve + mat-vec + ADMM (+ bias/objective) through the C-ABI and
writes this rank's outputs to <out>/P<world>_r<rank>.npz.

    torchrun --nproc-per-node P tests/_shard_worker.py OUTDIR CFG N [CAP] [BETA] [MAXIT] [sketch|ann]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    out, cfg_id, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    cap = int(sys.argv[4]) if len(sys.argv) > 4 else None
    beta = float(sys.argv[5]) if len(sys.argv) > 5 else 1e4
    max_it = int(sys.argv[6]) if len(sys.argv) > 6 else 60
    sampling = sys.argv[7] if len(sys.argv) > 7 else "sketch"
    interp = sys.argv[8] if len(sys.argv) > 8 else "id"       # N4: "spd"
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    import datagen
    import paper_2108_04167_b200 as P
    torch.cuda.set_device(0)
    comm = None
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        comm = P.Comm.host()
    cfg = datagen.get_config(cfg_id)
    if cap is not None:
        cfg["cap"], cfg["s"] = cap, cap + 16
    F, y, _, _ = datagen.generate(cfg_id, n=n, n_test=0)
    Ft = datagen.generate(cfg_id, n=n, n_test=301)[2]   # test points of a separate draw
    dev = torch.device("cuda:0")
    Fd, yd = torch.from_numpy(F).to(dev), torch.from_numpy(y).to(dev)
    h = cfg["h"][2] if isinstance(cfg["h"], list) else cfg["h"]
    H = P.hss_build(Fd, h, leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"],
                    max_rank=cfg["cap"], oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"],
                    tree_seed=cfg["seed_tree"], comm=comm, sampling=sampling,
                    ann_neighbors=cfg["ann_neighbors"], ann_trees=cfg["ann_trees"], ann_leaf=cfg["ann_leaf"],
                    ann_seed=cfg["ann_seed"], interp=interp)
    U = P.hss_ulv_factor(H, beta)
    g = np.random.default_rng(7)
    b = torch.from_numpy(g.standard_normal((n, 2))).to(dev)
    x = U.solve(b)
    kv = H.matvec(b)
    Cs = [0.5, 1.0, 10.0]
    res = P.admm_svm_train(U, yd, Cs, max_it, trace_every=20)
    hi = H.info()
    # a11 with the test points sharded over the ranks (svm_predict's comm)
    dv, lab = P.svm_predict(Fd, yd, res["z"], h, res["bias"], torch.from_numpy(Ft).to(dev), comm=comm)
    # the end-to-end host call (the bench's e2e path) with the same communicator
    e2e = P.svm_train_predict_host(F, y, h, beta, Cs, max_it, Ftest=Ft, leaf_size=cfg["leaf"],
                                   rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"], max_rank=cfg["cap"],
                                   oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"],
                                   tree_seed=cfg["seed_tree"], comm=comm, sampling=sampling, interp=interp,
                                   ann_neighbors=cfg["ann_neighbors"], ann_trees=cfg["ann_trees"],
                                   ann_leaf=cfg["ann_leaf"], ann_seed=cfg["ann_seed"])
    np.savez(os.path.join(out, f"P{world}_r{rank}.npz"), x=x.cpu().numpy(), kv=kv.cpu().numpy(),
             e2e_z=e2e["z"], e2e_bias=e2e["bias"], e2e_lab=e2e["labels"],
             dv=dv.cpu().numpy(), lab=lab.cpu().numpy(),
             z=res["z"].cpu().numpy(), mu=res["mu"].cpu().numpy(), bias=res["bias"], obj=res["obj"],
             trace_z=res["trace_z"].cpu().numpy(), w1=res["stats"]["w1"], perm=hi["perm"],
             cap_hits=hi["cap_hits"], passthrough=hi["passthrough"], max_rank=hi["max_rank_used"],
             gen_bytes=hi["generator_bytes"], graph=res["stats"]["graph"])
    U.free()
    H.free()
    if comm is not None:
        comm.free()
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
