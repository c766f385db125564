"""One rank of a torch.distributed NCCL group driving the library's own NCCL communicator
(Comm.nccl: 128-byte id from rank 0, broadcast over the group, ncclCommInitRank inside
libsvmhss).  Writes the ADMM outputs of a build/factor/train with and without the comm."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    out = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    import datagen
    import paper_2108_04167_b200 as P
    comm = P.Comm.nccl()
    info = comm.info()
    # N3: one exchange through the per-iteration path (NCCL device API when available: NVLink
    # stores into the peers' symmetric windows + LSA barrier; with one rank, the same kernel on
    # a one-rank team), and once more with the device API disabled (ncclAllGather)
    send = torch.arange(7, dtype=torch.float64, device="cuda") + 100.0 * rank
    ex_dev = comm.exchange_test(send).cpu().numpy()
    os.environ["SVMHSS_NCCL_DEVICE"] = "0"
    comm0 = P.Comm.nccl()
    info0 = comm0.info()
    ex_ag = comm0.exchange_test(send).cpu().numpy()
    comm0.free()
    del os.environ["SVMHSS_NCCL_DEVICE"]
    cfg = datagen.get_config(3)
    F, y, _, _ = datagen.generate(3, n=4096, n_test=0)
    Fd, yd = torch.from_numpy(F).cuda(), torch.from_numpy(y).cuda()
    res = {}
    for tag, c in (("comm", comm), ("none", None)):
        H = P.hss_build(Fd, cfg["h"], leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], max_rank=cfg["cap"],
                        oversample=16, omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"], comm=c)
        U = P.hss_ulv_factor(H, 1e3)
        r = P.admm_svm_train(U, yd, [1.0], 40)
        res[tag] = (r["z"].cpu().numpy(), r["obj"], r["stats"]["graph"])
        U.free()
        H.free()
    np.savez(os.path.join(out, f"nccl_r{rank}.npz"), z_comm=res["comm"][0], z_none=res["none"][0],
             obj_comm=res["comm"][1], obj_none=res["none"][1], graph=res["comm"][2],
             device_api=info["device_api"], device_api_off=info0["device_api"], ex_dev=ex_dev, ex_ag=ex_ag)
    comm.free()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
