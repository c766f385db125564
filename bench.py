#!/usr/bin/env python
"""bench.py — ADMM + HSS SVM hot path on B200 (BASELINE.json metric: "ADMM iters/sec and HSS
build+ULV time at n=524k; fraction of HBM/FP64 peak").

One STEP = one pass of the whole hot path over config 3
(n = 524,288 train / 131,072 test points, r = 54): tree + Omega + fused DMMA sketch + per-level
ID compression (hss_build), ULV factorization (hss_ulv_factor), precompute + MaxIt = 1000 ADMM
iterations + bias/objective (admm_svm_train), prediction of the test set (svm_predict).
Inputs are resident in HBM before the timed region; the factor (GBs) exceeds L2 (126 MB).

value       = ADMM iterations per second (whole job: sum over ranks), timed with CUDA events
              on the launching stream inside the library, max over ranks;
hss_build_ulv_s = build + factor seconds per step (the metric's second number);
e2e         = the same metric through the HOST-buffer C-ABI call svm_train_predict_host,
              host<->device copies inside the timed region (iterations / call seconds);
roofline    = dominant kernel (the sketch kmm_kernel, FP64 tensor cores);
roofline_solve = the per-iteration ULV solve sweeps (HBM);
cpu_baseline = the CPU oracle on a bounded sample (rank 0, N = 1 only).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cuda|reference] [--config 3]
Multi-GPU (torchrun, one process per GPU): subtree sharding (DESIGN.md
"Multi-GPU"): rank g owns tree node g at level log2(N); one NCCL allgather per build / factor
phase and one per ADMM iteration (inside the CUDA graph); scaling "strong" (the n-point problem
is fixed); test points split across ranks.  Config 4: h sharded across ranks (independent).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "ADMM iters/sec and HSS build+ULV time at n=524k; fraction of HBM/FP64 peak"
FP64_NOMINAL_TF, BF16_NOMINAL_TF = 45.0, 2250.0  # blackwell_cuda_programming.md (B200 FP64 tensor 45)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region (B200_PROFILING.md)."""

    def __init__(self, index=0):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 8]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        load = [x for x in sm if x > 0.5 * (max(mx) if mx else 1)]
        return {"sm_mhz": float(np.median(load if load else sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def _traffic(kernel, workload):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the committed ncu
    capture (profiles/traffic.json), if it was taken on this workload; else None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p)).get(kernel)
    if not d or d.get("workload") != workload:
        return None
    if d.get("dram_bytes") is not None:
        return d["dram_bytes"]
    return d["dram_bytes_read"] + d["dram_bytes_write"]


def measure_dgemm(dev, N=8192, reps=5):
    """cuBLAS fp64 GEMM (torch.matmul) TFLOP/s on this GPU, best of `reps` (the FP64 peak the
    DMMA sketch kernel is compared with; MEASURED_PEAKS.json has no FP64 figure)."""
    import torch
    a = torch.randn(N, N, dtype=torch.float64, device=dev)
    b = torch.randn(N, N, dtype=torch.float64, device=dev)
    c = torch.empty_like(a)
    torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    del a, b, c
    torch.cuda.empty_cache()
    return 2.0 * N ** 3 / best / 1e12


def cfg_opts(cfg, sampling="sketch", interp="id"):
    o = dict(leaf_size=cfg["leaf"], rel_tol=cfg["rel_tol"], abs_tol=cfg["abs_tol"], max_rank=cfg["cap"],
             oversample=cfg["s"] - cfg["cap"], omega_seed=cfg["seed_omega"], tree_seed=cfg["seed_tree"])
    if interp == "spd":
        o.update(interp="spd", spd_eps=SPD_EPS)
    if sampling == "ann":
        o.update(sampling="ann", ann_neighbors=cfg["ann_neighbors"], ann_trees=cfg["ann_trees"],
                 ann_leaf=cfg["ann_leaf"], ann_seed=cfg["ann_seed"])
    return o


SPD_EPS = 1e-12  # N4 jitter on K(J,J) (relative to K_ii = 1)


def node_shapes(ranks, n, leaf):
    """(level, R_t, k_t) of every non-root node from the exported ranks (level-major BFS) and the
    uniform T1 split: R = leaf size at the leaves, the children's k above."""
    L = 0
    while leaf * (1 << L) < n:
        L += 1
    sizes = [n]
    for _ in range(L):
        sizes = [x for v in sizes for x in (v // 2, v - v // 2)]
    k = {}
    out = []
    for lvl in range(L, 0, -1):
        for i in range(1 << lvl):
            t = (1 << lvl) - 1 + i
            R = sizes[i] if lvl == L else k[2 * t + 1] + k[2 * t + 2]
            k[t] = int(ranks[t])
            out.append((lvl, R, k[t]))
    root_R = k[1] + k[2] if L > 0 else n
    return out, root_R


def solve_algorithmic_bytes(shapes, root_R, n, nC):
    """one ULV solve reads each compressing node's compact factor twice (forward and
    backward): V (R k - k(k-1)/2, unit-diagonal Householder vectors), T (k(k+1)/2), L_r
    ((R-k)(R-k+1)/2), L_sr (k (R-k)); the root's Cholesky triangle R0(R0+1)/2; plus 8 n-vectors of
    nC columns (rhs, solution, y, w, z, mu and the epilogue's q / next rhs)."""
    per = 0
    for _, R, k in shapes:
        if k >= R:
            continue  # pass-through: no transform
        e = R - k
        per += R * k - k * (k - 1) // 2 + k * (k + 1) // 2 + e * (e + 1) // 2 + k * e
    per += root_R * (root_R + 1) // 2
    return 2.0 * 8.0 * per + 64.0 * n * nC


def compress_work(shapes, s):
    """per CPQR'd node 4 s R k + 4 k^2 s flops (pivoted Householder on the s x R
    sample block, R11^-1 R12, Omega' = U^T Omega^); algorithmic bytes: the node's sample block read
    and written once (16 R s)."""
    fl = sum(4.0 * s * R * k + 4.0 * k * k * s for _, R, k in shapes)
    by = sum(16.0 * R * s for _, R, k in shapes)
    return fl, by


def host_info():
    """CPU model, host DGEMM GFLOP/s (numpy 2048^3) and a STREAM-like copy GB/s (256 MB) on the
    cores the oracle uses: the denominators of the CPU baseline."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    a = np.random.default_rng(0).standard_normal((2048, 2048))
    a @ a
    t = time.perf_counter()
    for _ in range(3):
        a @ a
    gf = 3 * 2.0 * 2048 ** 3 / (time.perf_counter() - t) / 1e9
    x = np.ones(1 << 25)
    y = np.empty_like(x)
    np.copyto(y, x)
    t = time.perf_counter()
    for _ in range(5):
        np.copyto(y, x)
    gbs = 5 * 2.0 * x.nbytes / (time.perf_counter() - t) / 1e9
    return {"cpu_model": model, "cores": len(os.sched_getaffinity(0)), "host_dgemm_gflops": gf,
            "host_copy_gbs": gbs}


def oracle_offline(cfg_id):
    """The oracle's MEASURED full-size phase times, from the committed golden run
    (scripts/make_fullsize_goldens.py: oracle only, on the dev container's host)."""
    p = os.path.join(ROOT, "tests", "golden", f"cfg{cfg_id}_full.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    t = d.get("oracle_timings_s", {})
    return {"n": d["n"], "host": d.get("host"), "tree_s": t.get("tree"), "sketch_s": t.get("sketch"),
            "compress_after_sketch_s": t.get("compress_after_sketch"), "factor_s": t.get("factor"),
            "admm_per_iter_s": t.get("admm_per_iter"), "admm_iters_per_s": 1.0 / t["admm_per_iter"]
            if t.get("admm_per_iter") else None, "bias_objective_s": t.get("bias_objective"),
            "predict_1024_s": t.get("predict_1024"),
            "note": "measured at the full config size by the oracle-only golden script (not on this box)"}


def oracle_phases(cfg_id, n_sample, iters, sketch_rows=512):
    """The oracle (as it stands) timed per phase on this box's cores, on bounded samples of the
    config: HSS build + ULV of an n_sample-point draw (same knobs) and `iters` ADMM iterations on it
    (an iteration is linear in n at fixed node shapes: projected by n / n_sample), and `sketch_rows`
    full-length rows of the sketch S = K Omega (projected by n / sketch_rows).  Every projected
    number is labelled as such."""
    import datagen
    from threadpoolctl import threadpool_limits

    from oracle import admm, hss, kernel, pipeline, rng, svm, ulv
    cfg = datagen.get_config(cfg_id)
    n = cfg["n"]
    n_sample = min(n_sample, n)   # config 0 (n = 2000): the whole config, nothing projected
    F, y, Ft, _ = datagen.generate(cfg_id, n=n_sample, n_test=256)
    tm = {}
    # per-node phases (small LAPACK/BLAS calls in Python loops) run with one BLAS thread: the
    # multithreaded BLAS is 10-20x SLOWER on these shapes (measured); the sketch uses every core
    # through its row-chunk thread pool
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        perm, ranges, Om, H = pipeline.build(F, cfg, timings=tm)
        t1 = time.perf_counter()
        fac = ulv.factor(H, cfg["beta"])
        t2 = time.perf_counter()
        yp = y[perm]
        solve = lambda b: ulv.solve(fac, b)  # noqa: E731
        t3 = time.perf_counter()
        out = admm.run(solve, yp, cfg["C"][0], cfg["beta"], iters)
        t4 = time.perf_counter()
        mv = lambda v: hss.matvec(H, v)  # noqa: E731
        b = svm.bias(mv, out["z"], yp, cfg["C"][0])
        t5 = time.perf_counter()
    # sketch rows at the full size (the dominant phase): rows of K(F, F) Omega over all n points
    Ff, _, _, _ = datagen.generate(cfg_id)
    idx = np.arange(sketch_rows)
    Omf = rng.omega(cfg["seed_omega"], np.arange(n), cfg["s"])
    t6 = time.perf_counter()
    kernel.sketch_rows(Ff, cfg["h"], Omf, idx)
    t7 = time.perf_counter()
    del Ff, Omf
    inv = np.empty_like(perm)
    inv[perm] = np.arange(n_sample)
    t8 = time.perf_counter()
    svm.decision_values(F, y * out["z"][inv], cfg["h"], b, Ft)
    t9 = time.perf_counter()
    per_it = (t4 - t3) / iters
    sc = n / n_sample
    return {
        "admm_iters_per_s_projected": 1.0 / (per_it * sc),
        "phases_s_projected": {
            "sketch": (t7 - t6) * n / sketch_rows,
            "compress_excl_sketch": (t1 - t0 - tm.get("tree", 0.0)) * sc,
            "factor": (t2 - t1) * sc,
            "admm_per_iter": per_it * sc,
            "bias_objective": (t5 - t4) * sc,
            "predict_per_test_point": (t9 - t8) / Ft.shape[0] * sc},
        "threads": {"sketch_rows": "numpy default BLAS threads", "per_node_phases": 1},
        "sample": (f"oracle (NumPy/SciPy fp64): HSS build + ULV + {iters} ADMM iterations + bias on an "
                   f"n={n_sample} config-{cfg_id} draw (same leaf/cap/s/tol/seeds; times x n/n_sample = "
                   f"{sc:.1f}: per-node shapes equal the full config's), {sketch_rows} full-length sketch "
                   f"rows (x n/{sketch_rows}), 256 test points; all PROJECTED to n={n}")}


# ----------------------------------------------------------------------------- reference arm
def oracle_sample(cfg_id, n_sample, iters, steps=1, warmup=0):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload: build + factor
    once, then `steps` timed blocks of `iters` ADMM iterations.  Returns a dict in the
    metric's unit: ADMM iters/s scaled to the full n (one iteration is O(n): per-node work
    over n / leaf nodes)."""
    import datagen
    from threadpoolctl import threadpool_limits

    from oracle import admm, pipeline, ulv
    cfg = datagen.get_config(cfg_id)
    n_sample = min(n_sample, cfg["n"])
    F, y, _, _ = datagen.generate(cfg_id, n=n_sample, n_test=0)
    with threadpool_limits(limits=1):   # per-node phases: one BLAS thread (see oracle_phases)
        t0 = time.perf_counter()
        perm, ranges, Om, H = pipeline.build(F, cfg)
        fac = ulv.factor(H, cfg["beta"])
        t_build = time.perf_counter() - t0
        yp = y[perm]
        solve = lambda b: ulv.solve(fac, b)  # noqa: E731
        for _ in range(warmup):
            admm.run(solve, yp, cfg["C"][0], cfg["beta"], iters)
        times = []
        for _ in range(max(1, steps)):
            t = time.perf_counter()
            admm.run(solve, yp, cfg["C"][0], cfg["beta"], iters)
            times.append(time.perf_counter() - t)
    per_it = float(np.median(times)) / iters
    scale = n_sample / cfg["n"]
    return dict(value=scale / per_it, unit="iters/s", build_ulv_s_sample=t_build, per_iter_s_sample=per_it,
                times=times, cores=len(os.sched_getaffinity(0)),
                sample=f"oracle (NumPy/SciPy fp64) HSS build+ULV on n={n_sample} config-{cfg_id} points "
                       f"(same leaf/cap/s/tol/seeds), then {iters} ADMM iterations per step; iters/s "
                       f"scaled by n_sample/n = {scale:.5f} (ADMM iteration cost is linear in n)")


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import datagen
    cfg = datagen.get_config(args.config)
    r = oracle_sample(args.config, args.ref_n, args.ref_iters, steps=args.steps, warmup=args.warmup)
    hinfo = host_info()
    line = {"metric": METRIC, "value": r["value"], "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * float(np.median(r["times"])),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg["name"], "n": cfg["n"], "r": cfg["r"], "max_it": cfg["max_it"],
                       "leaf": cfg["leaf"], "cap": cfg["cap"], "s": cfg["s"], "sample_n": args.ref_n},
            "cpu_baseline": {"value": r["value"], "unit": "iters/s", "cores": r["cores"], "kind": "oracle",
                             "sample": r["sample"], "projected": True, **hinfo,
                             "offline_full_size": oracle_offline(args.config)},
            "e2e": {"value": r["value"], "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "hss_build_ulv_s_sample": r["build_ulv_s_sample"]}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- config 4 grid
def bench_grid(args, rank, world, dev):
    """Config 4: the (h, C) grid, h sharded across ranks (independent problems, no data-path
    collective), one build + factor per h reused for all 6 C (batched right-hand sides)."""
    import torch
    import torch.distributed as dist

    import datagen
    from paper_2108_04167_b200.grid import run_grid, shard_h
    cfg = datagen.get_config(4)
    if args.max_it:
        cfg["max_it"] = args.max_it
    F, y, Ft, yt = datagen.generate(4, n=args.n, n_test=None if args.n is None else max(1, args.n // 4))
    for _ in range(args.warmup):
        run_grid(F, y, Ft, yt, cfg, rank, world)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        out = run_grid(F, y, Ft, yt, cfg, rank, world)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    if rank == 0:
        iters = len(cfg["h"]) * len(cfg["C"]) * cfg["max_it"]
        best = max(out, key=lambda r: r["accuracy"])
        line = {"metric": METRIC, "value": iters / (ms / 1e3), "unit": "iters/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": cfg["name"], "n": F.shape[0], "h": cfg["h"], "C": cfg["C"],
                           "max_it": cfg["max_it"], "parallelism": f"h-sharded over {world}",
                           "h_per_rank": [shard_h(cfg["h"], r, world) for r in range(world)]},
                "grid_sweep_s": ms / 1e3, "best": best,
                "grid": [{k: r[k] for k in ("h", "C", "accuracy", "compress_ms", "factor_ms", "admm_ms")}
                         for r in out]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- CUDA arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=None, help="debug: override n (not a bench line)")
    ap.add_argument("--max-it", type=int, default=None, help="debug: override MaxIt")
    ap.add_argument("--beta", type=float, default=None, help="debug: override beta (not a bench line)")
    ap.add_argument("--ref-n", type=int, default=8192)
    ap.add_argument("--ref-iters", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-predict", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the HSS-ANN variant sub-line")
    ap.add_argument("--interp", default="id", choices=["id", "spd"],
                    help="interpolation of the compression: the paper's ID (default) or the SPD-preserving "
                         "kernel interpolant (SURVEY 8(f) N4; beta = the paper's schedule)")
    ap.add_argument("--sampling", default="sketch", choices=["sketch", "ann"],
                    help="compression sampling: the randomized sketch (north star, default) or HSS-ANN "
                         "column sampling (SURVEY 8(f) N1)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    # the library's memory pool stays reserved between steps (a process that rebuilds repeatedly;
    # the default trims it when the last handle is freed, and each build then re-maps ~30 GB)
    os.environ.setdefault("SVMHSS_POOL_KEEP", "1")
    import torch
    import torch.distributed as dist

    import datagen
    import paper_2108_04167_b200 as P

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # NCCL's communicator-init lines (rank count, transports, NVLS) on stderr, init only, so the
        # driver can see N ranks; the JSON line stays the only stdout line of rank 0
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=dev)
    if args.config == 4:
        return bench_grid(args, rank, world, dev)
    cfg = datagen.get_config(args.config)
    if args.sampling == "ann":
        cfg["beta"] = cfg["beta_ann"]  # AMB-9 calibrated on the ANN K~ (datagen/configs.py)
    if args.interp == "spd":
        cfg["beta"] = datagen.configs.beta_schedule(args.n or cfg["n"])  # N4: K~ PSD, no calibration
    if args.beta is not None:
        cfg["beta"] = args.beta
    n = args.n or cfg["n"]
    nt = cfg["n_test"] if args.n is None else max(1, n // 4)
    max_it = args.max_it or cfg["max_it"]
    h = cfg["h"] if not isinstance(cfg["h"], list) else cfg["h"][2]
    Cs = cfg["C"][:1]
    F, y, Ft, yt = datagen.generate(args.config, n=n, n_test=nt)
    # N > 1: subtree sharding over the library's NCCL communicator; every rank
    # holds all n training points (the tree's top levels are replicated), the test points are
    # split across ranks for prediction (independent, no collective)
    comm = P.Comm.nccl() if world > 1 else None
    t0, t1 = rank * nt // world, (rank + 1) * nt // world
    Fd, yd, Ftd = (torch.from_numpy(a).to(dev) for a in (F, y, np.ascontiguousarray(Ft[t0:t1])))
    stream = torch.cuda.current_stream()
    opts = cfg_opts(cfg, args.sampling, args.interp)
    opts["comm"] = comm

    def step():
        H = P.hss_build(Fd, h, **opts)
        U = P.hss_ulv_factor(H, cfg["beta"])
        res = P.admm_svm_train(U, yd, Cs, max_it, want_mu=False)
        st = dict(res["stats"])
        st["ms_predict"] = None
        if not args.no_predict and Ftd.shape[0] > 0:
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record(stream)
            _, lab = P.svm_predict(Fd, yd, res["z"], h, res["bias"], Ftd)
            p1.record(stream)
            p1.synchronize()
            st["ms_predict"] = p0.elapsed_time(p1)
            st["labels"] = lab
        hi, ui = H.info(), U.info()
        U.free()
        H.free()
        return hi, ui, st

    dgemm_tf = measure_dgemm(dev)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = ClockSampler(local)
    clk.start()
    l0 = P.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    recs = [step() for _ in range(args.steps)]
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = P.launch_count() - l0
    clocks = clk.stop()
    if world > 1:
        dist.barrier()
    ms_total = ev0.elapsed_time(ev1)
    loop_ms = float(np.median([a["ms_loop"] for _, _, a in recs]))
    build_ms = float(np.median([hi["ms_tree"] + hi["ms_omega"] + hi["ms_sketch"] + hi["ms_compress"] + ui["ms_factor"]
                                for hi, ui, _ in recs]))
    sketch_ms = float(np.median([hi["ms_sketch"] for hi, _, _ in recs]))
    t = torch.tensor([ms_total, loop_ms, build_ms, sketch_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total, loop_ms, build_ms, sketch_ms = t.tolist()
    hi, ui, ast = (dict(d) for d in recs[-1])
    # test accuracy of the last step's labels against the synthetic test labels (after the timed
    # region; each rank holds its share of the test points)
    acc = None
    if "labels" in ast:
        lab = ast.pop("labels")
        hit = torch.tensor([float((lab[:, 0].cpu().numpy() == yt[t0:t1]).sum()), float(t1 - t0)],
                           dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(hit)
        acc = hit[0].item() / max(1.0, hit[1].item())
    # phase times: per-phase medians over the timed steps (one step can hit a memory-pool growth)
    for j, d in enumerate((hi, ui, ast)):
        for k in list(d):
            if k.startswith("ms_") and all(r[j].get(k) is not None for r in recs):
                d[k] = float(np.median([r[j][k] for r in recs]))
    value = max_it * len(Cs) / (loop_ms / 1e3)  # iterations of the whole (sharded) problem
    peaks, peak_src = _peaks()
    rp = (cfg["r"] + 3) // 4 * 4
    sk_flops = 2.0 * n * n * (rp + cfg["s"]) / world  # this rank's rows of the sketch (n / world)
    fp64_derived = peaks["bf16_tflops_sustained"] * FP64_NOMINAL_TF / BF16_NOMINAL_TF
    fp64_peak = max(dgemm_tf, fp64_derived)
    ach_tf = sk_flops / (sketch_ms / 1e3) / 1e12
    shapes, root_R = node_shapes(hi["ranks"], n, cfg["leaf"])
    solve_alg = solve_algorithmic_bytes(shapes, root_R, n, len(Cs))
    solve_expl = 2.0 * ui["factor_bytes"] + 64.0 * n * len(Cs)
    ach_gbs = solve_alg * max_it / (loop_ms / 1e3) / 1e9
    cf_flops, cf_bytes = compress_work(shapes, cfg["s"])
    tree_bytes = 3.0 * hi["L"] * 8.0 * n * cfg["r"]
    # the committed captures are of the dense-sketch build (scripts/admm_profile.py sketch)
    solve_traffic = _traffic("admm_iteration", cfg["name"]) if args.n is None and args.sampling == "sketch" else None
    line = {"metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"] + ("" if args.sampling == "sketch" else "+ann")
                       + ("" if args.interp == "id" else "+spd"),
                       "sampling": args.sampling, "interp": args.interp, "n": n, "n_test": nt, "r": cfg["r"], "h": h, "C": Cs,
                       "beta": cfg["beta"], "max_it": max_it, "leaf": cfg["leaf"], "cap": cfg["cap"],
                       "s": cfg["s"], "rel_tol": cfg["rel_tol"],
                       "parallelism": (f"subtree-sharded over {world}: per-iteration exchange "
                                       + ("in-kernel via the NCCL device API (N3)" if comm is not None and comm.info()["device_api"]
                                          else "ncclAllGather in the iteration graph"))
                       if world > 1 else "1 GPU",
                       "pool": "library memory pool kept between steps (SVMHSS_POOL_KEEP=%s)" % os.environ.get("SVMHSS_POOL_KEEP"),
                       "l2": "inputs larger than L2 (factor %.2f GB, sketch operands %.2f GB)" % (
                           ui["factor_bytes"] / 1e9, 16.0 * n * cfg["s"] / 1e9)},
            "hss_build_ulv_s": build_ms / 1e3,
            "test_accuracy": acc,
            "phases_ms": {"tree": hi["ms_tree"], "omega": hi["ms_omega"], "sketch": hi["ms_sketch"],
                          "compress": hi["ms_compress"], "factor": ui["ms_factor"],
                          "admm_precompute": ast["ms_precompute"], "admm_loop": ast["ms_loop"],
                          "bias": ast["ms_bias"], "predict": ast["ms_predict"]},
            "hss": {"L": hi["L"], "max_rank": hi["max_rank_used"], "cap_hits": hi["cap_hits"],
                    "passthrough": hi["passthrough"], "generator_bytes": hi["generator_bytes"],
                    "factor_bytes": ui["factor_bytes"]},
            "gpu_launches": int(launches),
            "launches_per_admm_iter": int(ast["kernel_launches_per_iter"]),
            "roofline": {"bound": "tensor", "kernel": "kmm_kernel (sketch S = K Omega, DMMA)",
                         "achieved": ach_tf, "peak": fp64_peak, "unit": "TFLOP/s", "frac": ach_tf / fp64_peak,
                         "traffic": _traffic("kmm_kernel", cfg["name"]) if args.n is None else None,
                         "traffic_unit": "bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                                         "profiles/traffic.json)",
                         "peak_source": "max(cuBLAS fp64 DGEMM 8192^3 measured in this run = %.2f, %s bf16_tflops_sustained x FP64/BF16 nominal %g/%g = %.2f)" % (
                             dgemm_tf, peak_src, FP64_NOMINAL_TF, BF16_NOMINAL_TF, fp64_derived),
                         "work": "2 (n / n_gpus) n (r_pad + s) flops per launch (this rank's rows)"},
            "roofline_solve": {"bound": "hbm", "kernel": "ulv_fwd_kernel + ulv_bwd_kernel (+ epilogue)",
                               "achieved": ach_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                               "frac": ach_gbs / peaks["hbm_gbs"],
                               "algorithmic_bytes_per_iter": solve_alg,
                               "explicit_operator_bytes_per_iter": solve_expl,
                               "explicit_over_algorithmic": solve_expl / solve_alg,
                               "dram_bytes_per_iter_ncu": solve_traffic,
                               "work": "SURVEY 8(d) a9 algorithmic bytes: 2 x sum over compressing nodes 8[Rk - "
                                       "k(k-1)/2 + k(k+1)/2 + (R-k)(R-k+1)/2 + k(R-k)] + 2 x 8 R0(R0+1)/2 (root) "
                                       "+ 64 n nC per iteration; the library streams explicit R x R operators "
                                       "(explicit_operator_bytes_per_iter), ncu DRAM bytes beside it"},
            "roofline_compress": {"bound": "fp64 (CPQR: FP64 ALU) / hbm",
                                  "phase": "per-level ID (a6): blocked CPQR + R11^-1 R12 + U^T Omega + B + sibling update",
                                  "achieved": cf_flops / (hi["ms_compress"] / 1e3) / 1e12, "peak": fp64_peak,
                                  "unit": "TFLOP/s",
                                  "frac": cf_flops / (hi["ms_compress"] / 1e3) / 1e12 / fp64_peak,
                                  "hbm_achieved_gbs": cf_bytes / (hi["ms_compress"] / 1e3) / 1e9,
                                  "hbm_frac": cf_bytes / (hi["ms_compress"] / 1e3) / 1e9 / peaks["hbm_gbs"],
                                  "cpqr_dram_bytes_ncu": _traffic("cpqr_level_sum", cfg["name"]) if args.n is None and args.sampling == "sketch" else None,
                                  "work": "SURVEY 8(d) a6: sum over CPQR'd nodes 4sRk + 4k^2 s flops = %.3e; "
                                          "algorithmic bytes 16 R s per node (sample block read + written once) "
                                          "= %.3e" % (cf_flops, cf_bytes)},
            "roofline_tree": {"bound": "hbm", "phase": "cluster tree (a2): per level mean, covariance, power "
                                                      "iteration, projections, stable sorts",
                              "achieved": tree_bytes / (hi["ms_tree"] / 1e3) / 1e9, "peak": peaks["hbm_gbs"],
                              "unit": "GB/s", "frac": tree_bytes / (hi["ms_tree"] / 1e3) / 1e9 / peaks["hbm_gbs"],
                              "work": "SURVEY 8(d) a2: 3 passes over F per level, 3 L 8 n r = %.3e bytes" % tree_bytes},
            "roofline_factor": {"bound": "fp64 (DMMA)", "phase": "hss_ulv_factor (batched QR, WY GEMMs, POTRF, TRSM)",
                                "achieved": ui["factor_flops"] / (ui["ms_factor"] / 1e3) / 1e12,
                                "peak": fp64_peak, "unit": "TFLOP/s",
                                "frac": ui["factor_flops"] / (ui["ms_factor"] / 1e3) / 1e12 / fp64_peak,
                                "hbm_gbs": ui["factor_bytes"] / (ui["ms_factor"] / 1e3) / 1e9,
                                "work": "sum over nodes 2Rk^2 + 8R^2k + (R-k)^3/3 + k(R-k)^2 + k^2(R-k) + 4k^3 "
                                        "(SURVEY 8(d) a7), flops %.3e" % ui["factor_flops"]},
            "roofline_predict": None if ast["ms_predict"] is None else {
                "bound": "tensor", "phase": "svm_predict (predict_kernel: distance DMMA + exp + coefficient sums)",
                "achieved": 2.0 * Ftd.shape[0] * n * (rp + len(Cs)) / (ast["ms_predict"] / 1e3) / 1e12,
                "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": 2.0 * Ftd.shape[0] * n * (rp + len(Cs)) / (ast["ms_predict"] / 1e3) / 1e12 / fp64_peak,
                "work": "2 m n (r_pad + nC) flops + m n exp (incl. padding/norm/finish kernels in the time)"},
            "roofline_bias": {"bound": "hbm", "phase": "bias + objective: one HSS mat-vec with 2 nC columns",
                              "achieved": hi["generator_bytes"] / (ast["ms_bias"] / 1e3) / 1e9,
                              "peak": peaks["hbm_gbs"], "unit": "GB/s",
                              "frac": hi["generator_bytes"] / (ast["ms_bias"] / 1e3) / 1e9 / peaks["hbm_gbs"],
                              "work": "generator bytes (D, U, B) read once"},
            "clocks": clocks}
    if args.sampling == "ann":
        # no dense sketch in HSS-ANN mode: the dominant kernel of the step is the ULV sweep pair
        line["roofline_sketch_mode_only"] = line.pop("roofline")
        line["roofline_sketch_mode_only"] = {"note": "HSS-ANN sampling: no K*Omega sketch in this step",
                                             "ann_ms": line["phases_ms"]["sketch"]}
        line["roofline"] = dict(line["roofline_solve"], traffic=None)
        line["phases_ms"]["ann"] = line["phases_ms"].pop("sketch")
    if not args.no_e2e and args.n is None:
        # every rank makes the host-buffer call (with the communicator when N > 1: the library
        # shards the subtrees and the test points itself); time = max over ranks
        pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
        Fh, yh, Fth = pin(F), pin(y), pin(Ft)
        P.svm_train_predict_host(Fh, yh, h, cfg["beta"], Cs, max_it, Ftest=Fth, **opts)  # warm
        if world > 1:
            dist.barrier()
        e = P.svm_train_predict_host(Fh, yh, h, cfg["beta"], Cs, max_it, Ftest=Fth, **opts)
        tt = torch.tensor([e["timings_ms"]["total"]], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tot = tt.item()
        line["e2e"] = {"value": max_it * len(Cs) / (tot / 1e3), "unit": "iters/s",
                       "h2d_bytes_per_step": int(world * (Fh.nbytes + yh.nbytes + Fth.nbytes)),
                       "d2h_bytes_per_step": int(world * (n * len(Cs) * 8 + nt * len(Cs))),
                       "timings_ms": e["timings_ms"],
                       "note": "svm_train_predict_host on pinned host buffers: h2d + build + factor + "
                               "ADMM + bias + predict + d2h; iterations / total call time (max over "
                               "ranks; bytes summed over ranks: every rank copies F, y and F_test in "
                               "and z and the labels out)"}
    hi_a = None
    if world == 1 and args.sampling == "sketch" and not args.no_variants and args.n is None:
        # the same step with HSS-ANN compression (the paper's P:186-187 construction),
        # its own calibrated beta; one warm-up + one timed step, device-timed like the main line
        opts_a = cfg_opts(cfg, "ann")
        beta_a = cfg["beta_ann"]

        def step_ann():
            H = P.hss_build(Fd, h, **opts_a)
            try:
                U = P.hss_ulv_factor(H, beta_a)
                try:
                    res = P.admm_svm_train(U, yd, Cs, max_it, want_mu=False)
                    return H.info(), U.info(), res["stats"]
                finally:
                    U.free()
            finally:
                H.free()

        try:
            step_ann()
            hi_a, ui_a, st_a = step_ann()
        except P.HssError as ex:   # e.g. a config whose ANN K~ has no calibrated beta (only cfg 3 has one)
            hi_a = None
            line["variants"] = {"ann": {"sampling": "ann", "beta": beta_a, "error": str(ex)}}
    if hi_a is not None:
        line["variants"] = {"ann": {
            "sampling": "ann", "beta": beta_a, "admm_iters_per_s": max_it * len(Cs) / (st_a["ms_loop"] / 1e3),
            "hss_build_ulv_s": (hi_a["ms_tree"] + hi_a["ms_sketch"] + hi_a["ms_compress"] + ui_a["ms_factor"]) / 1e3,
            "phases_ms": {"tree": hi_a["ms_tree"], "ann": hi_a["ms_sketch"], "compress": hi_a["ms_compress"],
                          "factor": ui_a["ms_factor"], "admm_loop": st_a["ms_loop"]},
            "solve_gbs": (2.0 * ui_a["factor_bytes"] + 64.0 * n * len(Cs)) * max_it / (st_a["ms_loop"] / 1e3) / 1e9,
            "ranks_max": hi_a["max_rank_used"], "passthrough": hi_a["passthrough"],
            "factor_bytes": ui_a["factor_bytes"],
            "note": "HSS-ANN sampling (ann_neighbors/trees/leaf from datagen/configs.py); not the north-star "
                    "dense sketch - reported beside it"}}
    if world == 1 and args.sampling == "sketch" and args.interp == "id" and not args.no_variants and args.n is None:
        # N4: the same dense-sketch step with the SPD-preserving interpolation at the
        # paper's beta schedule - K~ is PSD, so no calibration; one warm-up + one timed step
        opts_s = cfg_opts(cfg, "sketch", "spd")
        beta_s = datagen.configs.beta_schedule(n)

        def step_spd():
            H = P.hss_build(Fd, h, **opts_s)
            try:
                U = P.hss_ulv_factor(H, beta_s)
                try:
                    res = P.admm_svm_train(U, yd, Cs, max_it, want_mu=False)
                    _, lab = P.svm_predict(Fd, yd, res["z"], h, res["bias"], Ftd)
                    acc_s = float((lab[:, 0].cpu().numpy() == yt[t0:t1]).mean())
                    return H.info(), U.info(), res["stats"], acc_s
                finally:
                    U.free()
            finally:
                H.free()

        step_spd()
        hi_s, ui_s, st_s, acc_s = step_spd()
        line.setdefault("variants", {})["spd"] = {
            "interp": "spd", "beta": beta_s, "test_accuracy": acc_s,
            "test_accuracy_id": acc, "beta_id": cfg["beta"],
            "admm_iters_per_s": max_it * len(Cs) / (st_s["ms_loop"] / 1e3),
            "hss_build_ulv_s": (hi_s["ms_tree"] + hi_s["ms_omega"] + hi_s["ms_sketch"] + hi_s["ms_compress"]
                                + ui_s["ms_factor"]) / 1e3,
            "phases_ms": {"tree": hi_s["ms_tree"], "sketch": hi_s["ms_sketch"], "compress": hi_s["ms_compress"],
                          "factor": ui_s["ms_factor"], "admm_loop": st_s["ms_loop"]},
            "ranks_max": hi_s["max_rank_used"], "passthrough": hi_s["passthrough"],
            "note": "N4 SPD-preserving compression (H3's skeletons, U = K(A,J)(K(J,J)+eps I)^-1): K~ PSD, "
                    "beta = the paper's schedule; test_accuracy on the synthetic test points vs the "
                    "main line's (ID form at the calibrated beta)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.n is None:
        r = oracle_phases(args.config, args.ref_n, args.ref_iters)
        hinfo = host_info()
        line["cpu_baseline"] = {"value": r["admm_iters_per_s_projected"], "unit": "iters/s",
                                "cores": hinfo["cores"], "kind": "oracle", "projected": True,
                                "sample": r["sample"], **hinfo, "phases_s_projected": r["phases_s_projected"],
                                "offline_full_size": oracle_offline(args.config)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
