"""bench.py's reference arm (the CPU oracle on a bounded sample, BASELINE contract): one JSON
line with the contract's keys from rank 0, nothing (exit 0) from the other ranks."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0",
           "--ref-n", "1024", "--ref-iters", "2"]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)


def test_reference_arm_json_line():
    r = _run({"RANK": "0", "WORLD_SIZE": "1"})
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["unit"] == "iters/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_reference_arm_other_ranks_silent():
    r = _run({"RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip() == ""


def test_solve_algorithmic_bytes_formula():
    """roofline_solve's byte count: with every rank at the cap (config 3: leaves
    pass-through, every other node R = 512, k = 256) it reproduces the survey's independently
    computed 7.56 GB per iteration; one more compressing leaf adds exactly its compact factor
    twice; the compression flop count matches 4 s R k + 4 k^2 s per node."""
    sys.path.insert(0, ROOT)
    import bench
    n, leaf, L = 524288, 256, 11
    ranks = [-1] + [256] * (2 ** (L + 1) - 2)
    shapes, root_R = bench.node_shapes(ranks, n, leaf)
    assert root_R == 512 and len(shapes) == 2 ** (L + 1) - 2
    b = bench.solve_algorithmic_bytes(shapes, root_R, n, 1)
    assert abs(b / 1e9 - 7.557) < 0.001
    ranks2 = list(ranks)
    ranks2[2 ** L - 1] = 200                   # first leaf compresses: R = 256, k = 200
    shapes2, r2 = bench.node_shapes(ranks2, n, leaf)
    R, k = 256, 200
    e = R - k
    leafb = R * k - k * (k - 1) // 2 + k * (k + 1) // 2 + e * (e + 1) // 2 + k * e
    # its parent now has R = 456: compact factor changes too
    Rp, kp = 456, 256
    ep = Rp - kp
    par_new = Rp * kp - kp * (kp - 1) // 2 + kp * (kp + 1) // 2 + ep * (ep + 1) // 2 + kp * ep
    par_old = 512 * 256 - 256 * 255 // 2 + 256 * 257 // 2 + 256 * 257 // 2 + 256 * 256
    b2 = bench.solve_algorithmic_bytes(shapes2, r2, n, 1)
    assert b2 - b == 16 * (leafb + par_new - par_old)
    fl, by = bench.compress_work([(1, 512, 256)], 272)
    assert fl == 4 * 272 * 512 * 256 + 4 * 256 * 256 * 272 and by == 16 * 512 * 272
