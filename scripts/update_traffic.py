"""Fill profiles/traffic.json (the ncu DRAM bytes bench.py reports beside its rooflines) from
committed launch lists:
  admm_iteration  : scripts/admm_profile.py capture (precompute solve + prologue + 3 iterations +
                    bias): an iteration = the launches after one admm_leaf_kernel up to and
                    including the next (forward L-1..0, backward 0..L-1, fused leaf kernel),
                    averaged over the complete iterations
  cpqr_level_sum  : scripts/build_profile.py capture: sum over the CPQR launches of one build
    python scripts/update_traffic.py ADMM_CSV BUILD_CSV TAG"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = [l for l in open(path) if l.startswith('"')]
    cur = {}
    for r in csv.DictReader(rows):
        key = (r["ID"], r["Kernel Name"])
        cur.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return [(k[1], v) for k, v in cur.items()]


def main():
    admm_csv, build_csv, tag = sys.argv[1:4]
    p = os.path.join(ROOT, "profiles", "traffic.json")
    d = json.load(open(p))
    L = launches(admm_csv)
    by = lambda v: v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)  # noqa: E731
    leaf = [i for i, (k, _) in enumerate(L) if "admm_leaf_kernel" in k]
    its = [L[a + 1:b + 1] for a, b in zip(leaf, leaf[1:])]
    assert its, "no complete ADMM iteration (fused leaf kernel) in the capture"
    nb = sum(sum(by(v) for _, v in it) for it in its) / len(its)
    nt = sum(sum(v.get("gpu__time_duration.sum", 0) for _, v in it) for it in its) / len(its)
    d["admm_iteration"] = {"workload": "cfg3_mixed524k", "dram_bytes": nb, "launches": len(its[0]),
                           "ncu_serialised_us": nt / 1e3,
                           "source": f"{admm_csv} ({tag}): ncu dram__bytes_read.sum + dram__bytes_write.sum over "
                                     f"the launches of one iteration (forward L-1..0, backward 0..L-1, fused leaf "
                                     f"kernel), mean of {len(its)} complete iterations"}
    B = launches(build_csv)
    cp = [(k, v) for k, v in B if "cpqr" in k]
    d["cpqr_level_sum"] = {"workload": "cfg3_mixed524k", "dram_bytes": sum(by(v) for _, v in cp),
                           "launches": len(cp), "ncu_serialised_ms": sum(v.get("gpu__time_duration.sum", 0)
                                                                          for _, v in cp) / 1e6,
                           "source": f"{build_csv} ({tag}): every CPQR launch of one config-3 build"}
    json.dump(d, open(p, "w"), indent=2)
    print(json.dumps({k: d[k] for k in ("admm_iteration", "cpqr_level_sum")}, indent=1))


if __name__ == "__main__":
    main()
