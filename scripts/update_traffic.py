"""Fill profiles/traffic.json (the ncu DRAM bytes bench.py reports beside its rooflines) from
committed launch lists:
  admm_iteration  : scripts/admm_profile.py capture (precompute solve + 3 iterations + bias):
                    per iteration = sum(ulv_* kernels) / 4 + sum(admm_epilogue) / 3
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
    ulv = sum(by(v) for k, v in L if "ulv_" in k)
    epi = sum(by(v) for k, v in L if "admm_epilogue" in k)
    t_ulv = sum(v.get("gpu__time_duration.sum", 0) for k, v in L if "ulv_" in k)
    t_epi = sum(v.get("gpu__time_duration.sum", 0) for k, v in L if "admm_epilogue" in k)
    d["admm_iteration"] = {"workload": "cfg3_mixed524k", "dram_bytes_read": None, "dram_bytes_write": None,
                           "dram_bytes": ulv / 4 + epi / 3, "ncu_serialised_us": (t_ulv / 4 + t_epi / 3) / 1e3,
                           "source": f"{admm_csv} ({tag}): ncu dram__bytes_read.sum + dram__bytes_write.sum over "
                                     "the ULV sweep and epilogue kernels; sum(ulv_*) / 4 (precompute solve + 3 "
                                     "iterations) + sum(epilogue) / 3"}
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
