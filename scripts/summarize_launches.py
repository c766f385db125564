"""Summarize an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel shares.

    python scripts/summarize_launches.py gpurun_out/<tag>_launches.csv [title] > profiles/<tag>_launches_summary.txt
Per-launch times from ncu are cold-cache and serialised: compare SHARES, not absolutes.
"""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name[:60]


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    rows = [l for l in open(path) if l.startswith('"')]
    rd = csv.DictReader(rows)
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(r["Metric Unit"], 1e-6)
        tot[k] += v * scale
        cnt[k] += 1
    all_ms = sum(tot.values())
    print(title)
    print("unit: ms (ncu gpu__time_duration.sum, cold-cache, serialised: compare SHARES only)\n")
    print(f"{'kernel':60s} {'launches':>8s} {'total_ms':>11s} {'share':>7s}")
    for k in sorted(tot, key=lambda x: -tot[x]):
        print(f"{k:60s} {cnt[k]:8d} {tot[k]:11.3f} {100 * tot[k] / all_ms:6.2f}%")
    print(f"{'TOTAL':60s} {sum(cnt.values()):8d} {all_ms:11.3f}")


if __name__ == "__main__":
    main()
