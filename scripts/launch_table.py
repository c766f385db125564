"""Per-launch table of an ncu launch list with time and DRAM bytes:
    python scripts/launch_table.py gpurun_out/<tag>_launches.csv [kernel-substring ...]"""
import csv
import sys

rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
pats = sys.argv[2:]
cur = {}
for r in csv.DictReader(rows):
    key = (r["ID"], r["Kernel Name"][:44], r["Grid Size"])
    cur.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
tot = 0.0
for k, v in cur.items():
    if pats and not any(p in k[1] for p in pats):
        continue
    t = v.get("gpu__time_duration.sum", 0) / 1e3
    tot += t
    rb = v.get("dram__bytes_read.sum", 0) / 1e6
    wb = v.get("dram__bytes_write.sum", 0) / 1e6
    print(f"{k[1]:44s} {k[2]:16s} {t:10.1f}us  R {rb:10.1f}MB W {wb:10.1f}MB  {(rb + wb) / max(t, 1e-9):6.2f} TB/s")
print(f"total {tot / 1e3:.2f} ms")
