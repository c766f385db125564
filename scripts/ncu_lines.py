"""Per-CUDA-source-line stall samples of one kernel in an ncu report (--import-source on):
    python scripts/ncu_lines.py REP KERNEL_REGEX [TOP]"""
import csv
import io
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", "regex:" + kre, "-c", "1"], capture_output=True, text=True).stdout
    f = lambda x: float(x) if x not in ("", "-") else 0.0
    fname, hdr, agg = None, None, {}
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0].isdigit() and len(r) > 4 and r[2] == "-":
            agg[(fname, int(r[0]))] = (f(r[4]), r[1].strip()[:90], f(r[7]))
    tot = sum(v[0] for v in agg.values()) or 1.0
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[0]}:{k[1]:5d} {100 * v[0] / tot:5.1f}%  exec={v[2]:10.0f} | {v[1]}")


if __name__ == "__main__":
    main()
