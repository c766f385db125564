"""Text summary of an `ncu --set full` report (one block per captured launch): duration, DRAM
bytes and throughput, FP64 / tensor pipe utilisation, occupancy, registers, shared-memory bank
conflicts, and the top warp-stall reasons.

    python scripts/ncu_summary.py gpurun_out/<tag>.ncu-rep [title] > profiles/<tag>_ncu_summary.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "compute-memory throughput %"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("smsp__pipe_tensor_subpipe_dmma_cycles_active.avg", "dmma subpipe active cycles (avg/SMSP)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "fp64 (DFMA) pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block", "shared mem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(title)
    print(f"source: {rep} (ncu --set full; per-launch, replayed, cold caches)\n")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"== {d.get('Kernel Name', '?')[:110]}")
        for k, name in KEYS:
            hit = k if k in d else next((h for h in hdr if h.endswith("." + k) or h.endswith(k)), None)
            if hit and d.get(hit) not in ("", None):
                print(f"   {name:42s} {d[hit]} {u.get(hit, '')}")
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", ""))
              for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not k.endswith("not_issued") and v not in ("", "0")}
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda x: -x[1])[:6]
        print("   stalls (share of samples): " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))
        print()


if __name__ == "__main__":
    main()
