"""Key metrics + warp-stall breakdown per kernel from an ncu report:
    python tools/ncu_summary.py gpurun_out/prof_C3.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "inst"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")][:70]
        print("==", name)
        vals = []
        for k, short in KEYS:
            if k in h:
                vals.append(f"{short}={r[h.index(k)]}")
        print("  ", " ".join(vals))
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v > 0.05:
                    stalls.append((v, k.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")))
        stalls.sort(reverse=True)
        print("   stalls (warps per issue):", ", ".join(f"{n} {v:.2f}" for v, n in stalls[:8]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
