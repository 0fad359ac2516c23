"""Top SASS instructions by warp-stall samples from an ncu report (needs -lineinfo):
    python tools/ncu_sass_hot.py gpurun_out/prof_C5.ncu-rep [kernel-substring] [N]
"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
filt = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')
for b in blocks[1:]:
    lines = b.splitlines()
    name = lines[0].strip(",").strip('"')
    if filt not in name:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    si = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, k in enumerate(h) if k.startswith("stall_")]
    data = []
    total = 0
    for r in rows[1:]:
        try:
            v = float(r[si])
        except (ValueError, IndexError):
            continue
        total += v
        reasons = sorted(((float(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:2]
        data.append((v, r[0], r[1], reasons))
    data.sort(reverse=True)
    print("==", name[:100], "total samples", total)
    for v, addr, src, reasons in data[:top]:
        rs = ", ".join(f"{n} {x:.0f}" for x, n in reasons if x > 0)
        print(f"{100 * v / total:5.1f}%  {addr}  {src[:60]:60s} {rs}")
