"""Registers / spills / stack per kernel from `nvcc -Xptxas -v` output.

    python tools/ptxas_report.py paper_2412_10910_b200/csrc/nnmg_transfer.cu [name-filter]
"""
import re
import subprocess
import sys

src = sys.argv[1]
filt = sys.argv[2] if len(sys.argv) > 2 else ""
cmd = ["nvcc", "-std=c++17", "--extended-lambda", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
       "-Xcompiler", "-fPIC", "-Iinclude", "-c", src, "-o", "/tmp/ptxas_report.o", "-Xptxas", "-v"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
name = None
rows = {}
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        rows[name] = {}
        continue
    if name is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
    if m:
        rows[name]["stack"], rows[name]["spill"] = int(m.group(1)), int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[name]["regs"] = int(m.group(1))
for n, r in rows.items():
    if filt in n:
        short = n.replace("nnmg::", "")
        short = short[: short.index("(")] if "(" in short else short
        print(f"{r.get('regs', '?'):>4} regs {r.get('spill', 0):>5} B spill {r.get('stack', 0):>5} B stack  {short}")
