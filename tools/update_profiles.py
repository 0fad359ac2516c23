"""Copy the evidence written by tools/gpu/evidence.sh (gpurun_out/) into profiles/ (tracked):
bench lines, launch lists + summaries, full-capture summaries / raw pages / SASS stall lists,
and traffic.json (DRAM bytes per launch of the hot kernels).   python tools/update_profiles.py r1"""
import csv
import json
import os
import shutil
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
G, P = "gpurun_out", "profiles"
for c in ["C1", "C2", "C3", "C4", "C5"]:
    if os.path.exists(f"{G}/bench_{c}.json"):
        shutil.copy(f"{G}/bench_{c}.json", f"{P}/{tag}_bench_{c}.json")
if os.path.exists(f"{G}/bench_ref.json"):
    shutil.copy(f"{G}/bench_ref.json", f"{P}/{tag}_bench_reference_C3.json")
traffic = {"source": f"profiles/{tag}_C*_hot_ncu_raw.csv (ncu --set full of the isolated hot kernels: "
                     "dram__bytes_read.sum + dram__bytes_write.sum per launch, bytes)"}
for c in ["C3", "C4", "C5"]:
    if os.path.exists(f"{G}/launches_{c}.csv"):
        shutil.copy(f"{G}/launches_{c}.csv", f"{P}/{tag}_launches_{c}.csv")
        out = subprocess.run([sys.executable, "tools/launch_summary.py", f"{G}/launches_{c}.csv"], capture_output=True,
                             text=True).stdout
        open(f"{P}/{tag}_launches_{c}_summary.txt", "w").write(out)
    for src, dst in [("summary.txt", "hot_ncu_full.txt"), ("sass_hot.txt", "hot_sass_stalls.txt"),
                     ("raw.csv", "hot_ncu_raw.csv")]:
        if os.path.exists(f"{G}/full_{c}_{src}"):
            shutil.copy(f"{G}/full_{c}_{src}", f"{P}/{tag}_{c}_{dst}")
    raw = f"{P}/{tag}_{c}_hot_ncu_raw.csv"
    if not os.path.exists(raw):
        continue
    rows = list(csv.reader(open(raw)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        kind = "apply" if "k_apply" in name else ("prolongate" if "prolong" in name else
                                                   ("restrict" if "restrict" in name else None))
        if kind is None:
            continue
        tot = 0.0
        for m in ["dram__bytes_read.sum", "dram__bytes_write.sum"]:
            i = h.index(m)
            tot += float(r[i].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[i]]
        traffic[f"{c}_{kind}"] = tot
json.dump(traffic, open(f"{P}/traffic.json", "w"), indent=1)
print(json.dumps(traffic, indent=1))
