"""CPU baseline rate of the reference V-cycle (oracle/_ref: the unmodified
nnmg package; the NumPy oracle port where that is absent) at several sample
scales of a config, single-threaded: shows the DoFs/s rate does not depend on
the sample size, so the bench's 1/5-scale CPU sample stands in for the full
configuration.   python tools/cpu_rate_vs_scale.py C3 8 6 5 4"""
import os, sys, time
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2412_10910_b200.configs import get_config

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
for scale in [int(s) for s in (sys.argv[2:] or ["8", "6", "5", "4", "3"])]:
    rate, n, k, el, kind = bench.cpu_vcycle_rate(cfg, scale, 20.0)
    print(f"{cfg.name} 1/{scale}: {n} fine DoFs, {k} V-cycles in {el:.1f} s: {rate * 1e3:.4f} MDoF/s "
          f"= {rate:.6f} GDoF/s (1 core, {kind})", flush=True)
