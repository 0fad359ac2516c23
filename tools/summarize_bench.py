"""One-line summaries of bench.py JSON outputs: python tools/summarize_bench.py gpurun_out/bench_C*.log"""
import json
import sys

for path in sys.argv[1:]:
    try:
        lines = [ln for ln in open(path).read().strip().splitlines() if ln.startswith("{")]
        d = json.loads(lines[-1])
    except Exception:
        print(path, "FAILED:", open(path).read()[-600:].replace("\n", " | "))
        continue
    k = d["kernels"]
    cfg = d["config"]
    print(f"{cfg['config']}: V {d['value']:.3f} GDoF/s {d['ms_per_step']:.3f} ms | e2e {d['e2e']['value']:.3f} | "
          f"vmult {d['roofline']['avg_launch_ms']:.3f} ms {100 * d['roofline']['frac']:.0f}% | "
          f"pro {k['prolongate_ms']:.3f} ms {100 * k['prolongate_frac']:.0f}% ({100 * k.get('prolongate_roof_frac', 0):.0f}% {k.get('prolongate_bound', '')}) | "
          f"res {k['restrict_ms']:.3f} ms {100 * k['restrict_frac']:.0f}% ({100 * k.get('restrict_roof_frac', 0):.0f}% {k.get('restrict_bound', '')}) | fp64 {k.get('fp64_peak_tflops', 0):.1f} TF | coarse its {cfg['coarse_cg_iterations']} | "
          f"solve {d.get('solve')} | setup {cfg['setup_s']}s | clocks {d['clocks'].get('sm_mhz')}")
