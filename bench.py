#!/usr/bin/env python
"""Benchmark: fp64 V-cycle GDoF/s (BASELINE.json metric) on a BASELINE config.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

A step is one V-cycle ``H.precondition(r)`` (Alg. 1: Chebyshev-Jacobi pre/post
smoothing, residual, non-nested restriction/prolongation, device-resident
coarse CG) on the finest level of the configuration.  ``value`` = fine DoFs x
steps / device time with the input resident in HBM (replayed CUDA graph);
``e2e`` = the same through the public call with pinned-host input, H2D + cycle
+ D2H of every step inside the timed region, serialised as a PCG caller's
dependent chain (the pipelined rate with independent inputs is reported beside
it as an upper bound).  The roofline object describes the dominant kernel (the
fine-level matrix-free apply) measured live with CUDA events on its stream.
``--impl reference`` times the reference's own hierarchy (oracle/_ref, the
unmodified NumPy package; the oracle port where that is absent) on a bounded
sample of the same configuration.

Multi-GPU (torchrun): the cell-partitioned hierarchy (strong scaling, same
global problem as N=1), halo exchange and dots over NCCL; timing is the max
over ranks.  The CPU arms run one single-threaded oracle process per host core
(the reference is single-threaded NumPy) and report the aggregate throughput.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_TEXT = {
    "C1": "2D Poisson Q1, 128^2/45^2/17^2 jittered +-0.25h, Chebyshev 4",
    "C2": "2D Poisson Q2, 512^2/181^2/64^2 jittered +-0.2h, Chebyshev 4",
    "C3": "3D Poisson Q2 hex, 128^3/47^3/17^3 jittered +-0.2h, Chebyshev 4",
    "C4": "3D Poisson Q4 curved, 64^3/23^3/8^3 jittered +-0.15h, Chebyshev 4",
    "C5": "3D elasticity vector Q2 beam, 256x32^2/93x12^2/33x4^2 jittered +-0.2h, Chebyshev 5",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--scale", type=int, default=1, help="divide cells per axis (1 = full config)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-scale", type=int, default=5, help="sample scale for the CPU baseline")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-solve", action="store_true", help="skip the full PCG solve (host in / host out)")
    ap.add_argument("--no-mixed", action="store_true", help="skip the mixed-precision V-cycle measurement")
    ap.add_argument("--profile", action="store_true", help="profiler range around one cycle + hot kernels, then exit")
    ap.add_argument("--distributed", action="store_true", help="use the cell-partitioned path even on one rank")
    ap.add_argument("--coarse", default="auto", choices=["auto", "cg", "direct"],
                    help="coarsest-level solver: the reference's CG, the exact direct solve, or the faster")
    return ap.parse_args()


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: start N ranks over
    NCCL on this node, exactly as the driver's torchrun command does."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout carries the one JSON line
    raise SystemExit(subprocess.call(cmd, env=env))


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------------------
# algorithmic byte / flop model
# ---------------------------------------------------------------------------
def vmult_bytes(dim, p, ncomp, n_dofs, n_cells, physics):
    nloc = (p + 1) ** dim
    g = dim * (dim + 1) // 2 if physics == "poisson" else dim * dim + 1
    return 16 * n_dofs + 4 * n_cells * nloc + 8 * n_cells * nloc * g


def transfer_bytes(dim, p, ncomp, npts, n_dofs_coarse, n_cells_coarse):
    nloc = (p + 1) ** dim
    return npts * (4 + 4 + 8 * dim + 8 * ncomp) + 8 * n_dofs_coarse + 4 * n_cells_coarse * nloc


def vmult_flops(dim, p, ncomp, n_cells, physics):
    """F = nc [4 d^2 ncomp n1^(d+1) + nq f_qp]."""
    n1 = p + 1
    fqp = 2 * dim * dim + dim if physics == "poisson" else 150
    return n_cells * (4 * dim * dim * ncomp * n1 ** (dim + 1) + n1 ** dim * fqp)


def transfer_flops(dim, p, ncomp, npts):
    """contraction + 1D basis evaluation from xhat."""
    n1 = p + 1
    return npts * ncomp * 2 * sum(n1 ** k for k in range(1, dim + 1)) + npts * dim * n1 * 2 * (n1 - 1)


def roof_frac(t, nbytes, flops, hbm_gbs, fp64_tflops):
    """t_roof / t with t_roof = max(B / HBM, F / FP64) and the binding resource."""
    tb = nbytes / (hbm_gbs * 1e9)
    tf = flops / (fp64_tflops * 1e12) if fp64_tflops else 0.0
    return max(tb, tf) / t, ("hbm" if tb >= tf else "fp64")


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def reference_pin(cname, key):
    """A value the reference computed at full size (tests/golden/full_<C>.npz,
    written by tests/golden/make_fullsize_pins.py in the build container)."""
    path = os.path.join(ROOT, "tests", "golden", f"full_{cname}.npz")
    if not os.path.exists(path):
        return None
    with np.load(path) as z:
        if key not in z.files:
            return None
        v = z[key]
        return v.item() if v.ndim == 0 else v.tolist()


def traffic_from_profiles(kernel_key):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        with open(path) as fh:
            return json.load(fh).get(kernel_key)
    return None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"nnmg_clocks_{os.getpid()}.csv")

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
            # the sampler is live before the timed region starts (its first
            # line takes ~0.1-0.3 s), so short regions still get the samples
            # that bracket them
            t_end = time.time() + 5.0
            while time.time() < t_end and os.path.getsize(self.path) == 0 and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        self.t0 = time.time()
        return self

    def __exit__(self, *a):
        self.elapsed = time.time() - self.t0
        if self.proc is not None and self.elapsed < 0.1:
            time.sleep(0.06)  # one more sample right at the end of a short region
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, flags in rows for i, f in enumerate(flags) if f == "Active"})
        out = {"sm_mhz": float(np.median([r[0] for r in rows])), "sm_max_mhz": rows[0][1], "reasons": reasons,
               "samples": len(rows)}
        if getattr(self, "elapsed", 1.0) < 0.1:
            out["note"] = (f"timed region {self.elapsed * 1e3:.1f} ms, shorter than the 50 ms sampling interval: "
                           "samples taken just before and after it")
        return out


# ---------------------------------------------------------------------------
# CPU baseline: the oracle (NumPy port of the reference path) on a sample
# ---------------------------------------------------------------------------
def _cpu_hierarchy(cfg, scale):
    """(precondition, rhs, n_dofs, kind): the reference's own NumPy hierarchy
    (oracle/_ref, installed by oracle/build_ref.py: kind "reference") when it
    travelled with the repo, else the oracle port (kind "port")."""
    from oracle import build_ref

    h0 = min((hi - lo) / n for (lo, hi), n in zip(cfg.extent, cfg.level_grid(0, scale)))
    nnmg = build_ref.import_reference()
    if nnmg is not None:
        import nnmg.geosearch
        import nnmg.mfoperator
        import nnmg.multigrid

        rm = [nnmg.mesh.Mesh(m.dim, m.vertices, m.cells, m.boundary_faces, validate=False)
              for m in cfg.make_meshes(scale=scale, validate=False)]
        kw = dict(problem=cfg.problem, dirichlet_ids=cfg.dirichlet_ids, lame=cfg.lame,
                  config=nnmg.multigrid.HierarchyConfig(chebyshev_degree=cfg.chebyshev_degree))
        try:
            H = nnmg.multigrid.build_hp_hierarchy(rm, cfg.degree, **kw)
        except nnmg.geosearch.GeosearchError:
            # coarse sample meshes of the curved config miss boundary points: widen
            # the box padding to 0.1 h_coarse as SURVEY.md §8(c) prescribes
            H = nnmg.multigrid.build_hp_hierarchy(rm, cfg.degree, search=nnmg.geosearch.SearchConfig(eps_box=0.1 * h0),
                                                  **kw)
        sp = H.finest.space
        if cfg.body_force:
            f = np.array(cfg.body_force, dtype=float)
            b = nnmg.mfoperator.assemble_rhs(sp, lambda x: np.broadcast_to(f, (len(x), len(f))))
        else:
            b = nnmg.mfoperator.assemble_rhs(sp, 1.0)
        return H.precondition, b, sp.n_dofs, "reference"
    from oracle import nnmg_oracle as O

    meshes = [O.jittered_mesh(cfg.level_grid(l, scale), cfg.extent, cfg.amplitude, 1000 * cfg.index + l + 1,
                              cfg.warp) for l in range(len(cfg.levels))]
    args = (meshes, cfg.degree, cfg.problem, cfg.dirichlet_ids, cfg.lame or (1.0, 1.0), cfg.chebyshev_degree)
    try:
        H, spaces = O.build_hierarchy(*args)
    except O.LocateError:
        H, spaces = O.build_hierarchy(*args, search={"eps_box": 0.1 * h0})
    b = O.assemble_rhs_const(spaces[-1], cfg.body_force if cfg.body_force else 1.0)
    return H.precondition, b, spaces[-1].n_dofs, "port"


def cpu_vcycle_rate(cfg, scale, seconds, steps=None, warmup=1, barrier=None):
    precondition, b, n, kind = _cpu_hierarchy(cfg, scale)
    for _ in range(max(1, warmup)):
        precondition(b)  # warm-up
    if barrier is not None:
        barrier.wait()  # all worker processes start timing together
    t0 = time.perf_counter()
    k = 0
    while True:
        precondition(b)
        k += 1
        el = time.perf_counter() - t0
        if (steps is not None and k >= steps) or (steps is None and el >= seconds):
            break
    return n * k / el / 1e9, n, k, el, kind


_THREAD_VARS = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")
_KIND_TEXT = {"reference": "the reference's own nnmg.multigrid.MultigridHierarchy (unmodified NumPy package, oracle/_ref)",
              "port": "NumPy oracle port of nnmg (oracle/_ref absent)"}


def _cpu_worker(cfg_name, scale, seconds, steps, warmup, barrier, queue):
    from paper_2412_10910_b200.configs import get_config

    _, n, k, el, kind = cpu_vcycle_rate(get_config(cfg_name), scale, seconds, steps, warmup, barrier)
    queue.put((n, k, el, kind))


def cpu_vcycle_rate_all_cores(cfg, scale, seconds, steps=None, warmup=1, procs=None):
    """The oracle V-cycle on every host core: one single-threaded process per
    core, each timing its own V-cycles on the same sample after a common
    start; aggregate throughput = sum of DoFs x cycles / the longest run."""
    import multiprocessing as mp

    procs = max(1, min(procs or os.cpu_count() or 1, 32))
    if procs == 1:
        rate, n, k, el, kind = cpu_vcycle_rate(cfg, scale, seconds, steps, warmup)
        return rate, n, k, el, 1, kind
    ctx = mp.get_context("spawn")
    saved = {v: os.environ.get(v) for v in _THREAD_VARS}
    for v in _THREAD_VARS:
        os.environ[v] = "1"
    try:
        barrier, queue = ctx.Barrier(procs), ctx.Queue()
        ps = [ctx.Process(target=_cpu_worker, args=(cfg.name, scale, seconds, steps, warmup, barrier, queue))
              for _ in range(procs)]
        for p in ps:
            p.start()
        res = [queue.get() for _ in ps]
        for p in ps:
            p.join()
    finally:
        for v, val in saved.items():
            if val is None:
                os.environ.pop(v, None)
            else:
                os.environ[v] = val
    n = res[0][0]
    work = sum(r[0] * r[1] for r in res)
    el = max(r[2] for r in res)
    return work / el / 1e9, n, sum(r[1] for r in res), el, procs, res[0][3]


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    rate, n, k, el, procs, kind = cpu_vcycle_rate_all_cores(cfg, args.cpu_scale, args.cpu_seconds,
                                                            steps=max(1, args.steps), warmup=args.warmup)
    sample = (f"{cfg.name} at 1/{args.cpu_scale} cells per axis ({n} fine DoFs), {k} V-cycles over {procs} "
              f"single-threaded processes ({max(1, args.steps)} each), {_KIND_TEXT[kind]}")
    line = {
        "impl": "reference", "metric": "fp64 V-cycle GDoF/s", "value": rate, "unit": "GDoF/s", "n_gpus": 0,
        "steps": max(1, args.steps), "warmup": max(1, args.warmup), "ms_per_step": el / max(1, args.steps) * 1e3,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SURVEY §8(d) meshes)",
        "config": {"workload": CONFIG_TEXT[cfg.name] + f" (CPU sample 1/{args.cpu_scale})", "config": cfg.name},
        "cpu_baseline": {"value": rate, "unit": "GDoF/s", "cores": procs, "kind": kind, "sample": sample},
        "e2e": {"value": rate, "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_ours(args, cfg):
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    from paper_2412_10910_b200 import _lib
    from paper_2412_10910_b200 import multigrid, solvers

    t_setup = time.perf_counter()
    meshes = cfg.make_meshes(scale=args.scale, validate=False)
    coarse_direct = {"auto": "auto", "cg": False, "direct": True}[args.coarse]
    H = multigrid.build_hp_hierarchy(meshes, cfg.degree, problem=cfg.problem, dirichlet_ids=cfg.dirichlet_ids,
                                     lame=cfg.lame, config=multigrid.HierarchyConfig(
                                         chebyshev_degree=cfg.chebyshev_degree, coarse_direct=coarse_direct),
                                     device=dev)
    fine = H.finest.operator
    b = fine.load_vector(cfg.body_force if cfg.body_force else 1.0)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    n = fine.n_dofs
    stream = torch.cuda.Stream(device=dev)
    z = torch.empty_like(b)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    # warm-up (captures the CUDA graph)
    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            H.v_cycle_into(b, z)
    stream.synchronize()

    if args.profile:
        # profiler range for `ncu --profile-from-start off`: one V-cycle
        # (graph), then one isolated fine apply / prolongate / restrict
        u = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).to(dev)
        v = torch.empty_like(u)
        T = H.transfers[-1]
        rc = torch.empty(T.coarse_space.n_dofs, dtype=torch.float64, device=dev)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        with torch.cuda.stream(stream):
            torch.cuda.nvtx.range_push("vcycle")
            H.v_cycle_into(b, z)
            torch.cuda.nvtx.range_pop()
            torch.cuda.nvtx.range_push("hot")
            fine.apply_into(u, v)
            T.prolongate_into(rc, v)
            T.restrict_into(u, rc)
            torch.cuda.nvtx.range_pop()
        stream.synchronize()
        torch.cuda.profiler.stop()
        if rank == 0:
            print(json.dumps({"profile": True, "config": cfg.name, "kernels_per_cycle": H.kernels_per_cycle()}))
        return

    # ---- timed region: K V-cycles ----
    # Configurations whose fine-level working set exceeds L2 (C3-C5: >1 GB per
    # apply) are timed back to back.  Smaller ones (C1, C2 fit in the 126 MB
    # L2) get an L2 flush (a 2x L2 buffer written) before every cycle, timed
    # per cycle with events around the cycle only; their L2-resident
    # back-to-back rate is reported beside it.
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    l2_bytes = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 << 20))
    finfo = fine.info()
    nloc_f = (H.finest.space.degree + 1) ** H.finest.space.mesh.dim
    working = finfo["geometry_bytes"] + 4 * H.finest.space.mesh.n_cells * nloc_f + 8 * 6 * n
    flush_mode = working < 2 * l2_bytes
    flush_buf = torch.empty(2 * l2_bytes // 4, dtype=torch.float32, device=dev) if flush_mode else None
    barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    t_resident = None
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            if flush_mode:
                starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
                ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
                for k in range(args.steps):
                    flush_buf.fill_(float(k))
                    starts[k].record(stream)
                    H.v_cycle_into(b, z)
                    ends[k].record(stream)
            else:
                e0.record(stream)
                for _ in range(args.steps):
                    H.v_cycle_into(b, z)
                e1.record(stream)
        stream.synchronize()
    launches = _lib.launch_count() - launches0
    if flush_mode:
        t_dev = sum(a.elapsed_time(c) for a, c in zip(starts, ends)) * 1e-3
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(args.steps):
                H.v_cycle_into(b, z)
            e1.record(stream)
        stream.synchronize()
        t_resident = e0.elapsed_time(e1) * 1e-3
    barrier()
    if not flush_mode:
        t_dev = e0.elapsed_time(e1) * 1e-3
    t_max = t_dev
    if world > 1:
        import torch.distributed as dist

        tt = torch.tensor([t_dev], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    value = world * n * args.steps / t_max / 1e9

    # ---- e2e (headline): a dependent chain through the public call ----
    # every step copies its input from pinned host memory, runs the V-cycle
    # and reads the result back before the next step starts (a PCG caller's
    # pattern: each preconditioner input depends on the previous output)
    hin = [b.cpu().pin_memory(), (2.0 * b).cpu().pin_memory()]
    hout = [torch.empty_like(hin[0]).pin_memory() for _ in range(2)]
    bin1, z1 = torch.empty_like(b), torch.empty_like(b)
    with torch.cuda.stream(stream):
        bin1.copy_(hin[0], non_blocking=True)
        H.v_cycle_into(bin1, z1)
        hout[0].copy_(z1, non_blocking=True)
    stream.synchronize()
    barrier()
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        e0.record(stream)
        for k in range(args.steps):
            bin1.copy_(hin[k % 2], non_blocking=True)
            H.v_cycle_into(bin1, z1)
            hout[k % 2].copy_(z1, non_blocking=True)
        e1.record(stream)
    stream.synchronize()
    t_chain = e0.elapsed_time(e1) * 1e-3
    if world > 1:
        tt = torch.tensor([t_chain], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_chain = float(tt.item())
    e2e_chain = world * n * args.steps / t_chain / 1e9

    # ---- e2e upper bound: independent right-hand sides streamed ----
    # the copies of steps k+1 (H2D) and k-1 (D2H) run on their own streams /
    # copy engines while the V-cycle of step k computes (two device buffer
    # pairs, event-ordered): a throughput bound for callers with independent
    # inputs, not what a PCG loop sees
    hin = [b.cpu().pin_memory(), (2.0 * b).cpu().pin_memory()]
    hout = [torch.empty_like(hin[0]).pin_memory() for _ in range(2)]
    bin_ = [torch.empty_like(b) for _ in range(2)]
    zz = [torch.empty_like(b) for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        for i in range(2):  # warm-up: one cycle per buffer pair (graph capture)
            bin_[i].copy_(hin[i], non_blocking=True)
            H.v_cycle_into(bin_[i], zz[i])
            hout[i].copy_(zz[i], non_blocking=True)
    stream.synchronize()
    barrier()
    torch.cuda.synchronize()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_cp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    e0.record(stream)
    s_in.wait_event(e0)
    s_out.wait_event(e0)
    for k in range(args.steps):
        i = k % 2
        with torch.cuda.stream(s_in):
            if k >= 2:
                s_in.wait_event(ev_cp[i])  # cycle k-2 has consumed bin_[i]
            bin_[i].copy_(hin[i], non_blocking=True)
            ev_in[i].record(s_in)
        with torch.cuda.stream(stream):
            stream.wait_event(ev_in[i])
            if k >= 2:
                stream.wait_event(ev_out[i])  # result k-2 has left zz[i]
            H.v_cycle_into(bin_[i], zz[i])
            ev_cp[i].record(stream)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_cp[i])
            hout[i].copy_(zz[i], non_blocking=True)
            ev_out[i].record(s_out)
    for i in range(min(2, args.steps)):
        stream.wait_event(ev_out[i])
    e1.record(stream)
    torch.cuda.synchronize()
    t_e2e = e0.elapsed_time(e1) * 1e-3
    if args.steps >= 2:  # the pipeline delivered the right results (input 2b -> 2z up to the coarse tolerance)
        err = float((hout[1] - 2.0 * hout[0]).norm() / (2.0 * hout[0]).norm())
        if not err <= 1e-7:
            raise RuntimeError(f"pipelined e2e results inconsistent (rel {err:.2e})")
    if world > 1:
        tt = torch.tensor([t_e2e], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    e2e = world * n * args.steps / t_e2e / 1e9

    # ---- dominant kernel: fine-level apply, CUDA events on its stream ----
    u = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).to(dev)
    v = torch.empty_like(u)
    reps = 20
    with torch.cuda.stream(stream):
        for _ in range(3):
            fine.apply_into(u, v)
        e0.record(stream)
        for _ in range(reps):
            fine.apply_into(u, v)
        e1.record(stream)
    stream.synchronize()
    t_apply = e0.elapsed_time(e1) * 1e-3 / reps
    info = fine.info()
    sp = H.finest.space
    ncomp = sp.n_components
    B = vmult_bytes(sp.mesh.dim, sp.degree, ncomp, n, sp.mesh.n_cells, cfg.problem)
    peak, peak_kind = measured_peaks()
    achieved = B / t_apply / 1e9
    # transfers (fine pair)
    T = H.transfers[-1]
    uc = torch.from_numpy(np.random.default_rng(0).standard_normal(T.coarse_space.n_dofs)).to(dev)
    rc = torch.empty_like(uc)
    with torch.cuda.stream(stream):
        for _ in range(3):
            T.prolongate_into(uc, v)
            T.restrict_into(u, rc)
        e0.record(stream)
        for _ in range(reps):
            T.prolongate_into(uc, v)
        e1.record(stream)
        e2 = torch.cuda.Event(enable_timing=True)
        for _ in range(reps):
            T.restrict_into(u, rc)
        e2.record(stream)
    stream.synchronize()
    t_pro = e0.elapsed_time(e1) * 1e-3 / reps
    t_res = e1.elapsed_time(e2) * 1e-3 / reps
    cm = T.coarse_space.mesh
    BT = transfer_bytes(sp.mesh.dim, T.coarse_space.degree, ncomp, len(T.cells), T.coarse_space.n_dofs, cm.n_cells)
    FT = transfer_flops(sp.mesh.dim, T.coarse_space.degree, ncomp, len(T.cells))
    FV = vmult_flops(sp.mesh.dim, sp.degree, ncomp, sp.mesh.n_cells, cfg.problem)
    fp64 = _lib.fp64_peak(local)
    v_rf, v_bound = roof_frac(t_apply, B, FV, peak, fp64)
    p_rf, p_bound = roof_frac(t_pro, BT, FT, peak, fp64)
    r_rf, r_bound = roof_frac(t_res, BT, FT, peak, fp64)
    # fine applies per V-cycle: (m1 + m2) sweeps of degree k, the residual
    # after pre-smoothing taken from the smoother's recurrence (one apply of
    # the k pre-smoothing applies) -> 2k (8 for C3)
    applies_per_cycle = (H.m1 + H.m2) * cfg.chebyshev_degree

    # ---- full PCG solve through the public call, host in / host out ----
    # cg_solve(A, b_numpy, precond=H.precondition, target_reduction=1e-8)
    # (solvers.py:129-164): the H2D copy of b and the D2H copy of x are inside
    # the timed region; iterations beside the reference's (tests/golden pins)
    solve = None
    if not args.no_solve:
        b_host = b.cpu().numpy()
        solvers.cg_solve(fine, b_host, precond=H.precondition, target_reduction=1e-8)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = solvers.cg_solve(fine, b_host, precond=H.precondition, target_reduction=1e-8)
        t_solve = time.perf_counter() - t0
        solve = {"iterations": res.iterations, "converged": res.converged, "seconds": t_solve,
                 "final_rel_residual": res.residual_norms[-1] / res.residual_norms[0],
                 "reference_iterations": reference_pin(cfg.name, "iterations"),
                 "gdofs_per_s_x_iterations": n * res.iterations / t_solve / 1e9,
                 "timing": "wall clock around cg_solve (host b in, host x out; every dot synchronises)"}
    cit, cconv, _ = H.coarse_solver.status() if not H.coarse_solver.dense else (None, None, None)

    # ---- mixed-precision V-cycle beside it ----
    # fp32 storage of vectors / geometry / transfer records above the coarsest
    # level, fp64 arithmetic and coarse solve; same device timing as `value`;
    # parity by the outer PCG iteration count
    mixed = None
    if not args.no_mixed:
        H.set_precision(32)
        with torch.cuda.stream(stream):
            for _ in range(max(args.warmup, 3)):
                H.v_cycle_into(b, z)
            if flush_mode:
                t32 = 0.0
                for k in range(args.steps):
                    flush_buf.fill_(float(k))
                    e0.record(stream)
                    H.v_cycle_into(b, z)
                    e1.record(stream)
                    e1.synchronize()
                    t32 += e0.elapsed_time(e1) * 1e-3
            else:
                e0.record(stream)
                for _ in range(args.steps):
                    H.v_cycle_into(b, z)
                e1.record(stream)
        stream.synchronize()
        if not flush_mode:
            t32 = e0.elapsed_time(e1) * 1e-3
        if world > 1:
            tt = torch.tensor([t32], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t32 = float(tt.item())
        res32 = solvers.cg_solve(fine, b, precond=H.precondition, target_reduction=1e-8)
        mixed = {"value": world * n * args.steps / t32 / 1e9, "unit": "GDoF/s",
                 "ms_per_step": t32 / args.steps * 1e3, "solve_iterations": res32.iterations,
                 "solve_converged": res32.converged, "reference_iterations": reference_pin(cfg.name, "iterations"),
                 "storage": "fp32 level vectors, geometry, inverse diagonals, transfer xhat (levels >= 2), "
                            "single-precision arithmetic in the applies and transfers (NNMG_MIXED_ARITH=64: fp64), "
                            "coarse solve from the packed inverse in fp32 tiles where faster, fp64 coarse vectors "
                            "and outer CG",
                 "coarse_solver": H.coarse_solver.info()}
        H.set_precision(64)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, ncpu, k, el, procs, kind = cpu_vcycle_rate_all_cores(cfg, args.cpu_scale, args.cpu_seconds)
        cpu = {"value": rate, "unit": "GDoF/s", "cores": procs, "kind": kind,
               "sample": f"{cfg.name} at 1/{args.cpu_scale} cells per axis ({ncpu} fine DoFs), {k} V-cycles in "
                         f"{el:.1f} s over {procs} single-threaded processes (one per host core), "
                         f"{_KIND_TEXT[kind]}"}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": "fp64 V-cycle GDoF/s", "value": value, "unit": "GDoF/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": t_max / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded SURVEY §8(d) jittered meshes, f=1 load vector)",
            "config": {"workload": CONFIG_TEXT[cfg.name] + ("" if args.scale == 1 else f" at 1/{args.scale}"),
                       "config": cfg.name, "fine_dofs": n, "levels_dofs": [lev.operator.n_dofs for lev in H.levels],
                       "l2": (f"L2 flushed before every cycle (fine working set {working / 1e6:.0f} MB < 2x L2); "
                              f"L2-resident back-to-back rate in value_l2_resident") if flush_mode
                             else f"inputs larger than L2 (fine working set {working / 1e9:.2f} GB per apply)",
                       "value_l2_resident": (world * n * args.steps / t_resident / 1e9) if t_resident else None,
                       "parallelism": "single GPU" if world == 1 else f"replicated x{world}",
                       "graph": True, "setup_s": round(setup_s, 2),
                       "coarse_cg_iterations": cit, "coarse_solver": H.coarse_solver.info()},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic_from_profiles(f"{cfg.name}_apply"),
                         "kernel": "k_apply (fine-level matrix-free vmult)", "bytes_per_launch": B,
                         "avg_launch_ms": t_apply * 1e3, "peak_kind": peak_kind,
                         "share_of_step": applies_per_cycle * t_apply / (t_max / args.steps)},
            "kernels": {
                "vmult_gdofs": n / t_apply / 1e9, "vmult_frac": achieved / peak,
                "prolongate_ms": t_pro * 1e3, "prolongate_frac": BT / t_pro / 1e9 / peak,
                "restrict_ms": t_res * 1e3, "restrict_frac": BT / t_res / 1e9 / peak,
                "transfer_bytes": BT, "geometry_bytes": info["geometry_bytes"],
                "fp64_peak_tflops": fp64, "vmult_flops": FV, "transfer_flops": FT,
                "vmult_roof_frac": v_rf, "vmult_bound": v_bound,
                "prolongate_roof_frac": p_rf, "prolongate_bound": p_bound,
                "restrict_roof_frac": r_rf, "restrict_bound": r_bound,
            },
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_chain, "unit": "GDoF/s", "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                    "pattern": "dependent chain: H2D of the step's input, V-cycle, D2H of its result, serialised "
                               "on one stream (a PCG caller's pattern)",
                    "pipelined_upper_bound": e2e,
                    "pipelined_pattern": "independent inputs: H2D of step k+1 and D2H of step k-1 on separate "
                                         "streams during cycle k"},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if solve is not None:
            line["solve"] = solve
        if mixed is not None:
            line["mixed_precision"] = mixed
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def run_distributed(args, cfg):
    """N ranks, one GPU each: the hierarchy's cells are partitioned (strong
    scaling, same global problem as N=1); halo exchange and dots over NCCL."""
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if "RANK" not in os.environ:  # plain `python bench.py --distributed`: a world of one
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # NCCL's version / debug lines stay off stdout
    dist.init_process_group("nccl", device_id=dev)
    from paper_2412_10910_b200 import _lib, distributed, fespace

    t_setup = time.perf_counter()
    meshes = cfg.make_meshes(scale=args.scale, validate=False)
    ncomp = cfg.dim if cfg.problem == "elasticity" else 1
    spaces = []
    for m in meshes:
        sp = fespace.build_space(m, cfg.degree, ncomp)
        sp.constraints = fespace.dirichlet_constraints(sp, cfg.dirichlet_ids)
        spaces.append(sp)
    bk = distributed.GpuBackend(dev)
    DH = distributed.build_distributed_hierarchy(spaces, bk, cfg.problem, cfg.lame, cfg.chebyshev_degree)
    fine = DH.finest
    b = fine.op.load_vector(cfg.body_force if cfg.body_force else 1.0)  # local load vector, owned part exact
    from paper_2412_10910_b200.distributed import halo_export_add

    halo_export_add(fine.exp, b)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    n_global = spaces[-1].n_dofs
    for _ in range(max(args.warmup, 3)):
        DH.precondition(b)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            DH.precondition(b)
        e1.record()
        torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1) * 1e-3], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    value = n_global * args.steps / t_max / 1e9
    # per-GPU roofline of the dominant kernel: this rank's local fine apply (no halo), events on its stream
    info = fine.op.info()
    B_local = vmult_bytes(cfg.dim, cfg.degree, ncomp, fine.n, info["n_cells"], cfg.problem)
    xa, ya = b.clone(), torch.empty_like(b)
    for _ in range(3):
        fine.op.apply_into(xa, ya)
    e0.record()
    for _ in range(10):
        fine.op.apply_into(xa, ya)
    e1.record()
    torch.cuda.synchronize()
    t_apply = torch.tensor([e0.elapsed_time(e1) * 1e-3 / 10], device=dev)
    dist.all_reduce(t_apply, op=dist.ReduceOp.MAX)
    t_apply = float(t_apply.item())
    hbm, hbm_kind = measured_peaks()
    # e2e: each rank's owned share from pinned host memory
    hb = b.cpu().pin_memory()
    hz = torch.empty_like(hb).pin_memory()
    dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        bd = hb.to(dev, non_blocking=True)
        z = DH.precondition(bd)
        hz.copy_(z, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) * 1e-3], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e = n_global * args.steps / float(t.item()) / 1e9
    if rank == 0:
        line = {
            "metric": "fp64 V-cycle GDoF/s", "value": value, "unit": "GDoF/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded SURVEY §8(d) jittered meshes, f=1 load vector)",
            "config": {"workload": CONFIG_TEXT[cfg.name], "config": cfg.name, "fine_dofs": n_global,
                       "parallelism": f"cell-partitioned x{world} (Morton), replicated coarse level",
                       "l2": "inputs larger than L2", "setup_s": round(setup_s, 2),
                       "owned_fine_dofs_rank0": fine.n_owned},
            "roofline": {"bound": "hbm", "achieved": B_local / t_apply / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": B_local / t_apply / 1e9 / hbm, "traffic": None,
                         "kernel": "k_apply (this rank's fine-level cells, max over ranks)",
                         "bytes_per_launch": B_local, "avg_launch_ms": t_apply * 1e3,
                         "peak_kind": hbm_kind},
            "cpu_baseline": None,
            "e2e": {"value": e2e, "unit": "GDoF/s", "h2d_bytes_per_step": 8 * fine.n,
                    "d2h_bytes_per_step": 8 * fine.n},
            "gpu_launches": launches, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    from paper_2412_10910_b200.configs import get_config

    cfg = get_config(args.config)
    if args.gpus > 1 and dist_env()[1] == 1 and "RANK" not in os.environ:
        relaunch_under_torchrun(args)
    if args.gpus != dist_env()[1] and "RANK" in os.environ:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={dist_env()[1]}")
    if args.impl == "reference":
        run_reference(args, cfg)
    elif dist_env()[1] > 1 or args.distributed:
        run_distributed(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
