"""Coarsest-level solve: the reference's Jacobi-PCG (k_coarse_cg1) vs the
direct packed-symmetric inverse (k_symv_tiles + k_symv_reduce) on the
coarse level of every BASELINE config; CUDA-event times, achieved GB/s."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2412_10910_b200 import configs, fespace, mfoperator, solvers

def timeit(cs, b, x, reps=20):
    s = torch.cuda.current_stream()
    for _ in range(3):
        cs.solve_into(b, x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        cs.solve_into(b, x)
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps

for name in sys.argv[1:] or ["C2", "C3", "C4", "C5"]:
    cfg = configs.get_config(name)
    m = cfg.make_meshes(validate=False)[0]
    ncomp = cfg.dim if cfg.problem == "elasticity" else 1
    sp = fespace.build_space(m, cfg.degree, ncomp)
    sp.constraints = fespace.dirichlet_constraints(sp, cfg.dirichlet_ids)
    op = (mfoperator.ElasticityOperator(sp, *cfg.lame) if cfg.problem == "elasticity"
          else mfoperator.LaplaceOperator(sp))
    b = torch.from_numpy(np.random.default_rng(0).standard_normal(sp.n_dofs)).cuda()
    b[torch.from_numpy(sp.constraints.dofs).cuda()] = 0
    cg = solvers.CoarseSolver(op, direct=False)
    x1 = torch.empty_like(b)
    t_cg = timeit(cg, b, x1)
    its = cg.status()[0]
    import time
    t0 = time.perf_counter()
    dr = solvers.CoarseSolver(op, direct=True)
    setup = time.perf_counter() - t0
    x2 = torch.empty_like(b)
    t_dr = timeit(dr, b, x2)
    nf = sp.n_dofs - len(sp.constraints.dofs)
    by = solvers.direct_solve_bytes(nf)
    r = float((x1 - x2).norm() / x2.norm())
    print(f"{name}: n={sp.n_dofs} free={nf} CG {its} its {t_cg*1e3:.3f} ms ({t_cg/its*1e6:.2f} us/it) | "
          f"direct {t_dr*1e3:.3f} ms, {by/1e9:.3f} GB -> {by/t_dr/1e9:.0f} GB/s, setup {setup:.1f} s | "
          f"rel diff {r:.2e}", flush=True)
    del dr, cg
    torch.cuda.empty_cache()
