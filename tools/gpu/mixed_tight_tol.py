"""Outer PCG with the mixed-precision cycle at tight tolerances (the fp32 V-cycle is only the
preconditioner; the fp64 residual decides): python tools/gpu/mixed_tight_tol.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2412_10910_b200 import configs, multigrid, solvers

for cname, scale in [("C3", 4), ("C5", 4), ("C4", 2), ("C2", 2)]:
    cfg = configs.get_config(cname)
    H = multigrid.build_hp_hierarchy(cfg.make_meshes(scale=scale, validate=False), cfg.degree, problem=cfg.problem,
                                     dirichlet_ids=cfg.dirichlet_ids, lame=cfg.lame,
                                     config=multigrid.HierarchyConfig(chebyshev_degree=cfg.chebyshev_degree,
                                                                      coarse_direct="auto"))
    b = H.finest.operator.load_vector(cfg.body_force if cfg.body_force else 1.0)
    for tol in (1e-8, 1e-10, 1e-12):
        out = []
        for bits in (64, 32):
            H.set_precision(bits)
            r = solvers.cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=tol, max_iter=60)
            res = b - H.finest.operator.apply(r.x)
            out.append((r.iterations, r.converged, float(res.norm() / b.norm())))
        print(f"{cname} 1/{scale} tol {tol:g}: fp64 its {out[0][0]} ({out[0][2]:.1e})  mixed its {out[1][0]} "
              f"({out[1][2]:.1e}) converged {out[1][1]}", flush=True)
    H.set_precision(64)
