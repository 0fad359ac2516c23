"""Small hierarchies through every solver path, for compute-sanitizer
(memcheck / racecheck / synccheck): fp64 V-cycle with the persistent coarse
CG (one grid barrier per iteration, rotating buffers), the direct coarse
solve, the mixed-precision cycle, deterministic mode, elasticity, Q4."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2412_10910_b200 import configs, multigrid, solvers

for name, scale in (("C3", 8), ("C5", 8), ("C4", 4), ("C2", 8)):
    cfg = configs.get_config(name)
    meshes = cfg.make_meshes(scale=scale, validate=False)
    for kw in (dict(coarse_dense_limit=0), dict(coarse_dense_limit=0, coarse_direct=True),
               dict(vcycle_precision=32), dict(deterministic=True)):
        H = multigrid.build_hp_hierarchy(meshes, cfg.degree, problem=cfg.problem, dirichlet_ids=cfg.dirichlet_ids,
                                         lame=cfg.lame, config=multigrid.HierarchyConfig(
                                             chebyshev_degree=cfg.chebyshev_degree, **kw))
        b = H.finest.operator.load_vector(cfg.body_force if cfg.body_force else 1.0)
        res = solvers.cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-8)
        z = H.v_cycle(b, executor=kw.get("vcycle_precision", 64) == 32)
        torch.cuda.synchronize()
        print(name, kw, "its", res.iterations, "conv", res.converged, flush=True)
print("sanitize-ok")
