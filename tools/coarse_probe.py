"""Probe the coarse CG kernel variants on the C3 coarse level (diagnostic)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10910_b200 import configs, fespace, mfoperator, solvers

cfg = configs.get_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
m = cfg.make_meshes(scale=1, validate=False)[0]
ncomp = cfg.dim if cfg.problem == "elasticity" else 1
sp = fespace.build_space(m, cfg.degree, ncomp)
sp.constraints = fespace.dirichlet_constraints(sp, cfg.dirichlet_ids)
op = (mfoperator.LaplaceOperator(sp) if cfg.problem == "poisson" else mfoperator.ElasticityOperator(sp, *cfg.lame))
b = torch.from_numpy(np.random.default_rng(2).standard_normal(op.n_dofs)).cuda()
x = torch.empty_like(b)
cs = solvers.CoarseSolver(op, dense_limit=10)
for _ in range(3):
    cs.solve_into(b, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    cs.solve_into(b, x)
e1.record()
torch.cuda.synchronize()
it, conv, _ = cs.status()
ms = e0.elapsed_time(e1) / 10
print(f"{cfg.name} coarse n={op.n_dofs} barrier={os.environ.get('NNMG_COARSE_BARRIER','0')} its={it} conv={conv} "
      f"{ms:.3f} ms/solve {1e3*ms/it:.2f} us/it info={cs.info()}")
