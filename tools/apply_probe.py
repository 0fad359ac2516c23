"""Time the fine-level matrix-free apply of a configuration (diagnostic).

    NNMG_APPLY_KERNEL=pencil|reg python tools/apply_probe.py C3 [scale]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10910_b200 import configs, fespace, mfoperator  # noqa: E402

cfg = configs.get_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 1
m = cfg.make_meshes(scale=scale, validate=False)[-1]
ncomp = cfg.dim if cfg.problem == "elasticity" else 1
sp = fespace.build_space(m, cfg.degree, ncomp)
sp.constraints = fespace.dirichlet_constraints(sp, cfg.dirichlet_ids)
op = mfoperator.LaplaceOperator(sp) if cfg.problem == "poisson" else mfoperator.ElasticityOperator(sp, *cfg.lame)
n = op.n_dofs
u = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
v = torch.empty_like(u)
for _ in range(3):
    op.apply_into(u, v)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record()
for _ in range(reps):
    op.apply_into(u, v)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
nloc = (cfg.degree + 1) ** cfg.dim
g = cfg.dim * (cfg.dim + 1) // 2 if cfg.problem == "poisson" else cfg.dim ** 2 + 1
B = 16 * n + 4 * m.n_cells * nloc + 8 * m.n_cells * nloc * g
print(f"{cfg.name} 1/{scale} kernel={os.environ.get('NNMG_APPLY_KERNEL', 'default')} n={n} apply {ms:.4f} ms "
      f"{B / ms / 1e6:.0f} GB/s {n / ms / 1e6:.2f} GDoF/s checksum {float(v.double().square().sum()):.12e}")
