"""Fine-level apply time of a config in the default (atomic scatter) and the
deterministic (cell buffer + fixed-order gather) modes; CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2412_10910_b200 import configs, fespace, mfoperator

for name in sys.argv[1:] or ["C3", "C4", "C5"]:
    cfg = configs.get_config(name)
    m = cfg.make_meshes(validate=False)[-1]
    sp = fespace.build_space(m, cfg.degree, cfg.dim if cfg.problem == "elasticity" else 1)
    sp.constraints = fespace.dirichlet_constraints(sp, cfg.dirichlet_ids)
    u = torch.from_numpy(np.random.default_rng(0).standard_normal(sp.n_dofs)).cuda()
    s = torch.cuda.Stream()
    out = {}
    for det in (False, True):
        op = (mfoperator.ElasticityOperator(sp, *cfg.lame, deterministic=det) if cfg.problem == "elasticity"
              else mfoperator.LaplaceOperator(sp, deterministic=det))
        v = torch.empty_like(u)
        with torch.cuda.stream(s):
            for _ in range(3):
                op.apply_into(u, v)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(20):
                op.apply_into(u, v)
            e1.record(s)
        s.synchronize()
        out[det] = (e0.elapsed_time(e1) / 20, v.cpu().numpy())
        del op
        torch.cuda.empty_cache()
    err = np.linalg.norm(out[True][1] - out[False][1]) / np.linalg.norm(out[False][1])
    print(f"{name}: apply atomic {out[False][0] * 1e3:.1f} us, deterministic {out[True][0] * 1e3:.1f} us "
          f"(x{out[True][0] / out[False][0]:.2f}), rel diff {err:.1e}", flush=True)
