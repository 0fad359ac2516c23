"""C5 fine elasticity apply variants (env switches read at level creation):
   python tools/gpu/elast_variants.py NNMG_ELAST_XCH=0 NNMG_ELAST_XCH=1 NNMG_ELAST_XCH=1,NNMG_ELAST_TMA=1"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2412_10910_b200 import configs, fespace, mfoperator

cfg = configs.get_config("C5")
m = cfg.make_meshes(validate=False)[-1]
sp = fespace.build_space(m, 2, 3)
sp.constraints = fespace.dirichlet_constraints(sp, cfg.dirichlet_ids)
u = torch.from_numpy(np.random.default_rng(0).standard_normal(sp.n_dofs)).cuda()
s = torch.cuda.Stream()
ref = None
combos = sys.argv[1:] or ["NNMG_ELAST_XCH=0", "NNMG_ELAST_XCH=1", "NNMG_ELAST_XCH=1,NNMG_ELAST_TMA=1"]
for xch in combos:
    for k in [k for k in os.environ if k.startswith("NNMG_ELAST")]:
        del os.environ[k]
    for kv in xch.split(","):
        k, v = kv.split("=")
        os.environ[k] = v
    op = mfoperator.ElasticityOperator(sp, 1.0, 1.0)
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
    vv = v.cpu().numpy()
    ref = vv if ref is None else ref
    print(f"{xch}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us  rel diff {np.linalg.norm(vv - ref) / np.linalg.norm(ref):.1e}",
          flush=True)
    del op
