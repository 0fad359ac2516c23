"""One fp64 and one mixed-precision V-cycle of a config (graph off), for an
ncu launch list: python tools/gpu/mixed_profile.py C3"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2412_10910_b200 import configs, multigrid

cfg = configs.get_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
H = multigrid.build_hp_hierarchy(cfg.make_meshes(validate=False), cfg.degree, problem=cfg.problem,
                                 dirichlet_ids=cfg.dirichlet_ids, lame=cfg.lame,
                                 config=multigrid.HierarchyConfig(chebyshev_degree=cfg.chebyshev_degree,
                                                                  coarse_direct="auto"))
b = H.finest.operator.load_vector(cfg.body_force if cfg.body_force else 1.0)
z = torch.empty_like(b)
H.use_graph(False)
for bits in (64, 32):
    H.set_precision(bits)
    H.v_cycle_into(b, z)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push(f"cycle{bits}")
    torch.cuda.profiler.start()
    H.v_cycle_into(b, z)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    torch.cuda.nvtx.range_pop()
print("done")
