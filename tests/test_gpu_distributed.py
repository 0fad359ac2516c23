"""The distributed V-cycle through the production GPU backend (NCCL, world
size 1 on the single available GPU): local spaces, GPU operators on local
numbering, transfers built from located records, the replicated coarse level
and the fused Chebyshev kernels must reproduce the single-GPU hierarchy.
(Halo exchanges between ranks are covered by tests/test_distributed_gloo.py.)"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("cname,scale", [("C3", 8), ("C5", 8)])
def test_distributed_gpu_backend_world1(cname, scale):
    import torch.distributed as dist

    from paper_2412_10910_b200 import configs, distributed, fespace, multigrid
    from paper_2412_10910_b200.mfoperator import assemble_rhs

    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1, device_id=dev)
    try:
        cfg = configs.get_config(cname)
        meshes = cfg.make_meshes(scale=scale)
        ncomp = cfg.dim if cfg.problem == "elasticity" else 1
        spaces = []
        for m in meshes:
            sp = fespace.build_space(m, cfg.degree, ncomp)
            sp.constraints = fespace.dirichlet_constraints(sp, cfg.dirichlet_ids)
            spaces.append(sp)
        DH = distributed.build_distributed_hierarchy(spaces, distributed.GpuBackend(dev), cfg.problem, cfg.lame,
                                                     cfg.chebyshev_degree)
        H = multigrid.build_hp_hierarchy(meshes, cfg.degree, problem=cfg.problem, dirichlet_ids=cfg.dirichlet_ids,
                                         lame=cfg.lame,
                                         config=multigrid.HierarchyConfig(chebyshev_degree=cfg.chebyshev_degree))
        b = assemble_rhs(spaces[-1], cfg.body_force if cfg.body_force else 1.0)
        fine = DH.finest
        for lev_d, lev in zip(DH.levels[1:], H.levels[1:]):
            assert abs(lev_d.lam_max - lev.smoother.lam_max) <= 1e-10 * lev.smoother.lam_max
        zd = fine.gather_global(DH.precondition(fine.from_global(b)))
        zh = H.v_cycle(b, executor=False)
        assert np.linalg.norm(zd - zh) <= 1e-10 * np.linalg.norm(zh)
        # the cycle ran as a replayed CUDA graph with the split apply (interior
        # blocks on the compute stream, ghost import forked to a side stream)
        assert DH.use_graph and DH._graph is not None
        assert fine.layout.n_interior_cells > 0 and fine.overlap
        # and equals the unsplit distributed cycle run eagerly
        for lev in DH.levels:
            lev.overlap = False
        DH.use_graph, DH._graph = False, None
        z0 = fine.gather_global(DH.precondition(fine.from_global(b)))
        assert np.linalg.norm(zd - z0) <= 1e-12 * np.linalg.norm(z0)
        # ... and to the explicit-residual form of multigrid.py:97, 101 (rounding-level difference)
        DH.recurrence = False
        z1 = fine.gather_global(DH.precondition(fine.from_global(b)))
        assert np.linalg.norm(z1 - z0) <= 1e-11 * np.linalg.norm(z0)
        DH.recurrence = True
        for lev in DH.levels:
            lev.overlap = True
        DH.use_graph = True
        x, its, conv, _ = distributed.dist_cg_solve(fine, fine.from_global(b), DH.precondition, 1e-8)
        from paper_2412_10910_b200.solvers import cg_solve

        ref = cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-8)
        assert conv and abs(its - ref.iterations) <= 1
    finally:
        dist.destroy_process_group()
