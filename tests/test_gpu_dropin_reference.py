"""Drop-in proof: the GPU components inside the REFERENCE's own classes.

The unmodified reference package (installed into oracle/_ref by
oracle/build_ref.py; test infrastructure) builds its all-NumPy hierarchy with
``nnmg.multigrid.build_hp_hierarchy`` (multigrid.py:145-203).  The same
reference ``FESpace`` objects are then handed to this repo's GPU operator,
``ChebyshevJacobi``, ``CoarseSolver`` and
``TwoLevelTransferNonNested.from_reference`` (the reference's own located
records), and those objects are plugged into the reference's
``nnmg.multigrid.MultigridHierarchy`` (multigrid.py:32-117) and the reference's
``cg_solve`` (solvers.py:129-164): NumPy in, NumPy out, no other glue.

Gates: V-cycle within 1e-9 relative l2 of the NumPy reference, operator
applies / transfers 1e-11, outer CG iterations +-1 and the same solution.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [("C1", 1), ("C2", 8), ("C3", 8), ("C4", 4), ("C5", 8)]


@pytest.fixture(scope="module")
def ref():
    from oracle import build_ref

    nnmg = build_ref.import_reference()
    if nnmg is None:
        pytest.skip("oracle/_ref not installed (run oracle/build_ref.py where /root/reference exists)")
    import nnmg.fespace  # noqa: F401
    import nnmg.mfoperator  # noqa: F401
    import nnmg.multigrid  # noqa: F401
    import nnmg.solvers  # noqa: F401
    import nnmg.transfer  # noqa: F401

    return nnmg


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2412_10910_b200 as pkg
    from paper_2412_10910_b200 import configs, mfoperator, multigrid, solvers, transfer  # noqa: F401

    return pkg


def _reference_hierarchy(ref, cfg, scale, dense_limit=2000):
    meshes = cfg.make_meshes(scale=scale)
    rmeshes = [ref.mesh.Mesh(m.dim, m.vertices, m.cells, m.boundary_faces) for m in meshes]
    rcfg = ref.multigrid.HierarchyConfig(chebyshev_degree=cfg.chebyshev_degree, coarse_dense_limit=dense_limit)
    search = None
    if cfg.warp:
        # the curved config's coarse sample meshes need the wider box padding
        h = min((hi - lo) / n for (lo, hi), n in zip(cfg.extent, cfg.level_grid(0, scale)))
        search = ref.geosearch.SearchConfig(eps_box=0.1 * h)
    return ref.multigrid.build_hp_hierarchy(rmeshes, cfg.degree, problem=cfg.problem, dirichlet_ids=cfg.dirichlet_ids,
                                            lame=cfg.lame, search=search, config=rcfg)


def _gpu_inside_reference(ref, P, Href, cfg, dense_limit=2000):
    levels = []
    for lev in Href.levels:
        if cfg.problem == "elasticity":
            op = P.mfoperator.ElasticityOperator(lev.space, *cfg.lame)
        else:
            op = P.mfoperator.LaplaceOperator(lev.space)
        sm = P.solvers.ChebyshevJacobi(op, degree=cfg.chebyshev_degree)
        levels.append(ref.multigrid.Level(lev.space, op, sm))
    transfers = [P.transfer.TwoLevelTransferNonNested.from_reference(T, levels[i].operator, levels[i + 1].operator)
                 for i, T in enumerate(Href.transfers)]
    cs = P.solvers.CoarseSolver(levels[0].operator, dense_limit=dense_limit)
    return ref.multigrid.MultigridHierarchy(levels, transfers, cs, m1=Href.m1, m2=Href.m2)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("cname,scale", CASES)
def test_gpu_components_inside_reference_hierarchy(ref, P, cname, scale):
    cfg = P.configs.get_config(cname)
    Href = _reference_hierarchy(ref, cfg, scale)
    Hgpu = _gpu_inside_reference(ref, P, Href, cfg)
    assert isinstance(Hgpu, ref.multigrid.MultigridHierarchy)
    sp = Href.finest.space
    f = np.array(cfg.body_force) if cfg.body_force else 1.0
    if cfg.body_force:
        b = ref.mfoperator.assemble_rhs(sp, lambda x: np.broadcast_to(f, (len(x), len(f))))
    else:
        b = ref.mfoperator.assemble_rhs(sp, 1.0)
    rng = np.random.default_rng(0)
    # per-component parity through the reference protocol (NumPy in / out)
    for l, (lr, lg) in enumerate(zip(Href.levels, Hgpu.levels)):
        u = rng.standard_normal(lr.space.n_dofs)
        assert _rel(lg.operator.apply(u), lr.operator.apply(u)) <= 1e-11
        assert _rel(lg.operator.diagonal(), lr.operator.diagonal()) <= 1e-12
        assert abs(lg.smoother.lam_max - lr.smoother.lam_max) <= 1e-9 * lr.smoother.lam_max
        assert _rel(lg.smoother.smooth(u), lr.smoother.smooth(u)) <= 1e-10
    for Tr, Tg in zip(Href.transfers, Hgpu.transfers):
        uc = rng.standard_normal(Tr.coarse_space.n_dofs)
        rf = rng.standard_normal(Tr.fine_space.n_dofs)
        assert _rel(Tg.prolongate(uc), Tr.prolongate(uc)) <= 1e-11
        assert _rel(Tg.restrict(rf), Tr.restrict(rf)) <= 1e-11
    # the reference's V-cycle recursion (multigrid.py:83-113) over GPU parts
    z_ref = Href.precondition(b)
    z_gpu = Hgpu.precondition(b)
    assert isinstance(z_gpu, np.ndarray)
    assert _rel(z_gpu, z_ref) <= 1e-9
    rows = Hgpu.timing_rows()
    assert {r[1] for r in rows} == set(ref.multigrid.V_CYCLE_COMPONENTS)
    # the reference's cg_solve preconditioned by it (solvers.py:129-164)
    res_ref = ref.solvers.cg_solve(Href.finest.operator, b, precond=Href.precondition, target_reduction=1e-8)
    res_gpu = ref.solvers.cg_solve(Hgpu.finest.operator, b, precond=Hgpu.precondition, target_reduction=1e-8)
    assert res_ref.converged and res_gpu.converged
    assert abs(res_gpu.iterations - res_ref.iterations) <= 1
    assert _rel(res_gpu.x, res_ref.x) <= 1e-6


def test_gpu_setup_on_reference_spaces_matches_reference_records(ref, P):
    """GPU point location on reference spaces reproduces the reference's
    records bit-exactly (transfer.py:67-85), and our own hierarchy builder
    accepts reference meshes."""
    cfg = P.configs.get_config("C3")
    Href = _reference_hierarchy(ref, cfg, 8)
    for T in Href.transfers:
        Tg = P.transfer.setup_nonnested(T.coarse_space, T.fine_space)
        assert np.array_equal(Tg.point_dofs, T.point_dofs)
        assert np.array_equal(Tg.cells, T.cells)
        assert np.array_equal(Tg.projected, T.projected)
        assert np.abs(Tg.xhat - T.xhat).max() <= 1e-10


@pytest.mark.parametrize("cname,scale", [("C3", 8), ("C5", 8)])
def test_gpu_coarse_cg_inside_reference_hierarchy(ref, P, cname, scale):
    """Same drop-in with the coarse level above the dense limit on both sides:
    the reference's Jacobi-PCG coarse solve (solvers.py:193-206) against the
    persistent coarse CG kernel."""
    cfg = P.configs.get_config(cname)
    Href = _reference_hierarchy(ref, cfg, scale, dense_limit=50)
    Hgpu = _gpu_inside_reference(ref, P, Href, cfg, dense_limit=50)
    assert not Hgpu.coarse_solver.dense
    rng = np.random.default_rng(1)
    b = rng.standard_normal(Href.finest.space.n_dofs)
    b[Href.finest.space.constraints.dofs] = 0.0
    bc = rng.standard_normal(Href.levels[0].space.n_dofs)
    bc[Href.levels[0].space.constraints.dofs] = 0.0
    xr, xg = Href.coarse_solver.solve(bc), Hgpu.coarse_solver.solve(bc)
    assert _rel(xg, xr) <= 1e-6  # both stop at a 1e-8 residual reduction
    assert _rel(Hgpu.precondition(b), Href.precondition(b)) <= 1e-6
    res_ref = ref.solvers.cg_solve(Href.finest.operator, b, precond=Href.precondition, target_reduction=1e-8)
    res_gpu = ref.solvers.cg_solve(Hgpu.finest.operator, b, precond=Hgpu.precondition, target_reduction=1e-8)
    assert res_ref.converged and res_gpu.converged
    assert abs(res_gpu.iterations - res_ref.iterations) <= 1
