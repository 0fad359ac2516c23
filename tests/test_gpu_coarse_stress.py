"""Stress of the persistent coarse CG kernel (one grid barrier per iteration,
r/s double- and w triple-buffered across CTAs): compute-sanitizer is closed
on this GPU pool (profiles/r2_sanitizer_unavailable.txt), so cross-CTA races
are hunted by repetition instead.  Every one of many back-to-back solves of
the same right-hand side must converge to the reference tolerance with the
same iteration count (+-1: the cell scatter inside the kernel uses fp64
atomics) and the same solution to rounding, matching the oracle's Jacobi-PCG
(solvers.py:193-206).  Also the configuration path of ADVICE r1 (more than
256 cell blocks: the single-barrier kernel is not used and the multi-barrier
fallback must launch with its own configuration)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2412_10910_b200 as P

    return P


def coarse_level(P, cname):
    cfg = P.configs.get_config(cname)
    m = cfg.make_meshes(validate=False)[0]
    sp = P.fespace.build_space(m, cfg.degree, cfg.dim if cfg.problem == "elasticity" else 1)
    sp.constraints = P.fespace.dirichlet_constraints(sp, cfg.dirichlet_ids)
    op = (P.mfoperator.ElasticityOperator(sp, *cfg.lame) if cfg.problem == "elasticity"
          else P.mfoperator.LaplaceOperator(sp))
    return cfg, m, sp, op


@pytest.mark.parametrize("cname", ["C2", "C3", "C5"])
def test_coarse_cg_repeated_solves(P, oracle, cname):
    cfg, m, sp, op = coarse_level(P, cname)
    cs = P.solvers.CoarseSolver(op)
    assert not cs.dense and not cs.direct
    rng = np.random.default_rng(5)
    b = rng.standard_normal(sp.n_dofs)
    b[sp.constraints.dofs] = 0.0
    bd = torch.from_numpy(b).cuda()
    xs, its = [], []
    x = torch.empty_like(bd)
    for k in range(60):
        cs.solve_into(bd, x)
        it, conv, indef = cs.status()
        assert conv and not indef, (k, it)
        its.append(it)
        xs.append(x.clone())
    assert max(its) - min(its) <= 1, its
    x0 = xs[0]
    for xk in xs[1:]:
        assert float((xk - x0).norm() / x0.norm()) <= 1e-7
    r = b - op.apply(x0.cpu().numpy())
    assert np.linalg.norm(r) <= 1.01e-8 * np.linalg.norm(b)
    # the oracle's Jacobi-PCG on the same level
    om = oracle.jittered_mesh(m.grid, cfg.extent, cfg.amplitude, 1000 * cfg.index + 1, cfg.warp)
    osp = oracle.make_space(om, cfg.degree, sp.n_components, cfg.dirichlet_ids)
    oop = oracle.OOperator(osp, cfg.problem, *(cfg.lame or (1.0, 1.0)))
    oc = oracle.OCoarse(oop)
    xo = oc.solve(b)
    assert np.linalg.norm(x0.cpu().numpy() - xo) <= 1e-6 * np.linalg.norm(xo)
    assert abs(np.mean(its) - oc.last_iterations) <= 1


def test_coarse_cg_many_cell_blocks(P):
    """3D Q1 with 13,824 cells (432 cell blocks > 256): the CG path must
    configure the multi-barrier kernel consistently and converge."""
    m = P.mesh.jittered_box_mesh((24, 24, 24), [(0.0, 1.0)] * 3, 0.2, seed=9)
    sp = P.fespace.build_space(m, 1)
    sp.constraints = P.fespace.dirichlet_constraints(sp, "all")
    op = P.mfoperator.LaplaceOperator(sp)
    cs = P.solvers.CoarseSolver(op)
    assert not cs.dense
    b = np.random.default_rng(6).standard_normal(sp.n_dofs)
    b[sp.constraints.dofs] = 0.0
    x = cs.solve(b)
    it, conv, _ = cs.status()
    assert conv and it > 0
    assert np.linalg.norm(b - op.apply(x)) <= 1.01e-8 * np.linalg.norm(b)
