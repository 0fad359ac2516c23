"""Degenerate inputs on the GPU path: levels without free DoFs, transfers
without points, zero right-hand sides, single-cell meshes, coarse meshes finer
than the fine one.  The reference's behaviour is the oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2412_10910_b200 as P

    return P


UNIT2 = ((0.0, 1.0), (0.0, 1.0))
UNIT3 = ((0.0, 1.0), (0.0, 1.0), (0.0, 1.0))


def _space(P, grid, extent, p, seed, ncomp=1, dirichlet="all", amp=0.2):
    m = P.mesh.jittered_box_mesh(grid, extent, amp, seed)
    sp = P.fespace.build_space(m, p, ncomp)
    if dirichlet is not None:
        sp.constraints = P.fespace.dirichlet_constraints(sp, dirichlet)
    return sp


def test_single_cell_q1_all_constrained(pkg):
    """Every DoF constrained: A = identity-out, diag = 1, the transfer has no
    points (prolongation and restriction are zero)."""
    sc = _space(pkg, (1, 1), UNIT2, 1, 1)
    sf = _space(pkg, (1, 1), UNIT2, 1, 2)
    op = pkg.mfoperator.LaplaceOperator(sf)
    u = np.random.default_rng(0).standard_normal(sf.n_dofs)
    assert np.array_equal(op.apply(u), u)  # zero-in / identity-out
    assert np.array_equal(op.diagonal(), np.ones(sf.n_dofs))
    T = pkg.transfer.setup_nonnested(sc, sf)
    assert len(T.point_dofs) == 0
    assert np.array_equal(T.prolongate(np.ones(sc.n_dofs)), np.zeros(sf.n_dofs))
    assert np.array_equal(T.restrict(np.ones(sf.n_dofs)), np.zeros(sc.n_dofs))


def test_zero_rhs_solve_and_vcycle(pkg):
    meshes = [pkg.mesh.jittered_box_mesh(g, UNIT3, 0.2, 90 + i) for i, g in enumerate([(2, 2, 2), (4, 4, 4)])]
    H = pkg.multigrid.build_hp_hierarchy(meshes, 2)
    b = np.zeros(H.finest.operator.n_dofs)
    assert np.array_equal(H.precondition(b), b)
    res = pkg.solvers.cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-8)
    assert res.converged and res.iterations == 0 and np.array_equal(res.x, b)  # solvers.py:141-142


def test_coarse_finer_than_fine_and_single_cell_fine(pkg, oracle):
    """Coarse 6x5 cells, fine ONE cell (Q3): most coarse cells own no point."""
    sc = _space(pkg, (6, 5), UNIT2, 2, 3)
    sf = _space(pkg, (1, 1), UNIT2, 2, 4, amp=0.0)
    T = pkg.transfer.setup_nonnested(sc, sf)
    oc = oracle.make_space(oracle.jittered_mesh((6, 5), UNIT2, 0.2, 3), 2)
    of = oracle.make_space(oracle.jittered_mesh((1, 1), UNIT2, 0.0, 4), 2)
    OT = oracle.OTransfer(oc, of)
    rng = np.random.default_rng(5)
    r, u = rng.standard_normal(sf.n_dofs), rng.standard_normal(sc.n_dofs)
    assert np.allclose(T.restrict(r), OT.restrict(r), rtol=0, atol=1e-13)
    assert np.allclose(T.prolongate(u), OT.prolongate(u), rtol=0, atol=1e-13)


def test_coarse_solver_with_no_free_dofs(pkg):
    sp = _space(pkg, (1, 1), UNIT2, 1, 7)
    cs = pkg.solvers.CoarseSolver(pkg.mfoperator.LaplaceOperator(sp))
    b = np.arange(1.0, sp.n_dofs + 1)
    assert np.allclose(cs.solve(b), b)  # A = I on constrained rows


def test_elasticity_single_cell_clamped(pkg, oracle):
    sp = _space(pkg, (1, 1, 1), UNIT3, 2, 8, ncomp=3, dirichlet=[0])
    op = pkg.mfoperator.ElasticityOperator(sp, 1.0, 1.0)
    osp = oracle.make_space(oracle.jittered_mesh((1, 1, 1), UNIT3, 0.2, 8), 2, 3, [0])
    oop = oracle.OOperator(osp, "elasticity", 1.0, 1.0)
    u = np.random.default_rng(9).standard_normal(sp.n_dofs)
    want = oop.apply(u)
    assert np.linalg.norm(op.apply(u) - want) <= 1e-11 * np.linalg.norm(want)
