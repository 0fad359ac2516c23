"""Smoother, coarse-solver and transfer properties restated from the
reference's tests (pkg/tests/test_solvers.py:67-97, 160-169;
test_transfer.py:192-205) on the GPU objects."""

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


UNIT2 = [(-1.0, 1.0), (-1.0, 1.0)]


def _laplace(P, cells, p, oracle=None, seed=None):
    m = (P.mesh.structured_box_mesh((cells, cells), UNIT2) if seed is None
         else P.mesh.jittered_box_mesh((cells, cells), UNIT2, 0.2, seed))
    sp = P.fespace.build_space(m, p)
    sp.constraints = P.fespace.dirichlet_constraints(sp, "all")
    op = P.mfoperator.LaplaceOperator(sp)
    A = None
    if oracle is not None:
        om = (oracle.box_mesh((cells, cells), UNIT2) if seed is None
              else oracle.jittered_mesh((cells, cells), UNIT2, 0.2, seed))
        A = oracle.OOperator(oracle.make_space(om, p)).assemble_dense()
    return sp, op, A


def test_smoother_damps_high_frequency(pkg, oracle):
    """test_solvers.py:74-85: the highest mode of D^-1 A is reduced 5x by one
    degree-3 pass of the error propagation (b = 0)."""
    sp, op, A = _laplace(pkg, 6, 2, oracle, seed=11)
    s = pkg.solvers.ChebyshevJacobi(op, degree=3)
    d = np.diag(A)
    w, V = np.linalg.eigh(A / np.sqrt(d)[:, None] / np.sqrt(d)[None, :])
    v = V[:, -1] / np.sqrt(d)
    v /= np.linalg.norm(v)
    e = s.smooth(np.zeros(sp.n_dofs), x0=v.copy())
    assert np.linalg.norm(e) <= 0.2 * np.linalg.norm(v)


def test_smoother_linear_in_residual(pkg):
    """test_solvers.py:88-97: smooth(b, x0) == x0 + smooth(b - A x0)."""
    sp, op, _ = _laplace(pkg, 5, 2, seed=12)
    s = pkg.solvers.ChebyshevJacobi(op)
    rng = np.random.default_rng(0)
    free = ~sp.constrained_mask()
    for _ in range(5):
        b = rng.standard_normal(sp.n_dofs) * free
        x0 = rng.standard_normal(sp.n_dofs) * free
        direct = s.smooth(b, x0=x0.copy())
        shifted = x0 + s.smooth(b - op.apply(x0))
        assert np.abs(direct - shifted).max() <= 1e-11 * max(1, np.abs(direct).max())


def test_coarse_solver_single_free_dof(pkg, oracle):
    """test_solvers.py:160-169: one free DoF, x = b / a."""
    sp, op, A = _laplace(pkg, 2, 1, oracle)
    b = pkg.mfoperator.assemble_rhs(sp, f=1.0)
    x = pkg.solvers.CoarseSolver(op).solve(b)
    free = ~sp.constrained_mask()
    assert free.sum() == 1
    assert np.isclose(x[free][0], b[free][0] / A[free][:, free][0, 0], rtol=1e-13)


def test_transfer_locality(pkg):
    """test_transfer.py:192-205: P e_j touches only fine points located in
    coarse cells carrying DoF j."""
    ext = [(0.0, 1.0), (0.0, 1.0)]
    sc = pkg.fespace.build_space(pkg.mesh.jittered_box_mesh((3, 3), ext, 0.2, 21), 2)
    sf = pkg.fespace.build_space(pkg.mesh.jittered_box_mesh((7, 6), ext, 0.2, 22), 2)
    sc.constraints = pkg.fespace.dirichlet_constraints(sc, "all")
    sf.constraints = pkg.fespace.dirichlet_constraints(sf, "all")
    T = pkg.transfer.setup_nonnested(sc, sf)
    cd = np.asarray(sc.cell_dofs)
    cons = set(np.asarray(sc.constraints.dofs).tolist())
    for j in range(0, sc.n_dofs, 5):
        e = np.zeros(sc.n_dofs)
        e[j] = 1.0
        touched = np.abs(T.prolongate(e)) > 0
        allowed = np.zeros(sf.n_dofs, dtype=bool)
        if j not in cons:
            allowed[T.point_dofs[np.isin(T.cells, np.nonzero((cd == j).any(axis=1))[0])]] = True
        assert not np.any(touched & ~allowed)
