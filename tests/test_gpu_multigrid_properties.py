"""V-cycle properties of the GPU hierarchy, restated from the reference's
multigrid tests (pkg/tests/test_multigrid.py:13-115) on this package: single
level = coarse solve, level-independent contraction, linearity, zero input,
symmetry, hp-level structure, nested sanity iteration counts and the
equivalence of nested and non-nested transfers on nested meshes."""

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


def nested_meshes(P, dim, n_levels, extent=(-1.0, 1.0)):
    """generate_hypercube(dim, extent, r) for r < n_levels (mesh.py:357-363)"""
    return [P.mesh.structured_box_mesh((2**r,) * dim, [extent] * dim) for r in range(n_levels)]


def test_single_level_equals_coarse_solve(pkg):
    H = pkg.multigrid.build_hp_hierarchy(nested_meshes(pkg, 2, 1), 2)
    b = pkg.mfoperator.assemble_rhs(H.finest.space, f=1.0)
    assert np.array_equal(H.v_cycle(b), H.coarse_solver.solve(b))


@pytest.mark.parametrize("n_levels", [2, 3, 4])
def test_v_cycle_contraction_level_independent(pkg, n_levels):
    rng = np.random.default_rng(0)
    H = pkg.multigrid.build_hp_hierarchy(nested_meshes(pkg, 2, n_levels), 1)
    op = H.finest.operator
    free = ~H.finest.space.constrained_mask()
    x_exact = rng.standard_normal(op.n_dofs) * free
    x = H.v_cycle(op.apply(x_exact))

    def a_norm(v):
        return np.sqrt(abs(v @ op.apply(v)))

    assert a_norm(x_exact - x) / a_norm(x_exact) < 0.2


def test_v_cycle_linear_and_zero(pkg):
    H = pkg.multigrid.build_hp_hierarchy(nested_meshes(pkg, 2, 3), 2)
    rng = np.random.default_rng(1)
    n = H.finest.operator.n_dofs
    f, g = rng.standard_normal(n), rng.standard_normal(n)
    lhs = H.v_cycle(0.7 * f - 2.3 * g)
    rhs = 0.7 * H.v_cycle(f) - 2.3 * H.v_cycle(g)
    assert np.abs(lhs - rhs).max() <= 1e-12 * max(1, np.abs(rhs).max())
    z = H.precondition(np.zeros(n))
    assert np.array_equal(z, np.zeros_like(z))


def test_preconditioner_symmetry_probe(pkg):
    H = pkg.multigrid.build_hp_hierarchy(nested_meshes(pkg, 2, 3), 2)
    rng = np.random.default_rng(2)
    n = H.finest.operator.n_dofs
    for _ in range(20):
        u, v = rng.standard_normal(n), rng.standard_normal(n)
        mu, mv = H.precondition(u), H.precondition(v)
        scale = np.linalg.norm(mu) * np.linalg.norm(v) + np.linalg.norm(u) * np.linalg.norm(mv)
        assert abs(mu @ v - u @ mv) <= 1e-9 * scale


def test_hp_hierarchy_structure_and_h_only(pkg):
    meshes = nested_meshes(pkg, 2, 3)
    H = pkg.multigrid.build_hp_hierarchy(meshes, 3, mode="hp", nested=True)
    assert [lev.space.degree for lev in H.levels] == [1, 2, 3, 3, 3]
    lm = [lev.space.mesh for lev in H.levels]
    assert lm[0] is meshes[0] and lm[1] is meshes[0] and lm[2] is meshes[0]
    assert lm[3] is meshes[1] and lm[4] is meshes[2]
    H1 = pkg.multigrid.build_hp_hierarchy(nested_meshes(pkg, 2, 1), 2, mode="h")
    assert H1.n_levels == 1 and not H1.transfers


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_nested_sanity_iteration_counts(pkg, p):
    H = pkg.multigrid.build_hp_hierarchy(nested_meshes(pkg, 2, 4), p, nested=True)
    b = pkg.mfoperator.assemble_rhs(H.finest.space, f=1.0)
    res = pkg.solvers.cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-4)
    assert res.converged and 2 <= res.iterations <= 4


@pytest.mark.parametrize("p", [1, 3])
def test_nested_equivalence_paths(pkg, p):
    counts, sols = [], []
    meshes = nested_meshes(pkg, 2, 4)
    for nested in (True, False):
        H = pkg.multigrid.build_hp_hierarchy(meshes, p, nested=nested)
        b = pkg.mfoperator.assemble_rhs(H.finest.space, f=1.0)
        res = pkg.solvers.cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-4)
        counts.append(res.iterations)
        sols.append(res.x)
    assert counts[0] == counts[1]
    assert np.linalg.norm(sols[0] - sols[1]) <= 1e-10 * max(1, np.linalg.norm(sols[0]))
