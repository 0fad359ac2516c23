"""Deterministic (atomic-free) summation, SURVEY §7 hard part 1 and the
reference's serial-order scatter (mfoperator.py:88-90): with
``deterministic=True`` every apply / diagonal / load vector sums the cell
contributions of each DoF in a fixed order (cell buffer + k_cell_gather), the
coarse solve is exact (packed inverse), the restriction is the fixed-order
two-phase one and the dots are fixed-order.  Results are then bitwise
reproducible run to run and across independently built hierarchies, and stay
within the parity tolerances of the reference."""

import numpy as np
import pytest

from conftest import dirichlet_arg, golden, golden_names

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2412_10910_b200 as P

    return P


def space_of(P, g):
    v = g["mesh_vertices"]
    m = P.mesh.Mesh(v.shape[1], v, g["mesh_cells"], g["mesh_faces"], validate=False)
    problem = str(g["problem"])
    sp = P.fespace.build_space(m, int(g["p"]), v.shape[1] if problem == "elasticity" else 1)
    d = dirichlet_arg(g["dirichlet"])
    if d is not None:
        sp.constraints = P.fespace.dirichlet_constraints(sp, d)
    return sp, problem


@pytest.mark.parametrize("name", golden_names("op_"))
def test_deterministic_apply_matches_reference_bitwise_repeatable(P, name):
    g = golden(name)
    sp, problem = space_of(P, g)
    kw = dict(deterministic=True)
    op = (P.mfoperator.ElasticityOperator(sp, *g["lame"], **kw) if problem == "elasticity"
          else P.mfoperator.LaplaceOperator(sp, **kw))
    U = np.random.default_rng(0).standard_normal((len(g["apply"]), sp.n_dofs))
    for u, want in zip(U, g["apply"]):
        v1 = op.apply(u)
        assert rel(v1, want) <= 1e-11
        assert np.array_equal(v1, op.apply(u))
    assert rel(op.diagonal(), g["diag"]) <= 1e-12
    # residual form (dst -= A src) through the smoother path: r = b - A x
    b = torch.from_numpy(U[0]).cuda()
    x = torch.from_numpy(U[-1]).cuda()
    r1, r2 = torch.empty_like(b), torch.empty_like(b)
    op.residual_into(b, x, r1)
    op.residual_into(b, x, r2)
    assert torch.equal(r1, r2)
    assert rel(r1.cpu().numpy(), U[0] - op.apply(U[-1])) <= 1e-13


@pytest.mark.parametrize("tag", ["C2_s8", "C3_s8", "C5_s8"])
def test_deterministic_hierarchy_bitwise_across_builds(P, tag):
    g = golden("mg_" + tag)
    cfg = P.configs.get_config(tag[:2])
    meshes = []
    for l, row in enumerate(g["grids"]):
        grid = tuple(int(x) for x in row[: cfg.dim])
        meshes.append(P.mesh.jittered_box_mesh(grid, cfg.extent, cfg.amplitude, 1000 * cfg.index + l + 1))
    out = []
    for _ in range(2):
        H = P.multigrid.build_hp_hierarchy(
            meshes, cfg.degree, problem=cfg.problem, dirichlet_ids=cfg.dirichlet_ids, lame=cfg.lame,
            config=P.multigrid.HierarchyConfig(chebyshev_degree=cfg.chebyshev_degree, deterministic=True))
        b = H.finest.operator.load_vector(cfg.body_force if cfg.body_force else 1.0)
        z1 = H.precondition(b)
        z2 = H.precondition(b)
        assert torch.equal(z1, z2)  # graph replays
        res = P.solvers.cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-8)
        out.append((b.clone(), z1.clone(), res.x.clone(), res.iterations, [lev.smoother.lam_max for lev in H.levels]))
        st = int(g["stride"])
        assert rel(b.cpu().numpy()[::st], g["rhs"]) <= 1e-12
        assert rel(z1.cpu().numpy()[::st], g["vcycle"]) <= 1e-9
        assert abs(res.iterations - int(g["iterations"])) <= 1
        del H
    (b1, z1, x1, i1, l1), (b2, z2, x2, i2, l2) = out
    assert torch.equal(b1, b2) and torch.equal(z1, z2) and torch.equal(x1, x2)
    assert i1 == i2 and l1 == l2
