"""Direct coarsest-level solve (nnmg_coarse_direct_*, packed symmetric inverse
tiles) against the exact dense solve of the oracle's matrix, and its use in
hierarchies (CoarseSolver(direct=...), a documented deviation from the
reference's Jacobi-PCG, solvers.py:193-206)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2412_10910_b200 as P

    return P


def level(P, O, grid, p, problem="poisson", dirichlet="all", extent=None, seed=5):
    dim = len(grid)
    extent = extent or [(0.0, 1.0)] * dim
    ncomp = dim if problem == "elasticity" else 1
    m = P.mesh.jittered_box_mesh(grid, extent, 0.2, seed=seed)
    sp = P.fespace.build_space(m, p, ncomp)
    if dirichlet is not None:
        sp.constraints = P.fespace.dirichlet_constraints(sp, dirichlet)
    op = (P.mfoperator.ElasticityOperator(sp, 1.0, 1.0) if problem == "elasticity"
          else P.mfoperator.LaplaceOperator(sp))
    om = O.jittered_mesh(grid, extent, 0.2, seed)
    osp = O.make_space(om, p, ncomp, dirichlet)
    A = O.OOperator(osp, problem).assemble_dense() if problem == "elasticity" else O.OOperator(osp).assemble_dense()
    return sp, op, A


@pytest.mark.parametrize("case", [((30, 30), 2, "poisson", "all"),      # n = 3721: 59 tiles, padded
                                  ((5, 2, 2), 2, "elasticity", [0]),    # vector field, 825 DoFs
                                  ((3, 3), 1, "poisson", "all")])      # n = 16 < one tile
def test_direct_matches_dense_solve(pkg, oracle, case):
    grid, p, problem, dirichlet = case
    sp, op, A = level(pkg, oracle, grid, p, problem, dirichlet)
    cs = pkg.solvers.CoarseSolver(op, dense_limit=0, direct=True)
    assert cs.direct and cs.info()["kind"] == "direct"
    rng = np.random.default_rng(11)
    for _ in range(2):
        b = rng.standard_normal(sp.n_dofs)
        x = cs.solve(b)
        assert rel(x, np.linalg.solve(A, b)) <= 1e-10
    # bitwise reproducible (no atomics), symmetric operator
    bd = torch.from_numpy(b).cuda()
    x1 = torch.empty_like(bd)
    x2 = torch.empty_like(bd)
    cs.solve_into(bd, x1)
    cs.solve_into(bd, x2)
    assert torch.equal(x1, x2)
    c = rng.standard_normal(sp.n_dofs)
    lhs, rhs = float(np.dot(cs.solve(b), c)), float(np.dot(b, cs.solve(c)))
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(b) * np.linalg.norm(c) * np.linalg.norm(np.linalg.inv(A), 2)


def test_direct_singular_raises(pkg, oracle):
    sp, op, _ = level(pkg, oracle, (6, 6), 2, dirichlet=None)
    with pytest.raises(pkg.solvers.SingularCoarseSystemError):
        pkg.solvers.CoarseSolver(op, dense_limit=0, direct=True)


def test_auto_choice_and_bad_argument(pkg, oracle):
    sp, op, A = level(pkg, oracle, (30, 30), 2)
    cs = pkg.solvers.CoarseSolver(op, dense_limit=0, direct="auto")
    info = cs.info()
    assert info["kind"] in ("cg", "direct") and info["cg_s"] > 0 and info["direct_predicted_s"] > 0
    b = np.random.default_rng(1).standard_normal(sp.n_dofs)
    x = cs.solve(b)
    assert np.linalg.norm(A @ x - b) <= 1e-7 * np.linalg.norm(b)
    with pytest.raises(ValueError):
        pkg.solvers.CoarseSolver(op, direct="maybe")


def test_hierarchy_with_direct_coarse_converges_like_cg(pkg):
    """C2 at 1/4 scale has a 32^2 Q2 coarse level (3969 DoFs, above the
    dense limit): PCG iterations with the direct coarse solve equal the CG
    coarse solve's within 1."""
    from paper_2412_10910_b200 import configs, multigrid, solvers

    cfg = configs.get_config("C2")
    meshes = cfg.make_meshes(scale=2, validate=False)
    its = {}
    for mode in (False, True):
        H = multigrid.build_hp_hierarchy(meshes, cfg.degree, config=multigrid.HierarchyConfig(
            chebyshev_degree=4, coarse_direct=mode))
        assert H.coarse_solver.direct == mode
        b = H.finest.operator.load_vector(1.0)
        res = solvers.cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-8)
        assert res.converged
        its[mode] = res.iterations
        # the native executor and the Python recursion agree with the direct solve too
        z1 = H.v_cycle(b)
        z2 = H.v_cycle(b, executor=False)
        assert rel(z1.cpu().numpy(), z2.cpu().numpy()) <= 1e-12
    assert abs(its[True] - its[False]) <= 1


def test_mixed_cycle_uses_fp32_tile_coarse_solve(pkg):
    """The mixed-precision cycle attaches the packed inverse in fp32 tiles
    (nnmg_coarse_direct_create_f32) where the direct path is allowed: same
    outer iterations as the fp64 cycle, cycle within single-precision rounding
    of the fp64 one; the parity mode (coarse_direct=False) keeps one solver."""
    from paper_2412_10910_b200 import configs, multigrid, solvers

    cfg = configs.get_config("C2")
    meshes = cfg.make_meshes(scale=2, validate=False)
    H = multigrid.build_hp_hierarchy(meshes, cfg.degree, config=multigrid.HierarchyConfig(
        chebyshev_degree=4, coarse_direct=True))
    b = H.finest.operator.load_vector(1.0)
    z64 = H.v_cycle(b).cpu().numpy()
    r64 = solvers.cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-8)
    H.set_precision(32)
    assert H.coarse_solver._h32 is not None
    assert H.coarse_solver.info().get("mixed_direct_predicted_s", 0) > 0
    z32 = H.v_cycle(b).cpu().numpy()
    assert 0 < rel(z32, z64) <= 2e-4
    r32 = solvers.cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-8)
    assert r32.converged and abs(r32.iterations - r64.iterations) <= 1
    H.set_precision(64)
    assert rel(H.v_cycle(b).cpu().numpy(), z64) <= 1e-14  # the fp64 cycle keeps its own solver
    Hp = multigrid.build_hp_hierarchy(meshes, cfg.degree, config=multigrid.HierarchyConfig(
        chebyshev_degree=4, coarse_direct=False, vcycle_precision=32))
    Hp.v_cycle(b)
    assert Hp.coarse_solver._h32 is None and not Hp.coarse_solver.direct


@pytest.mark.parametrize("n_shares", [2, 3, 8])
def test_direct_tile_shares_add_up(pkg, oracle, n_shares):
    """Cell-partitioned runs split the inverse tiles across ranks
    (nnmg_coarse_direct_create_share): the shares' outputs add up to the full
    solve (identity rows from share 0 only), in a fixed order per share."""
    sp, op, A = level(pkg, oracle, (30, 30), 2)
    full = pkg.solvers.CoarseSolver(op, dense_limit=0, direct=True)
    parts = [pkg.solvers.CoarseSolver(op, dense_limit=0, direct=True, share=(i, n_shares)) for i in range(n_shares)]
    assert all(p.partial for p in parts) and not full.partial
    b = np.random.default_rng(3).standard_normal(sp.n_dofs)
    want = full.solve(b)
    got = sum(p.solve(b) for p in parts)
    assert rel(got, want) <= 1e-14
    assert rel(got, np.linalg.solve(A, b)) <= 1e-10
    cd = np.asarray(sp.constraints.dofs)
    assert np.array_equal(parts[0].solve(b)[cd], b[cd]) and not parts[1].solve(b)[cd].any()
    with pytest.raises(ValueError):
        pkg.solvers.CoarseSolver(op, dense_limit=0, direct=True, share=(2, 2))
