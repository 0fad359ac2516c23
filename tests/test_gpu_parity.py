"""GPU path vs the reference (golden fixtures) and the CPU oracle.

Tolerances (BASELINE.json north star): bit-exact index/map data, 1e-11
relative l2 for individual applies and transfers, CG iterations +-1 to a 1e-8
relative residual."""

import numpy as np
import pytest

from conftest import dirichlet_arg, golden, golden_names

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

APPLY_TOL = 1e-11


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2412_10910_b200 as P

    return P


def product_space(P, g, prefix="mesh", p=None, ncomp=1, dirichlet="all"):
    v = g[f"{prefix}_vertices"]
    m = P.mesh.Mesh(v.shape[1], v, g[f"{prefix}_cells"], g[f"{prefix}_faces"], validate=False)
    sp = P.fespace.build_space(m, int(g["p"]) if p is None else p, ncomp)
    if dirichlet is not None:
        sp.constraints = P.fespace.dirichlet_constraints(sp, dirichlet)
    return sp


def make_op(P, sp, problem, lame):
    if problem == "elasticity":
        return P.mfoperator.ElasticityOperator(sp, *lame)
    return P.mfoperator.LaplaceOperator(sp)


# ---------------------------------------------------------------------------
# operators (mfoperator.py:108-122, 171-202, 92-95)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", golden_names("op_"))
def test_apply_and_diagonal_match_reference(pkg, name):
    g = golden(name)
    problem = str(g["problem"])
    dim = g["mesh_vertices"].shape[1]
    sp = product_space(pkg, g, ncomp=dim if problem == "elasticity" else 1,
                       dirichlet=dirichlet_arg(g["dirichlet"]))
    assert np.array_equal(sp.cell_dofs, g["cell_dofs"])
    op = make_op(pkg, sp, problem, tuple(g["lame"]))
    U = np.random.default_rng(0).standard_normal((len(g["apply"]), sp.n_dofs))
    for u, want in zip(U, g["apply"]):
        u0 = u.copy()
        v = op.apply(u)
        assert isinstance(v, np.ndarray) and v.shape == u.shape
        assert np.array_equal(u, u0)  # input untouched
        assert rel(v, want) <= APPLY_TOL, rel(v, want)
    d = op.diagonal()
    assert np.abs(d - g["diag"]).max() <= 1e-12 * np.abs(g["diag"]).max()
    # device-tensor path returns a device tensor with the same values
    ud = torch.from_numpy(U[0]).cuda()
    vd = op.apply(ud)
    assert vd.is_cuda and rel(vd.cpu().numpy(), g["apply"][0]) <= APPLY_TOL


def test_apply_rejects_wrong_length(pkg):
    g = golden("op_2d_q2")
    op = make_op(pkg, product_space(pkg, g), "poisson", (1, 1))
    with pytest.raises(ValueError):
        op.apply(np.zeros(op.n_dofs + 1))


def test_operator_symmetry_probe_and_columns(pkg, oracle):
    # test_mfoperator.py:68-77, 90-100
    g = golden("op_3d_q2")
    sp = product_space(pkg, g)
    op = make_op(pkg, sp, "poisson", (1, 1))
    rng = np.random.default_rng(4)
    for _ in range(5):
        u, v = rng.standard_normal(sp.n_dofs), rng.standard_normal(sp.n_dofs)
        au, av = op.apply(u), op.apply(v)
        assert abs(au @ v - u @ av) <= 1e-11 * np.linalg.norm(au) * np.linalg.norm(v)
    osp = oracle.make_space(oracle.OMesh(3, g["mesh_vertices"], g["mesh_cells"], g["mesh_faces"]), 2, 1, "all")
    A = oracle.OOperator(osp).assemble_dense()
    from paper_2412_10910_b200.solvers import assemble_dense

    B = assemble_dense(op)
    assert np.abs(A - B).max() <= 1e-12 * np.abs(A).max()


def test_constant_in_kernel_and_rigid_modes(pkg):
    g = golden("op_3d_q2_neumann")
    op = make_op(pkg, product_space(pkg, g, dirichlet=None), "poisson", (1, 1))
    assert np.abs(op.apply(np.ones(op.n_dofs))).max() <= 1e-11 * np.abs(op.diagonal()).max()
    # rigid-body modes of free elasticity (test_mfoperator.py:195-205)
    g = golden("op_ref_cube3d_el")
    sp = product_space(pkg, g, ncomp=3, dirichlet=None)
    el = make_op(pkg, sp, "elasticity", (0.5769, 0.3846))
    pts = sp.support_points
    ns = sp.n_scalar_dofs
    modes = []
    for a in range(3):
        m = np.zeros((ns, 3))
        m[:, a] = 1.0
        modes.append(m.ravel())
    x, y, z = pts[:, 0], pts[:, 1], pts[:, 2]
    for cols in [(0 * x, z, -y), (-z, 0 * x, x), (y, -x, 0 * x)]:
        modes.append(np.stack(cols, axis=1).ravel())
    na = np.abs(el.diagonal()).max()
    for m in modes:
        assert np.linalg.norm(el.apply(m)) <= 1e-10 * na * np.linalg.norm(m)


# ---------------------------------------------------------------------------
# point location and transfers (geosearch.py:163-227, transfer.py:31-124)
# ---------------------------------------------------------------------------
def _transfer_setup(pkg, g):
    p, ncomp = int(g["p"]), int(g["ncomp"])
    d = dirichlet_arg(g["dirichlet"])
    sc = product_space(pkg, g, "coarse", p, ncomp, d)
    sf = product_space(pkg, g, "fine", p, ncomp, d)
    eps_box = None if float(g["eps_box"]) < 0 else float(g["eps_box"])
    search = pkg.geosearch.SearchConfig(eps_box=eps_box)
    if ncomp == 1:
        return sc, sf, pkg.transfer.setup_nonnested(sc, sf, search)
    cop = pkg.mfoperator.ElasticityOperator(sc, 1.0, 1.0)
    fop = pkg.mfoperator.ElasticityOperator(sf, 1.0, 1.0)
    return sc, sf, pkg.transfer.setup_nonnested(sc, sf, search, coarse_operator=cop, fine_operator=fop)


@pytest.mark.parametrize("name", golden_names("tr_"))
def test_transfer_matches_reference(pkg, name):
    g = golden(name)
    sc, sf, T = _transfer_setup(pkg, g)
    assert np.array_equal(T.point_dofs, g["point_dofs"])
    assert np.array_equal(T.cells, g["cells"])  # bit-exact owning cells
    assert np.array_equal(T.projected, g["projected"])
    assert np.abs(T.xhat - g["xhat"]).max() <= 1e-12
    rng = np.random.default_rng(1)
    uc = rng.standard_normal((3, sc.n_dofs))
    rf = rng.standard_normal((3, sf.n_dofs))
    for u, want in zip(uc, g["prolongate"]):
        assert rel(T.prolongate(u), want) <= APPLY_TOL
    for r, want in zip(rf, g["restrict"]):
        got = T.restrict(r)
        assert rel(got, want) <= APPLY_TOL
        assert np.array_equal(got, T.restrict(r))  # deterministic, bitwise
    # exact transpose (test_transfer.py:80-87)
    rng = np.random.default_rng(31)
    for _ in range(5):
        u, r = rng.standard_normal(sc.n_dofs), rng.standard_normal(sf.n_dofs)
        a, b = T.prolongate(u) @ r, u @ T.restrict(r)
        assert abs(a - b) <= 1e-12 * max(1.0, abs(a), np.linalg.norm(u) * np.linalg.norm(r))


def test_partition_of_unity_and_polynomial_reproduction(pkg):
    # test_transfer.py:115-138
    g = golden("tr_2d_q3_free")
    sc, sf, T = _transfer_setup(pkg, g)
    assert np.abs(T.prolongate(np.ones(sc.n_dofs)) - 1).max() <= 1e-12

    def poly(x):
        return (0.3 + x[:, 0]) ** 3 + (x[:, 1] - 0.1) ** 3 + x[:, 0] * x[:, 1]

    uf = T.prolongate(pkg.fespace.interpolate(sc, poly))
    assert np.abs(uf - pkg.fespace.interpolate(sf, poly)).max() <= 1e-11


def test_prolongate_accumulate_and_linearity(pkg):
    g = golden("tr_3d_q2")
    sc, sf, T = _transfer_setup(pkg, g)
    rng = np.random.default_rng(5)
    u, v = rng.standard_normal(sc.n_dofs), rng.standard_normal(sc.n_dofs)
    lhs = T.prolongate(0.37 * u - 1.25 * v)
    rhs = 0.37 * T.prolongate(u) - 1.25 * T.prolongate(v)
    assert np.abs(lhs - rhs).max() <= 1e-13 * max(1, np.abs(rhs).max())
    x = torch.from_numpy(rng.standard_normal(sf.n_dofs)).cuda()
    x0 = x.clone()
    T.prolongate_into(torch.from_numpy(u).cuda(), x, accumulate=True)
    assert rel((x - x0).cpu().numpy(), T.prolongate(u)) <= 1e-14
    assert np.array_equal(T.restrict(np.zeros(sf.n_dofs)), np.zeros(sc.n_dofs))


def test_transfer_timing_rows(pkg):
    # the reference's per-call rows (transfer.py:29, 43, 100-101, 122-123):
    # "calls" counts prolongations, both time rows grow on every public call,
    # and the _into calls of the V-cycle leave them alone (no events in a capture)
    g = golden("tr_3d_q2")
    sc, sf, T = _transfer_setup(pkg, g)
    assert T.timings == {"evaluate": 0.0, "gather_scatter": 0.0, "calls": 0}
    rng = np.random.default_rng(9)
    T.prolongate(rng.standard_normal(sc.n_dofs))
    t1 = dict(T.timings)
    assert t1["calls"] == 1 and t1["evaluate"] > 0.0 and t1["gather_scatter"] > 0.0
    T.restrict(rng.standard_normal(sf.n_dofs))
    t2 = dict(T.timings)
    assert t2["calls"] == 1 and t2["evaluate"] > t1["evaluate"] and t2["gather_scatter"] > t1["gather_scatter"]
    assert t2["evaluate"] < 1.0 and t2["gather_scatter"] < 1.0  # device seconds of two small kernels
    x = torch.zeros(sf.n_dofs, dtype=torch.float64, device="cuda")
    T.prolongate_into(torch.from_numpy(rng.standard_normal(sc.n_dofs)).cuda(), x)
    assert T.timings == t2


# ---------------------------------------------------------------------------
# smoother, CG, coarse solver, V-cycle, full solve (solvers.py, multigrid.py)
# ---------------------------------------------------------------------------
def _hierarchy(pkg, tag, timing=False):
    g = golden("mg_" + tag)
    cfg = pkg.configs.get_config(tag[:2])
    meshes = []
    for l, row in enumerate(g["grids"]):
        grid = tuple(int(x) for x in row[: cfg.dim])
        meshes.append(pkg.mesh.jittered_box_mesh(grid, cfg.extent, cfg.amplitude, 1000 * cfg.index + l + 1,
                                                 pkg.mesh.sine_warp if cfg.warp else None))
    eps_box = None if float(g["eps_box"]) < 0 else float(g["eps_box"])
    H = pkg.multigrid.build_hp_hierarchy(
        meshes, cfg.degree, problem=cfg.problem, dirichlet_ids=cfg.dirichlet_ids, lame=cfg.lame,
        search=pkg.geosearch.SearchConfig(eps_box=eps_box),
        config=pkg.multigrid.HierarchyConfig(chebyshev_degree=cfg.chebyshev_degree), timing=timing)
    b = pkg.mfoperator.assemble_rhs(H.finest.space, cfg.body_force if cfg.body_force else 1.0)
    return g, cfg, H, b


@pytest.mark.parametrize("tag", ["C1_full", "C2_s8", "C3_s8", "C4_s4", "C5_s8"])
def test_hierarchy_vcycle_and_solve_match_reference(pkg, tag):
    g, cfg, H, b = _hierarchy(pkg, tag)
    st = int(g["stride"])
    for i, T in enumerate(H.transfers):
        assert np.array_equal(T.cells, g[f"t{i}_cells"])
    lam = np.array([lev.smoother.lam_max for lev in H.levels])
    assert np.allclose(lam, g["lam_max"], rtol=1e-9), (lam, g["lam_max"])
    assert rel(b[::st], g["rhs"]) <= 1e-13
    # GPU body-load kernel (k_load_vector) vs the reference's assemble_rhs
    bl = H.finest.operator.load_vector(cfg.body_force if cfg.body_force else 1.0).cpu().numpy()
    assert rel(bl[::st], g["rhs"]) <= 1e-12
    z_exec = H.v_cycle(b, executor=True)
    z_py = H.v_cycle(b, executor=False)
    assert rel(z_exec[::st], g["vcycle"]) <= 1e-9
    assert rel(z_py, z_exec) <= 1e-12
    res = pkg.solvers.cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-8)
    assert res.converged
    assert abs(res.iterations - int(g["iterations"])) <= 1, (res.iterations, int(g["iterations"]))
    assert rel(res.x[::st], g["x"]) <= 1e-7
    if "coarse_random_iterations" in g:
        cs = H.coarse_solver
        rb = np.random.default_rng(2).standard_normal(cs.op.n_dofs)
        xc = cs.solve(rb)
        it, conv, indef = cs.status()
        assert conv and not indef
        assert abs(it - int(g["coarse_random_iterations"])) <= 1
        sc = max(1, cs.op.n_dofs // 8192)
        assert rel(xc[::sc], g["coarse_random_x"]) <= 1e-7


@pytest.mark.parametrize("smoother_residual,post", [("1", "1"), ("1", "0"), ("0", "1")])
def test_vcycle_timing_rows_and_graph_replay(pkg, monkeypatch, smoother_residual, post):
    """Native executor (residual from the smoother recurrence or f - A x
    explicitly; post-smoothing started from that residual or from a copy of
    f) and its graph replay against the Python recursion."""
    monkeypatch.setenv("NNMG_SMOOTHER_RESIDUAL", smoother_residual)
    monkeypatch.setenv("NNMG_POST_FROM_RESIDUAL", post)
    g, cfg, H, b = _hierarchy(pkg, "C2_s8", timing=True)
    H.v_cycle(b)
    comps = {(lvl, c) for lvl, c, _, _ in H.timing_rows()}
    assert (1, "coarse_solve") in comps
    for lvl in (2, 3):
        for c in pkg.multigrid.V_CYCLE_COMPONENTS:
            if c != "coarse_solve":
                assert (lvl, c) in comps
    H.timing = False
    f = torch.from_numpy(b).cuda()
    x1 = torch.empty_like(f)
    x2 = torch.empty_like(f)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        H.v_cycle_into(f, x1)
        H.v_cycle_into(f, x2)  # graph replay
    s.synchronize()
    assert rel(x1.cpu().numpy(), x2.cpu().numpy()) <= 1e-13
    assert rel(x1.cpu().numpy(), H.v_cycle(b, executor=False)) <= 1e-12
    assert H.kernels_per_cycle() > 10


def test_chebyshev_matches_oracle(pkg, oracle):
    g = golden("op_2d_q3")
    sp = product_space(pkg, g)
    op = make_op(pkg, sp, "poisson", (1, 1))
    sm = pkg.solvers.ChebyshevJacobi(op, degree=4)
    osp = oracle.make_space(oracle.OMesh(2, g["mesh_vertices"], g["mesh_cells"], g["mesh_faces"]), 3, 1, "all")
    oop = oracle.OOperator(osp)
    ocheb = oracle.OChebyshev(oop, 4)
    assert abs(sm.lam_max - ocheb.lam_max) <= 1e-9 * ocheb.lam_max
    ocheb.lam_max, ocheb.lam_min = sm.lam_max, sm.lam_min
    rng = np.random.default_rng(0)
    b, x0 = rng.standard_normal(sp.n_dofs), rng.standard_normal(sp.n_dofs)
    assert rel(sm.smooth(b), ocheb.smooth(b)) <= 1e-11
    assert rel(sm.smooth(b, x0=x0, n_sweeps=2), ocheb.smooth(b, x0, 2)) <= 1e-11
    assert np.array_equal(sm.smooth(np.zeros(sp.n_dofs)), np.zeros(sp.n_dofs))


def test_coarse_solver_dense_and_singular(pkg, oracle):
    g = golden("op_2d_q2")
    sp = product_space(pkg, g)
    op = make_op(pkg, sp, "poisson", (1, 1))
    cs = pkg.solvers.CoarseSolver(op)
    assert cs.dense
    b = np.random.default_rng(3).standard_normal(sp.n_dofs)
    osp = oracle.make_space(oracle.OMesh(2, g["mesh_vertices"], g["mesh_cells"], g["mesh_faces"]), 2, 1, "all")
    xr = np.linalg.solve(oracle.OOperator(osp).assemble_dense(), b)
    assert rel(cs.solve(b), xr) <= 1e-10
    # CG path on the same level
    cg = pkg.solvers.CoarseSolver(op, dense_limit=10)
    x = cg.solve(b)
    assert np.linalg.norm(b - op.apply(x)) <= 1e-7 * np.linalg.norm(b)
    # all-Neumann coarse system is singular (test_solvers.py:167-172)
    spn = product_space(pkg, g, dirichlet=None)
    with pytest.raises(pkg.solvers.SingularCoarseSystemError):
        pkg.solvers.CoarseSolver(make_op(pkg, spn, "poisson", (1, 1)))


def test_cg_indefinite_and_max_iter(pkg):
    g = golden("op_2d_q2")
    op = make_op(pkg, product_space(pkg, g), "poisson", (1, 1))
    b = np.ones(op.n_dofs)
    res = pkg.solvers.cg_solve(op, b, target_reduction=1e-14, max_iter=3)
    assert not res.converged and res.iterations == 3 and len(res.residual_norms) == 4

    class Neg:
        n_dofs = op.n_dofs
        device = op.device

        def apply(self, u):
            return -op.apply(u)

    with pytest.raises(pkg.solvers.IndefiniteOperatorError):
        pkg.solvers.cg_solve(Neg(), b)
