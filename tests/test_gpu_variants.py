"""Every kernel variant the library can select (environment switches read at
handle creation) against the reference fixtures and the CPU oracle.

The defaults are tuned per configuration on B200; the alternatives stay
selectable for measurement, so each one must meet the same parity bar
(1e-11 relative l2, bit-exact determinism of the restriction)."""

import numpy as np
import pytest

from conftest import dirichlet_arg, golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

TOL = 1e-11


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2412_10910_b200 as P

    return P


def _space(P, g, prefix="mesh", ncomp=1, dirichlet="all", p=None):
    v = g[f"{prefix}_vertices"]
    m = P.mesh.Mesh(v.shape[1], v, g[f"{prefix}_cells"], g[f"{prefix}_faces"], validate=False)
    sp = P.fespace.build_space(m, int(g["p"]) if p is None else p, ncomp)
    if dirichlet is not None:
        sp.constraints = P.fespace.dirichlet_constraints(sp, dirichlet)
    return sp


# (fixture, environment) pairs: register / pencil / split / shared-memory geometry
APPLY_VARIANTS = [
    ("op_3d_q2", {"NNMG_APPLY_KERNEL": "pencil"}),
    ("op_3d_q2", {"NNMG_REG_MINB": "3"}),
    ("op_2d_q2", {"NNMG_APPLY_KERNEL": "pencil"}),
    ("op_3d_el_q2", {"NNMG_APPLY_KERNEL": "pencil"}),
    ("op_3d_el_q2", {"NNMG_APPLY_KERNEL": "pencil", "NNMG_APPLY_SPLIT": "2"}),
    ("op_3d_el_q1", {"NNMG_APPLY_KERNEL": "pencil"}),
    ("op_3d_el_q2", {"NNMG_ELAST_RECOMPUTE": "1"}),
    ("op_3d_el_q2", {"NNMG_ELAST_RECOMPUTE": "0"}),
    ("op_3d_el_q2", {"NNMG_ELAST_TMA": "1"}),
    ("op_3d_el_q2", {"NNMG_ELAST_TMA": "0"}),
    ("op_ref_cube3d_el", {"NNMG_ELAST_TMA": "1"}),
    ("op_3d_el_q1", {"NNMG_ELAST_TMA": "1"}),
    ("op_3d_el_q2", {"NNMG_ELAST_XNB": "1"}),
    ("op_3d_el_q1", {"NNMG_ELAST_XNB": "1"}),
    ("op_ref_cube3d_el", {"NNMG_ELAST_XNB": "1"}),
    ("op_3d_el_q2", {"NNMG_ELAST_XNB": "0"}),
    ("op_3d_el_q2", {"NNMG_ELAST_BLN": "1"}),
    ("op_3d_el_q2", {"NNMG_ELAST_BLN": "1", "NNMG_ELAST_TMA": "1"}),
    ("op_3d_el_q1", {"NNMG_ELAST_BLN": "1"}),
    ("op_ref_cube3d_el", {"NNMG_ELAST_BLN": "1"}),
    ("op_ref_cube3d_el", {"NNMG_ELAST_RECOMPUTE": "1"}),
    ("op_3d_q4", {"NNMG_APPLY_RECOMPUTE": "0"}),
    ("op_3d_q4", {"NNMG_APPLY_RECOMPUTE": "0", "NNMG_APPLY_SPLIT": "1"}),
    ("op_3d_q4", {"NNMG_APPLY_RECOMPUTE": "1", "NNMG_APPLY_SPLIT": "4"}),
    ("op_3d_q4", {"NNMG_APPLY_RECOMPUTE": "1", "NNMG_APPLY_SPLIT": "2"}),
    ("op_3d_q4", {"NNMG_APPLY_RECOMPUTE": "1", "NNMG_APPLY_SPLIT": "1"}),
    ("op_3d_q3", {"NNMG_APPLY_RECOMPUTE": "0"}),
    ("op_3d_q3", {"NNMG_APPLY_RECOMPUTE": "1", "NNMG_APPLY_SPLIT": "2"}),
    ("op_3d_q2", {"NNMG_RECOMPUTE_MOD": "2"}),
    ("op_3d_q2", {"NNMG_REG_RECOMPUTE": "1"}),
    ("op_3d_q2", {"NNMG_REG_TMA": "1"}),
    ("op_3d_q1", {"NNMG_REG_TMA": "1"}),
    ("op_3d_q1", {"NNMG_REG_RECOMPUTE": "1"}),
    ("op_3d_q4", {"NNMG_APPLY_RECOMPUTE": "0", "NNMG_APPLY_GEOS": "1", "NNMG_APPLY_SPLIT": "4"}),
    ("op_3d_q4", {"NNMG_APPLY_RECOMPUTE": "0", "NNMG_APPLY_GEOS": "1", "NNMG_APPLY_SPLIT": "8"}),
    ("op_3d_q3", {"NNMG_APPLY_RECOMPUTE": "0", "NNMG_APPLY_GEOS": "1", "NNMG_APPLY_SPLIT": "4"}),
    # x-adjacent cells of a warp share their face nodes (shuffles instead of gathers / atomics)
    ("op_3d_q2", {"NNMG_REG_XNB": "1"}),
    ("op_3d_q1", {"NNMG_REG_XNB": "1"}),
    ("op_2d_q2", {"NNMG_REG_XNB": "1"}),
    ("op_2d_q1", {"NNMG_REG_XNB": "1"}),
    ("op_2d_q3", {"NNMG_REG_XNB": "1"}),
    ("op_3d_q2_neumann", {"NNMG_REG_XNB": "1"}),
    ("op_ref_lshape_q2", {"NNMG_REG_XNB": "1"}),
    ("op_3d_q2", {"NNMG_REG_XNB": "2"}),
    ("op_3d_q2_neumann", {"NNMG_REG_XNB": "2"}),
    ("op_2d_q2", {"NNMG_REG_XNB": "2"}),
    ("op_2d_q2", {"NNMG_REG_XNB": "0"}),
    ("op_2d_q1", {"NNMG_REG_XNB": "0"}),
    # constrained rows by the separate copy / subtract kernels instead of the cell kernels' prologue
    ("op_3d_q2", {"NNMG_FUSE_CONSTRAINED": "0"}),
    ("op_2d_q2", {"NNMG_FUSE_CONSTRAINED": "0"}),
    ("op_3d_el_q2", {"NNMG_FUSE_CONSTRAINED": "0"}),
]


@pytest.mark.parametrize("name,env", APPLY_VARIANTS, ids=[f"{n}-{'-'.join(f'{k[5:]}={v}' for k, v in e.items())}"
                                                          for n, e in APPLY_VARIANTS])
def test_apply_variant_matches_reference(pkg, monkeypatch, name, env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = golden(name)
    problem = str(g["problem"])
    dim = g["mesh_vertices"].shape[1]
    sp = _space(pkg, g, ncomp=dim if problem == "elasticity" else 1, dirichlet=dirichlet_arg(g["dirichlet"]))
    op = (pkg.mfoperator.ElasticityOperator(sp, *tuple(g["lame"])) if problem == "elasticity"
          else pkg.mfoperator.LaplaceOperator(sp))
    U = np.random.default_rng(0).standard_normal((len(g["apply"]), sp.n_dofs))
    for u, want in zip(U, g["apply"]):
        assert rel(op.apply(u), want) <= TOL


def _transfer(pkg, g):
    p, ncomp = int(g["p"]), int(g["ncomp"])
    dirichlet = dirichlet_arg(g["dirichlet"])
    sc = _space(pkg, g, "coarse", ncomp, dirichlet, p)
    sf = _space(pkg, g, "fine", ncomp, dirichlet, p)
    eps_box = None if float(g["eps_box"]) < 0 else float(g["eps_box"])
    search = pkg.geosearch.SearchConfig(eps_box=eps_box)
    if ncomp == 1:
        return sc, sf, pkg.transfer.setup_nonnested(sc, sf, search)
    cop = pkg.mfoperator.ElasticityOperator(sc, 1.0, 1.0)
    fop = pkg.mfoperator.ElasticityOperator(sf, 1.0, 1.0)
    return sc, sf, pkg.transfer.setup_nonnested(sc, sf, search, coarse_operator=cop, fine_operator=fop)


# restriction: lane-owned local vector with 1 / 2 / 3 points per lane and
# round (0 / 1 / 3), shared-memory staged groups (2); several cell chunks
RESTRICT_VARIANTS = [(n, k, c) for n in ("tr_3d_q2", "tr_2d_q2", "tr_2d_q1") for k in ("0", "1", "2", "3")
                     for c in ("1", "3")] + [(n, "1", c) for n in ("tr_3d_el_q2", "tr_3d_q4_warp", "tr_2d_q3_free")
                                             for c in ("1", "2", "5")]


@pytest.mark.parametrize("name,kernel,chunk", RESTRICT_VARIANTS)
def test_transfer_variant_matches_reference(pkg, monkeypatch, name, kernel, chunk):
    monkeypatch.setenv("NNMG_RESTRICT_KERNEL", kernel)
    monkeypatch.setenv("NNMG_RESTRICT_CHUNK", chunk)
    g = golden(name)
    sc, sf, T = _transfer(pkg, g)
    rng = np.random.default_rng(1)
    uc = rng.standard_normal((3, sc.n_dofs))
    rf = rng.standard_normal((3, sf.n_dofs))
    for u, want in zip(uc, g["prolongate"]):
        assert rel(T.prolongate(u), want) <= TOL
    for r, want in zip(rf, g["restrict"]):
        got = T.restrict(r)
        assert rel(got, want) <= TOL
        assert np.array_equal(got, T.restrict(r))  # deterministic, bitwise


@pytest.mark.parametrize("wide", ["0", "1"])
@pytest.mark.parametrize("name,chunk", [("tr_3d_el_q2", c) for c in ("1", "3", "6")])
def test_restriction_wide_lane_matches_reference(pkg, monkeypatch, name, chunk, wide):
    """32 < NLOC*NCOMP <= 81 (3D Q2 elasticity: 81 outputs, three 32-output
    tiles in the cell-end reduction): the lane-owned local vector with the tiled cell-end reduction
    (NNMG_RESTRICT_WIDE=1) against the staged groups, both against the reference."""
    monkeypatch.setenv("NNMG_RESTRICT_WIDE", wide)
    monkeypatch.setenv("NNMG_RESTRICT_CHUNK", chunk)
    g = golden(name)
    sc, sf, T = _transfer(pkg, g)
    rng = np.random.default_rng(1)
    rng.standard_normal((3, sc.n_dofs))  # the golden draws the coarse inputs first
    rf = rng.standard_normal((3, sf.n_dofs))
    for r, want in zip(rf, g["restrict"]):
        got = T.restrict(r)
        assert rel(got, want) <= TOL
        assert np.array_equal(got, T.restrict(r))


@pytest.mark.parametrize("pl", ["1", "2"])
@pytest.mark.parametrize("name,chunk,maxp", [("tr_3d_el_q2", "1", None), ("tr_3d_el_q2", "4", "64"),
                                             ("tr_3d_q4_warp", "1", None), ("tr_3d_q4_warp", "3", "64")])
def test_restriction_planes_per_lane_matches_reference(pkg, monkeypatch, name, chunk, maxp, pl):
    """Staged restriction with one or two planes of the outermost axis per
    lane (NNMG_RESTRICT_PL): slots of ceil(N1 / PL) lanes share a staged point."""
    monkeypatch.setenv("NNMG_RESTRICT_PL", pl)
    monkeypatch.setenv("NNMG_RESTRICT_CHUNK", chunk)
    if maxp:
        monkeypatch.setenv("NNMG_TRANSFER_MAXP", maxp)
    g = golden(name)
    sc, sf, T = _transfer(pkg, g)
    rng = np.random.default_rng(1)
    rng.standard_normal((3, sc.n_dofs))  # the golden draws the coarse inputs first
    rf = rng.standard_normal((3, sf.n_dofs))
    for r, want in zip(rf, g["restrict"]):
        got = T.restrict(r)
        assert rel(got, want) <= TOL
        assert np.array_equal(got, T.restrict(r))


@pytest.mark.parametrize("name,maxp,kernel", [(n, m, k) for n in ("tr_3d_q2", "tr_3d_q4_warp", "tr_3d_el_q2", "tr_2d_q2")
                                               for m in ("32", "64") for k in ("1", "2")])
def test_transfer_split_cells_match_reference(pkg, monkeypatch, name, maxp, kernel):
    """Coarse cells split into work items of at most `maxp` points (small
    levels): partial local vectors per item, summed in the fixed-order gather."""
    monkeypatch.setenv("NNMG_TRANSFER_MAXP", maxp)
    monkeypatch.setenv("NNMG_RESTRICT_KERNEL", kernel)
    g = golden(name)
    sc, sf, T = _transfer(pkg, g)
    rng = np.random.default_rng(1)
    uc = rng.standard_normal((3, sc.n_dofs))
    rf = rng.standard_normal((3, sf.n_dofs))
    for u, want in zip(uc, g["prolongate"]):
        assert rel(T.prolongate(u), want) <= TOL
    for r, want in zip(rf, g["restrict"]):
        got = T.restrict(r)
        assert rel(got, want) <= TOL
        assert np.array_equal(got, T.restrict(r))


@pytest.mark.parametrize("kernel,chunk", [("1", "1"), ("1", "4"), ("2", "3"), ("0", "7")])
def test_restriction_with_pointless_coarse_cells(pkg, oracle, monkeypatch, kernel, chunk):
    """A coarse mesh finer than the fine one: most coarse cells own no fine
    point, so their partial local vectors must be written as zeros."""
    monkeypatch.setenv("NNMG_RESTRICT_KERNEL", kernel)
    monkeypatch.setenv("NNMG_RESTRICT_CHUNK", chunk)
    ext = ((0.0, 1.0), (0.0, 1.0))
    mc = pkg.mesh.jittered_box_mesh((9, 7), ext, 0.2, 77)
    mf = pkg.mesh.jittered_box_mesh((3, 2), ext, 0.2, 78)
    sc, sf = pkg.fespace.build_space(mc, 2), pkg.fespace.build_space(mf, 2)
    sc.constraints = pkg.fespace.dirichlet_constraints(sc, "all")
    sf.constraints = pkg.fespace.dirichlet_constraints(sf, "all")
    T = pkg.transfer.setup_nonnested(sc, sf)
    oc = oracle.make_space(oracle.jittered_mesh((9, 7), ext, 0.2, 77), 2)
    of = oracle.make_space(oracle.jittered_mesh((3, 2), ext, 0.2, 78), 2)
    OT = oracle.OTransfer(oc, of)
    assert np.array_equal(T.cells, OT.cells)
    rng = np.random.default_rng(3)
    for _ in range(2):
        r = rng.standard_normal(sf.n_dofs)
        u = rng.standard_normal(sc.n_dofs)
        assert rel(T.restrict(r), OT.restrict(r)) <= TOL
        assert rel(T.prolongate(u), OT.prolongate(u)) <= TOL


# device-resident coarse Jacobi-PCG (solvers.py:193-206): owner-warp and
# dot-product variants against the oracle CG (same iterations +-1, residual)
COARSE_VARIANTS = [{"NNMG_COARSE_OWNER_WARPS": "0", "NNMG_COARSE_ATOMIC_DOTS": "1"},
                   {"NNMG_COARSE_OWNER_WARPS": "1", "NNMG_COARSE_ATOMIC_DOTS": "1"},
                   {"NNMG_COARSE_OWNER_WARPS": "0", "NNMG_COARSE_ATOMIC_DOTS": "0"},
                   {"NNMG_COARSE_OWNER_WARPS": "1", "NNMG_COARSE_ATOMIC_DOTS": "0"}]


@pytest.mark.parametrize("name", ["op_2d_q2", "op_3d_q2", "op_3d_el_q2", "op_3d_q4"])
@pytest.mark.parametrize("env", COARSE_VARIANTS, ids=lambda e: "ow{}-atomic{}".format(
    e["NNMG_COARSE_OWNER_WARPS"], e["NNMG_COARSE_ATOMIC_DOTS"]))
def test_coarse_cg_variants_match_oracle(pkg, oracle, monkeypatch, name, env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = golden(name)
    problem = str(g["problem"])
    dim = g["mesh_vertices"].shape[1]
    ncomp = dim if problem == "elasticity" else 1
    d = dirichlet_arg(g["dirichlet"])
    sp = _space(pkg, g, ncomp=ncomp, dirichlet=d)
    op = (pkg.mfoperator.ElasticityOperator(sp, *tuple(g["lame"])) if problem == "elasticity"
          else pkg.mfoperator.LaplaceOperator(sp))
    cs = pkg.solvers.CoarseSolver(op, dense_limit=0)
    b = np.random.default_rng(7).standard_normal(sp.n_dofs)
    x = cs.solve(b)
    its, conv = cs.status()[:2]
    assert conv
    assert np.linalg.norm(b - op.apply(x)) <= 1.1e-8 * np.linalg.norm(b)
    om = oracle.OMesh(dim, g["mesh_vertices"], g["mesh_cells"], g["mesh_faces"])
    osp = oracle.make_space(om, int(g["p"]), ncomp, d)
    oop = oracle.OOperator(osp, problem, *tuple(g["lame"]))
    oc = oracle.OCoarse(oop, dense_limit=0)
    xo = oc.solve(b)
    assert abs(its - oc.last_iterations) <= 1, (its, oc.last_iterations)
    assert rel(x, xo) <= 1e-6
