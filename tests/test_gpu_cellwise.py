"""GPU nested / polynomial transfers and hp / nested hierarchies against the
reference's own outputs (tests/golden/make_golden_cellwise.py).

The reference builds these transfers as per-cell embeddings with claim masks
(transfer.py:127-251); the GPU package builds them on the point-evaluation
kernels (the same operator for nested Lagrange spaces, see transfer.py here).
Tolerances as everywhere: 1e-11 relative l2 per transfer, V-cycle 1e-9, CG
iterations +-1."""

import numpy as np
import pytest

from conftest import dirichlet_arg, golden, golden_names

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


def _mesh(P, g, prefix):
    v = g[f"{prefix}_vertices"]
    return P.mesh.Mesh(v.shape[1], v, g[f"{prefix}_cells"], g[f"{prefix}_faces"], validate=False)


def _space(P, mesh, p, ncomp, dirichlet):
    sp = P.fespace.build_space(mesh, p, ncomp)
    if dirichlet is not None:
        sp.constraints = P.fespace.dirichlet_constraints(sp, dirichlet)
    return sp


@pytest.mark.parametrize("name", golden_names("trc_"))
def test_cellwise_transfer_matches_reference(pkg, name):
    g = golden(name)
    kind, pc, pf, nc = str(g["kind"]), int(g["pc"]), int(g["pf"]), int(g["ncomp"])
    d = dirichlet_arg(g["dirichlet"])
    mc = _mesh(pkg, g, "coarse")
    mf = mc if kind == "poly" else _mesh(pkg, g, "fine")
    sc, sf = _space(pkg, mc, pc, nc, d), _space(pkg, mf, pf, nc, d)
    ops = {}
    if nc > 1:
        ops = {"coarse_operator": pkg.mfoperator.ElasticityOperator(sc, 1.0, 1.0),
               "fine_operator": pkg.mfoperator.ElasticityOperator(sf, 1.0, 1.0)}
    T = pkg.transfer.setup_polynomial(sc, sf, **ops) if kind == "poly" else pkg.transfer.setup_nested(sc, sf, **ops)
    rng = np.random.default_rng(1)
    uc = rng.standard_normal((3, sc.n_dofs))
    rf = rng.standard_normal((3, sf.n_dofs))
    for u, want in zip(uc, g["prolongate"]):
        assert rel(T.prolongate(u), want) <= TOL
    for r, want in zip(rf, g["restrict"]):
        got = T.restrict(r)
        assert rel(got, want) <= TOL
        assert np.array_equal(got, T.restrict(r))


def test_cellwise_transfer_argument_checks(pkg):
    g = golden("trc_poly_2d_q1q2")
    m = _mesh(pkg, g, "coarse")
    s1, s2, s3 = (_space(pkg, m, p, 1, "all") for p in (1, 2, 3))
    with pytest.raises(ValueError):  # degree must drop by exactly one (transfer.py:233-234)
        pkg.transfer.setup_polynomial(s1, s3)
    with pytest.raises(ValueError):  # fine degree >= 2 (transfer.py:265-266)
        pkg.transfer.setup_polynomial(s1, s1)
    m2 = _mesh(pkg, g, "fine")
    with pytest.raises(ValueError):  # one shared mesh (transfer.py:231-232)
        pkg.transfer.setup_polynomial(s1, _space(pkg, m2, 2, 1, "all"))
    with pytest.raises(ValueError):  # nested keeps the degree (transfer.py:176-177)
        pkg.transfer.setup_nested(s1, s2)


@pytest.mark.parametrize("name", golden_names("mgc_"))
def test_hp_and_nested_hierarchies_match_reference(pkg, name):
    g = golden(name)
    meshes = [_mesh(pkg, g, f"m{i}") for i in range(int(g["n_meshes"]))]
    H = pkg.multigrid.build_hp_hierarchy(meshes, int(g["degree"]), mode=str(g["mode"]), nested=bool(g["nested"]),
                                         config=pkg.multigrid.HierarchyConfig(chebyshev_degree=4))  # as generated
    assert [lev.space.degree for lev in H.levels] == list(g["degrees"])
    assert [lev.operator.n_dofs for lev in H.levels] == list(g["n_dofs"])
    b = pkg.mfoperator.assemble_rhs(H.finest.space, 1.0)
    assert rel(b, g["rhs"]) <= 1e-13
    lam = np.array([lev.smoother.lam_max for lev in H.levels])
    assert np.allclose(lam[1:], g["lam_max"][1:], rtol=1e-9)
    z = H.precondition(b)
    assert rel(z, g["vcycle"]) <= 1e-9
    res = pkg.solvers.cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-8)
    assert res.converged and abs(res.iterations - int(g["iterations"])) <= 1
    assert rel(res.x, g["x"]) <= 1e-7
