"""Parity at the BASELINE full sizes (C3: 16.97M DoFs, C5: 6.5M DoFs).

The CPU oracle cannot run these sizes whole, so the GPU path is checked on
sampled rows against the oracle restricted to the touched cells, plus
size-independent properties: symmetry, exact transpose, bitwise determinism
of the restriction, V-cycle symmetry, and CG convergence to 1e-8."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module", params=["C3", "C5"])
def full(request):
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2412_10910_b200 import configs, mfoperator, multigrid

    cfg = configs.get_config(request.param)
    meshes = cfg.make_meshes(scale=1, validate=False)
    H = multigrid.build_hp_hierarchy(meshes, cfg.degree, problem=cfg.problem, dirichlet_ids=cfg.dirichlet_ids,
                                     lame=cfg.lame,
                                     config=multigrid.HierarchyConfig(chebyshev_degree=cfg.chebyshev_degree))
    b = H.finest.operator.load_vector(cfg.body_force if cfg.body_force else 1.0)
    yield cfg, H, b
    del H
    torch.cuda.empty_cache()


def test_fullsize_apply_sampled_rows_vs_oracle(full, oracle):
    cfg, H, _ = full
    op = H.finest.operator
    sp = H.finest.space
    n = op.n_dofs
    rng = np.random.default_rng(0)
    u = rng.standard_normal(n)
    v = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    rows = np.concatenate([rng.choice(n, 150, replace=False), sp.constraints.dofs[:10]])
    want = oracle.sampled_apply_rows(sp.mesh.vertices, sp.mesh.cells, np.asarray(sp.cell_dofs), sp.constraints.dofs,
                                     sp.degree, rows, u, cfg.problem, *(cfg.lame or (1.0, 1.0)),
                                     ncomp=sp.n_components)
    assert rel(v[rows], want) <= 1e-11


def test_fullsize_apply_symmetry(full):
    _, H, _ = full
    op = H.finest.operator
    rng = np.random.default_rng(4)
    u = torch.from_numpy(rng.standard_normal(op.n_dofs)).cuda()
    w = torch.from_numpy(rng.standard_normal(op.n_dofs)).cuda()
    au, aw = op.apply(u), op.apply(w)
    lhs, rhs = float(torch.dot(au, w)), float(torch.dot(u, aw))
    assert abs(lhs - rhs) <= 1e-11 * float(au.norm() * w.norm())


def test_fullsize_transfer_sampled_and_transpose(full, oracle):
    cfg, H, _ = full
    T = H.transfers[-1]
    sc, sf = T.coarse_space, T.fine_space
    ncomp = sf.n_components
    rng = np.random.default_rng(1)
    uc = rng.standard_normal(sc.n_dofs)
    uf = T.prolongate(torch.from_numpy(uc).cuda()).cpu().numpy()
    pick = rng.choice(len(T.point_dofs), 2000, replace=False)
    want = oracle.sampled_prolongate(np.asarray(sc.cell_dofs), sc.constraints.dofs, sc.degree, sc.mesh.dim,
                                     T.cells[pick], T.xhat[pick], uc, ncomp)
    got = uf.reshape(-1, ncomp)[T.point_dofs[pick]]
    assert rel(got, want) <= 1e-11
    # exact transpose: (P u).r == u.(P^T r)
    r = torch.from_numpy(rng.standard_normal(sf.n_dofs)).cuda()
    u = torch.from_numpy(uc).cuda()
    a = float(torch.dot(T.prolongate(u), r))
    rc = T.restrict(r)
    b = float(torch.dot(u, rc))
    assert abs(a - b) <= 1e-12 * float(u.norm() * r.norm())
    assert torch.equal(rc, T.restrict(r))  # deterministic restriction, bitwise


def test_fullsize_vcycle_symmetry_and_solve(full):
    cfg, H, b = full
    n = H.finest.operator.n_dofs
    rng = np.random.default_rng(2)
    u = torch.from_numpy(rng.standard_normal(n)).cuda()
    w = torch.from_numpy(rng.standard_normal(n)).cuda()
    # symmetrised inputs: constrained entries zero (the V-cycle acts on residuals)
    cd = torch.from_numpy(H.finest.space.constraints.dofs).cuda()
    u[cd] = 0.0
    w[cd] = 0.0
    mu, mw = H.precondition(u), H.precondition(w)
    lhs, rhs = float(torch.dot(mu, w)), float(torch.dot(u, mw))
    assert abs(lhs - rhs) <= 1e-9 * (float(mu.norm() * w.norm()) + float(u.norm() * mw.norm()))
    from paper_2412_10910_b200 import solvers

    res = solvers.cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-8)
    assert res.converged and res.iterations <= 14
    x = res.x
    r = b - H.finest.operator.apply(x)
    assert float(r.norm()) <= 1.01e-8 * float(b.norm())
