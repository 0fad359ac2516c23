"""Split apply of the distributed levels ("overlap interior
cells with the exchange"): ``nnmg_level_apply_begin`` + ``nnmg_level_apply_cells``
over complementary cell-block ranges must reproduce ``nnmg_level_apply``
(mfoperator.py:108-122, 171-202) on every operator golden, and the
world-size-1 distributed level (interior cells on the compute stream, ghost
import on a side stream, fork / join captured in the cycle's CUDA graph) must
match the single-GPU operator."""

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


def operator_of(P, g, **kw):
    v = g["mesh_vertices"]
    m = P.mesh.Mesh(v.shape[1], v, g["mesh_cells"], g["mesh_faces"], validate=False)
    problem = str(g["problem"])
    sp = P.fespace.build_space(m, int(g["p"]), v.shape[1] if problem == "elasticity" else 1)
    d = dirichlet_arg(g["dirichlet"])
    if d is not None:
        sp.constraints = P.fespace.dirichlet_constraints(sp, d)
    op = (P.mfoperator.ElasticityOperator(sp, *g["lame"], **kw) if problem == "elasticity"
          else P.mfoperator.LaplaceOperator(sp, **kw))
    return sp, op


@pytest.mark.parametrize("name", golden_names("op_"))
def test_split_apply_equals_apply_and_reference(P, name):
    g = golden(name)
    sp, op = operator_of(P, g)
    nb = op.n_cell_blocks
    assert nb == -(-sp.mesh.n_cells // op.info()["cells_per_block"])
    u = torch.from_numpy(np.random.default_rng(0).standard_normal(sp.n_dofs)).cuda()
    want = torch.empty_like(u)
    op.apply_into(u, want)
    for cut in sorted({0, nb // 3, nb // 2, nb}):
        v = torch.full_like(u, 7.0)  # begin overwrites everything
        op.apply_begin_into(u, v)
        op.apply_cells_into(u, v, cut, nb)  # boundary range first: the pieces commute
        op.apply_cells_into(u, v, 0, cut)
        assert rel(v.cpu().numpy(), want.cpu().numpy()) <= 1e-14
        assert rel(v.cpu().numpy(), g["apply"][0]) <= 1e-11
        # residual form r -= A u in place (the distributed smoother's pieces)
        f = torch.from_numpy(np.random.default_rng(3).standard_normal(sp.n_dofs)).cuda()
        r = f.clone()
        op.apply_begin_into(u, r, negate=True)
        op.apply_cells_into(u, r, 0, cut, negate=True)
        op.apply_cells_into(u, r, cut, nb, negate=True)
        assert rel((f - r).cpu().numpy(), want.cpu().numpy()) <= 1e-13
    # constrained rows: identity-out from begin alone, untouched by the cell pieces
    cd = np.asarray(sp.constraints.dofs)
    if len(cd):
        v = torch.empty_like(u)
        op.apply_begin_into(u, v)
        vh = v.cpu().numpy()
        assert np.array_equal(vh[cd], u.cpu().numpy()[cd])
        free = np.ones(sp.n_dofs, bool)
        free[cd] = False
        assert not vh[free].any()


def test_split_apply_argument_checks(P):
    g = golden(golden_names("op_")[0])
    sp, op = operator_of(P, g)
    u = torch.zeros(sp.n_dofs, dtype=torch.float64, device="cuda")
    v = torch.zeros_like(u)
    with pytest.raises(ValueError):
        op.apply_cells_into(u, v, 0, op.n_cell_blocks + 1)
    with pytest.raises(ValueError):
        op.apply_cells_into(u, v, 2, 1)
    with pytest.raises(ValueError):
        op.apply_cells_into(u, u, 0, 1)
    sp2, det = operator_of(P, g, deterministic=True)
    with pytest.raises(Exception):  # status 3: unsupported in deterministic mode
        det.apply_cells_into(u, v, 0, 1)
