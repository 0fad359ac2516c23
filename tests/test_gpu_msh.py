"""Unstructured meshes through the GPU path: ``read_msh`` ->
generic numbering -> GPU operators / non-nested hierarchy, against the
reference's outputs on the same msh files (tests/golden/make_golden_msh.py)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, dirichlet_arg, golden

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


@pytest.mark.parametrize("name", ["lshape_q2", "cube_q3", "cube_el_q2"])
def test_msh_operator_matches_reference(P, name):
    g = golden("mshref_" + name)
    m = P.mesh.read_msh(os.path.join(GOLDEN, f"msh_{name}.msh"))
    problem = str(g["problem"])
    ncomp = m.dim if problem == "elasticity" else 1
    sp = P.fespace.build_space(m, int(g["p"]), ncomp)
    sp.constraints = P.fespace.dirichlet_constraints(sp, dirichlet_arg(g["dirichlet"]))
    assert np.array_equal(sp.cell_dofs, g["cell_dofs"])
    op = (P.mfoperator.ElasticityOperator(sp, *g["lame"]) if problem == "elasticity"
          else P.mfoperator.LaplaceOperator(sp))
    U = np.random.default_rng(0).standard_normal((len(g["apply"]), sp.n_dofs))
    for u, want in zip(U, g["apply"]):
        assert rel(op.apply(u), want) <= 1e-11
    assert rel(op.diagonal(), g["diag"]) <= 1e-12


def test_msh_hierarchy_matches_reference(P):
    g = golden("mshref_h2d_q2")
    meshes = [P.mesh.read_msh(os.path.join(GOLDEN, f"msh_h2d_q2_l{l}.msh")) for l in range(int(g["n_levels"]))]
    H = P.multigrid.build_hp_hierarchy(meshes, int(g["p"]), config=P.multigrid.HierarchyConfig(chebyshev_degree=4))
    for i, T in enumerate(H.transfers):
        assert np.array_equal(T.point_dofs, g[f"t{i}_point_dofs"])
        assert np.array_equal(T.cells, g[f"t{i}_cells"])
    assert np.allclose([lev.smoother.lam_max for lev in H.levels], g["lam_max"], rtol=1e-9)
    b = P.mfoperator.assemble_rhs(H.finest.space, 1.0)
    assert rel(b, g["rhs"]) <= 1e-13
    # the GPU body-load kernel on an unstructured mesh
    assert rel(H.finest.operator.load_vector(1.0).cpu().numpy(), g["rhs"]) <= 1e-12
    assert rel(H.precondition(b), g["vcycle"]) <= 1e-9
    res = P.solvers.cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-8)
    assert res.converged and abs(res.iterations - int(g["iterations"])) <= 1
    assert rel(res.x, g["x"]) <= 1e-7
