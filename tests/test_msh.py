"""Unstructured ingestion on the host: ``read_msh`` /
``write_msh`` (reference mesh.py:448-569) against the reference's own reading
of files its ``write_msh`` produced (tests/golden/make_golden_msh.py), the
generic DoF numbering on those meshes, and the reference's msh tests
(test_mesh.py:162-205) restated."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, golden

CASES = ["lshape_q2", "cube_q3", "cube_el_q2"]


@pytest.fixture(scope="module")
def M():
    from paper_2412_10910_b200 import mesh

    return mesh


@pytest.mark.parametrize("name", CASES)
def test_read_msh_matches_reference(M, name):
    g = golden("mshref_" + name)
    m = M.read_msh(os.path.join(GOLDEN, f"msh_{name}.msh"))
    assert m.grid is None  # unstructured: generic numbering path
    assert np.array_equal(m.vertices, g["vertices"])
    assert np.array_equal(m.cells, g["cells"])
    assert np.array_equal(m.boundary_faces, g["faces"])


@pytest.mark.parametrize("name", CASES)
def test_generic_numbering_on_msh_meshes(M, name):
    from conftest import dirichlet_arg
    from paper_2412_10910_b200 import fespace

    g = golden("mshref_" + name)
    m = M.read_msh(os.path.join(GOLDEN, f"msh_{name}.msh"))
    ncomp = m.dim if str(g["problem"]) == "elasticity" else 1
    sp = fespace.build_space(m, int(g["p"]), ncomp)
    sp.constraints = fespace.dirichlet_constraints(sp, dirichlet_arg(g["dirichlet"]))
    assert np.array_equal(sp.cell_dofs, g["cell_dofs"])
    assert np.array_equal(sp.support_points, g["support"])
    assert np.array_equal(sp.constraints.dofs, g["cdofs"])


def test_hierarchy_meshes_number_like_reference(M):
    from paper_2412_10910_b200 import fespace

    g = golden("mshref_h2d_q2")
    for l in range(int(g["n_levels"])):
        m = M.read_msh(os.path.join(GOLDEN, f"msh_h2d_q2_l{l}.msh"))
        assert np.array_equal(fespace.build_space(m, int(g["p"])).cell_dofs, g[f"l{l}_cell_dofs"])


def test_roundtrip_identity(M, tmp_path):
    for m in [M.structured_box_mesh((2, 2), [(-1, 1), (-1, 1)]),
              M.jittered_box_mesh((4, 4), [(-1, 1), (-1, 1)], 0.2, 5),
              M.structured_box_mesh((2, 2, 2), [(0, 2)] * 3)]:
        path = tmp_path / "m.msh"
        M.write_msh(m, path)
        back = M.read_msh(path)
        assert np.array_equal(back.vertices, m.vertices)
        assert np.array_equal(back.cells, m.cells)
        assert np.array_equal(back.boundary_faces, m.boundary_faces)


def test_single_quad_and_errors(M, tmp_path):
    head = "$MeshFormat\n2.2 0 8\n$EndMeshFormat\n"
    p = tmp_path / "one.msh"
    p.write_text(head + "$Nodes\n4\n1 0 0 0\n2 1 0 0\n3 1 1 0\n4 0 1 0\n$EndNodes\n"
                 "$Elements\n1\n1 3 2 0 1 1 2 3 4\n$EndElements\n")
    m = M.read_msh(p)
    assert m.n_cells == 1 and m.n_vertices == 4 and m.dim == 2
    assert sorted(m.boundary_faces[:, 1].tolist()) == [0, 1, 2, 3] and set(m.boundary_faces[:, 2]) == {0}
    p.write_text(head + "$Nodes\n3\n1 0 0 0\n2 1 0 0\n3 0 1 0\n$EndNodes\n"
                 "$Elements\n1\n1 2 2 0 1 1 2 3\n$EndElements\n")
    with pytest.raises(M.MeshError, match="unsupported element type"):
        M.read_msh(p)
    p.write_text(head + "$Nodes\nnot-a-number\n$EndNodes\n")
    with pytest.raises(M.MeshError):
        M.read_msh(p)
    p.write_text(head + "$Nodes\n1\n1 0 0 0\n")
    with pytest.raises(M.MeshError, match="missing"):
        M.read_msh(p)
    p.write_text(head + "$Nodes\n4\n1 0 0 0\n2 1 0 0\n3 1 1 0\n4 0 1 0\n$EndNodes\n"
                 "$Elements\n2\n1 1 2 7 1 1 3\n2 3 2 0 2 1 2 3 4\n$EndElements\n")
    with pytest.raises(M.MeshError, match="boundary element"):
        M.read_msh(p)
