"""Host-side setup of the GPU path vs the reference (golden) and the oracle:
mesh generation, DoF numbering (closed form and generic), constraints.  CPU only."""

import numpy as np
import pytest

from conftest import dirichlet_arg, golden, golden_names
from paper_2412_10910_b200 import fespace as F
from paper_2412_10910_b200 import mesh as M
from paper_2412_10910_b200.configs import CONFIGS, get_config


def product_mesh(g, prefix="mesh"):
    v = g[f"{prefix}_vertices"]
    return M.Mesh(v.shape[1], v, g[f"{prefix}_cells"], g[f"{prefix}_faces"], validate=False)


@pytest.mark.parametrize("name", golden_names("op_"))
def test_generic_numbering_matches_reference(name):
    g = golden(name)
    m = product_mesh(g)
    ncomp = m.dim if str(g["problem"]) == "elasticity" else 1
    sp = F.build_space(m, int(g["p"]), ncomp)
    sp.constraints = F.dirichlet_constraints(sp, dirichlet_arg(g["dirichlet"])) if str(g["dirichlet"]) != "None" \
        else F.DirichletConstraints()
    assert np.array_equal(sp.cell_dofs, g["cell_dofs"])
    assert np.array_equal(sp.constraints.dofs, g["cdofs"])
    assert np.abs(sp.support_points - g["support"]).max() <= 1e-14


@pytest.mark.parametrize("name", [n for n in golden_names("op_") if not n.startswith("op_ref")])
def test_structured_numbering_matches_reference(name):
    """Rebuild the SURVEY-recipe mesh with the structured generator: the
    closed-form numbering must equal the reference's geometric matching."""
    g = golden(name)
    v = g["mesh_vertices"]
    dim = v.shape[1]
    lo, hi = v.min(axis=0), v.max(axis=0)
    cells = g["mesh_cells"]
    # grid from the lexicographic vertex strides of the first cell
    nvx = int(cells[0][2])
    nv = [nvx] + ([int(cells[0][4]) // nvx] if dim == 3 else [])
    nv.append(len(v) // int(np.prod(nv)))
    grid = [n - 1 for n in nv]
    base = M.structured_box_mesh(grid, [(0.0, 1.0)] * dim, validate=False)
    assert np.array_equal(base.cells, cells)
    m = M.Mesh(dim, v, cells, g["mesh_faces"], grid=grid, validate=False)
    ncomp = dim if str(g["problem"]) == "elasticity" else 1
    sp = F.build_space(m, int(g["p"]), ncomp)
    assert np.array_equal(sp.cell_dofs, g["cell_dofs"])
    assert np.abs(sp.support_points - g["support"]).max() <= 1e-14
    assert np.array_equal(base.boundary_faces, g["mesh_faces"])


@pytest.mark.parametrize("cname", sorted(CONFIGS))
def test_config_meshes_match_oracle_recipe(oracle, cname):
    cfg = get_config(cname)
    for l, m in enumerate(cfg.make_meshes(scale=8, validate=True)):
        om = oracle.jittered_mesh(m.grid, cfg.extent, cfg.amplitude, 1000 * cfg.index + l + 1, cfg.warp)
        assert np.array_equal(m.vertices, om.vertices)
        assert np.array_equal(m.cells, om.cells)
        assert np.array_equal(m.boundary_faces, om.boundary_faces)


@pytest.mark.parametrize("tag", ["C1_full", "C2_s8", "C3_s8", "C4_s4", "C5_s8"])
def test_config_meshes_match_golden_hierarchies(tag):
    """Product meshes + numbering reproduce the reference hierarchy's sizes."""
    g = golden("mg_" + tag)
    cfg = get_config(tag[:2])
    ncomp = cfg.dim if cfg.problem == "elasticity" else 1
    for l, row in enumerate(g["grids"]):
        grid = tuple(int(x) for x in row[: cfg.dim])
        from paper_2412_10910_b200.mesh import jittered_box_mesh, sine_warp

        m = jittered_box_mesh(grid, cfg.extent, cfg.amplitude, 1000 * cfg.index + l + 1,
                              sine_warp if cfg.warp else None)
        sp = F.build_space(m, cfg.degree, ncomp)
        assert sp.n_dofs == int(g["n_dofs"][l])


def test_dirichlet_unknown_id_rejected():
    m = M.structured_box_mesh((2, 2), [(0, 1), (0, 1)])
    sp = F.build_space(m, 1)
    with pytest.raises(ValueError):
        F.dirichlet_constraints(sp, [42])


def test_shape1d_matches_oracle(oracle):
    for p in (1, 2, 3, 4):
        t = np.linspace(-0.1, 1.1, 17)
        s = F.Shape1D(p)
        assert np.array_equal(s.values(t), oracle.shape_values(p, t))
        assert np.abs(s.derivatives(t) - oracle.shape_derivatives(p, t)).max() <= 1e-12
        assert np.abs(s.values(s.nodes) - np.eye(p + 1)).max() <= 1e-14
