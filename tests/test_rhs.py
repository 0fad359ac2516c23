"""Load vectors with body loads and Neumann boundary terms (host setup,
mfoperator.py:313-414) against the reference's own outputs
(tests/golden/make_golden_rhs.py).  CPU only: assemble_rhs is NumPy host code."""

import numpy as np
import pytest

from conftest import dirichlet_arg, golden, golden_names

# the callables of make_golden_rhs.py
G = {
    "xn": lambda x, n: (x * n).sum(axis=1),
    "sin": lambda x, n: np.sin(3.0 * x[:, 0]) + x[:, 1] ** 2,
    "vec": lambda x, n: np.stack([n[:, 0] + x[:, 1], 0.5 * n[:, 1], -x[:, 0] * n[:, -1]], axis=1),
}
F = {
    "poly": lambda x: 1.0 + x[:, 0] * x[:, 1],
    "down": lambda x: np.tile(np.array([0.0, 0.0, -1.0]), (len(x), 1)),
    "1.0": 1.0,
    "None": None,
}


def _value(s):
    s = str(s)
    if s.startswith("'") and s.strip("'") in G:
        return G[s.strip("'")]
    if s.startswith("("):
        kind, mag = s.strip("()").split(",")
        return (kind.strip().strip("'"), float(mag))
    return float(s)


@pytest.mark.parametrize("name", golden_names("rhs_"))
def test_assemble_rhs_with_neumann_matches_reference(name):
    from paper_2412_10910_b200 import fespace, mesh, mfoperator

    g = golden(name)
    v = g["mesh_vertices"]
    m = mesh.Mesh(v.shape[1], v, g["mesh_cells"], g["mesh_faces"], validate=False)
    sp = fespace.build_space(m, int(g["p"]), int(g["ncomp"]))
    d = dirichlet_arg(g["dirichlet"])
    if d is not None:
        sp.constraints = fespace.dirichlet_constraints(sp, d)
    neumann = {int(i): _value(s) for i, s in zip(g["neumann_ids"], g["neumann_vals"])}
    b = mfoperator.assemble_rhs(sp, f=F[str(g["f"])], neumann=neumann)
    want = g["b"]
    assert np.linalg.norm(b - want) <= 1e-13 * max(1.0, np.linalg.norm(want))


def test_neumann_unknown_boundary_id_raises():
    from paper_2412_10910_b200 import fespace, mesh, mfoperator

    g = golden("rhs_2d_q2")
    v = g["mesh_vertices"]
    m = mesh.Mesh(v.shape[1], v, g["mesh_cells"], g["mesh_faces"], validate=False)
    sp = fespace.build_space(m, 2, 1)
    with pytest.raises(ValueError):
        mfoperator.assemble_rhs(sp, f=1.0, neumann={99: 1.0})
