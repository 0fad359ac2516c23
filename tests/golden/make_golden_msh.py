"""Unstructured ingestion fixtures: meshes written by the
REFERENCE's ``write_msh`` (mesh.py:448-474) and the reference's outputs on
the meshes its ``read_msh`` (mesh.py:477-569) returns.

Run in the build container (the reference exists only here):

    python tests/golden/make_golden_msh.py

Writes ``tests/golden/msh_<name>.msh`` (the files) and
``tests/golden/mshref_<name>.npz`` (reference read_msh arrays, DoF numbering,
constraints, applies, diagonal; for the hierarchy case the V-cycle of the load
vector and the PCG iteration count).
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as mg  # noqa: E402,F401  (puts the reference on sys.path)

from nnmg.fespace import build_space, dirichlet_constraints  # noqa: E402
from nnmg.mesh import generate_hypercube, generate_lshape, generate_perturbed, read_msh, write_msh  # noqa: E402
from nnmg.mfoperator import ElasticityOperator, LaplaceOperator, assemble_rhs  # noqa: E402
from nnmg.multigrid import HierarchyConfig, build_hp_hierarchy  # noqa: E402
from nnmg.solvers import cg_solve  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def mesh_arrays(m):
    return {"vertices": m.vertices, "cells": m.cells, "faces": m.boundary_faces}


def op_case(name, mesh, p, problem="poisson", dirichlet="all", lame=(1.0, 1.0)):
    path = os.path.join(OUT, f"msh_{name}.msh")
    write_msh(mesh, path)
    m = read_msh(path)
    ncomp = m.dim if problem == "elasticity" else 1
    sp = build_space(m, p, n_components=ncomp)
    if dirichlet is not None:
        sp.constraints = dirichlet_constraints(sp, dirichlet)
    op = LaplaceOperator(sp) if problem == "poisson" else ElasticityOperator(sp, *lame)
    U = np.random.default_rng(0).standard_normal((2, sp.n_dofs))
    out = {"p": p, "problem": problem, "dirichlet": str(dirichlet), "lame": np.array(lame),
           "cell_dofs": sp.cell_dofs, "support": sp.support_points, "cdofs": sp.constraints.dofs,
           "apply": np.stack([op.apply(u) for u in U]), "diag": op.diagonal()}
    out.update(mesh_arrays(m))
    np.savez_compressed(os.path.join(OUT, f"mshref_{name}.npz"), **out)
    print("msh op", name, sp.n_dofs)


def hierarchy_case(name, meshes, p):
    paths = []
    for l, mesh in enumerate(meshes):
        path = os.path.join(OUT, f"msh_{name}_l{l}.msh")
        write_msh(mesh, path)
        paths.append(path)
    ms = [read_msh(path) for path in paths]
    H = build_hp_hierarchy(ms, degree=p, config=HierarchyConfig(chebyshev_degree=4))
    b = assemble_rhs(H.finest.space, f=1.0)
    z = H.precondition(b)
    res = cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-8)
    out = {"p": p, "n_levels": len(ms), "rhs": b, "vcycle": z, "iterations": res.iterations,
           "x": res.x, "lam_max": np.array([lev.smoother.lam_max for lev in H.levels])}
    for i, T in enumerate(H.transfers):
        out[f"t{i}_cells"] = T.cells
        out[f"t{i}_point_dofs"] = T.point_dofs
    for l, m in enumerate(ms):
        out[f"l{l}_cell_dofs"] = H.levels[l].space.cell_dofs
    np.savez_compressed(os.path.join(OUT, f"mshref_{name}.npz"), **out)
    print("msh hierarchy", name, [lev.operator.n_dofs for lev in H.levels], "its", res.iterations)


def main():
    # L-shape (2D, cells removed: not a full tensor grid), Q2 Laplace
    op_case("lshape_q2", generate_lshape(2, 2, 1), 2)
    # perturbed 3D cube, Q3 Laplace, and vector Q2 elasticity clamped on face 0
    cube = generate_perturbed(generate_hypercube(3, (-1.0, 1.0), 2), 0.1, seed=3)
    op_case("cube_q3", cube, 3)
    op_case("cube_el_q2", cube, 2, "elasticity", [0], (0.5769, 0.3846))
    # non-nested 2D hierarchy from three independently perturbed msh meshes
    meshes = [generate_perturbed(generate_hypercube(2, (-1.0, 1.0), r), 0.3 * 2.0 ** -r, seed=10 + r)
              for r in (2, 3, 5)]
    hierarchy_case("h2d_q2", meshes, 2)


if __name__ == "__main__":
    main()
