"""Generate tests/golden/rhs_*.npz: reference load vectors with body loads
and Neumann boundary terms (mfoperator.py:313-414), by running the REFERENCE.

    python tests/golden/make_golden_rhs.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import OUT, mesh_arrays, ref_jittered  # noqa: E402  (puts the reference on sys.path)

from nnmg.fespace import build_space, dirichlet_constraints  # noqa: E402
from nnmg.mfoperator import assemble_rhs  # noqa: E402

# the callables are restated by name in tests/test_rhs.py
G = {
    "xn": lambda x, n: (x * n).sum(axis=1),
    "sin": lambda x, n: np.sin(3.0 * x[:, 0]) + x[:, 1] ** 2,
    "vec": lambda x, n: np.stack([n[:, 0] + x[:, 1], 0.5 * n[:, 1], -x[:, 0] * n[:, -1]], axis=1),
}
F = {
    "poly": lambda x: 1.0 + x[:, 0] * x[:, 1],
    "down": lambda x: np.tile(np.array([0.0, 0.0, -1.0]), (len(x), 1)),
}


def case(name, mesh, p, ncomp, dirichlet, f, neumann):
    sp = build_space(mesh, p, ncomp)
    if dirichlet is not None:
        sp.constraints = dirichlet_constraints(sp, dirichlet)
    fv = F[f] if isinstance(f, str) else f
    nv = {bid: (G[g] if isinstance(g, str) and g in G else g) for bid, g in neumann.items()}
    b = assemble_rhs(sp, f=fv, neumann=nv)
    out = {"p": p, "ncomp": ncomp, "dirichlet": str(dirichlet), "f": str(f), "b": b,
           "neumann_ids": np.array(list(neumann.keys())),
           "neumann_vals": np.array([repr(v) for v in neumann.values()])}
    out.update(mesh_arrays("mesh", mesh))
    np.savez_compressed(os.path.join(OUT, f"rhs_{name}.npz"), **out)
    print("rhs", name, sp.n_dofs, float(np.linalg.norm(b)))


def main():
    case("2d_q2", ref_jittered((5, 4), [(0, 1), (0, 1)], 0.2, 71), 2, 1, [0, 2], "poly", {1: 1.5, 3: "sin"})
    case("3d_q1", ref_jittered((3, 3, 2), [(0, 1)] * 3, 0.2, 72), 1, 1, [0], 1.0, {1: "xn", 5: -2.0})
    case("3d_el_q2", ref_jittered((4, 1, 1), [(0, 4), (0, 1), (0, 1)], 0.2, 73), 2, 3, [0], "down",
         {1: ("normal", -0.7), 3: "vec"})
    case("2d_q3_neumann_only", ref_jittered((3, 3), [(0, 1), (0, 1)], 0.2, 74), 3, 1, None, None, {0: "xn", 2: 0.25})


if __name__ == "__main__":
    main()
