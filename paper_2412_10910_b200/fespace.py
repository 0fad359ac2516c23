"""Continuous Q^p spaces: 1D Lagrange shapes, DoF numbering, Dirichlet constraints.

Host-side setup feeding the GPU path.  Semantics follow the reference
``nnmg.fespace`` (``/root/reference/pkg/src/nnmg/fespace.py``):

* Gauss-Legendre / Gauss-Lobatto rules on [0,1] (fespace.py:11-25);
* ``Shape1D`` Lagrange basis at the Lobatto nodes (fespace.py:28-71);
* global DoF ids by first occurrence in a cell-major, local-lexicographic scan
  (``build_space``, fespace.py:137-163).  For structured meshes the numbering
  is produced in closed form (bit-exact with the geometric matching, pinned by
  tests/test_setup_parity.py); other meshes use tolerance matching as the
  reference does;
* vector DoF = scalar DoF * n_components + component (fespace.py:125-131);
* ``dirichlet_constraints`` constrains every DoF whose support point lies on a
  face carrying a wanted boundary id (fespace.py:175-207).
"""

from __future__ import annotations

import numpy as np

from .mesh import tensor_points, vertex_bits


def gauss_legendre(n):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def gauss_lobatto(n):
    if n < 2:
        raise ValueError("need at least 2 points")
    t = np.linspace(0.0, 1.0, n)
    if n > 2:
        r = np.polynomial.legendre.Legendre.basis(n - 1).deriv(1).roots()
        t[1:-1] = 0.5 * (r + 1.0)
    return t


class Shape1D:
    """Degree-p Lagrange basis on the Gauss-Lobatto nodes of [0,1]."""

    def __init__(self, p):
        if p < 1:
            raise ValueError("degree must be >= 1")
        self.p = int(p)
        self.nodes = gauss_lobatto(p + 1)
        diff = self.nodes[:, None] - self.nodes[None, :]
        np.fill_diagonal(diff, 1.0)
        self._denom = diff.prod(axis=1)

    def values(self, t):
        t = np.atleast_1d(np.asarray(t, dtype=float))
        n = self.p + 1
        m = t[:, None] - self.nodes[None, :]
        out = np.empty((len(t), n))
        for i in range(n):
            keep = [j for j in range(n) if j != i]
            out[:, i] = m[:, keep].prod(axis=1) / self._denom[i]
        return out

    def derivatives(self, t):
        t = np.atleast_1d(np.asarray(t, dtype=float))
        n = self.p + 1
        m = t[:, None] - self.nodes[None, :]
        out = np.zeros((len(t), n))
        for i in range(n):
            for k in range(n):
                if k == i:
                    continue
                keep = [j for j in range(n) if j not in (i, k)]
                out[:, i] += m[:, keep].prod(axis=1) if keep else 1.0
            out[:, i] /= self._denom[i]
        return out


class DirichletConstraints:
    """Sorted constrained global DoFs with their values."""

    def __init__(self, dofs=None, values=None):
        dofs = np.asarray([] if dofs is None else dofs, dtype=np.int64).ravel()
        values = np.asarray([] if values is None else values, dtype=float).ravel()
        order = np.argsort(dofs, kind="stable")
        self.dofs = dofs[order]
        self.values = values[order] if len(values) else np.zeros(len(dofs))
        if len(self.dofs) != len(self.values):
            raise ValueError("dofs and values must align")

    def __len__(self):
        return len(self.dofs)

    def mask(self, n_dofs):
        m = np.zeros(n_dofs, dtype=bool)
        m[self.dofs] = True
        return m


class FESpace:
    """Scalar or vector Q^p space; components interleaved fastest."""

    def __init__(self, mesh, degree, n_components, cell_dofs, support_points):
        self.mesh = mesh
        self.degree = int(degree)
        self.n_components = int(n_components)
        self.shape1d = Shape1D(degree)
        self.cell_dofs = cell_dofs
        self.support_points = support_points
        self.n_scalar_dofs = len(support_points)
        self.n_dofs = self.n_scalar_dofs * self.n_components
        self.constraints = DirichletConstraints()
        self.reference_nodes = tensor_points(self.shape1d.nodes, mesh.dim)
        for a in (self.cell_dofs, self.support_points):
            a.setflags(write=False)

    @property
    def n_local_dofs(self):
        return (self.degree + 1) ** self.mesh.dim

    def cell_dofs_full(self):
        nc = self.n_components
        if nc == 1:
            return self.cell_dofs
        full = self.cell_dofs[:, :, None] * nc + np.arange(nc)[None, None, :]
        return full.reshape(len(self.cell_dofs), -1)

    def constrained_mask(self):
        return self.constraints.mask(self.n_dofs)


# ----------------------------------------------------------------------------
# DoF numbering
# ----------------------------------------------------------------------------

def _structured_numbering(grid, p):
    """Closed-form first-occurrence numbering on a lexicographic tensor mesh.

    Local point a of cell i is *new* in the scan iff a_j > 0 or i_j == 0 for
    every axis j.  A point that is not new was introduced by the cell with
    i_j -> i_j - 1 (a_j -> p) on every axis where a_j == 0 < i_j; that cell has
    the smallest index among the cells containing it.  Returns
    (cell_dofs int64 (nc, nloc), owner cell and local index of every DoF).
    """
    dim = len(grid)
    n1 = p + 1
    grid = [int(g) for g in grid]
    nc = int(np.prod(grid))
    # new points per cell and the exclusive prefix sum over cells (x fastest)
    per_axis = [np.where(np.arange(g) == 0, n1, p).astype(np.int64) for g in grid]
    n_new = per_axis[0]
    for j in range(1, dim):
        n_new = (per_axis[j][:, None] * n_new[None, :]).ravel()
    offset = np.zeros(nc + 1, dtype=np.int64)
    np.cumsum(n_new, out=offset[1:])
    # every lattice point X (X_j in [0, p*n_j]) is owned by the cell
    # i_j = max(0, ceil(X_j / p) - 1) at local a_j = X_j - p*i_j
    lat = [p * g + 1 for g in grid]
    oi = [np.maximum(0, (np.arange(L) + p - 1) // p - 1) for L in lat]
    oa = [np.arange(L) - p * oi[j] for j, L in enumerate(lat)]
    cstride = np.cumprod([1] + grid[:-1]).astype(np.int64)
    # rank of local a in the owner's new points; separable per axis
    lo = [np.where(oi[j] == 0, 0, 1) for j in range(dim)]
    width = [np.where(oi[j] == 0, n1, p) for j in range(dim)]
    ocell = np.zeros(1, dtype=np.int64)
    rank = np.zeros(1, dtype=np.int64)
    mult = np.ones(1, dtype=np.int64)
    for j in range(dim):  # build x-fastest tables over the lattice
        ocell = (oi[j][:, None] * cstride[j] + ocell[None, :]).ravel()
        rank = ((oa[j] - lo[j])[:, None] * mult[None, :] + rank[None, :]).ravel()
        mult = (width[j][:, None] * mult[None, :]).ravel()
    ids = offset[ocell] + rank  # DoF id of every lattice point
    n_dofs = int(offset[-1])
    # cell_dofs[c, l] = ids[lattice index of (p*i + a)]
    lstride = np.cumprod([1] + lat[:-1]).astype(np.int64)
    cbase = np.zeros(1, dtype=np.int64)
    for j in range(dim):
        cbase = ((p * np.arange(grid[j], dtype=np.int64) * lstride[j])[:, None] + cbase[None, :]).ravel()
    loc = tensor_points(np.arange(n1), dim).astype(np.int64)
    loff = (loc * lstride[None, :]).sum(axis=1)
    cell_dofs = ids[cbase[:, None] + loff[None, :]]
    first_cell = np.empty(n_dofs, dtype=np.int64)
    first_local = np.empty(n_dofs, dtype=np.int64)
    first_cell[ids] = ocell
    lloc = np.zeros(1, dtype=np.int64)
    for j in range(dim):
        lloc = ((oa[j] * n1**j)[:, None] + lloc[None, :]).ravel()
    first_local[ids] = lloc
    return cell_dofs, first_cell, first_local


def _support_points(mesh, cells, local, ref):
    """Mapped support point of each DoF, taken at its first occurrence."""
    n_dofs = len(cells)
    dim = mesh.dim
    bits = vertex_bits(dim)
    W = np.where(bits[None] == 1, ref[:, None, :], 1.0 - ref[:, None, :]).prod(axis=2)  # (nloc, 2^d)
    out = np.empty((n_dofs, dim))
    # group DoFs by the local index of their first occurrence: one weight row
    # per group, the sum over corners in vertex order as map_points does
    order = np.argsort(local, kind="stable")
    bounds = np.searchsorted(local[order], np.arange(len(ref) + 1))
    for l in range(len(ref)):
        sel = order[bounds[l]:bounds[l + 1]]
        if len(sel) == 0:
            continue
        cv = mesh.cells[cells[sel]]
        acc = np.zeros((len(sel), dim))
        for v in range(2**dim):
            if W[l, v] != 0.0:
                acc += W[l, v] * mesh.vertices[cv[:, v]]
        out[sel] = acc
    return out


def _matched_numbering(mesh, ref):
    """Tolerance matching of mapped Lobatto points (general meshes)."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    from scipy.spatial import cKDTree

    pts = mesh.map_points(ref)
    nc, nloc, dim = pts.shape
    flat = pts.reshape(-1, dim)
    n = len(flat)
    tol = 1e-10 * mesh.min_edge_length()
    pairs = cKDTree(flat).query_pairs(r=tol, output_type="ndarray")
    if len(pairs):
        g = coo_matrix((np.ones(len(pairs)), (pairs[:, 0], pairs[:, 1])), shape=(n, n)).tocsr()
        ncomp, labels = connected_components(g, directed=False)
    else:
        ncomp, labels = n, np.arange(n)
    first = np.full(ncomp, n, dtype=np.int64)
    np.minimum.at(first, labels, np.arange(n))
    order = np.argsort(first, kind="stable")
    newid = np.empty(ncomp, dtype=np.int64)
    newid[order] = np.arange(ncomp)
    return newid[labels].reshape(nc, nloc), flat[first[order]]


def build_space(mesh, degree, n_components=1):
    """Number global DoFs by first occurrence (fespace.py:137-163)."""
    shape = Shape1D(degree)
    ref = tensor_points(shape.nodes, mesh.dim)
    if getattr(mesh, "grid", None) is not None:
        cell_dofs, fcell, floc = _structured_numbering(tuple(mesh.grid), degree)
        support = _support_points(mesh, fcell, floc, ref)
    else:
        cell_dofs, support = _matched_numbering(mesh, ref)
    return FESpace(mesh, degree, n_components, cell_dofs, support)


def face_local_dofs(degree, dim, face):
    n = degree + 1
    j, s = divmod(face, 2)
    idx = np.arange(n**dim)
    return idx[((idx // n**j) % n) == (0 if s == 0 else degree)]


def dirichlet_constraints(space, boundary_ids, g=0.0):
    """Constrain all DoFs on faces with the given boundary ids (or "all")."""
    mesh = space.mesh
    known = set(mesh.boundary_ids().tolist())
    if isinstance(boundary_ids, str) and boundary_ids == "all":
        wanted = known
    else:
        wanted = set(int(b) for b in np.atleast_1d(boundary_ids))
        missing = wanted - known
        if missing:
            raise ValueError(f"boundary ids {sorted(missing)} not present on the mesh")
    bf = mesh.boundary_faces
    sel = bf[np.isin(bf[:, 2], sorted(wanted))]
    if len(sel) == 0:
        return DirichletConstraints()
    chunks = []
    for f in np.unique(sel[:, 1]):
        cells = sel[sel[:, 1] == f, 0]
        chunks.append(space.cell_dofs[cells][:, face_local_dofs(space.degree, mesh.dim, int(f))].ravel())
    scalar = np.unique(np.concatenate(chunks))
    nc = space.n_components
    pts = space.support_points[scalar]
    if callable(g):
        vals = np.asarray(g(pts), dtype=float)
    else:
        vals = np.full((len(scalar), nc) if nc > 1 else len(scalar), float(g))
    if nc == 1:
        return DirichletConstraints(scalar, vals.reshape(len(scalar)))
    vals = np.broadcast_to(vals.reshape(len(scalar), -1), (len(scalar), nc))
    dofs = scalar[:, None] * nc + np.arange(nc)[None, :]
    return DirichletConstraints(dofs.ravel(), vals.ravel())


def interpolate(space, f):
    """Nodal interpolant at the support points."""
    pts = space.support_points
    nc = space.n_components
    vals = np.asarray(f(pts), dtype=float) if callable(f) else np.full(
        (len(pts), nc) if nc > 1 else len(pts), float(f))
    if nc == 1:
        return vals.reshape(space.n_scalar_dofs).copy()
    return np.broadcast_to(vals.reshape(len(pts), -1), (len(pts), nc)).ravel().copy()
