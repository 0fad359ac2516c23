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
    nc = int(np.prod(grid))
    cidx = np.indices(grid[::-1]).reshape(dim, -1)[::-1].T  # (nc, dim), x fastest
    first = cidx == 0  # (nc, dim)
    per_axis = np.where(first, n1, p)
    n_new = per_axis.prod(axis=1)
    offset = np.zeros(nc + 1, dtype=np.int64)
    np.cumsum(n_new, out=offset[1:])
    loc = tensor_points(np.arange(n1), dim).astype(np.int64)  # (nloc, dim)
    nloc = len(loc)
    strides = np.cumprod([1] + list(grid[:-1])).astype(np.int64)
    cell_dofs = np.empty((nc, nloc), dtype=np.int64)
    n_dofs = int(offset[-1])
    first_cell = np.empty(n_dofs, dtype=np.int64)
    first_local = np.empty(n_dofs, dtype=np.int64)
    chunk = max(1, (1 << 22) // nloc)
    for s in range(0, nc, chunk):
        e = min(nc, s + chunk)
        ci = cidx[s:e][:, None, :]  # (m,1,dim)
        a = np.broadcast_to(loc[None], (e - s, nloc, dim))
        back = (a == 0) & (ci > 0)
        oi = ci - back  # owner cell coordinates
        oa = np.where(back, p, a)  # owner local coordinates
        ofirst = oi == 0
        lo = np.where(ofirst, 0, 1)
        width = np.where(ofirst, n1, p)
        rank = np.zeros((e - s, nloc), dtype=np.int64)
        mult = np.ones((e - s, nloc), dtype=np.int64)
        for j in range(dim):
            rank += (oa[..., j] - lo[..., j]) * mult
            mult *= width[..., j]
        ocell = (oi * strides).sum(axis=2)
        ids = offset[ocell] + rank
        cell_dofs[s:e] = ids
        new = ~back.any(axis=2)
        first_cell[ids[new]] = np.broadcast_to(np.arange(s, e)[:, None], new.shape)[new]
        first_local[ids[new]] = np.broadcast_to(np.arange(nloc)[None, :], new.shape)[new]
    return cell_dofs, first_cell, first_local


def _support_points(mesh, cells, local, ref):
    """Mapped support point of each DoF, taken at its first occurrence."""
    n_dofs = len(cells)
    bits = vertex_bits(mesh.dim)
    xr = ref[local]  # (n_dofs, dim)
    w = np.where(bits[None] == 1, xr[:, None, :], 1.0 - xr[:, None, :]).prod(axis=2)
    out = np.empty((n_dofs, mesh.dim))
    chunk = 1 << 21
    for s in range(0, n_dofs, chunk):
        e = min(n_dofs, s + chunk)
        cv = mesh.vertices[mesh.cells[cells[s:e]]]  # (m, 2^d, d)
        out[s:e] = np.einsum("pv,pvd->pd", w[s:e], cv)
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
