"""Quad/hex meshes for the GPU path (host-side setup, not hot path).

Mirrors the parts of the reference ``nnmg.mesh`` that the hot path consumes
(``/root/reference/pkg/src/nnmg/mesh.py``):

* ``Mesh`` attributes ``dim``, ``vertices``, ``cells``, ``boundary_faces`` and
  the geometric helpers ``map_points``/``jacobians`` (mesh.py:94-202);
* local vertex ``v`` of a cell sits at reference coordinates
  ``(bit_0(v), .., bit_{d-1}(v))`` and local face ``2j+s`` is the side where
  reference coordinate ``j`` equals ``s`` (mesh.py:5-7);
* structured tensor meshes are numbered lexicographically with x fastest, both
  vertices and cells (``_tensor_mesh``, mesh.py:315-336), and box faces carry
  boundary id ``2j+s`` (``_assign_box_boundary_ids``, mesh.py:339-354).

Structured meshes additionally remember their grid (cells per axis) so that
``fespace.build_space`` can use the closed-form first-occurrence numbering.
"""

from __future__ import annotations

import numpy as np


class MeshError(Exception):
    pass


def tensor_points(nodes, dim):
    """dim-fold tensor grid of 1D nodes, x fastest (mesh.py:20-25)."""
    nodes = np.asarray(nodes, dtype=float)
    n = len(nodes)
    idx = np.arange(n**dim)
    return np.stack([nodes[(idx // n**j) % n] for j in range(dim)], axis=1)


def vertex_bits(dim):
    v = np.arange(2**dim)
    return np.stack([(v >> j) & 1 for j in range(dim)], axis=1)


def corner_weights(dim, xhat):
    """Multilinear vertex weights at reference points, (npts, 2^dim)."""
    xhat = np.atleast_2d(np.asarray(xhat, dtype=float))
    bits = vertex_bits(dim)
    f = np.where(bits[None] == 1, xhat[:, None, :], 1.0 - xhat[:, None, :])
    return f.prod(axis=2)


def corner_weight_gradients(dim, xhat):
    """d(weight_v)/d(xhat_k), shape (npts, 2^dim, dim)."""
    xhat = np.atleast_2d(np.asarray(xhat, dtype=float))
    bits = vertex_bits(dim)
    f = np.where(bits[None] == 1, xhat[:, None, :], 1.0 - xhat[:, None, :])
    sgn = np.where(bits == 1, 1.0, -1.0)
    out = np.empty((len(xhat), 2**dim, dim))
    for k in range(dim):
        rest = np.ones((len(xhat), 2**dim))
        for j in range(dim):
            if j != k:
                rest = rest * f[:, :, j]
        out[:, :, k] = rest * sgn[None, :, k]
    return out


def face_vertex_indices(dim, face):
    j, s = divmod(face, 2)
    return np.nonzero(vertex_bits(dim)[:, j] == s)[0]


class Mesh:
    """Conforming multilinear quad/hex mesh (immutable after construction)."""

    def __init__(self, dim, vertices, cells, boundary_faces, grid=None, extent=None,
                 validate=True):
        self.dim = int(dim)
        self.vertices = np.ascontiguousarray(vertices, dtype=np.float64)
        self.cells = np.ascontiguousarray(cells, dtype=np.int64)
        self.boundary_faces = np.ascontiguousarray(boundary_faces, dtype=np.int64).reshape(-1, 3)
        if self.vertices.ndim != 2 or self.vertices.shape[1] != self.dim:
            raise MeshError(f"vertices must have shape (n, {self.dim})")
        if self.cells.ndim != 2 or self.cells.shape[1] != 2**self.dim:
            raise MeshError(f"cells must have shape (n, {2 ** self.dim})")
        # structured metadata: cells per axis (x first) and the box extent
        self.grid = None if grid is None else tuple(int(g) for g in grid)
        self.extent = extent
        for a in (self.vertices, self.cells, self.boundary_faces):
            a.setflags(write=False)
        self._min_edge = None
        if validate:
            self.validate()

    # -- sizes ---------------------------------------------------------------
    @property
    def n_cells(self):
        return len(self.cells)

    @property
    def n_vertices(self):
        return len(self.vertices)

    # -- geometry --------------------------------------------------------------
    def cell_vertex_coords(self, cells=None):
        if cells is None:
            return self.vertices[self.cells]
        return self.vertices[self.cells[cells]]

    def map_points(self, xhat, cells=None):
        w = corner_weights(self.dim, xhat)
        if cells is None:
            return np.einsum("pv,cvd->cpd", w, self.cell_vertex_coords())
        return np.einsum("pv,pvd->pd", w, self.cell_vertex_coords(cells))

    def jacobians(self, xhat, cells=None):
        g = corner_weight_gradients(self.dim, xhat)
        if cells is None:
            return np.einsum("pvb,cva->cpab", g, self.cell_vertex_coords())
        return np.einsum("pvb,pva->pab", g, self.cell_vertex_coords(cells))

    def bounding_box(self):
        return self.vertices.min(axis=0), self.vertices.max(axis=0)

    def diameter(self):
        lo, hi = self.bounding_box()
        return float(np.linalg.norm(hi - lo))

    def min_edge_length(self):
        if self._min_edge is None:
            bits = vertex_bits(self.dim)
            lmin = np.inf
            for j in range(self.dim):
                a = np.nonzero(bits[:, j] == 0)[0]
                for s in range(0, self.n_cells, 1 << 20):
                    cv = self.vertices[self.cells[s:s + (1 << 20)]]
                    lmin = min(lmin, float(np.linalg.norm(cv[:, a] - cv[:, a + 2**j], axis=2).min()))
            self._min_edge = lmin
        return self._min_edge

    def boundary_ids(self):
        return np.unique(self.boundary_faces[:, 2])

    def validate(self):
        if self.cells.size and (self.cells.min() < 0 or self.cells.max() >= self.n_vertices):
            raise MeshError("cell vertex index out of range")
        # det J > 0 at the 2^d Gauss points (mesh.py:190-195), chunked
        g = 0.5 / np.sqrt(3.0)
        pts = tensor_points([0.5 - g, 0.5 + g], self.dim)
        for s in range(0, self.n_cells, 1 << 18):
            idx = np.arange(s, min(s + (1 << 18), self.n_cells))
            J = np.einsum("pvb,cva->cpab", corner_weight_gradients(self.dim, pts),
                          self.cell_vertex_coords(idx))
            det = np.linalg.det(J)
            if det.size and det.min() <= 0.0:
                bad = idx[np.nonzero(det.min(axis=1) <= 0.0)[0]]
                raise MeshError(f"non-positive Jacobian in cells {bad[:10].tolist()}")


def structured_box_mesh(grid, extent, validate=True):
    """Tensor mesh of a box with per-face boundary ids 2j+s.

    grid: cells per axis (x first); extent: [(lo, hi)] per axis.  Vertex and
    cell numbering is lexicographic with x fastest, as ``_tensor_mesh`` +
    ``_assign_box_boundary_ids`` produce (mesh.py:315-354).
    """
    dim = len(grid)
    grid = [int(g) for g in grid]
    axes = [np.linspace(lo, hi, n + 1) for (lo, hi), n in zip(extent, grid)]
    nv = [n + 1 for n in grid]
    vidx = np.indices(nv[::-1]).reshape(dim, -1)[::-1]  # (dim, nverts), x fastest
    vertices = np.stack([axes[j][vidx[j]] for j in range(dim)], axis=1)
    strides = np.cumprod([1] + nv[:-1])
    cidx = np.indices(grid[::-1]).reshape(dim, -1)[::-1].T  # (nc, dim), x fastest
    bits = vertex_bits(dim)
    cells = ((cidx[:, None, :] + bits[None, :, :]) * strides).sum(axis=2)
    # boundary faces in (cell, local face) order, id 2j+s
    rows = []
    nc = len(cidx)
    cell_ids = np.arange(nc)
    for f in range(2 * dim):
        j, s = divmod(f, 2)
        on = cidx[:, j] == (0 if s == 0 else grid[j] - 1)
        c = cell_ids[on]
        rows.append(np.stack([c, np.full(len(c), f), np.full(len(c), f)], axis=1))
    faces = np.concatenate(rows, axis=0)
    order = np.lexsort((faces[:, 1], faces[:, 0]))
    faces = faces[order]
    return Mesh(dim, vertices, cells, faces, grid=grid, extent=[tuple(e) for e in extent],
                validate=validate)


def interior_vertex_mask(mesh):
    """Vertices not on any boundary face."""
    interior = np.ones(mesh.n_vertices, dtype=bool)
    for f in range(2 * mesh.dim):
        sel = mesh.boundary_faces[mesh.boundary_faces[:, 1] == f]
        if len(sel):
            interior[mesh.cells[sel[:, 0]][:, face_vertex_indices(mesh.dim, f)].ravel()] = False
    return interior


def jittered_box_mesh(grid, extent, amplitude, seed, warp=None, validate=True):
    """SURVEY.md §8(d) recipe: structured box, interior vertices displaced by
    i.i.d. U(-a*h_j, a*h_j) drawn from ``default_rng(seed)`` for ALL vertices
    in vertex order, optional warp applied to all vertices afterwards."""
    base = structured_box_mesh(grid, extent, validate=False)
    h = np.array([(hi - lo) / n for (lo, hi), n in zip(extent, grid)])
    rng = np.random.default_rng(seed)
    disp = rng.uniform(-1.0, 1.0, size=base.vertices.shape) * (amplitude * h)[None]
    v = base.vertices + disp * interior_vertex_mask(base)[:, None]
    if warp is not None:
        v = warp(v)
    return Mesh(base.dim, v, base.cells, base.boundary_faces, grid=base.grid,
                extent=base.extent, validate=validate)


def sine_warp(v):
    """C4 curved-domain map x+=0.05 sin(2πy) sin(2πz), cyclic in (x,y,z),
    all three evaluated on the pre-warp coordinates."""
    x, y, z = v[:, 0], v[:, 1], v[:, 2]
    tp = 2.0 * np.pi
    out = np.empty_like(v)
    out[:, 0] = x + 0.05 * np.sin(tp * y) * np.sin(tp * z)
    out[:, 1] = y + 0.05 * np.sin(tp * z) * np.sin(tp * x)
    out[:, 2] = z + 0.05 * np.sin(tp * x) * np.sin(tp * y)
    return out


def from_reference(mesh):
    """Wrap a reference ``nnmg.mesh.Mesh`` (duck-typed) without re-validation."""
    return Mesh(mesh.dim, mesh.vertices, mesh.cells, mesh.boundary_faces, validate=False)


# ---------------------------------------------------------------------------
# gmsh ASCII v2.2 I/O (mesh.py:440-569): unstructured ingestion
# ---------------------------------------------------------------------------
# gmsh lists quad corners counter-clockwise and hex corners bottom-CCW then
# top-CCW; swapping local corners 2<->3 (and 6<->7) maps that to the
# lexicographic order used here, in both directions.
_MSH_CORNER_SWAP = {2: np.array([0, 1, 3, 2]), 3: np.array([0, 1, 3, 2, 4, 5, 7, 6])}
_MSH_CELL = {2: 3, 3: 5}   # element type: 3 = 4-node quad, 5 = 8-node hex
_MSH_FACE = {2: 1, 3: 3}   # element type: 1 = 2-node line, 3 = 4-node quad
_MSH_NODES = {1: 2, 2: 3, 3: 4, 4: 4, 5: 8, 15: 1}  # accepted element types -> node count


def boundary_faces_of(cells, dim):
    """(cell, local face) pairs of faces that belong to exactly one cell,
    sorted by (cell, face)."""
    cells = np.asarray(cells, dtype=np.int64)
    nc = len(cells)
    fv = np.stack([cells[:, face_vertex_indices(dim, f)] for f in range(2 * dim)], axis=1)  # (nc, 2d, 2^(d-1))
    keys = np.sort(fv.reshape(nc * 2 * dim, -1), axis=1)
    _, inv, cnt = np.unique(keys, axis=0, return_inverse=True, return_counts=True)
    on = np.nonzero(cnt[inv.ravel()] == 1)[0]
    return np.stack([on // (2 * dim), on % (2 * dim)], axis=1), keys[on]


def write_msh(mesh, path):
    """ASCII msh v2.2: nodes, one tagged line/quad element per boundary face
    (physical tag = boundary id), then the cells (mesh.py:448-474)."""
    dim = mesh.dim
    out = ["$MeshFormat", "2.2 0 8", "$EndMeshFormat", "$Nodes", str(mesh.n_vertices)]
    pad = np.zeros((mesh.n_vertices, 3))
    pad[:, :dim] = mesh.vertices
    out += [f"{i + 1} {x:.17g} {y:.17g} {z:.17g}" for i, (x, y, z) in enumerate(pad)]
    out += ["$EndNodes", "$Elements", str(len(mesh.boundary_faces) + mesh.n_cells)]
    eid = 0
    for cell, face, bid in mesh.boundary_faces:
        fv = mesh.cells[cell][face_vertex_indices(dim, face)]
        if dim == 3:
            fv = fv[[0, 1, 3, 2]]
        eid += 1
        out.append(f"{eid} {_MSH_FACE[dim]} 2 {bid} {eid} " + " ".join(str(v + 1) for v in fv))
    swap = _MSH_CORNER_SWAP[dim]
    for cell in mesh.cells:
        eid += 1
        out.append(f"{eid} {_MSH_CELL[dim]} 2 0 {eid} " + " ".join(str(v + 1) for v in cell[swap]))
    out.append("$EndElements")
    with open(path, "w") as fh:
        fh.write("\n".join(out) + "\n")


def _msh_sections(text):
    sections, name, body = {}, None, None
    for line in text.split("\n"):
        s = line.strip()
        if name is None:
            if s.startswith("$") and not s.startswith("$End"):
                name, body = s[1:], []
        elif s == f"$End{name}":
            sections[name] = body
            name = None
        else:
            body.append(s)
    if name is not None:
        raise MeshError(f"malformed section {name}: missing $End{name}")
    return sections


def read_msh(path, validate=True):
    """Quad/hex mesh from an ASCII msh v2.2 file (mesh.py:477-569): unused
    nodes dropped (remaining ones keep their file order), cells in file order
    with lexicographic corners, boundary faces = faces of exactly one cell,
    boundary id = physical tag of the matching line/quad element (0 if none),
    sorted by (cell, face).  Simplices are rejected.  The result has no
    structured grid, so ``build_space`` numbers it by geometric matching."""
    with open(path) as fh:
        sec = _msh_sections(fh.read())
    if "Nodes" not in sec or "Elements" not in sec:
        raise MeshError("malformed msh file: missing $Nodes or $Elements")
    try:
        nn = int(sec["Nodes"][0])
        tab = np.array(" ".join(sec["Nodes"][1:1 + nn]).split(), dtype=float).reshape(nn, 4)
    except (ValueError, IndexError) as exc:
        raise MeshError(f"malformed $Nodes section: {exc}") from exc
    node_row = {int(i): k for k, i in enumerate(tab[:, 0].astype(np.int64))}
    try:
        ne = int(sec["Elements"][0])
        rows = [[int(t) for t in sec["Elements"][1 + k].split()] for k in range(ne)]
    except (ValueError, IndexError) as exc:
        raise MeshError(f"malformed $Elements section: {exc}") from exc
    elems = []
    for r in rows:
        etype, ntag = r[1], r[2]
        if etype not in _MSH_NODES:
            raise MeshError(f"unsupported element type {etype}")
        nodes = r[3 + ntag:]
        if len(nodes) != _MSH_NODES[etype]:
            raise MeshError(f"malformed element line: expected {_MSH_NODES[etype]} nodes")
        try:
            elems.append((etype, r[3] if ntag else 0, [node_row[n] for n in nodes]))
        except KeyError as exc:
            raise MeshError(f"element references unknown node {exc}") from exc
    kinds = {e[0] for e in elems}
    if kinds & {2, 4}:
        raise MeshError("unsupported element type: simplex elements are not handled")
    dim = 3 if 5 in kinds else 2 if 3 in kinds else None
    if dim is None:
        raise MeshError("no quad or hex cells found")
    cells = np.array([e[2] for e in elems if e[0] == _MSH_CELL[dim]], dtype=np.int64)[:, _MSH_CORNER_SWAP[dim]]
    used = np.unique(cells)
    renum = np.full(nn, -1, dtype=np.int64)
    renum[used] = np.arange(len(used))
    cells = renum[cells]
    vertices = tab[used, 1:1 + dim]
    pairs, keys = boundary_faces_of(cells, dim)
    ids = np.zeros(len(pairs), dtype=np.int64)
    lookup = {tuple(k): i for i, k in enumerate(keys.tolist())}
    for etype, tag, nodes in elems:
        if etype != _MSH_FACE[dim]:
            continue
        key = tuple(sorted(renum[np.array(nodes)].tolist()))
        i = lookup.get(key)
        if i is None or -1 in key:
            raise MeshError("boundary element does not match any boundary face")
        ids[i] = tag
    faces = np.concatenate([pairs, ids[:, None]], axis=1)
    return Mesh(dim, vertices, cells, faces, validate=validate)
