"""GPU matrix-free Poisson and linear-elasticity operators.

Drop-in twins of the reference ``LaplaceOperator`` / ``ElasticityOperator``
(``/root/reference/pkg/src/nnmg/mfoperator.py:98-252``): same constructor
arguments, the operator protocol ``{n_dofs, apply, diagonal, space,
constraints}`` (test_solvers.py:17-31) and the zero-in / identity-out
constraint convention (mfoperator.py:1-7, 114-121).  The space may be this
package's ``FESpace`` or the reference's (duck-typed: ``mesh.vertices``,
``mesh.cells``, ``degree``, ``n_components``, ``cell_dofs``,
``constraints.dofs``).

Work runs in ``libnnmg_cuda.so`` (K1/K2 apply, K3 diagonal, K4 geometry);
there is no CPU fallback.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _device as D
from . import _lib

PHYSICS_LAPLACE = 0
PHYSICS_ELASTICITY = 1


def lame_parameters(E, nu):
    """(lambda, mu) from Young's modulus and Poisson ratio (mfoperator.py:18-22)."""
    lam = E * nu / ((1 - 2 * nu) * (1 + nu))
    mu = E / (2 * (1 + nu))
    return lam, mu


class _GpuOperatorBase:
    _physics = PHYSICS_LAPLACE

    def __init__(self, space, lam=0.0, mu=0.0, device=None, deterministic=False):
        self.space = space
        self.deterministic = bool(deterministic)
        self.device = D.resolve_device(device)
        mesh = space.mesh
        dim = int(mesh.dim)
        ncomp = int(space.n_components)
        verts = _lib.as_f64(mesh.vertices)
        cells = _lib.as_i64(mesh.cells)
        cell_dofs = _lib.as_i64(space.cell_dofs)
        cons = _lib.as_i64(space.constraints.dofs)
        h = ctypes.c_void_p()
        with self._on_device():
            _lib.call(
                "nnmg_level_create", self.device.index, dim, int(space.degree), ncomp, self._physics,
                len(cells), len(verts), _lib.host_ptr(verts), _lib.host_ptr(cells), int(space.n_scalar_dofs),
                _lib.host_ptr(cell_dofs), len(cons), _lib.host_ptr(cons), float(lam), float(mu), ctypes.byref(h),
            )
        self._h = h
        if self.deterministic:
            # fixed-order summation of the cell contributions (cell buffer +
            # gather) instead of fp64 atomics: bitwise reproducible results, as
            # the reference's serial bincount scatter (mfoperator.py:88-90)
            _lib.call("nnmg_level_set_deterministic", h, 1)
        self._n = int(space.n_dofs)
        self._constraint_snapshot = cons
        self._diag = None

    def _on_device(self):
        import torch

        return torch.cuda.device(self.device)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and _lib._lib is not None:  # not at interpreter exit
            _lib.load().nnmg_level_destroy(h)
            self._h = None

    # -- protocol ------------------------------------------------------------
    @property
    def handle(self):
        return self._h

    @property
    def n_dofs(self):
        return self._n

    @property
    def constraints(self):
        return self.space.constraints

    def info(self):
        vals = [ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()]
        _lib.call("nnmg_level_info", self._h, *[ctypes.byref(v) for v in vals])
        return {"n_dofs": vals[0].value, "n_cells": vals[1].value, "cells_per_block": vals[2].value,
                "geometry_bytes": vals[3].value, "index_bytes": vals[4].value}

    def apply_into(self, u, v):
        """v = A u on device tensors (no allocation, no checks)."""
        _lib.call("nnmg_level_apply", self._h, u.data_ptr(), v.data_ptr(), D.stream_ptr(self.device))
        return v

    def apply_begin_into(self, u, v, negate=False):
        """First piece of a split apply: v = 0 plus identity-out on the
        constrained rows (the distributed levels' interior / boundary split);
        negate: the residual form v -= A u (subtracts u on the constrained rows)."""
        _lib.call("nnmg_level_apply_begin", self._h, u.data_ptr(), v.data_ptr(), 1 if negate else 0,
                  D.stream_ptr(self.device))
        return v

    def apply_cells_into(self, u, v, block0, block1, negate=False):
        """v += (negate: -=) contributions of the cell blocks [block0, block1) to the free rows."""
        _lib.call("nnmg_level_apply_cells", self._h, u.data_ptr(), v.data_ptr(), int(block0), int(block1),
                  1 if negate else 0, D.stream_ptr(self.device))
        return v

    @property
    def n_cell_blocks(self):
        i = self.info()
        return -(-i["n_cells"] // i["cells_per_block"])

    def apply(self, u):
        """v = A u; new output, input untouched (mfoperator.py:108-122)."""
        ud, host = D.to_device(u, self._n, self.device)
        v = D.empty(self._n, self.device)
        self.apply_into(ud, v)
        return D.from_device(v, host)

    def residual_into(self, f, x, r):
        _lib.call("nnmg_level_residual", self._h, f.data_ptr(), x.data_ptr(), r.data_ptr(),
                  D.stream_ptr(self.device))
        return r

    def load_vector(self, f):
        """Device b = (f, phi_i) for a constant (per-component) body load,
        constrained entries 0 (body-load part of mfoperator.py:313-355)."""
        fv = np.broadcast_to(np.atleast_1d(np.asarray(f, dtype=float)), (self.space.n_components,)).copy()
        b = D.empty(self._n, self.device)
        _lib.call("nnmg_level_load_vector", self._h, _lib.host_ptr(fv), b.data_ptr(), D.stream_ptr(self.device))
        return b

    def _ensure_diagonal(self):
        if self._diag is None:
            _lib.call("nnmg_level_compute_diagonal", self._h, D.stream_ptr(self.device))
            d = D.empty(self._n, self.device)
            _lib.call("nnmg_level_diagonal", self._h, d.data_ptr(), D.stream_ptr(self.device))
            self._diag = d

    def diagonal_device(self):
        """Cached exact diagonal as a device tensor (do not modify)."""
        self._ensure_diagonal()
        return self._diag

    def diagonal(self):
        """Exact diagonal, constrained entries 1; a host copy (mfoperator.py:92-95)."""
        self._ensure_diagonal()
        return self._diag.cpu().numpy()


class LaplaceOperator(_GpuOperatorBase):
    """Matrix-free scalar Laplacian, Gauss-Legendre (p+1)^d (mfoperator.py:98-122)."""

    _physics = PHYSICS_LAPLACE

    def __init__(self, space, device=None, deterministic=False):
        if space.n_components != 1:
            raise ValueError("LaplaceOperator is scalar; use ElasticityOperator")
        super().__init__(space, device=device, deterministic=deterministic)


class ElasticityOperator(_GpuOperatorBase):
    """sigma = lam tr(eps) I + 2 mu eps (mfoperator.py:160-202)."""

    _physics = PHYSICS_ELASTICITY

    def __init__(self, space, lam, mu, device=None, deterministic=False):
        if space.n_components != space.mesh.dim:
            raise ValueError("elasticity needs one component per space dimension")
        self.lam = float(lam)
        self.mu = float(mu)
        super().__init__(space, lam=self.lam, mu=self.mu, device=device, deterministic=deterministic)


def compute_diagonal(op):
    return op.diagonal()


def assemble_rhs(space, f=None, neumann=None, chunk=1 << 16):
    """Load vector b_i = (f, phi_i) + (g, phi_i)_GammaN, constrained entries
    zeroed (host setup, mfoperator.py:313-414).  f: constant, per-component
    constant sequence, or callable of batched points returning (npts,) or
    (npts, ncomp).  neumann: {boundary id: g} with g a constant, a callable of
    (points, outward unit normals), or ("normal", m) for the traction m n."""
    from .fespace import gauss_legendre
    from .mesh import tensor_points

    mesh = space.mesh
    dim, p, ncomp = mesh.dim, space.degree, space.n_components
    b = np.zeros(space.n_dofs)
    bm = b.reshape(space.n_scalar_dofs, ncomp)
    if neumann:
        _add_neumann(space, neumann, bm)
    if f is None:
        b[space.constraints.dofs] = 0.0
        return b
    q1, w1 = gauss_legendre(p + 1)
    qpts = tensor_points(q1, dim)
    wq = tensor_points(w1, dim).prod(axis=1)
    S = space.shape1d.values(q1)
    n1 = p + 1
    cell_dofs = np.asarray(space.cell_dofs)
    const = None if callable(f) else np.atleast_1d(np.asarray(f, dtype=float))
    for s in range(0, mesh.n_cells, chunk):
        cells = np.arange(s, min(s + chunk, mesh.n_cells))
        J = np.einsum("pvb,cva->cpab", _corner_grad(dim, qpts), mesh.vertices[mesh.cells[cells]])
        det = np.linalg.det(J)
        if const is None:
            xq = np.einsum("pv,cvd->cpd", _corner_w(dim, qpts), mesh.vertices[mesh.cells[cells]])
            fv = np.asarray(f(xq.reshape(-1, dim)), dtype=float).reshape(len(cells), len(qpts), -1)
        else:
            fv = np.broadcast_to(const[None, None, :], (len(cells), len(qpts), len(const)))
        if fv.shape[2] == 1 and ncomp > 1:
            fv = np.broadcast_to(fv, (len(cells), len(qpts), ncomp))
        scaled = fv * (det * wq[None, :])[:, :, None]
        t = scaled.reshape((len(cells),) + (n1,) * dim + (fv.shape[2],))
        for k in range(dim):
            ax = 1 + (dim - 1 - k)
            t = np.moveaxis(np.moveaxis(t, ax, -1) @ S, -1, ax)
        local = t.reshape(len(cells), -1, fv.shape[2])
        flat = cell_dofs[cells].ravel()
        for c in range(ncomp):
            bm[:, c] += np.bincount(flat, weights=local[:, :, min(c, fv.shape[2] - 1)].ravel(),
                                    minlength=space.n_scalar_dofs)
    b[space.constraints.dofs] = 0.0
    return b


def _add_neumann(space, neumann, bm):
    """Boundary term (g, phi_i) over the faces whose id has an entry in
    ``neumann`` (mfoperator.py:356-411): on face (j, s) of a cell (face id
    2j + s) the Gauss-Legendre rule of the other reference axes; surface
    element |dx/dt1| (2D) or |dx/dt1 x dx/dt2| (3D); outward unit normal
    J^-T (+-e_j) normalised."""
    from .fespace import gauss_legendre
    from .mesh import tensor_points

    mesh = space.mesh
    dim, p, ncomp = mesh.dim, space.degree, space.n_components
    known = set(int(i) for i in mesh.boundary_ids())
    for bid in neumann:
        if bid not in known:
            raise ValueError(f"unknown boundary id {bid}")
    q1, w1 = gauss_legendre(p + 1)
    tq = q1[:, None] if dim == 2 else tensor_points(q1, 2)
    tw = w1 if dim == 2 else tensor_points(w1, 2).prod(axis=1)
    bf = np.asarray(mesh.boundary_faces)
    cell_dofs = np.asarray(space.cell_dofs)
    for face in np.unique(bf[:, 1]):
        j, side = int(face) // 2, int(face) % 2
        tdims = [k for k in range(dim) if k != j]
        ref = np.empty((len(tq), dim))
        ref[:, j] = float(side)
        ref[:, tdims] = tq
        # local basis values at the face points (x fastest)
        tab = np.ones((len(ref), 1))
        for k in range(dim):
            tab = (tab[:, None, :] * space.shape1d.values(ref[:, k])[:, :, None]).reshape(len(ref), -1)
        cw, cg = _corner_w(dim, ref), _corner_grad(dim, ref)
        for bid, g in neumann.items():
            cells = bf[(bf[:, 1] == face) & (bf[:, 2] == bid), 0]
            if len(cells) == 0:
                continue
            X = mesh.vertices[mesh.cells[cells]]                       # (nf, 2^d, d)
            J = np.einsum("pvb,cva->cpab", cg, X)                        # dx_a / dxhat_b
            xq = np.einsum("pv,cvd->cpd", cw, X)
            if dim == 2:
                dA = np.linalg.norm(J[:, :, :, tdims[0]], axis=2)
            else:
                dA = np.linalg.norm(np.cross(J[:, :, :, tdims[0]], J[:, :, :, tdims[1]]), axis=2)
            e = np.zeros(dim)
            e[j] = 1.0 if side == 1 else -1.0
            nrm = np.linalg.solve(np.swapaxes(J, 2, 3), np.broadcast_to(e, J.shape[:2] + (dim,))[..., None])[..., 0]
            nrm /= np.linalg.norm(nrm, axis=2)[:, :, None]
            if isinstance(g, tuple) and g[0] == "normal":
                gv = float(g[1]) * nrm
            elif callable(g):
                gv = np.asarray(g(xq.reshape(-1, dim), nrm.reshape(-1, dim)), dtype=float)
                gv = gv.reshape(len(cells), len(ref), -1)
            else:
                gv = np.full((len(cells), len(ref), 1), float(g))
            contrib = np.einsum("fqc,ql->flc", gv * (dA * tw[None, :])[:, :, None], tab)
            flat = cell_dofs[cells].ravel()
            for c in range(ncomp):
                bm[:, c] += np.bincount(flat, weights=contrib[:, :, min(c, gv.shape[2] - 1)].ravel(),
                                        minlength=space.n_scalar_dofs)


def _corner_w(dim, x):
    from .mesh import corner_weights

    return corner_weights(dim, x)


def _corner_grad(dim, x):
    from .mesh import corner_weight_gradients

    return corner_weight_gradients(dim, x)
