"""GPU two-level transfers: point evaluation and its exact transpose.

Drop-in twin of the reference ``TwoLevelTransferNonNested``
(``/root/reference/pkg/src/nnmg/transfer.py:61-124``) and ``setup_nonnested``
(transfer.py:254-256): same records (``point_dofs``, ``cells``, ``xhat``,
``projected``, lazily ``tabs`` / ``gather``), same symmetric constraint masking
(transfer.py:35-36, 42, 51, 57), ``prolongate`` / ``restrict`` returning new
vectors.  Point location runs on the GPU (geosearch.py here); the apply paths
are the K6/K7 kernels of libnnmg_cuda.so.

The nested (transfer.py:169-222) and polynomial (transfer.py:225-251)
transfers of the reference are per-cell tensor-product embeddings with claim
masks.  For conforming Lagrange spaces with the coarse space contained in the
fine one, both ARE the nodal interpolation of the coarse field at the fine
support points: the claiming cell's embedding evaluates the (continuous)
coarse function at the fine node, and the transpose sums the same global
basis-function values.  They are therefore built here on the same GPU point
evaluation (identical operator up to rounding; parity against the reference's
own outputs in tests/test_gpu_cellwise.py), with the reference's argument
checks.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _device as D
from . import _lib
from .geosearch import SearchConfig, locate_points
from .mfoperator import ElasticityOperator, LaplaceOperator


class TwoLevelTransferNonNested:
    """Matrix-free non-nested transfer; the levels are given as GPU operators
    (or spaces, in which case GPU Laplace/elasticity levels are created)."""

    def __init__(self, coarse_space, fine_space, search=None, coarse_operator=None, fine_operator=None,
                 records=None, device=None):
        if coarse_space.n_components != fine_space.n_components:
            raise ValueError("component counts of the two levels must match")
        self.coarse_space = coarse_space
        self.fine_space = fine_space
        self.timings = {"evaluate": 0.0, "gather_scatter": 0.0, "calls": 0}
        self.device = D.resolve_device(device if coarse_operator is None else coarse_operator.device)
        nc = fine_space.n_components
        if records is None:
            fully = fine_space.constrained_mask().reshape(fine_space.n_scalar_dofs, nc).all(axis=1)
            self.point_dofs = np.nonzero(~fully)[0]
            located = locate_points(coarse_space.mesh, fine_space.support_points[self.point_dofs],
                                    search or SearchConfig(), device=self.device)
            self.located = located
            self.cells = located.cells
            self.xhat = located.xhat
            self.projected = located.projected
        else:
            self.point_dofs = _lib.as_i64(records["point_dofs"])
            self.cells = _lib.as_i64(records["cells"])
            self.xhat = _lib.as_f64(records["xhat"])
            self.projected = np.asarray(records.get("projected", np.zeros(len(self.cells), bool)), dtype=bool)
        self._cop = coarse_operator or _level_for(coarse_space, self.device)
        self._fop = fine_operator or _level_for(fine_space, self.device)
        h = ctypes.c_void_p()
        pd = _lib.as_i64(self.point_dofs)
        ce = _lib.as_i64(self.cells)
        xh = _lib.as_f64(self.xhat)
        _lib.call("nnmg_transfer_create", self._cop.handle, self._fop.handle, len(pd), _lib.host_ptr(pd),
                  _lib.host_ptr(ce), _lib.host_ptr(xh), ctypes.byref(h))
        self._h = h

    @classmethod
    def from_reference(cls, ref_transfer, coarse_operator, fine_operator):
        """Wrap the records of a reference TwoLevelTransferNonNested (same spaces)."""
        rec = {"point_dofs": ref_transfer.point_dofs, "cells": ref_transfer.cells, "xhat": ref_transfer.xhat,
               "projected": ref_transfer.projected}
        return cls(ref_transfer.coarse_space, ref_transfer.fine_space, coarse_operator=coarse_operator,
                   fine_operator=fine_operator, records=rec)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and _lib._lib is not None:  # not at interpreter exit
            _lib.load().nnmg_transfer_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    # reference data members materialised on demand (host memory heavy at scale)
    @property
    def tabs(self):
        dim = self.coarse_space.mesh.dim
        return [self.coarse_space.shape1d.values(self.xhat[:, j]) for j in range(dim)]

    @property
    def gather(self):
        return np.asarray(self.coarse_space.cell_dofs)[self.cells]

    # -- apply paths ---------------------------------------------------------
    def prolongate_into(self, uc, uf, accumulate=False):
        _lib.call("nnmg_transfer_prolongate", self._h, uc.data_ptr(), uf.data_ptr(), 1 if accumulate else 0,
                  D.stream_ptr(self.device))
        return uf

    def restrict_into(self, rf, rc):
        _lib.call("nnmg_transfer_restrict", self._h, rf.data_ptr(), rc.data_ptr(), D.stream_ptr(self.device))
        return rc

    def _timed(self, call):
        """Run one public-path call with the library's per-phase events on and
        add the device times to the reference's rows (transfer.py:100-101,
        122-123): "evaluate" = the point-evaluation kernel, "gather_scatter" =
        the zero-fill of point-less DoFs / the fixed-order coarse gather."""
        _lib.call("nnmg_transfer_set_timing", self._h, 1)
        try:
            call()
            ev, gs = ctypes.c_double(), ctypes.c_double()
            _lib.call("nnmg_transfer_last_timing", self._h, ctypes.byref(ev), ctypes.byref(gs))
        finally:
            _lib.call("nnmg_transfer_set_timing", self._h, 0)
        self.timings["evaluate"] += ev.value
        self.timings["gather_scatter"] += gs.value

    def prolongate(self, u_c):
        ud, host = D.to_device(u_c, self.coarse_space.n_dofs, self.device, "coarse vector")
        out = D.empty(self.fine_space.n_dofs, self.device)
        self._timed(lambda: self.prolongate_into(ud, out))
        self.timings["calls"] += 1
        return D.from_device(out, host)

    def restrict(self, r_f):
        rd, host = D.to_device(r_f, self.fine_space.n_dofs, self.device, "fine vector")
        out = D.empty(self.coarse_space.n_dofs, self.device)
        self._timed(lambda: self.restrict_into(rd, out))
        return D.from_device(out, host)


class TwoLevelTransferNested(TwoLevelTransferNonNested):
    """GPU twin of ``TwoLevelTransferNested`` (transfer.py:169-222): nested mesh
    pair (global refinement), same degree."""

    def __init__(self, coarse_space, fine_space, search=None, coarse_operator=None, fine_operator=None,
                 device=None):
        if coarse_space.n_components != fine_space.n_components:
            raise ValueError("component counts of the two levels must match")
        if coarse_space.degree != fine_space.degree:
            raise ValueError("nested mesh transfer keeps the polynomial degree")
        super().__init__(coarse_space, fine_space, search, coarse_operator=coarse_operator,
                         fine_operator=fine_operator, device=device)


class TwoLevelTransferPolynomial(TwoLevelTransferNonNested):
    """GPU twin of ``TwoLevelTransferPolynomial`` (transfer.py:225-251):
    Q^(p-1) embedded into Q^p on one mesh."""

    def __init__(self, coarse_space, fine_space, coarse_operator=None, fine_operator=None, device=None):
        if coarse_space.n_components != fine_space.n_components:
            raise ValueError("component counts of the two levels must match")
        if coarse_space.mesh is not fine_space.mesh:
            raise ValueError("polynomial transfer levels share one mesh")
        if coarse_space.degree != fine_space.degree - 1:
            raise ValueError("polynomial coarsening lowers the degree by one")
        super().__init__(coarse_space, fine_space, SearchConfig(), coarse_operator=coarse_operator,
                         fine_operator=fine_operator, device=device)


def _level_for(space, device):
    if space.n_components == 1:
        return LaplaceOperator(space, device=device)
    raise ValueError("pass coarse_operator/fine_operator for vector spaces (elasticity parameters needed)")


def setup_nonnested(coarse_space, fine_space, search=None, coarse_operator=None, fine_operator=None, device=None):
    """Locate the fine support points in the coarse mesh (transfer.py:254-256)."""
    return TwoLevelTransferNonNested(coarse_space, fine_space, search, coarse_operator=coarse_operator,
                                     fine_operator=fine_operator, device=device)


def setup_nested(coarse_space, fine_space, search=None, coarse_operator=None, fine_operator=None, device=None):
    """Nested mesh pair (transfer.py:259-260)."""
    return TwoLevelTransferNested(coarse_space, fine_space, search, coarse_operator=coarse_operator,
                                  fine_operator=fine_operator, device=device)


def setup_polynomial(coarse_space, fine_space, coarse_operator=None, fine_operator=None, device=None):
    """p -> p-1 transfer on a shared mesh; needs fine degree >= 2 (transfer.py:263-267)."""
    if fine_space.degree < 2:
        raise ValueError("polynomial coarsening needs degree >= 2")
    return TwoLevelTransferPolynomial(coarse_space, fine_space, coarse_operator=coarse_operator,
                                      fine_operator=fine_operator, device=device)
