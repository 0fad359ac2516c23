"""Point location for the non-nested transfer setup, on the GPU.

Same contract as the reference ``locate_points`` (geosearch.py:163-227):
candidates are the cells whose ``eps_box``-padded bounding box contains the
point (the reference finds them with an AABB tree; the tree only prunes, so a
bucket grid over the same padded boxes yields the same candidate set), each
candidate is inverted with the damped Newton iteration of
``invert_mapping_batch`` (mesh.py:235-287, tol 1e-12 x cell diameter), the
first candidate in ascending cell order that contains the point within
``eps_geo`` / ``eps_ref`` wins and its reference coordinates are clamped to
[0,1]; otherwise the converged candidate whose clamped image lies nearest
(ties to the lowest cell) is taken and the point is flagged ``projected``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib


class GeosearchError(Exception):
    pass


@dataclass
class SearchConfig:
    """Tolerances; None picks the reference's mesh-scaled defaults (geosearch.py:15-21)."""

    eps_box: float = None  # default 1e-6 * coarse-mesh diameter
    eps_geo: float = None  # default 1e-8 * coarse-mesh diameter
    eps_ref: float = 1e-10


class LocatedPoints:
    def __init__(self, points, cells, xhat, projected):
        self.points = points
        self.cells = cells
        self.xhat = xhat
        self.projected = projected

    def __len__(self):
        return len(self.cells)


def locate_points(mesh, points, search=None, device=None):
    search = search or SearchConfig()
    points = np.atleast_2d(np.asarray(points, dtype=float))
    if not np.isfinite(points).all():
        raise GeosearchError("points must be finite")
    dev = D.resolve_device(device)
    diam = mesh.diameter()
    eps_box = 1e-6 * diam if search.eps_box is None else float(search.eps_box)
    eps_geo = 1e-8 * diam if search.eps_geo is None else float(search.eps_geo)
    eps_ref = float(search.eps_ref)
    npts, dim = points.shape
    verts = _lib.as_f64(mesh.vertices)
    cells = _lib.as_i64(mesh.cells)
    pts = _lib.as_f64(points)
    out_cells = np.empty(npts, dtype=np.int64)
    out_xhat = np.empty((npts, dim), dtype=np.float64)
    out_proj = np.empty(npts, dtype=np.uint8)
    nfail = ctypes.c_int64(0)
    first = ctypes.c_int64(-1)
    st = _lib.load().nnmg_locate_points(
        dev.index, dim, len(verts), _lib.host_ptr(verts), len(cells), _lib.host_ptr(cells), npts,
        _lib.host_ptr(pts), eps_box, eps_geo, eps_ref, _lib.host_ptr(out_cells), _lib.host_ptr(out_xhat),
        _lib.host_ptr(out_proj), ctypes.byref(nfail), ctypes.byref(first),
    )
    if st == _lib.STATUS_SEARCH:
        i = int(first.value)
        raise GeosearchError(
            f"points outside padded domain: {nfail.value} point(s), first index {i}, "
            f"first point {points[i].tolist()}"
        )
    _lib.check(st)
    return LocatedPoints(points, out_cells, out_xhat, out_proj.astype(bool))
