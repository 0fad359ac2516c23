"""ctypes binding of libnnmg_cuda.so (include/nnmg_cuda.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make`` in
``csrc/``).  There is no CPU fallback: if the shared library is missing or no
CUDA device is present, every GPU object raises on construction.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int64, c_uint8, c_uint64, c_void_p

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# NNMG_LIB_PATH: load another build of the same library (A/B experiments)
LIB_PATH = os.environ.get("NNMG_LIB_PATH") or os.path.join(_HERE, "libnnmg_cuda.so")

STATUS_INVALID = 1
STATUS_CUDA = 2
STATUS_UNSUPPORTED = 3
STATUS_GEOMETRY = 4
STATUS_SEARCH = 5
STATUS_INDEFINITE = 6


class NnmgError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


_p_double = POINTER(c_double)
_p_int64 = POINTER(c_int64)
_handle = c_void_p

# name -> (argtypes)
_SIGNATURES = {
    "nnmg_abi_version": [],
    "nnmg_last_error": [],
    "nnmg_launch_count": [],
    "nnmg_measure_fp64_peak": [c_int, POINTER(c_double)],
    "nnmg_level_create": [c_int, c_int, c_int, c_int, c_int, c_int64, c_int64, c_void_p, c_void_p, c_int64,
                          c_void_p, c_int64, c_void_p, c_double, c_double, POINTER(_handle)],
    "nnmg_level_destroy": [_handle],
    "nnmg_level_info": [_handle, _p_int64, _p_int64, POINTER(c_int), _p_int64, _p_int64],
    "nnmg_level_apply": [_handle, c_void_p, c_void_p, c_void_p],
    "nnmg_level_apply_begin": [_handle, c_void_p, c_void_p, c_int, c_void_p],
    "nnmg_level_apply_cells": [_handle, c_void_p, c_void_p, c_int64, c_int64, c_int, c_void_p],
    "nnmg_level_residual": [_handle, c_void_p, c_void_p, c_void_p, c_void_p],
    "nnmg_level_compute_diagonal": [_handle, c_void_p],
    "nnmg_level_diagonal": [_handle, c_void_p, c_void_p],
    "nnmg_level_load_vector": [_handle, c_void_p, c_void_p, c_void_p],
    "nnmg_smoother_sweep": [_handle, c_double, c_double, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    "nnmg_cheb_start": [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_void_p, c_void_p, c_void_p,
                        c_void_p],
    "nnmg_cheb_start_t": [c_int64, c_void_p, c_void_p, c_void_p, c_double, c_void_p, c_void_p, c_void_p, c_void_p],
    "nnmg_cheb_step": [c_int64, c_void_p, c_void_p, c_double, c_double, c_void_p, c_void_p, c_void_p, c_void_p],
    "nnmg_dot_workspace": [],
    "nnmg_dot2": [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    "nnmg_axpby": [c_int64, c_double, c_void_p, c_double, c_void_p, c_void_p],
    "nnmg_sub": [c_int64, c_void_p, c_void_p, c_void_p, c_void_p],
    "nnmg_mul": [c_int64, c_void_p, c_void_p, c_void_p, c_void_p],
    "nnmg_cg_update": [c_int64, c_double, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    "nnmg_transfer_create": [_handle, _handle, c_int64, c_void_p, c_void_p, c_void_p, POINTER(_handle)],
    "nnmg_transfer_destroy": [_handle],
    "nnmg_transfer_prolongate": [_handle, c_void_p, c_void_p, c_int, c_void_p],
    "nnmg_transfer_restrict": [_handle, c_void_p, c_void_p, c_void_p],
    "nnmg_transfer_set_timing": [_handle, c_int],
    "nnmg_transfer_last_timing": [_handle, POINTER(c_double), POINTER(c_double)],
    "nnmg_locate_points": [c_int, c_int, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_double,
                           c_double, c_double, c_void_p, c_void_p, c_void_p, _p_int64, _p_int64],
    "nnmg_coarse_dense_create": [_handle, c_void_p, POINTER(_handle)],
    "nnmg_coarse_cg_create": [_handle, c_double, c_int, POINTER(_handle)],
    "nnmg_coarse_direct_create": [_handle, c_void_p, c_int64, POINTER(_handle)],
    "nnmg_coarse_direct_create_f32": [_handle, c_void_p, c_int64, POINTER(_handle)],
    "nnmg_coarse_direct_create_share": [_handle, c_void_p, c_int64, c_int, c_int, POINTER(_handle)],
    "nnmg_coarse_destroy": [_handle],
    "nnmg_coarse_solve": [_handle, c_void_p, c_void_p, c_void_p],
    "nnmg_coarse_status": [_handle, POINTER(c_int), POINTER(c_int), POINTER(c_int)],
    "nnmg_coarse_info": [_handle, POINTER(c_int), POINTER(c_int), POINTER(c_int)],
    "nnmg_vcycle_create": [c_int, c_void_p, c_void_p, _handle, c_void_p, c_void_p, c_void_p, c_int, c_int,
                           POINTER(_handle)],
    "nnmg_vcycle_destroy": [_handle],
    "nnmg_vcycle_run": [_handle, c_void_p, c_void_p, c_void_p],
    "nnmg_vcycle_use_graph": [_handle, c_int],
    "nnmg_vcycle_set_precision": [_handle, c_int],
    "nnmg_vcycle_set_mixed_coarse": [_handle, _handle],
    "nnmg_level_set_deterministic": [_handle, c_int],
    "nnmg_halo_pack": [c_int64, c_void_p, c_void_p, c_void_p, c_void_p],
    "nnmg_halo_unpack": [c_int64, c_void_p, c_void_p, c_void_p, c_int, c_void_p],
    "nnmg_vcycle_kernels_per_cycle": [_handle, _p_int64],
}

_RESTYPES = {"nnmg_last_error": ctypes.c_char_p, "nnmg_launch_count": c_uint64}

_lib = None


def exported_symbols():
    return sorted(_SIGNATURES)


def load(path=None):
    """Load (once) and return the ctypes library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not found: build the CUDA extension first (python -c 'import __graft_entry__ as g; g.build()')"
        )
    lib = ctypes.CDLL(path)
    for name, args in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, c_int)
    _lib = lib
    return lib


def check(status):
    if status != 0:
        msg = load().nnmg_last_error().decode(errors="replace")
        if status in (STATUS_INVALID, STATUS_GEOMETRY):
            raise ValueError(msg)
        if status == STATUS_UNSUPPORTED:
            raise NotImplementedError(msg)
        raise NnmgError(status, msg)


def call(name, *args):
    check(getattr(load(), name)(*args))


def launch_count():
    return int(load().nnmg_launch_count())


def host_ptr(a):
    """Pointer to a C-contiguous numpy array (caller keeps it alive)."""
    return c_void_p(a.ctypes.data) if a.size else c_void_p(None)


def as_i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def as_f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def fp64_peak(device=0):
    """Measured DFMA throughput (TFLOP/s) of ``device``: the FP64 roofline denominator."""
    out = ctypes.c_double(0.0)
    call("nnmg_measure_fp64_peak", int(device), ctypes.byref(out))
    return out.value
