"""V-cycle over GPU levels and its use as a CG preconditioner.

``MultigridHierarchy`` keeps the reference's interface and recursion
(``/root/reference/pkg/src/nnmg/multigrid.py:32-117``: Alg. 1, 1-based level
numbers, zero initial guess on coarse levels, per-(level, component) timers).
Two execution modes:

* ``executor=False``: the Python recursion of multigrid.py:83-113 calling the
  GPU components one by one, with per-component CUDA-event timers;
* ``executor=True`` (default for ``precondition``): the native V-cycle of
  libnnmg_cuda.so (nnmg_vcycle_*), replayed as one CUDA graph.

``build_hp_hierarchy`` mirrors multigrid.py:145-203 for the non-nested
``mode="h"`` hierarchies of the BASELINE configurations.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _lib
from .fespace import build_space, dirichlet_constraints
from .geosearch import SearchConfig
from .mfoperator import ElasticityOperator, LaplaceOperator
from .solvers import ChebyshevJacobi, CoarseSolver
from .transfer import setup_nested, setup_nonnested, setup_polynomial

V_CYCLE_COMPONENTS = (
    "pre_smooth",
    "residual",
    "restrict",
    "coarse_solve",
    "prolongate",
    "post_smooth",
)


@dataclass
class Level:
    space: object
    operator: object
    smoother: object


class MultigridHierarchy:
    """Ordered levels (coarsest first) with two-level transfers between them."""

    def __init__(self, levels, transfers, coarse_solver, m1=1, m2=1, timing=False):
        if len(transfers) != len(levels) - 1:
            raise ValueError("need one transfer per consecutive level pair")
        for i, t in enumerate(transfers):
            if t.coarse_space is not levels[i].space or t.fine_space is not levels[i + 1].space:
                raise ValueError(f"transfer {i} does not connect levels {i} and {i + 1}")
        self.levels = list(levels)
        self.transfers = list(transfers)
        self.coarse_solver = coarse_solver
        self.m1 = int(m1)
        self.m2 = int(m2)
        self.timings = {}
        self.timing = bool(timing)
        self.device = levels[-1].operator.device
        self._vc = None
        self._graph = True
        self.precision = 64

    @property
    def n_levels(self):
        return len(self.levels)

    @property
    def finest(self):
        return self.levels[-1]

    def reset_timers(self):
        self.timings = {}

    def _record(self, level, component, seconds):
        key = (level, component)
        t, c = self.timings.get(key, (0.0, 0))
        self.timings[key] = (t + seconds, c + 1)

    def timing_rows(self):
        rows = []
        for (level, comp), (secs, calls) in sorted(self.timings.items()):
            rows.append((level, comp, secs, calls))
        return rows

    # -- Python recursion with device tensors ----------------------------------
    def _timed(self, level, comp, fn):
        if not self.timing:
            return fn()
        s = torch.cuda.current_stream(self.device)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        out = fn()
        e1.record(s)
        e1.synchronize()
        self._record(level, comp, e0.elapsed_time(e1) * 1e-3)
        return out

    def _v(self, l, f):
        dev = self.device
        if l == 1:
            cs = self.coarse_solver
            x = D.empty(self.levels[0].operator.n_dofs, dev)
            return self._timed(1, "coarse_solve", lambda: cs.solve_into(f, x))
        lev = self.levels[l - 1]
        T = self.transfers[l - 2]
        n = lev.operator.n_dofs
        x = D.empty(n, dev)

        def pre():
            cur = None
            for _ in range(self.m1):
                lev.smoother.sweep_into(f, cur, x)
                cur = x
            if cur is None:
                x.zero_()
            return x

        self._timed(l, "pre_smooth", pre)
        r = D.empty(n, dev)
        self._timed(l, "residual", lambda: lev.operator.residual_into(f, x, r))
        rc = D.empty(T.coarse_space.n_dofs, dev)
        self._timed(l, "restrict", lambda: T.restrict_into(r, rc))
        delta = self._v(l - 1, rc)
        self._timed(l, "prolongate", lambda: T.prolongate_into(delta, x, accumulate=True))

        def post():
            for _ in range(self.m2):
                lev.smoother.sweep_into(f, x, x)
            return x

        self._timed(l, "post_smooth", post)
        return x

    # -- native executor ---------------------------------------------------------
    def _executor(self):
        if self._vc is None:
            n = self.n_levels
            lv = (ctypes.c_void_p * n)(*[lev.operator.handle.value for lev in self.levels])
            tr = (ctypes.c_void_p * max(1, n - 1))(*[t.handle.value for t in self.transfers])
            lmax = np.array([getattr(lev.smoother, "lam_max", 1.0) if i else 1.0 for i, lev in enumerate(self.levels)])
            lmin = np.array([getattr(lev.smoother, "lam_min", 0.1) if i else 0.1 for i, lev in enumerate(self.levels)])
            deg = np.array([getattr(lev.smoother, "degree", 1) if i else 1 for i, lev in enumerate(self.levels)],
                           dtype=np.int32)
            h = ctypes.c_void_p()
            _lib.call("nnmg_vcycle_create", n, ctypes.cast(lv, ctypes.c_void_p), ctypes.cast(tr, ctypes.c_void_p),
                      self.coarse_solver.handle, _lib.host_ptr(lmax), _lib.host_ptr(lmin), _lib.host_ptr(deg),
                      self.m1, self.m2, ctypes.byref(h))
            self._vc = h
            self._vc_keep = (lv, tr, lmax, lmin, deg)
            if self.precision != 64:
                self._attach_mixed_coarse()
                _lib.call("nnmg_vcycle_set_precision", h, int(self.precision))
        return self._vc

    def _attach_mixed_coarse(self):
        """The mixed-precision cycle's coarse solve: the packed inverse in fp32
        tiles where the coarse solver offers it (half the bytes of the fp64
        direct solve; on C3 faster than the coarse CG the fp64 cycle keeps)."""
        make = getattr(self.coarse_solver, "mixed_handle", None)
        h32 = make() if make is not None else None
        if h32 is not None and self._vc is not None:
            _lib.call("nnmg_vcycle_set_mixed_coarse", self._vc, h32)

    def set_precision(self, bits):
        """64: the fp64 V-cycle (default).  32: the paper's mixed-precision
        cycle: fp32 storage of level vectors, geometry,
        inverse diagonals and transfer coordinates above the coarsest level,
        single-precision arithmetic in the register applies and the transfers
        (NNMG_MIXED_ARITH=64: fp64 arithmetic on the fp32 storage), fp64
        coarse vectors; the cycle's input and output (and the outer CG) stay
        fp64.  Native executor only."""
        if bits not in (32, 64):
            raise ValueError("precision must be 32 or 64")
        self.precision = int(bits)
        if self._vc is not None:
            if bits == 32:
                self._attach_mixed_coarse()
            _lib.call("nnmg_vcycle_set_precision", self._vc, int(bits))

    def use_graph(self, enable=True):
        self._graph = bool(enable)

    def kernels_per_cycle(self):
        v = ctypes.c_int64()
        _lib.call("nnmg_vcycle_kernels_per_cycle", self._executor(), ctypes.byref(v))
        return v.value

    def v_cycle_into(self, f, x):
        """x = V-cycle(f) on the finest level through the native executor."""
        vc = self._executor()
        stream = D.stream_ptr(self.device)
        graph = self._graph and stream not in (0, None)
        _lib.call("nnmg_vcycle_use_graph", vc, 1 if graph else 0)
        _lib.call("nnmg_vcycle_run", vc, f.data_ptr(), x.data_ptr(), stream)
        return x

    def __del__(self):
        h = getattr(self, "_vc", None)
        if h is not None and h.value and _lib is not None and _lib._lib is not None:  # not at interpreter exit
            _lib.load().nnmg_vcycle_destroy(h)
            self._vc = None

    # -- public API ------------------------------------------------------------
    def v_cycle(self, f, level=None, executor=None):
        """One V-cycle for A_l x = f at 1-based level l; returns the correction."""
        l = self.n_levels if level is None else int(level)
        if not 1 <= l <= self.n_levels:
            raise ValueError(f"level must be in [1, {self.n_levels}]")
        n = self.levels[l - 1].operator.n_dofs
        fd, host = D.to_device(f, n, self.device)
        use_exec = (not self.timing) if executor is None else bool(executor)
        if self.precision != 64 and not (use_exec and l == self.n_levels):
            raise ValueError("the mixed-precision cycle runs in the native executor on the finest level only")
        if use_exec and l == self.n_levels:
            x = D.empty(n, self.device)
            self.v_cycle_into(fd, x)
        else:
            x = self._v(l, fd)
        return D.from_device(x, host)

    def precondition(self, r):
        """z = V-cycle(r) on the finest level, suitable inside CG."""
        return self.v_cycle(r)


@dataclass
class HierarchyConfig:
    """Solver configuration (multigrid.py:120-132)."""

    chebyshev_degree: int = 3
    m1: int = 1
    m2: int = 1
    window_ratio: float = 10.0
    safety: float = 1.1
    lanczos_iters: int = 12
    lanczos_seed: int = 0
    coarse_dense_limit: int = 2000
    coarse_cg_reduction: float = 1e-8
    # not in the reference: exact solve above the dense limit where faster
    # (False = the reference's CG, the parity mode; True; "auto")
    coarse_direct: object = False
    # 64: fp64 V-cycle; 32: the paper's mixed-precision cycle
    vcycle_precision: int = 64
    # fixed-order (atomic-free) summation in every apply / diagonal / load
    # vector and an exact coarse solve: bitwise reproducible V-cycles and
    # iteration counts (the reference's serial scatter, mfoperator.py:88-90)
    deterministic: bool = False


def _make_operator(space, problem, lame, device, deterministic=False):
    if problem == "poisson":
        return LaplaceOperator(space, device=device, deterministic=deterministic)
    if problem == "elasticity":
        if lame is None:
            raise ValueError("elasticity needs lame=(lambda, mu)")
        return ElasticityOperator(space, *lame, device=device, deterministic=deterministic)
    raise ValueError(f"unknown problem {problem!r}")


def build_hp_hierarchy(meshes, degree, mode="h", nested=False, problem="poisson", dirichlet_ids="all",
                       dirichlet_value=0.0, lame=None, search=None, config=None, device=None, timing=False):
    """GPU hierarchy over coarse-to-fine meshes (multigrid.py:145-203).

    mode "h" uses the meshes as given; mode "hp" prepends Q^1..Q^(degree-1)
    levels on the coarsest mesh below the geometric stack (polynomial
    transfers).  nested=True uses the nested transfer between meshes (global
    refinement), otherwise the non-nested point-evaluation transfer."""
    if mode not in ("h", "hp"):
        raise ValueError("mode must be 'h' or 'hp'")
    if not meshes:
        raise ValueError("need at least one mesh")
    cfg = config or HierarchyConfig()
    search = search or SearchConfig()
    dev = D.resolve_device(device)
    n_components = meshes[0].dim if problem == "elasticity" else 1
    # (degree, mesh, kind of the incoming transfer) as multigrid.py:166-175
    plan = []
    if mode == "hp":
        plan.append((1, meshes[0], None))
        for p in range(2, degree + 1):
            plan.append((p, meshes[0], "poly"))
    else:
        plan.append((degree, meshes[0], None))
    for m in meshes[1:]:
        plan.append((degree, m, "nested" if nested else "nonnested"))
    levels, transfers = [], []
    for p, mesh, kind in plan:
        space = build_space(mesh, p, n_components=n_components)
        if dirichlet_ids is not None:
            space.constraints = dirichlet_constraints(space, dirichlet_ids, dirichlet_value)
        op = _make_operator(space, problem, lame, dev, cfg.deterministic)
        smoother = ChebyshevJacobi(op, degree=cfg.chebyshev_degree, window_ratio=cfg.window_ratio,
                                   safety=cfg.safety, n_lanczos=cfg.lanczos_iters, seed=cfg.lanczos_seed)
        levels.append(Level(space, op, smoother))
        if kind is None:
            continue
        cop, cspace = levels[-2].operator, levels[-2].space
        if kind == "poly":
            transfers.append(setup_polynomial(cspace, space, coarse_operator=cop, fine_operator=op))
        elif kind == "nested":
            transfers.append(setup_nested(cspace, space, search, coarse_operator=cop, fine_operator=op))
        else:
            transfers.append(setup_nonnested(cspace, space, search, coarse_operator=cop, fine_operator=op))
    # the coarse CG kernel sums with atomics: deterministic mode solves exactly
    coarse = CoarseSolver(levels[0].operator, dense_limit=cfg.coarse_dense_limit,
                          cg_reduction=cfg.coarse_cg_reduction,
                          direct=True if cfg.deterministic else cfg.coarse_direct)
    H = MultigridHierarchy(levels, transfers, coarse, m1=cfg.m1, m2=cfg.m2, timing=timing)
    if cfg.vcycle_precision != 64:
        H.set_precision(cfg.vcycle_precision)
    return H
