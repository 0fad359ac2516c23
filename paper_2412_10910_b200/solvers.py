"""GPU Chebyshev-Jacobi smoother, Lanczos estimate, PCG and coarse solver.

Twins of the reference ``nnmg.solvers`` (``/root/reference/pkg/src/nnmg/solvers.py``)
with the same signatures, defaults, stopping rules and exceptions.  Vectors
live on the device; scalar recurrences (Lanczos tridiagonal, CG alpha/beta,
Chebyshev rho) are computed on the host exactly as the reference does.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import torch

from . import _device as D
from . import _lib


class SolverError(Exception):
    pass


class IndefiniteOperatorError(SolverError):
    pass


class SingularCoarseSystemError(SolverError):
    pass


def _apply_into(op, u, v):
    if hasattr(op, "apply_into"):
        return op.apply_into(u, v)
    v.copy_(op.apply(u))
    return v


def estimate_eigenvalues(op, diag=None, n_iter=12, seed=0, safety=1.1):
    """safety x largest Ritz value of D^-1/2 A D^-1/2 after n_iter Lanczos
    steps from a default_rng(seed) start (solvers.py:24-59)."""
    dev = op.device
    ops = D.vector_ops(dev)
    if diag is None:
        diag = op.diagonal_device()
    elif not isinstance(diag, torch.Tensor):
        diag = torch.from_numpy(np.ascontiguousarray(diag, dtype=np.float64)).to(dev)
    n = op.n_dofs
    dinv_sqrt = torch.from_numpy(1.0 / np.sqrt(diag.cpu().numpy())).to(dev)
    rng = np.random.default_rng(seed)
    v0 = rng.standard_normal(n)
    v0 /= np.linalg.norm(v0)
    v = torch.from_numpy(v0).to(dev)
    v_prev = D.zeros(n, dev)
    s = D.empty(n, dev)
    t = D.empty(n, dev)
    w = D.empty(n, dev)
    u = D.empty(n, dev)
    beta = 0.0
    alphas, betas = [], []
    for _ in range(n_iter):
        ops.mul(dinv_sqrt, v, s)
        _apply_into(op, s, t)
        ops.mul(dinv_sqrt, t, w)
        alpha = ops.dot(v, w)
        ops.axpby(beta, v_prev, 0.0, u)
        ops.axpby(alpha, v, 1.0, u)
        ops.sub(w, u, w)
        alphas.append(alpha)
        beta = float(np.sqrt(ops.dot(w, w)))
        if beta <= 1e-12 * max(abs(a) for a in alphas):
            break
        betas.append(beta)
        v_prev, v = v, v_prev
        ops.axpby(1.0 / beta, w, 0.0, v)
    if len(betas) == len(alphas):
        betas = betas[:-1]
    if len(alphas) == 1:
        ritz = alphas[0]
    else:
        ritz = scipy.linalg.eigh_tridiagonal(np.array(alphas), np.array(betas), eigvals_only=True)[-1]
    return safety * float(ritz)


DEFAULT_WINDOW_RATIO = 10.0


class ChebyshevJacobi:
    """Degree-k Chebyshev iteration with point-Jacobi preconditioning over the
    window [lam_max/window_ratio, lam_max] (solvers.py:68-114)."""

    def __init__(self, op, degree=3, window_ratio=DEFAULT_WINDOW_RATIO, safety=1.1, n_lanczos=12, seed=0,
                 lam_max=None):
        self.op = op
        self.degree = int(degree)
        self.device = op.device
        self._diag_dev = op.diagonal_device()
        if lam_max is None:
            lam_max = estimate_eigenvalues(op, self._diag_dev, n_iter=n_lanczos, seed=seed, safety=safety)
        self.lam_max = float(lam_max)
        self.lam_min = self.lam_max / float(window_ratio)
        self._work = None

    @property
    def diag(self):
        return self._diag_dev.cpu().numpy()

    @property
    def inv_diag(self):
        return 1.0 / self.diag

    def _workspace(self):
        if self._work is None:
            self._work = D.empty(3 * self.op.n_dofs, self.device)
        return self._work

    def sweep_into(self, b, x0, x):
        """One degree-k pass on device tensors; x0 may be None or alias x."""
        _lib.call("nnmg_smoother_sweep", self.op.handle, self.lam_max, self.lam_min, self.degree, b.data_ptr(),
                  None if x0 is None else x0.data_ptr(), x.data_ptr(), self._workspace().data_ptr(),
                  D.stream_ptr(self.device))
        return x

    def smooth(self, b, x0=None, n_sweeps=1):
        n = self.op.n_dofs
        bd, host = D.to_device(b, n, self.device)
        x = D.empty(n, self.device)
        if x0 is not None:
            xd, _ = D.to_device(x0, n, self.device)
            x.copy_(xd)
            cur = x
        else:
            cur = None
        for _ in range(n_sweeps):
            self.sweep_into(bd, cur, x)
            cur = x
        if cur is None:  # n_sweeps == 0 and no x0: the reference returns None
            return None
        return D.from_device(x, host)


def smooth(smoother, b, x0=None, n_sweeps=1):
    return smoother.smooth(b, x0, n_sweeps)


@dataclass
class CgResult:
    x: object
    iterations: int
    converged: bool
    residual_norms: list = field(default_factory=list)


def cg_solve(op, b, precond=None, target_reduction=1e-4, max_iter=1000, x0=None):
    """PCG on the unpreconditioned l2 residual (solvers.py:129-164).

    op: GPU operator (or callable on device tensors); precond: callable on
    device tensors returning a device tensor (e.g. MultigridHierarchy.precondition).
    Returns x as the same kind as b (NumPy in -> NumPy out)."""
    dev = op.device if hasattr(op, "device") else (b.device if isinstance(b, torch.Tensor) else
                                                   D.resolve_device())
    n = op.n_dofs if hasattr(op, "n_dofs") else len(b)
    bd, host = D.to_device(b, n, dev)
    ops = D.vector_ops(dev)
    apply_op = (lambda u, v: _apply_into(op, u, v)) if hasattr(op, "apply") else (lambda u, v: v.copy_(op(u)))
    ap = D.empty(n, dev)
    if x0 is None:
        x = D.zeros(n, dev)
        r = bd.clone()
    else:
        xd, _ = D.to_device(x0, n, dev)
        x = xd.clone()
        apply_op(x, ap)
        r = D.empty(n, dev)
        ops.sub(bd, ap, r)
    norm0 = float(np.sqrt(ops.dot(r, r)))
    history = [norm0]
    if norm0 == 0.0:
        return CgResult(D.from_device(x, host), 0, True, history)
    target = target_reduction * norm0
    z = precond(r) if precond is not None else r.clone()
    p = z.clone()
    rz = ops.dot(r, z)
    for k in range(1, max_iter + 1):
        apply_op(p, ap)
        pap = ops.dot(p, ap)
        if pap <= 0.0:
            raise IndefiniteOperatorError(f"p'Ap = {pap:.3e} at iteration {k}")
        alpha = rz / pap
        ops.cg_update(alpha, p, ap, x, r)
        norm = float(np.sqrt(ops.dot(r, r)))
        history.append(norm)
        if norm <= target:
            return CgResult(D.from_device(x, host), k, True, history)
        z = precond(r) if precond is not None else r.clone()
        rz_new = ops.dot(r, z)
        beta = rz_new / rz
        rz = rz_new
        ops.axpby(1.0, z, beta, p)
    return CgResult(D.from_device(x, host), max_iter, False, history)


def assemble_dense(op):
    """Dense matrix of a GPU operator by applying it to unit vectors.  Equals
    the reference's assemble_oracle(op).toarray() (mfoperator.py:255-285):
    zero-in / identity-out gives unit rows/columns on constrained DoFs."""
    n = op.n_dofs
    dev = op.device
    e = D.zeros(n, dev)
    A = torch.empty((n, n), dtype=torch.float64, device=dev)
    col = D.empty(n, dev)
    for j in range(n):
        e[j] = 1.0
        _apply_into(op, e, col)
        A[:, j] = col
        e[j] = 0.0
    return A.cpu().numpy()


class CoarseSolver:
    """Dense Cholesky below dense_limit DoFs, otherwise Jacobi-PCG to
    cg_reduction (solvers.py:167-206), both on the device."""

    def __init__(self, op, dense_limit=2000, cg_reduction=1e-8, cg_max_iter=10_000):
        self.op = op
        self.device = op.device
        self.cg_reduction = cg_reduction
        self.cg_max_iter = cg_max_iter
        self.dense = op.n_dofs <= dense_limit
        h = ctypes.c_void_p()
        if self.dense:
            if len(op.constraints) == 0:
                # pure Neumann Laplace / free elasticity: constants / rigid modes
                # span the kernel; the reference's factorisation test
                # (solvers.py:179-191) fails on exactly these systems, here we
                # decide structurally instead of on rounding-level pivots
                raise SingularCoarseSystemError(
                    "coarse matrix is numerically singular (all-Neumann system?); "
                    "pin the nullspace or add Dirichlet constraints"
                )
            A = assemble_dense(op)
            A = 0.5 * (A + A.T)
            try:
                chol = scipy.linalg.cho_factor(A)
            except scipy.linalg.LinAlgError as exc:
                raise SingularCoarseSystemError(
                    "coarse matrix is not positive definite (all-Neumann system?); "
                    "pin the nullspace or add Dirichlet constraints"
                ) from exc
            piv = np.abs(np.diag(chol[0]))
            if piv.min() <= 1e-8 * piv.max():
                raise SingularCoarseSystemError(
                    "coarse matrix is numerically singular (all-Neumann system?); "
                    "pin the nullspace or add Dirichlet constraints"
                )
            inv = np.ascontiguousarray(scipy.linalg.cho_solve(chol, np.eye(op.n_dofs)))
            _lib.call("nnmg_coarse_dense_create", op.handle, _lib.host_ptr(inv), ctypes.byref(h))
        else:
            op.diagonal_device()
            _lib.call("nnmg_coarse_cg_create", op.handle, float(cg_reduction), int(cg_max_iter), ctypes.byref(h))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and _lib._lib is not None:  # not at interpreter exit
            _lib.load().nnmg_coarse_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def solve_into(self, b, x):
        _lib.call("nnmg_coarse_solve", self._h, b.data_ptr(), x.data_ptr(), D.stream_ptr(self.device))
        return x

    def solve(self, b):
        bd, host = D.to_device(b, self.op.n_dofs, self.device)
        x = D.empty(self.op.n_dofs, self.device)
        self.solve_into(bd, x)
        if not self.dense:
            it, conv, indef = self.status()
            if indef:
                raise IndefiniteOperatorError(f"p'Ap <= 0 at coarse iteration {it}")
        return D.from_device(x, host)

    def status(self):
        """(iterations, converged, indefinite) of the last CG coarse solve."""
        it, cv, er = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _lib.call("nnmg_coarse_status", self._h, ctypes.byref(it), ctypes.byref(cv), ctypes.byref(er))
        return it.value, bool(cv.value), bool(er.value)

    def info(self):
        a, b, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _lib.call("nnmg_coarse_info", self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
        return {"cluster_ctas": a.value, "threads_per_cta": b.value, "subgroups": c.value}


def coarse_solve(solver, b):
    return solver.solve(b)
