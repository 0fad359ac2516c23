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


def assemble_dense_device(op, rows=None):
    """Dense matrix of a GPU operator on the device: row k = (A e_j)[rows]
    for j = rows[k] (A is symmetric; constrained rows/columns are unit
    vectors as in assemble_oracle, mfoperator.py:255-285).  rows=None: all."""
    n = op.n_dofs
    dev = op.device
    rows = np.arange(n) if rows is None else np.asarray(rows, dtype=np.int64)
    ri = torch.from_numpy(rows).to(dev)
    e = D.zeros(n, dev)
    col = D.empty(n, dev)
    A = torch.empty((len(rows), len(rows)), dtype=torch.float64, device=dev)
    for k, j in enumerate(rows.tolist()):
        e[j] = 1.0
        _apply_into(op, e, col)
        torch.index_select(col, 0, ri, out=A[k])
        e[j] = 0.0
    return A


# effective stream rate of the direct solve's packed symmetric GEMV (B200,
# measured: profiles/r2_coarse_direct.txt), used to predict its time
DIRECT_STREAM_BYTES_PER_S = 6.3e12


def direct_solve_bytes(n_free):
    nb = (n_free + 63) // 64
    return 8 * 4096 * nb * (nb + 1) // 2


class CoarseSolver:
    """Dense Cholesky below dense_limit DoFs, otherwise Jacobi-PCG to
    cg_reduction (solvers.py:167-206), both on the device.

    direct (not in the reference): above the dense limit, solve exactly with
    the SPD inverse streamed as packed symmetric tiles (nnmg_coarse_direct_*)
    instead of iterating.  False (default, the reference's semantics and the
    parity mode), True, or "auto": only where the predicted GEMV time
    (direct_solve_bytes / DIRECT_STREAM_BYTES_PER_S) beats 0.8x the measured
    time of one CG solve and the setup fits in device memory.  The inverse
    covers the free DoFs only (constrained rows are identity).  The V-cycle
    then differs from the reference's at the level of the coarse CG tolerance
    (1e-8); outer CG iteration counts are the parity gate."""

    def __init__(self, op, dense_limit=2000, cg_reduction=1e-8, cg_max_iter=10_000, direct=False, share=None):
        if direct not in (False, True, "auto"):
            raise ValueError("direct must be False, True or 'auto'")
        # share = (i, n): cell-partitioned runs with the direct path stream an
        # equal share of the inverse tiles per rank; solve_into then yields a
        # PARTIAL result and the caller sums the shares (all-reduce)
        if share is not None and not (len(share) == 2 and 0 <= share[0] < share[1]):
            raise ValueError("share must be (index, count) with 0 <= index < count")
        self.share = tuple(int(v) for v in share) if share is not None and share[1] > 1 else None
        self.op = op
        self.device = op.device
        self.cg_reduction = cg_reduction
        self.cg_max_iter = cg_max_iter
        self.dense = op.n_dofs <= dense_limit
        self.direct = False
        self._direct_mode = direct   # False: the reference's CG only (parity mode)
        self._h32 = None             # fp32-tile direct solve of the mixed-precision cycle (mixed_handle)
        self._h32_tried = False
        self.timing = None
        self.choice = "dense" if self.dense else "cg"
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
        if not self.dense and direct:
            nf = op.n_dofs - len(op.constraints.dofs)
            t_cg = self._time_cg() if direct == "auto" else None
            t_direct = direct_solve_bytes(nf) / DIRECT_STREAM_BYTES_PER_S
            mem = torch.cuda.mem_get_info(self.device)[0]
            if self.share is not None:
                t_direct /= self.share[1]
            fits = 3 * 8 * nf ** 2 + direct_solve_bytes(nf) < 0.8 * mem
            self.timing = {"cg_s": t_cg, "direct_predicted_s": t_direct}
            if direct is True or (fits and t_direct < 0.9 * t_cg):
                self._make_direct()
        self.partial = self.direct and self.share is not None  # solve_into returns this rank's share of x

    def _time_cg(self):
        """Device time of one CG solve on a random right-hand side (after one
        untimed solve); the CG iteration count barely depends on the RHS."""
        n = self.op.n_dofs
        rng = np.random.default_rng(7)
        b = torch.from_numpy(rng.standard_normal(n)).to(self.device)
        b[torch.from_numpy(_lib.as_i64(self.op.constraints.dofs)).to(self.device)] = 0.0
        x = D.empty(n, self.device)
        s = torch.cuda.current_stream(self.device)
        self.solve_into(b, x)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        self.solve_into(b, x)
        e1.record(s)
        e1.synchronize()
        return e0.elapsed_time(e1) * 1e-3

    def mixed_handle(self):
        """Coarse solver handle for the mixed-precision cycle, or None to share
        the fp64 one: the exact inverse packed in fp32 tiles
        (nnmg_coarse_direct_create_f32), half the bytes of the fp64 direct
        solve.  Built on first use where the direct path is allowed
        (direct=True / "auto") and predicted faster than the active solver."""
        if self.dense or not self._direct_mode or self.share is not None:
            return None
        if self._h32 is None and not self._h32_tried:
            self._h32_tried = True
            nf = self.op.n_dofs - len(self.op.constraints.dofs)
            t32 = 0.5 * direct_solve_bytes(nf) / DIRECT_STREAM_BYTES_PER_S
            if self.direct:
                t_now = direct_solve_bytes(nf) / DIRECT_STREAM_BYTES_PER_S
            else:
                t_now = (self.timing or {}).get("cg_s") or self._time_cg()
            mem = torch.cuda.mem_get_info(self.device)[0]
            fits = 3 * 8 * nf ** 2 + direct_solve_bytes(nf) // 2 < 0.8 * mem
            if self._direct_mode is True or (fits and t32 < 0.9 * t_now):
                self._h32 = self._make_direct(f32=True)
                self.timing = dict(self.timing or {}, mixed_direct_predicted_s=t32)
        return self._h32

    def _make_direct(self, f32=False):
        n = self.op.n_dofs
        cons = np.asarray(self.op.constraints.dofs, dtype=np.int64)
        if len(cons) == 0:
            # constants / rigid modes span the kernel (decided structurally, as
            # the dense path does; test_solvers.py:167-172)
            raise SingularCoarseSystemError(
                "coarse matrix is numerically singular (all-Neumann system?); "
                "pin the nullspace or add Dirichlet constraints"
            )
        free = np.setdiff1d(np.arange(n), cons)
        A = assemble_dense_device(self.op, free)
        A.add_(A.T.clone()).mul_(0.5)
        Lc, info = torch.linalg.cholesky_ex(A)
        del A
        if int(info.item()) != 0:
            raise SingularCoarseSystemError(
                "coarse matrix is not positive definite (all-Neumann system?); "
                "pin the nullspace or add Dirichlet constraints"
            )
        piv = Lc.diagonal().abs()
        if len(piv) and float(piv.min()) <= 1e-8 * float(piv.max()):
            raise SingularCoarseSystemError(
                "coarse matrix is numerically singular (all-Neumann system?); "
                "pin the nullspace or add Dirichlet constraints"
            )
        inv = torch.cholesky_inverse(Lc)
        del Lc
        h = ctypes.c_void_p()
        if self.share is not None and not f32:
            _lib.call("nnmg_coarse_direct_create_share", self.op.handle, inv.data_ptr(), len(free), self.share[0],
                      self.share[1], ctypes.byref(h))
        else:
            _lib.call("nnmg_coarse_direct_create_f32" if f32 else "nnmg_coarse_direct_create", self.op.handle,
                      inv.data_ptr(), len(free), ctypes.byref(h))
        torch.cuda.synchronize(self.device)
        del inv
        if f32:
            return h
        _lib.load().nnmg_coarse_destroy(self._h)
        self._h = h
        self.direct = True
        self.choice = "direct"

    def __del__(self):
        for name in ("_h", "_h32"):
            h = getattr(self, name, None)
            if h is not None and h.value and _lib is not None and _lib._lib is not None:  # not at interpreter exit
                _lib.load().nnmg_coarse_destroy(h)
                setattr(self, name, None)

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
        if not self.dense and not self.direct:
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
        out = {"kind": self.choice, "cluster_ctas": a.value, "threads_per_cta": b.value, "subgroups": c.value}
        if getattr(self, "timing", None):
            out.update(self.timing)
        return out


def coarse_solve(solver, b):
    return solver.solve(b)
