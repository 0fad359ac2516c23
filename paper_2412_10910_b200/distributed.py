"""Multi-GPU domain decomposition of the V-cycle hot path.

One process per GPU with ``torch.distributed`` (NCCL) for the plumbing:

* **Partition.** Each non-coarsest level's cells are split by the reference's
  Morton policy (``partition_morton``, metrics.py:24-38). A scalar DoF belongs
  to the rank of the lowest-index cell containing it (``dof_owner_cells``,
  metrics.py:60-64).
* **Local vectors** hold owned DoFs first, then ghosts; both are sorted by
  global id. The ghosts are every DoF of an owned cell plus, on coarse levels,
  every DoF of a coarse cell that owns one of this rank's fine transfer points.
* **Apply.** Import the ghost values (halo), run the local cell loop (the GPU
  kernels), then export-add the ghost partial sums to their owners.
  Constrained ghosts are never exported; the owner applies identity-out.
  A rank's cells are ordered interior first (every DoF owned), boundary last:
  the interior cell blocks run on the compute stream while the ghost import
  (pack kernel, NCCL point-to-point, unpack kernel) is in flight on a side
  stream; the boundary blocks wait for it (SURVEY §8(e) "overlap interior
  cells with the exchange").
* **Transfers.** Fine points are owned. Prolongation imports the coarse ghosts
  first. Restriction export-adds the coarse ghost partials; on the replicated
  coarsest level it all-reduces them.
* **Coarsest level** is replicated: every rank runs the identical
  device-resident coarse solve and needs no further communication.
* **Dots** are reduced locally over owned entries, then all-reduced.

All halo plans are built at setup from global (replicated) host data plus one
``all_gather_object`` of the per-rank ghost lists. Halo traffic uses batched
point-to-point ops, which NCCL and gloo both support. Local compute is
injected through a *backend*. ``GpuBackend`` (the default) runs the CUDA
kernels of ``libnnmg_cuda.so``. The world_size-2 tests in ``tests/`` inject
an oracle backend to check this host logic on CPU with gloo.
"""

from __future__ import annotations

import os

import numpy as np
import scipy.linalg
import torch
import torch.distributed as dist

from .fespace import DirichletConstraints, FESpace
from .mesh import Mesh

# ---------------------------------------------------------------------------
# partitioning (host, deterministic on every rank)
# ---------------------------------------------------------------------------


def _morton_codes(points, lo, hi, bits=16):
    """Interleaved-bit Z-order codes of quantised coordinates (metrics.py:11-21)."""
    span = np.where(hi > lo, hi - lo, 1.0)
    q = ((points - lo) / span * (2**bits - 1)).astype(np.uint64)
    codes = np.zeros(len(points), dtype=np.uint64)
    for b in range(bits):
        for j in range(points.shape[1]):
            codes |= ((q[:, j] >> np.uint64(b)) & np.uint64(1)) << np.uint64(b * points.shape[1] + j)
    return codes


def partition_morton(mesh, n_ranks):
    """Equal-count contiguous split of the cells along the Morton curve
    (metrics.py:24-38); returns the owner rank of every cell."""
    if n_ranks < 1 or n_ranks > mesh.n_cells:
        raise ValueError("need 1 <= n_ranks <= n_cells")
    lo, hi = mesh.vertices.min(axis=0), mesh.vertices.max(axis=0)
    cent = np.zeros((mesh.n_cells, mesh.dim))
    for v in range(mesh.cells.shape[1]):
        cent += mesh.vertices[mesh.cells[:, v]]
    cent /= mesh.cells.shape[1]
    order = np.lexsort((np.arange(mesh.n_cells), _morton_codes(cent, lo, hi)))
    counts = np.full(n_ranks, mesh.n_cells // n_ranks, dtype=np.int64)
    counts[: mesh.n_cells % n_ranks] += 1
    owner = np.empty(mesh.n_cells, dtype=np.int64)
    owner[order] = np.repeat(np.arange(n_ranks), counts)
    return owner


def partition_matching(mesh, fine_mesh, fine_owner, locate):
    """Owner of each cell = owner of the fine cell containing its centroid
    (metrics.py:41-46), so consecutive levels overlap spatially and the
    transfers stay mostly rank-local.  ``locate(mesh, points)`` returns the
    owning cells (the backend's point location)."""
    cent = np.zeros((mesh.n_cells, mesh.dim))
    for v in range(mesh.cells.shape[1]):
        cent += mesh.vertices[mesh.cells[:, v]]
    cent /= mesh.cells.shape[1]
    return np.asarray(fine_owner)[np.asarray(locate(fine_mesh, cent))]


def dof_owner_ranks(cell_dofs, cell_owner, n_scalar):
    """Rank of the lowest-index cell containing each scalar DoF."""
    nc, nloc = cell_dofs.shape
    first = np.full(n_scalar, nc, dtype=np.int64)
    np.minimum.at(first, cell_dofs.ravel(), np.repeat(np.arange(nc), nloc))
    return cell_owner[first]


# ---------------------------------------------------------------------------
# layouts and halo plans
# ---------------------------------------------------------------------------


# cells per block of the level handles (nnmg_level_info: 32 for every
# supported element); the interior / boundary split is aligned to it
CELL_ALIGN = 32


class LevelLayout:
    """Local numbering of one level on one rank: owned DoFs, then ghosts."""

    def __init__(self, space, cell_owner, dof_owner, rank, extra_dofs=None, replicated=False):
        self.rank = rank
        self.ncomp = space.n_components
        self.replicated = replicated
        self.n_global_scalar = space.n_scalar_dofs
        cell_dofs = np.asarray(space.cell_dofs)
        self.n_interior_cells = 0
        if replicated:
            self.owned_cells = np.arange(len(cell_dofs))
            self.owned = np.arange(space.n_scalar_dofs)
            self.ghosts = np.zeros(0, dtype=np.int64)
            self.cell_ghosts = self.ghosts
        else:
            oc = np.nonzero(cell_owner == rank)[0]
            # interior cells (no ghost DoF) first, boundary cells last, both in
            # ascending global order; the interior count is cut to whole cell
            # blocks so the two groups are block ranges of the level handle
            bnd = (dof_owner[cell_dofs[oc]] != rank).any(axis=1)
            self.owned_cells = np.concatenate([oc[~bnd], oc[bnd]])
            self.n_interior_cells = (int((~bnd).sum()) // CELL_ALIGN) * CELL_ALIGN
            self.owned = np.nonzero(dof_owner == rank)[0]
            touched = np.unique(cell_dofs[self.owned_cells])
            self.cell_ghosts = touched[dof_owner[touched] != rank]
            ghosts = self.cell_ghosts
            if extra_dofs is not None and len(extra_dofs):
                ex = np.unique(extra_dofs)
                ghosts = np.union1d(ghosts, ex[dof_owner[ex] != rank])
            self.ghosts = ghosts
        self.l2g = np.concatenate([self.owned, self.ghosts])
        self.n_owned = len(self.owned)
        self.n_local = len(self.l2g)
        self._g2l = np.full(self.n_global_scalar, -1, dtype=np.int64)
        self._g2l[self.l2g] = np.arange(self.n_local)
        cmask = np.zeros(space.n_dofs, dtype=bool)
        cmask[space.constraints.dofs] = True
        self.global_constrained_scalar = cmask.reshape(-1, self.ncomp).all(axis=1)
        loc_full = self.full(np.arange(self.n_local))
        self.local_constrained = np.nonzero(cmask[self.full_global(np.arange(self.n_local))])[0]
        del loc_full

    def g2l(self, g):
        out = self._g2l[np.asarray(g)]
        if (out < 0).any():
            raise KeyError("global DoF not present on this rank")
        return out

    def full(self, scalar_local):
        s = np.asarray(scalar_local, dtype=np.int64)
        return (s[:, None] * self.ncomp + np.arange(self.ncomp)[None]).ravel()

    def full_global(self, scalar_local):
        s = self.l2g[np.asarray(scalar_local, dtype=np.int64)]
        return (s[:, None] * self.ncomp + np.arange(self.ncomp)[None]).ravel()

    @property
    def n_owned_full(self):
        return self.n_owned * self.ncomp

    @property
    def n_local_full(self):
        return self.n_local * self.ncomp

    def local_space(self, space, cells_global):
        """FESpace over the given global cells in this rank's local numbering."""
        mesh = space.mesh
        sub = np.asarray(mesh.cells)[cells_global]
        used, inv = np.unique(sub, return_inverse=True)
        lmesh = Mesh(mesh.dim, mesh.vertices[used], inv.reshape(sub.shape), np.zeros((0, 3), np.int64),
                     validate=False)
        lcd = self.g2l(np.asarray(space.cell_dofs)[cells_global])
        lsp = FESpace(lmesh, space.degree, self.ncomp, lcd, np.asarray(space.support_points)[self.l2g])
        lsp.constraints = DirichletConstraints(self.local_constrained)
        return lsp


class HaloPlan:
    """Per-peer (send, recv) local index lists, full (component) indices."""

    def __init__(self, layout, mine, theirs_by_rank, dof_owner):
        """mine: global scalar ghosts this rank receives (import) or sends
        (export); theirs_by_rank[q]: the same list of rank q."""
        r = layout.rank
        self.peers = []
        self.send, self.recv = {}, {}
        for q, theirs in enumerate(theirs_by_rank):
            if q == r:
                continue
            mine_q = mine[dof_owner[mine] == q] if len(mine) else mine
            theirs_q = theirs[dof_owner[theirs] == r] if len(theirs) else theirs
            if len(mine_q) == 0 and len(theirs_q) == 0:
                continue
            self.peers.append(q)
            self.recv[q] = layout.full(layout.g2l(mine_q))
            self.send[q] = layout.full(layout.g2l(theirs_q))

    def to(self, device):
        self.send = {q: torch.from_numpy(v).to(device) for q, v in self.send.items()}
        self.recv = {q: torch.from_numpy(v).to(device) for q, v in self.recv.items()}
        # persistent per-peer message buffers (no allocation per exchange;
        # fixed addresses, so the exchange can live in a CUDA graph)
        f64 = dict(dtype=torch.float64, device=device)
        self.buf_send = {q: torch.empty(len(v), **f64) for q, v in self.send.items()}
        self.buf_recv = {q: torch.empty(len(v), **f64) for q, v in self.recv.items()}
        return self


def _pack(x, idx, out):
    """out[i] = x[idx[i]]: the K9 pack kernel on the GPU, index_select on CPU."""
    if x.is_cuda:
        from . import _device as D
        from . import _lib

        _lib.call("nnmg_halo_pack", idx.numel(), idx.data_ptr(), x.data_ptr(), out.data_ptr(),
                  D.stream_ptr(x.device))
    else:
        torch.index_select(x, 0, idx, out=out)


def _unpack(x, idx, buf, add):
    """x[idx[i]] = buf[i] (or +=): the K9 unpack kernel on the GPU."""
    if x.is_cuda:
        from . import _device as D
        from . import _lib

        _lib.call("nnmg_halo_unpack", idx.numel(), idx.data_ptr(), buf.data_ptr(), x.data_ptr(), 1 if add else 0,
                  D.stream_ptr(x.device))
    elif add:
        x.index_add_(0, idx, buf)
    else:
        x.index_copy_(0, idx, buf)


def _exchange(peers, sendbufs, recvbufs):
    ops = []
    for q in peers:
        if recvbufs[q].numel():
            ops.append(dist.P2POp(dist.irecv, recvbufs[q], q))
        if sendbufs[q].numel():
            ops.append(dist.P2POp(dist.isend, sendbufs[q], q))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def halo_import(plan, x):
    """Owner values -> ghost copies (x is a local vector)."""
    for q in plan.peers:
        _pack(x, plan.send[q], plan.buf_send[q])
    _exchange(plan.peers, plan.buf_send, plan.buf_recv)
    for q in plan.peers:
        _unpack(x, plan.recv[q], plan.buf_recv[q], add=False)


def halo_export_add(plan, y):
    """Ghost partial sums -> owners (added in fixed peer order)."""
    # for export the roles flip: we send what we hold as ghosts (plan.recv)
    # from the receive-side buffers and receive into the send-side ones
    for q in plan.peers:
        _pack(y, plan.recv[q], plan.buf_recv[q])
    _exchange(plan.peers, plan.buf_recv, plan.buf_send)
    for q in sorted(plan.peers):
        _unpack(y, plan.send[q], plan.buf_send[q], add=True)


# ---------------------------------------------------------------------------
# distributed level, transfer, hierarchy
# ---------------------------------------------------------------------------


class DistLevel:
    def __init__(self, layout, op, backend, import_plan, export_plan):
        self.layout = layout
        self.op = op
        self.bk = backend
        self.imp = import_plan
        self.exp = export_plan
        self.n = layout.n_local_full
        self.n_owned = layout.n_owned_full
        self.overlap = True  # interior cells overlap the ghost import (False: import, then all cells)
        self._t = backend.zeros(self.n)   # product scratch of the unsplit residual form
        self._tc = backend.zeros(self.n)  # prolongated correction of the V-cycle
        self._r = backend.zeros(self.n)  # smoother work vectors (fixed addresses: graph capture)
        self._d = backend.zeros(self.n)
        d = backend.diagonal_partial(op)
        if self.exp is not None:
            halo_export_add(self.exp, d)
        if len(layout.local_constrained):
            d[torch.from_numpy(layout.local_constrained).to(d.device)] = 1.0
        self.diag = d
        self.inv_diag = 1.0 / d  # owned entries are exact; ghost entries are never read
        self.lam_max = None

    def _split_cells(self, x, y, negate):
        """Local cell loop with the ghost import of x overlapped: interior
        cells never read a ghost entry of x, so they run while the import is
        in flight; the boundary cells follow it."""
        n_int = self.layout.n_interior_cells
        n_cells = len(self.layout.owned_cells)
        self.bk.apply_begin(self.op, x, y, negate)
        if self.imp is not None and n_int > 0:
            self.bk.overlapped(lambda: halo_import(self.imp, x),
                               lambda: self.bk.apply_cells(self.op, x, y, 0, n_int, negate))
            self.bk.apply_cells(self.op, x, y, n_int, n_cells, negate)
        else:
            if self.imp is not None:
                halo_import(self.imp, x)
            self.bk.apply_cells(self.op, x, y, 0, n_cells, negate)

    def _split(self):
        return self.overlap and self.bk.can_split(self.op)

    def apply_into(self, x, y):
        if self._split():
            self._split_cells(x, y, False)
        else:
            if self.imp is not None:
                halo_import(self.imp, x)
            self.bk.apply_into(self.op, x, y)
        if self.exp is not None:
            halo_export_add(self.exp, y)
        return y

    def apply_sub_into(self, x, r):
        """r -= A x on the owned rows, in place (the residual form of the
        smoother and of the V-cycle residual: no product vector is written and
        read back).  The ghost rows of r are scratch: zeroed, they collect this
        rank's partial sums, which the export adds to the owners."""
        if not self._split():
            self.apply_into(x, self._t)
            self.bk.sub(r, self._t, r)
            return r
        if self.n > self.n_owned:
            r[self.n_owned:].zero_()
        self._split_cells(x, r, True)
        if self.exp is not None:
            halo_export_add(self.exp, r)
        return r

    def dot(self, a, b):
        s = self.bk.dot(a[: self.n_owned], b[: self.n_owned])
        if self.layout.replicated:
            return s
        t = torch.tensor([s], dtype=torch.float64, device=self.bk.comm_device)
        dist.all_reduce(t)
        return float(t.item())

    def from_global(self, v_global):
        return torch.as_tensor(np.asarray(v_global)[self.layout.full_global(np.arange(self.layout.n_local))],
                               dtype=torch.float64).to(self.bk.device)

    def gather_global(self, x):
        """Owned parts of all ranks -> full global vector (host, every rank)."""
        mine = x[: self.n_owned].detach().cpu().numpy()
        if self.layout.replicated:
            return mine.copy()
        parts = [None] * dist.get_world_size()
        dist.all_gather_object(parts, (self.layout.full_global(np.arange(self.layout.n_owned)), mine))
        out = np.zeros(self.layout.n_global_scalar * self.layout.ncomp)
        for idx, val in parts:
            out[idx] = val
        return out

    # -- Chebyshev-Jacobi sweep (solvers.py:88-108) on local vectors --------
    def smooth_into(self, b, x0, x, degree, window, residual_out=False, t=None):
        """One degree-k sweep.  residual_out: one more residual-form apply
        leaves b - A x in self._r (the recurrence keeps r = b - A (x - d), so
        the V-cycle needs no copy of b and no extra vector for its residual).
        t: self._r already holds b - A x0 (left by residual_out) and the sweep
        starts from x0 + t, the prolongated correction: r -= A t, then
        x = (x0 + t) + d in the first vector kernel (no copy of b either)."""
        lam_max = self.lam_max
        lam_min = lam_max / window
        theta = (lam_max + lam_min) / 2.0
        delta = (lam_max - lam_min) / 2.0
        sigma = theta / delta
        r, d = self._r, self._d
        if t is not None:
            self.apply_sub_into(t, r)  # r = b - A (x0 + t)
            self.bk.cheb_start_t(t, x0, self.inv_diag, theta, r, d, x)
        elif x0 is None:
            self.bk.cheb_start(b, None, None, self.inv_diag, theta, r, d, x)
        else:
            r.copy_(b)
            self.apply_sub_into(x0, r)  # r = b - A x0
            self.bk.cheb_start(None, None, x0, self.inv_diag, theta, r, d, x)
        rho_old = 1.0 / sigma
        for _ in range(degree - 1):
            self.apply_sub_into(d, r)  # r -= A d
            rho = 1.0 / (2.0 * sigma - rho_old)
            self.bk.cheb_step(None, self.inv_diag, rho * rho_old, 2.0 * rho / delta, r, d, x)
            rho_old = rho
        if residual_out:
            self.apply_sub_into(d, r)  # r = b - A x
        return x

    def estimate_lam_max(self, n_iter=12, seed=0, safety=1.1):
        """Distributed Lanczos on D^-1/2 A D^-1/2 (solvers.py:24-59); the start
        vector is the reference's global default_rng(seed) vector."""
        n_global = self.layout.n_global_scalar * self.layout.ncomp
        v0 = np.random.default_rng(seed).standard_normal(n_global)
        v = self.from_global(v0)
        ds = 1.0 / torch.sqrt(self.diag.abs())
        v = v / np.sqrt(self.dot(v, v))
        vp = torch.zeros_like(v)
        beta = 0.0
        al, be = [], []
        w = self.bk.zeros(self.n)
        for _ in range(n_iter):
            s = ds * v
            self.apply_into(s, w)
            w = ds * w
            a = self.dot(v, w)
            w = w - (a * v + beta * vp)
            al.append(a)
            beta = float(np.sqrt(self.dot(w, w)))
            if beta <= 1e-12 * max(abs(t) for t in al):
                break
            be.append(beta)
            vp, v = v, w / beta
            w = self.bk.zeros(self.n)
        if len(be) == len(al):
            be = be[:-1]
        ritz = al[0] if len(al) == 1 else scipy.linalg.eigh_tridiagonal(np.array(al), np.array(be),
                                                                       eigvals_only=True)[-1]
        self.lam_max = safety * float(ritz)
        return self.lam_max


class DistTransfer:
    def __init__(self, coarse, fine, local_transfer, backend, coarse_import=None, coarse_export=None):
        self.coarse = coarse
        self.fine = fine
        self.t = local_transfer
        self.bk = backend
        self.cimp = coarse_import
        self.cexp = coarse_export

    def prolongate_into(self, uc, uf, accumulate):
        if self.cimp is not None:
            halo_import(self.cimp, uc)
        self.bk.prolongate_into(self.t, uc, uf, accumulate)
        return uf

    def restrict_into(self, rf, rc):
        self.bk.restrict_into(self.t, rf, rc)
        if self.coarse.layout.replicated:
            dist.all_reduce(rc)
        elif self.cexp is not None:
            halo_export_add(self.cexp, rc)
        return rc


class DistHierarchy:
    """Distributed twin of MultigridHierarchy (multigrid.py:83-117): level 1
    replicated, levels >= 2 partitioned."""

    def __init__(self, levels, transfers, coarse_solve, degree, window=10.0, m1=1, m2=1, graph=True):
        self.levels = levels
        self.transfers = transfers
        self.coarse_solve = coarse_solve
        self.degree = degree
        self.window = window
        self.m1, self.m2 = m1, m2
        # GPU: the whole distributed cycle (kernels, halo pack/unpack, NCCL
        # point-to-point and the coarse all-reduce) captured as one CUDA graph
        self.use_graph = bool(graph)
        self._graph = None
        # residuals from the smoother recurrence (False: the explicit form of multigrid.py:97, 101)
        self.recurrence = True

    @property
    def finest(self):
        return self.levels[-1]

    def _v(self, l, f):
        lev = self.levels[l - 1]
        if l == 1:
            x = lev.bk.zeros(lev.n)
            self.coarse_solve(f, x)
            return x
        T = self.transfers[l - 2]
        x = lev.bk.empty(lev.n)  # fully written by the first sweep
        rc = T.coarse.bk.zeros(T.coarse.n)
        if self.recurrence and self.m1 >= 1 and self.m2 >= 1:
            # residual after pre-smoothing from the smoother's recurrence and
            # the first post-smoothing sweep from that residual (as the native
            # executor): no copy of f, no read-modify-write of x by
            # the prolongation; the same applies as multigrid.py:93-111
            cur = None
            for k in range(self.m1):
                lev.smooth_into(f, cur, x, self.degree, self.window, residual_out=(k == self.m1 - 1))
                cur = x
            T.restrict_into(lev._r, rc)
            delta = self._v(l - 1, rc)
            T.prolongate_into(delta, lev._tc, accumulate=False)
            lev.smooth_into(f, x, x, self.degree, self.window, t=lev._tc)
            for _ in range(self.m2 - 1):
                lev.smooth_into(f, x, x, self.degree, self.window)
            return x
        cur = None
        for _ in range(self.m1):
            lev.smooth_into(f, cur, x, self.degree, self.window)
            cur = x
        if cur is None:
            x.zero_()
        r = lev.bk.empty(lev.n)
        r.copy_(f)
        lev.apply_sub_into(x, r)  # r = f - A x (multigrid.py:97)
        T.restrict_into(r, rc)
        delta = self._v(l - 1, rc)
        T.prolongate_into(delta, x, accumulate=True)
        for _ in range(self.m2):
            lev.smooth_into(f, x, x, self.degree, self.window)
        return x

    def precondition(self, r):
        """z = V-cycle(r).  On the GPU the cycle is captured once into a CUDA
        graph (static input/output buffers; the returned tensor is reused by
        the next call) and replayed; capture failures fall back to eager."""
        if self.use_graph and r.is_cuda:
            try:
                return self._replay(r)
            except RuntimeError:
                self.use_graph = False
                self._graph = None
        return self._v(len(self.levels), r)

    def _replay(self, r):
        if self._graph is None:
            self._gin = r.clone()
            side = torch.cuda.Stream(device=r.device)
            side.wait_stream(torch.cuda.current_stream(r.device))
            with torch.cuda.stream(side):
                self._v(len(self.levels), self._gin)  # warm-up outside the capture
            torch.cuda.current_stream(r.device).wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._gout = self._v(len(self.levels), self._gin)
            self._graph = g
        self._gin.copy_(r)
        self._graph.replay()
        return self._gout


def dist_cg_solve(level, b, precond=None, target_reduction=1e-4, max_iter=1000):
    """cg_solve (solvers.py:129-164) with distributed apply and dots."""
    bk = level.bk
    x = bk.zeros(level.n)
    r = b.clone()
    norm0 = float(np.sqrt(level.dot(r, r)))
    history = [norm0]
    if norm0 == 0.0:
        return x, 0, True, history
    target = target_reduction * norm0
    z = precond(r) if precond else r.clone()
    p = z.clone()
    rz = level.dot(r, z)
    ap = bk.zeros(level.n)
    for k in range(1, max_iter + 1):
        level.apply_into(p, ap)
        pap = level.dot(p, ap)
        if pap <= 0.0:
            raise RuntimeError(f"p'Ap = {pap:.3e} at iteration {k}")
        alpha = rz / pap
        bk.cg_update(alpha, p, ap, x, r)
        norm = float(np.sqrt(level.dot(r, r)))
        history.append(norm)
        if norm <= target:
            return x, k, True, history
        z = precond(r) if precond else r.clone()
        rz_new = level.dot(r, z)
        beta = rz_new / rz
        rz = rz_new
        bk.axpby(1.0, z, beta, p)
    return x, max_iter, False, history


# ---------------------------------------------------------------------------
# construction
# ---------------------------------------------------------------------------


def build_distributed_hierarchy(spaces, backend, problem="poisson", lame=None, cheb_degree=4, window=10.0,
                                search=None, m1=1, m2=1, partition=None, policy="matching", graph=None):
    """spaces: global FESpaces coarsest first (replicated host data on every
    rank).  Returns a DistHierarchy for this rank.  policy: "matching" (the
    finest level Morton-split, each coarser partitioned level takes the owner
    of the finer cell containing its centroid, metrics.py:41-46) or
    "default" (Morton on every level, metrics.py:24-38)."""
    if policy not in ("matching", "default"):
        raise ValueError("policy must be 'matching' or 'default'")
    rank, world = dist.get_rank(), dist.get_world_size()
    if graph is None:
        # graph=None: replay the cycle as a CUDA graph on one rank (measured);
        # with peers the captured NCCL point-to-point calls have never run on
        # hardware here (one GPU per run), so the eager cycle is the default
        # and NNMG_DIST_GRAPH=1 opts in
        graph = world == 1 or os.environ.get("NNMG_DIST_GRAPH", "0") == "1"
    nlev = len(spaces)
    owners = [None] * nlev
    dofown = [None] * nlev
    for l in range(nlev - 1, 0, -1):
        sp = spaces[l]
        if partition is not None:
            owners[l] = partition[l]
        elif policy == "matching" and l < nlev - 1:
            owners[l] = partition_matching(sp.mesh, spaces[l + 1].mesh, owners[l + 1],
                                           lambda m, pts: backend.locate(m, pts, None)[0])
            if np.bincount(owners[l], minlength=world).min() == 0:
                # a rank would own no cell of this level (coarse level with
                # fewer cells than ranks in a region): Morton split instead
                owners[l] = partition_morton(sp.mesh, world)
        else:
            owners[l] = partition_morton(sp.mesh, world)
        dofown[l] = dof_owner_ranks(np.asarray(sp.cell_dofs), owners[l], sp.n_scalar_dofs)
    # fine-side transfer records: this rank's owned points located in the coarse mesh
    recs = [None] * (nlev - 1)
    extra = [None] * nlev
    for l in range(1, nlev):
        cs, fs = spaces[l - 1], spaces[l]
        nc = fs.n_components
        fully = np.zeros(fs.n_dofs, bool)
        fully[fs.constraints.dofs] = True
        fully = fully.reshape(-1, nc).all(axis=1)
        pts = np.nonzero((~fully) & (dofown[l] == rank))[0]
        cells, xhat, proj = backend.locate(cs.mesh, np.asarray(fs.support_points)[pts], search)
        recs[l - 1] = (pts, cells, xhat, proj)
        if l - 1 >= 1:
            extra[l - 1] = np.unique(np.asarray(cs.cell_dofs)[np.unique(cells)])
    layouts = [LevelLayout(spaces[0], None, None, rank, replicated=True)]
    for l in range(1, nlev):
        layouts.append(LevelLayout(spaces[l], owners[l], dofown[l], rank, extra_dofs=extra[l]))
    # ghost lists of every rank (one all_gather_object)
    mine = [(lay.ghosts, lay.cell_ghosts[~lay.global_constrained_scalar[lay.cell_ghosts]],
             np.setdiff1d(extra[l], lay.owned) if extra[l] is not None else np.zeros(0, np.int64))
            for l, lay in enumerate(layouts)]
    allg = [None] * world
    dist.all_gather_object(allg, mine)
    levels = []
    for l, lay in enumerate(layouts):
        sp = spaces[l]
        if lay.replicated:
            lsp = sp
            imp = exp = None
        else:
            lsp = lay.local_space(sp, lay.owned_cells)
            imp = HaloPlan(lay, lay.ghosts, [allg[q][l][0] for q in range(world)], dofown[l]).to(backend.device)
            exp_mine = lay.cell_ghosts[~lay.global_constrained_scalar[lay.cell_ghosts]]
            exp = HaloPlan(lay, exp_mine, [allg[q][l][1] for q in range(world)], dofown[l]).to(backend.device)
        op = backend.make_operator(lsp, problem, lame)
        lev = DistLevel(lay, op, backend, imp, exp)
        lev.space = lsp
        levels.append(lev)
    for lev in levels[1:]:
        lev.estimate_lam_max()
    transfers = []
    for l in range(1, nlev):
        cl, fl = levels[l - 1], levels[l]
        pts, cells, xhat, proj = recs[l - 1]
        cs = spaces[l - 1]
        if cl.layout.replicated:
            tc_space, tc_op = cs, cl.op
            ucells = np.arange(cs.mesh.n_cells)
            local_cells = cells
            cimp = cexp = None
        else:
            ucells = np.unique(cells)
            tc_space = cl.layout.local_space(cs, ucells)
            tc_op = backend.make_operator(tc_space, problem, lame)
            local_cells = np.searchsorted(ucells, cells)
            lay = cl.layout
            t_mine = np.setdiff1d(np.unique(np.asarray(cs.cell_dofs)[ucells]), lay.owned)
            t_mine = t_mine[~lay.global_constrained_scalar[t_mine]]
            cexp = HaloPlan(lay, t_mine, [_free(allg[q][l - 1][2], lay) for q in range(world)],
                            dofown[l - 1]).to(backend.device)
            cimp = cl.imp
        rec = {"point_dofs": fl.layout.g2l(pts), "cells": local_cells, "xhat": xhat, "projected": proj}
        lt = backend.make_transfer(tc_space, fl.space, tc_op, fl.op, rec)
        transfers.append(DistTransfer(cl, fl, lt, backend, cimp, cexp))
    coarse = backend.make_coarse(levels[0].op)
    H = DistHierarchy(levels, transfers, coarse, cheb_degree, window, m1, m2, graph=graph)
    H.owners = owners
    return H


def _free(dofs, layout):
    return dofs[~layout.global_constrained_scalar[dofs]] if len(dofs) else dofs


# ---------------------------------------------------------------------------
# production backend: the CUDA kernels of libnnmg_cuda.so
# ---------------------------------------------------------------------------


class GpuBackend:
    """Local compute on this rank's GPU (no CPU path)."""

    def __init__(self, device):
        from . import _device as D

        self.device = torch.device(device)
        self.comm_device = self.device
        self._D = D
        self._ops = D.vector_ops(self.device)
        self._side = None

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.float64, device=self.device)

    def empty(self, n):
        return torch.empty(n, dtype=torch.float64, device=self.device)

    def make_operator(self, space, problem, lame):
        from .mfoperator import ElasticityOperator, LaplaceOperator

        if problem == "elasticity":
            return ElasticityOperator(space, *lame, device=self.device)
        return LaplaceOperator(space, device=self.device)

    def diagonal_partial(self, op):
        return op.diagonal_device().clone()

    def apply_into(self, op, x, y):
        op.apply_into(x, y)

    # split apply: y = 0 + constrained rows, then cell ranges (whole blocks)
    def can_split(self, op):
        return not op.deterministic

    def apply_begin(self, op, x, y, negate=False):
        op.apply_begin_into(x, y, negate)

    def apply_cells(self, op, x, y, cell0, cell1, negate=False):
        if cell1 > cell0:
            op.apply_cells_into(x, y, cell0 // CELL_ALIGN, -(-cell1 // CELL_ALIGN), negate)

    def overlapped(self, comm_fn, compute_fn):
        """comm_fn on a side stream forked from the current one, compute_fn on
        the current stream, then join (inside a graph capture the fork and the
        join become graph dependencies)."""
        cur = torch.cuda.current_stream(self.device)
        if self._side is None:
            self._side = torch.cuda.Stream(device=self.device)
        self._side.wait_stream(cur)
        with torch.cuda.stream(self._side):
            comm_fn()
        compute_fn()
        cur.wait_stream(self._side)

    def make_transfer(self, coarse_space, fine_space, coarse_op, fine_op, records):
        from .transfer import TwoLevelTransferNonNested

        return TwoLevelTransferNonNested(coarse_space, fine_space, coarse_operator=coarse_op, fine_operator=fine_op,
                                         records=records)

    def prolongate_into(self, t, uc, uf, accumulate):
        t.prolongate_into(uc, uf, accumulate)

    def restrict_into(self, t, rf, rc):
        t.restrict_into(rf, rc)

    def locate(self, mesh, points, search):
        from .geosearch import locate_points

        loc = locate_points(mesh, points, search, device=self.device)
        return loc.cells, loc.xhat, loc.projected

    def make_coarse(self, op):
        from .solvers import CoarseSolver

        world = dist.get_world_size() if dist.is_initialized() else 1
        if world == 1:
            cs = CoarseSolver(op, direct="auto")
        else:
            # with peers the direct path streams 1/world of the inverse tiles
            # per rank and the shares are summed by one all-reduce of the
            # coarse vector (the replicated CG otherwise): the coarse solve
            # then scales with the ranks instead of bounding the parallel
            # efficiency.  The choice is made collectively (slowest
            # CG time, smallest free memory) so every rank takes the same path.
            from .solvers import DIRECT_STREAM_BYTES_PER_S, direct_solve_bytes

            cs = CoarseSolver(op, direct=False)
            if not cs.dense:
                nf = op.n_dofs - len(op.constraints.dofs)
                mem = torch.cuda.mem_get_info(self.device)[0]
                v = torch.tensor([cs._time_cg(), -float(mem)], dtype=torch.float64, device=self.device)
                dist.all_reduce(v, op=dist.ReduceOp.MAX)
                t_cg, mem = float(v[0]), -float(v[1])
                t_direct = direct_solve_bytes(nf) / DIRECT_STREAM_BYTES_PER_S / world
                fits = 3 * 8 * nf ** 2 + direct_solve_bytes(nf) // world < 0.8 * mem
                if fits and t_direct < 0.9 * t_cg:
                    cs = CoarseSolver(op, direct=True, share=(dist.get_rank(), world))
                cs.timing = dict(cs.timing or {}, cg_s=t_cg, direct_predicted_s=t_direct)
        self.coarse_solver = cs
        if cs.partial:
            def solve(b, x):
                cs.solve_into(b, x)
                dist.all_reduce(x)
                return x

            return solve
        return lambda b, x: cs.solve_into(b, x)

    def dot(self, a, b):
        return self._ops.dot(a.contiguous(), b.contiguous())

    def sub(self, a, b, out):
        self._ops.sub(a, b, out)

    def cg_update(self, alpha, p, ap, x, r):
        self._ops.cg_update(alpha, p, ap, x, r)

    def axpby(self, alpha, x, beta, y):
        self._ops.axpby(alpha, x, beta, y)

    def cheb_start(self, b, ax, x0, inv_diag, theta, r, d, x):
        from . import _lib

        D = self._D
        _lib.call("nnmg_cheb_start", r.numel(), D.ptr(b), D.ptr(ax), D.ptr(x0), D.ptr(inv_diag), float(theta),
                  D.ptr(r), D.ptr(d), D.ptr(x), D.stream_ptr(self.device))

    def cheb_start_t(self, t, x0, inv_diag, theta, r, d, x):
        from . import _lib

        D = self._D
        _lib.call("nnmg_cheb_start_t", r.numel(), D.ptr(t), D.ptr(x0), D.ptr(inv_diag), float(theta), D.ptr(r),
                  D.ptr(d), D.ptr(x), D.stream_ptr(self.device))

    def cheb_step(self, ad, inv_diag, c1, c2, r, d, x):
        from . import _lib

        D = self._D
        _lib.call("nnmg_cheb_step", r.numel(), D.ptr(ad), D.ptr(inv_diag), float(c1), float(c2), D.ptr(r),
                  D.ptr(d), D.ptr(x), D.stream_ptr(self.device))
