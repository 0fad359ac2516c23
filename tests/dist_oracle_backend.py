"""Test-only backend for paper_2412_10910_b200.distributed: the local compute
runs in the CPU oracle so the distributed host logic (partitions, local
numbering, halo plans, export-add, replicated coarse level, distributed dots
and Lanczos) can be checked with gloo on CPU.  Never used by the product."""

import numpy as np
import torch

from oracle import nnmg_oracle as O


def _ospace(space):
    m = space.mesh
    om = O.OMesh(m.dim, m.vertices, m.cells, np.zeros((0, 3), np.int64))
    return O.OSpace(om, space.degree, space.n_components, np.asarray(space.cell_dofs),
                    np.asarray(space.support_points), np.asarray(space.constraints.dofs))


class OracleBackend:
    device = torch.device("cpu")
    comm_device = torch.device("cpu")

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def empty(self, n):
        return torch.full((n,), float("nan"), dtype=torch.float64)  # catches reads of unwritten entries

    def make_operator(self, space, problem, lame):
        op = O.OOperator(_ospace(space), problem, *(lame or (1.0, 1.0)))
        op._meta = (problem, lame or (1.0, 1.0))
        op._parts = {}
        return op

    # split apply (interior / boundary cell ranges of a distributed level)
    def can_split(self, op):
        return True

    def apply_begin(self, op, x, y, negate=False):
        cd = torch.from_numpy(op.space.cdofs)
        if negate:
            y[cd] -= x[cd]
            return
        y.zero_()
        y[cd] = x[cd]

    def apply_cells(self, op, x, y, cell0, cell1, negate=False):
        if cell1 <= cell0:
            return
        key = (cell0, cell1)
        if key not in op._parts:
            sp = op.space
            om = O.OMesh(sp.mesh.dim, sp.mesh.vertices, sp.mesh.cells[cell0:cell1], np.zeros((0, 3), np.int64))
            sub = O.OSpace(om, sp.degree, sp.n_components, sp.cell_dofs[cell0:cell1], sp.support_points, sp.cdofs)
            op._parts[key] = O.OOperator(sub, op._meta[0], *op._meta[1])
        part = op._parts[key].apply(x.numpy().copy())
        part[op.space.cdofs] = 0.0  # identity-out belongs to apply_begin
        if negate:
            y -= torch.from_numpy(part)
        else:
            y += torch.from_numpy(part)

    def overlapped(self, comm_fn, compute_fn):
        # worst-case order on CPU: the interior cells run BEFORE the ghost
        # import, so a misclassified interior cell would read stale ghosts
        compute_fn()
        comm_fn()

    def diagonal_partial(self, op):
        return torch.from_numpy(op.diagonal())

    def apply_into(self, op, x, y):
        y.copy_(torch.from_numpy(op.apply(x.numpy().copy())))

    def make_transfer(self, coarse_space, fine_space, coarse_op, fine_op, records):
        rec = (np.asarray(records["point_dofs"]), np.asarray(records["cells"]), np.asarray(records["xhat"]),
               np.asarray(records["projected"]))
        return O.OTransfer(coarse_op.space, fine_op.space, records=rec)

    def prolongate_into(self, t, uc, uf, accumulate):
        v = torch.from_numpy(t.prolongate(uc.numpy().copy()))
        if accumulate:
            uf += v
        else:
            uf.copy_(v)

    def restrict_into(self, t, rf, rc):
        rc.copy_(torch.from_numpy(t.restrict(rf.numpy().copy())))

    def locate(self, mesh, points, search):
        eps_box = None if search is None else search.eps_box
        om = O.OMesh(mesh.dim, mesh.vertices, mesh.cells, np.zeros((0, 3), np.int64))
        return O.locate(om, np.asarray(points), eps_box=eps_box)

    def make_coarse(self, op):
        cs = O.OCoarse(op)
        return lambda b, x: x.copy_(torch.from_numpy(cs.solve(b.numpy().copy())))

    def dot(self, a, b):
        return float((a * b).sum())

    def sub(self, a, b, out):
        torch.sub(a, b, out=out)

    def cg_update(self, alpha, p, ap, x, r):
        x.add_(alpha * p)
        r.sub_(alpha * ap)

    def axpby(self, alpha, x, beta, y):
        y.mul_(beta).add_(alpha * x)

    def cheb_start(self, b, ax, x0, inv_diag, theta, r, d, x):
        if b is not None:
            r.copy_(b - ax if ax is not None else b)
        d.copy_(inv_diag * r / theta)
        x.copy_(x0 + d if x0 is not None else d)

    def cheb_start_t(self, t, x0, inv_diag, theta, r, d, x):
        d.copy_(inv_diag * r / theta)
        x.copy_((x0 + t) + d)

    def cheb_step(self, ad, inv_diag, c1, c2, r, d, x):
        if ad is not None:
            r -= ad
        z = inv_diag * r
        d.copy_(c1 * d + c2 * z)
        x += d
