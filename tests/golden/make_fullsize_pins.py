"""Pin the five BASELINE configurations at FULL size by running the REFERENCE.

Run in the build container (the reference exists only here), one config per
process so a memory failure in one does not lose the others:

    python tests/golden/make_fullsize_pins.py C1 [maps|apply|solve ...]

Writes ``tests/golden/full_<C>.npz`` (merged with what an earlier run
wrote), holding only reference OUTPUTS:

* per level: SHA-256 of ``cell_dofs`` (int64) and of the constrained DoF list
  (fespace.py:137-207), n_dofs;
* per non-nested transfer: SHA-256 of ``point_dofs``, owning ``cells`` and
  ``projected`` (transfer.py:67-85, geosearch.py:163-227), a strided sample of
  ``xhat``;
* ``apply``: a strided sample and the norm of ``A u`` for u ~ N(0,1) from
  ``default_rng(0)`` on the finest level (mfoperator.py:108-122 / 171-202);
* ``transfer``: strided samples of ``P u_c`` and the whole ``P^T r_f`` for the
  finest transfer, inputs from ``default_rng(1)`` (transfer.py:31-58);
* ``rhs``: a strided sample and the norm of ``assemble_rhs`` (mfoperator.py:313-355);
* ``solve``: outer PCG iterations and residual history to a 1e-8 reduction,
  λmax per level, the V-cycle of b (strided sample + norm) and the coarse
  CG iteration count of every coarse solve in the first V-cycle
  (solvers.py:129-206, multigrid.py:83-113).

The maps of the two big 3D configurations are computed with the reference's
own ``build_tree`` / ``locate_points`` on point chunks (location is per
point, so chunking does not change a bit), and the big transfers are
evaluated by the reference's ``_prolongate_scalar`` / ``_restrict_scalar`` on
point chunks, so the int64 ``gather`` table (17 GB for C4) is never whole.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as mg  # noqa: E402  (puts the reference on sys.path)

from nnmg import solvers as ref_solvers  # noqa: E402
from nnmg.fespace import build_space, dirichlet_constraints  # noqa: E402
from nnmg.geosearch import SearchConfig, build_tree, locate_points  # noqa: E402
from nnmg.mfoperator import ElasticityOperator, LaplaceOperator, assemble_rhs  # noqa: E402
from nnmg.multigrid import HierarchyConfig, build_hp_hierarchy  # noqa: E402
from nnmg.transfer import TwoLevelTransferNonNested, _TransferBase  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
NSAMPLE = 6000
CHUNK = 1 << 20


def sha(a, dtype="<i8"):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a), dtype=dtype).tobytes()).hexdigest()


def stride_of(n):
    return max(1, n // NSAMPLE)


def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, flush=True)


def meshes_of(cname):
    dim, p, problem, levels, extent, a, warp, dirichlet, lame, body, cheb = mg.CONFIG[cname]
    cidx = int(cname[1])
    out = []
    for l, g in enumerate(levels):
        t = time.time()
        out.append(mg.ref_jittered(g, extent, a, 1000 * cidx + l + 1, warp))
        log(cname, "mesh", l, g, f"{time.time() - t:.0f}s")
    return out


def spaces_of(cname, meshes):
    dim, p, problem, levels, extent, a, warp, dirichlet, lame, body, cheb = mg.CONFIG[cname]
    ncomp = dim if problem == "elasticity" else 1
    sps = []
    for l, m in enumerate(meshes):
        t = time.time()
        sp = build_space(m, p, n_components=ncomp)
        sp.constraints = dirichlet_constraints(sp, dirichlet)
        sps.append(sp)
        log(cname, "space", l, sp.n_dofs, f"{time.time() - t:.0f}s")
    return sps


def rhs_of(cname, sp):
    dim, p, problem, levels, extent, a, warp, dirichlet, lame, body, cheb = mg.CONFIG[cname]
    if problem == "poisson":
        return assemble_rhs(sp, f=1.0)
    return assemble_rhs(sp, f=lambda x: np.tile(np.asarray(body)[None], (len(x), 1)))


def op_of(cname, sp):
    dim, p, problem, levels, extent, a, warp, dirichlet, lame, body, cheb = mg.CONFIG[cname]
    return LaplaceOperator(sp) if problem == "poisson" else ElasticityOperator(sp, *lame)


class ChunkedTransfer:
    """The reference's non-nested transfer data members, located and evaluated
    on point chunks (transfer.py:67-124 with geosearch.py:163-227)."""

    def __init__(self, sc, sf, search=None):
        search = search or SearchConfig()
        nc = sf.n_components
        fully = sf.constrained_mask().reshape(sf.n_scalar_dofs, nc).all(axis=1)
        self.sc, self.sf = sc, sf
        self.point_dofs = np.where(~fully)[0]
        tree = build_tree(sc.mesh, eps_box=search.eps_box)
        pts = sf.support_points[self.point_dofs]
        cells, xhat, proj = [], [], []
        for s in range(0, len(pts), CHUNK):
            loc = locate_points(tree, sc.mesh, pts[s:s + CHUNK], eps_geo=search.eps_geo, eps_ref=search.eps_ref)
            cells.append(loc.cells)
            xhat.append(loc.xhat)
            proj.append(loc.projected)
            log("  located", s + len(loc.cells), "/", len(pts))
        self.cells = np.concatenate(cells)
        self.xhat = np.concatenate(xhat)
        self.projected = np.concatenate(proj)

    def _piece(self, s, e):
        T = TwoLevelTransferNonNested.__new__(TwoLevelTransferNonNested)
        _TransferBase.__init__(T, self.sc, self.sf)
        T.point_dofs = self.point_dofs[s:e]
        T.cells = self.cells[s:e]
        T.xhat = self.xhat[s:e]
        T.tabs = [self.sc.shape1d.values(T.xhat[:, j]) for j in range(self.sc.mesh.dim)]
        T.gather = self.sc.cell_dofs[T.cells]
        return T

    def prolongate(self, uc):
        out = np.zeros(self.sf.n_dofs)
        for s in range(0, len(self.cells), CHUNK):
            out += self._piece(s, s + CHUNK).prolongate(uc)
        return out

    def restrict(self, rf):
        out = np.zeros(self.sc.n_dofs)
        for s in range(0, len(self.cells), CHUNK):
            out += self._piece(s, s + CHUNK).restrict(rf)
        return out


def save(cname, upd):
    path = os.path.join(OUT, f"full_{cname}.npz")
    old = dict(np.load(path, allow_pickle=False)) if os.path.exists(path) else {}
    old.update(upd)
    np.savez_compressed(path, **old)
    log(cname, "saved", sorted(upd))


def maps_and_kernels(cname, what):
    meshes = meshes_of(cname)
    sps = spaces_of(cname, meshes)
    out = {}
    for l, sp in enumerate(sps):
        out[f"l{l}_n_dofs"] = sp.n_dofs
        out[f"l{l}_cell_dofs_sha"] = sha(sp.cell_dofs)
        out[f"l{l}_cdofs_sha"] = sha(sp.constraints.dofs)
    save(cname, out)
    sf = sps[-1]
    if "apply" in what:
        t = time.time()
        op = op_of(cname, sf)
        u = np.random.default_rng(0).standard_normal(sf.n_dofs)
        v = op.apply(u)
        st = stride_of(sf.n_dofs)
        b = rhs_of(cname, sf)
        save(cname, {"apply_stride": st, "apply": v[::st], "apply_norm": np.linalg.norm(v),
                     "diag": op.diagonal()[::st],
                     "rhs_stride": st, "rhs": b[::st], "rhs_norm": np.linalg.norm(b)})
        log(cname, "apply/rhs", f"{time.time() - t:.0f}s")
        del op, v, b
    if "maps" in what:
        for l in range(1, len(sps)):
            t = time.time()
            T = ChunkedTransfer(sps[l - 1], sps[l])
            st = stride_of(len(T.cells))
            upd = {f"t{l - 1}_npts": len(T.cells), f"t{l - 1}_point_dofs_sha": sha(T.point_dofs),
                   f"t{l - 1}_cells_sha": sha(T.cells), f"t{l - 1}_projected_sha": sha(T.projected, "u1"),
                   f"t{l - 1}_n_projected": int(T.projected.sum()),
                   f"t{l - 1}_xhat_stride": st, f"t{l - 1}_xhat": T.xhat[::st]}
            if l == len(sps) - 1:
                rng = np.random.default_rng(1)
                uc = rng.standard_normal(sps[l - 1].n_dofs)
                rf = rng.standard_normal(sps[l].n_dofs)
                pu = T.prolongate(uc)
                sp_ = stride_of(len(pu))
                upd.update({"prolongate_stride": sp_, "prolongate": pu[::sp_],
                            "prolongate_norm": np.linalg.norm(pu), "restrict": T.restrict(rf)})
            save(cname, upd)
            log(cname, "transfer", l - 1, f"{time.time() - t:.0f}s")
            del T


def solve(cname):
    dim, p, problem, levels, extent, a, warp, dirichlet, lame, body, cheb = mg.CONFIG[cname]
    meshes = meshes_of(cname)
    t = time.time()
    H = build_hp_hierarchy(meshes, degree=p, problem=problem, dirichlet_ids=dirichlet, lame=lame,
                           config=HierarchyConfig(chebyshev_degree=cheb))
    log(cname, "hierarchy", f"{time.time() - t:.0f}s")
    b = rhs_of(cname, H.finest.space)
    # count the coarse CG iterations of the first V-cycle's coarse solve
    coarse_its = []
    real_cg = ref_solvers.cg_solve

    def counting_cg(*args, **kw):
        res = real_cg(*args, **kw)
        coarse_its.append(res.iterations)
        return res

    ref_solvers.cg_solve = counting_cg
    try:
        t = time.time()
        z = H.precondition(b)
        log(cname, "v-cycle", f"{time.time() - t:.0f}s")
    finally:
        ref_solvers.cg_solve = real_cg
    st = stride_of(len(b))
    out = {"vcycle_stride": st, "vcycle": z[::st], "vcycle_norm": np.linalg.norm(z),
           "vcycle_coarse_iterations": np.array(coarse_its, dtype=np.int64),
           "lam_max": np.array([lev.smoother.lam_max for lev in H.levels])}
    save(cname, out)
    t = time.time()
    res = real_cg(H.finest.operator, b, precond=H.precondition, target_reduction=1e-8)
    log(cname, "cg", res.iterations, f"{time.time() - t:.0f}s")
    save(cname, {"iterations": res.iterations, "residual_norms": np.array(res.residual_norms),
                 "x_stride": st, "x": res.x[::st], "x_norm": np.linalg.norm(res.x)})


def main():
    cname = sys.argv[1].upper()
    what = set(sys.argv[2:]) or {"maps", "apply", "solve"}
    if what & {"maps", "apply"}:
        maps_and_kernels(cname, what)
    if "solve" in what:
        solve(cname)


if __name__ == "__main__":
    main()
