"""World-size-2 gloo tests of the multi-GPU host logic (CPU only): the
distributed apply, transfers, V-cycle and PCG over a Morton-partitioned
hierarchy must reproduce the single-process oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cname, scale, q, policy="matching"):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from dist_oracle_backend import OracleBackend
        from oracle import nnmg_oracle as O
        from paper_2412_10910_b200 import configs, distributed, fespace
        from paper_2412_10910_b200.mfoperator import assemble_rhs

        cfg = configs.get_config(cname)
        meshes = cfg.make_meshes(scale=scale)
        ncomp = cfg.dim if cfg.problem == "elasticity" else 1
        spaces = []
        for m in meshes:
            sp = fespace.build_space(m, cfg.degree, ncomp)
            sp.constraints = fespace.dirichlet_constraints(sp, cfg.dirichlet_ids)
            spaces.append(sp)
        bk = OracleBackend()
        DH = distributed.build_distributed_hierarchy(spaces, bk, cfg.problem, cfg.lame, cfg.chebyshev_degree,
                                                     policy=policy)
        fine = DH.finest
        b_glob = assemble_rhs(spaces[-1], cfg.body_force if cfg.body_force else 1.0)
        u_glob = np.random.default_rng(0).standard_normal(len(b_glob))
        # distributed apply
        u = fine.from_global(u_glob)
        v = bk.zeros(fine.n)
        fine.apply_into(u, v)
        Au = fine.gather_global(v)
        # distributed V-cycle and PCG
        z = fine.gather_global(DH.precondition(fine.from_global(b_glob)))
        x, its, conv, hist = distributed.dist_cg_solve(fine, fine.from_global(b_glob), DH.precondition, 1e-8)
        xg = fine.gather_global(x)
        lam = [lev.lam_max for lev in DH.levels[1:]]
        owned = [int(lev.layout.n_owned) for lev in DH.levels]
        # interior / boundary split of this rank's cells (overlap of the ghost import)
        interior = []
        for lev in DH.levels[1:]:
            lay = lev.layout
            gh = np.zeros(lay.n_global_scalar, bool)
            gh[lay.ghosts] = True
            cd = np.asarray(spaces[DH.levels.index(lev)].cell_dofs)[lay.owned_cells]
            touches = gh[cd].any(axis=1)
            assert not touches[: lay.n_interior_cells].any()  # interior cells read no ghost
            assert lay.n_interior_cells % distributed.CELL_ALIGN == 0
            interior.append(int(lay.n_interior_cells))
        all_int = [None] * world
        dist.all_gather_object(all_int, interior)
        if rank == 0:
            # single-process oracle on the same meshes
            om = [O.jittered_mesh(m.grid, cfg.extent, cfg.amplitude, 1000 * cfg.index + l + 1, cfg.warp)
                  for l, m in enumerate(meshes)]
            OH, osp = O.build_hierarchy(om, cfg.degree, cfg.problem, cfg.dirichlet_ids, cfg.lame or (1, 1),
                                        cfg.chebyshev_degree)
            ref_Au = OH.ops[-1].apply(u_glob)
            ref_z = OH.precondition(b_glob)
            rx, rits, _, _ = O.cg(OH.ops[-1].apply, b_glob, OH.precondition, 1e-8)
            ref_lam = [s.lam_max for s in OH.smoothers[1:]]
            q.put(dict(Au=np.linalg.norm(Au - ref_Au) / np.linalg.norm(ref_Au),
                       z=np.linalg.norm(z - ref_z) / np.linalg.norm(ref_z),
                       x=np.linalg.norm(xg - rx) / np.linalg.norm(rx), its=its, rits=rits, conv=conv,
                       lam=np.max(np.abs(np.array(lam) - ref_lam) / np.array(ref_lam)), owned=owned,
                       interior=all_int))
    except Exception as exc:  # surface worker failures
        import traceback

        q.put({"error": f"rank {rank}: {exc}\n{traceback.format_exc()}"})
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cname,scale,world,policy", [("C2", 16, 2, "matching"), ("C3", 8, 2, "matching"),
                                                     ("C5", 16, 2, "matching"), ("C3", 8, 2, "default"),
                                                     ("C3", 8, 4, "matching")])
def test_distributed_matches_oracle(cname, scale, world, policy):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cname, scale, q, policy)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
    print(cname, res)
    assert "error" not in res, res.get("error")
    assert res["Au"] <= 1e-12, res
    assert res["lam"] <= 1e-9, res
    assert res["z"] <= 1e-9, res
    assert res["conv"] and abs(res["its"] - res["rits"]) <= 1, res
    assert res["x"] <= 1e-7, res
    assert min(res["owned"][1:]) > 0  # rank 0 owns part of every partitioned level
    # the overlapped apply (interior cells before the ghost import) ran on the finest level
    # (tiny cases: a rank whose every cell touches the interface has no interior block)
    assert any(r[-1] > 0 for r in res["interior"]), res["interior"]


def test_partition_morton_and_dof_owner():
    from paper_2412_10910_b200 import distributed, fespace, mesh

    m = mesh.structured_box_mesh((4, 4), [(0, 1), (0, 1)])
    own = distributed.partition_morton(m, 4)
    assert np.bincount(own).tolist() == [4, 4, 4, 4]
    # Morton quadrants of a 4x4 grid are the 2x2 corner blocks
    assert len(set(own.reshape(4, 4)[:2, :2].ravel())) == 1
    sp = fespace.build_space(m, 2)
    do = distributed.dof_owner_ranks(np.asarray(sp.cell_dofs), own, sp.n_scalar_dofs)
    first = np.full(sp.n_scalar_dofs, 10**9)
    for c in range(m.n_cells):
        for g in sp.cell_dofs[c]:
            first[g] = min(first[g], c)
    assert np.array_equal(do, own[first])


def test_partition_matching_follows_the_finer_level():
    """metrics.py:41-46: each coarse cell takes the rank of the fine cell
    containing its centroid; on nested box meshes that is the Morton owner
    of its children."""
    from paper_2412_10910_b200 import distributed, mesh

    fine = mesh.structured_box_mesh((8, 8), [(0, 1), (0, 1)])
    coarse = mesh.structured_box_mesh((4, 4), [(0, 1), (0, 1)])
    fo = distributed.partition_morton(fine, 4)

    def locate(m, pts):  # exact location on the uniform fine grid
        ij = np.minimum((pts * 8).astype(int), 7)
        return ij[:, 0] + 8 * ij[:, 1]

    co = distributed.partition_matching(coarse, fine, fo, locate)
    assert np.array_equal(co, distributed.partition_morton(coarse, 4))
