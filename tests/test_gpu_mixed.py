"""Mixed-precision V-cycle (the V-cycle in
single precision inside double-precision CG).  fp32 storage of level vectors,
geometry, inverse diagonals and transfer coordinates; fp64 arithmetic and
coarse solve.  Parity is by outer CG iteration count (+-1 of the reference's
fp64 solve, tests/golden/mg_*), the V-cycle agrees with the fp64 one to fp32
rounding, and the solve still reaches the 1e-8 reduction in fp64."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2412_10910_b200 as P

    return P


def _hierarchy(P, tag, precision):
    g = golden("mg_" + tag)
    cfg = P.configs.get_config(tag[:2])
    meshes = []
    for l, row in enumerate(g["grids"]):
        grid = tuple(int(x) for x in row[: cfg.dim])
        meshes.append(P.mesh.jittered_box_mesh(grid, cfg.extent, cfg.amplitude, 1000 * cfg.index + l + 1,
                                               P.mesh.sine_warp if cfg.warp else None))
    eps_box = None if float(g["eps_box"]) < 0 else float(g["eps_box"])
    H = P.multigrid.build_hp_hierarchy(
        meshes, cfg.degree, problem=cfg.problem, dirichlet_ids=cfg.dirichlet_ids, lame=cfg.lame,
        search=P.geosearch.SearchConfig(eps_box=eps_box),
        config=P.multigrid.HierarchyConfig(chebyshev_degree=cfg.chebyshev_degree, vcycle_precision=precision))
    b = P.mfoperator.assemble_rhs(H.finest.space, cfg.body_force if cfg.body_force else 1.0)
    return g, H, b


@pytest.mark.parametrize("arith", ["32", "64"])
@pytest.mark.parametrize("tag", ["C1_full", "C2_s8", "C3_s8", "C4_s4", "C5_s8"])
def test_mixed_precision_iterations_match_reference(pkg, monkeypatch, tag, arith):
    # NNMG_MIXED_ARITH: 32 (default) = single-precision arithmetic in the register
    # Laplace apply of the fp32 levels (the paper's fp32 V-cycle); 64 = fp64
    # arithmetic on fp32 storage everywhere
    monkeypatch.setenv("NNMG_MIXED_ARITH", arith)
    g, H, b = _hierarchy(pkg, tag, 32)
    assert H.precision == 32
    z32 = H.v_cycle(b)
    H.set_precision(64)
    z64 = H.v_cycle(b)
    assert rel(z64[:: int(g["stride"])], g["vcycle"]) <= 1e-9  # switching back restores the fp64 cycle
    dev = rel(z32, z64)
    print(tag, arith, "mixed vs fp64 V-cycle", dev)
    assert 0 < dev <= (2e-5 if arith == "64" else 2e-4)  # single-precision rounding (storage / + arithmetic)
    H.set_precision(32)
    res = pkg.solvers.cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-8)
    assert res.converged
    assert abs(res.iterations - int(g["iterations"])) <= 1, (res.iterations, int(g["iterations"]))
    r = b - H.finest.operator.apply(res.x)
    assert np.linalg.norm(r) <= 1.01e-8 * np.linalg.norm(b)


def test_mixed_precision_tma_staged_geometry(pkg, monkeypatch):
    # NNMG_REG_TMA=1: the fp32 register apply stages each warp's geometry chunk by one TMA bulk copy
    monkeypatch.setenv("NNMG_REG_TMA", "1")
    g, H, b = _hierarchy(pkg, "C3_s8", 32)
    z32 = H.v_cycle(b)
    H.set_precision(64)
    z64 = H.v_cycle(b)
    assert 0 < rel(z32, z64) <= 2e-4
    H.set_precision(32)
    res = pkg.solvers.cg_solve(H.finest.operator, b, precond=H.precondition, target_reduction=1e-8)
    assert res.converged and abs(res.iterations - int(g["iterations"])) <= 1


def test_mixed_precision_graph_replay_and_errors(pkg):
    g, H, b = _hierarchy(pkg, "C2_s8", 32)
    f = torch.from_numpy(b).cuda()
    x1, x2 = torch.empty_like(f), torch.empty_like(f)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        H.v_cycle_into(f, x1)  # captured
        H.v_cycle_into(f, x2)  # replayed
    s.synchronize()
    H.use_graph(False)
    x3 = torch.empty_like(f)
    H.v_cycle_into(f, x3)
    torch.cuda.synchronize()
    assert rel(x1.cpu().numpy(), x3.cpu().numpy()) <= 1e-6 and rel(x2.cpu().numpy(), x3.cpu().numpy()) <= 1e-6
    with pytest.raises(ValueError):
        H.v_cycle(b, executor=False)
    with pytest.raises(ValueError):
        H.set_precision(16)
