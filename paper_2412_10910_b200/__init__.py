"""B200-native (sm_100a, fp64) hot path of the matrix-free non-nested multigrid
method of arXiv 2412.10910.

Drop-in GPU twins of the reference ``nnmg`` operator / transfer / smoother /
solver / V-cycle API (see DESIGN.md and INTEGRATION.md).  Kernels live in
``libnnmg_cuda.so`` (built in-tree from ``csrc/``); there is no CPU fallback.
"""

from . import configs, fespace, mesh  # noqa: F401  (host setup, no GPU needed)

__all__ = ["configs", "fespace", "mesh", "mfoperator", "transfer", "solvers", "multigrid", "geosearch"]


def __getattr__(name):
    # GPU modules import torch / the CUDA library lazily
    if name in ("mfoperator", "transfer", "solvers", "multigrid", "geosearch", "distributed"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
