"""Device-vector plumbing: torch CUDA tensors carry the level vectors.

Public calls accept either NumPy float64 arrays (host; the result comes back
as a NumPy array, as the reference returns) or CUDA float64 tensors (the
result stays on the device).  Shape errors raise ValueError like the
reference (mfoperator.py:110-111, transfer.py:32-33).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2412_10910_b200 needs a CUDA device (no CPU fallback)")
    _lib.load()


def resolve_device(device=None):
    require_cuda()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError("device must be a CUDA device")
    return dev if dev.index is not None else torch.device("cuda", torch.cuda.current_device())


def stream_ptr(device):
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t):
    return t.data_ptr() if t is not None else None


def to_device(u, n, device, what="vector"):
    """Return (device tensor, was_host).  Never mutates u."""
    if isinstance(u, torch.Tensor):
        if u.shape != (n,):
            raise ValueError(f"expected {what} of length {n}")
        if u.device != device:
            raise ValueError(f"{what} lives on {u.device}, operator on {device}")
        if u.dtype != torch.float64:
            raise ValueError(f"{what} must be float64")
        return (u if u.is_contiguous() else u.contiguous()), False
    a = np.asarray(u)
    if a.shape != (n,):
        raise ValueError(f"expected {what} of length {n}")
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device, non_blocking=False)
    return t, True


def from_device(t, was_host):
    if was_host:
        return t.cpu().numpy()
    return t


def empty(n, device):
    return torch.empty(n, dtype=torch.float64, device=device)


def zeros(n, device):
    return torch.zeros(n, dtype=torch.float64, device=device)


class DeviceVectorOps:
    """Thin wrappers over the library's vector kernels on one device."""

    def __init__(self, device):
        self.device = device
        self._work = torch.empty(int(_lib.load().nnmg_dot_workspace()), dtype=torch.float64, device=device)
        self._out = torch.empty(2, dtype=torch.float64, device=device)

    def dot2_async(self, a, b, c=None, d=None, out=None):
        out = self._out if out is None else out
        _lib.call("nnmg_dot2", a.numel(), ptr(a), ptr(b), ptr(c), ptr(d), ptr(out), ptr(self._work),
                  stream_ptr(self.device))
        return out

    def dot(self, a, b):
        return float(self.dot2_async(a, b)[0].item())

    def dot2(self, a, b, c, d):
        o = self.dot2_async(a, b, c, d).cpu()
        return float(o[0]), float(o[1])

    def axpby(self, alpha, x, beta, y):
        _lib.call("nnmg_axpby", x.numel(), float(alpha), ptr(x), float(beta), ptr(y), stream_ptr(self.device))
        return y

    def sub(self, a, b, out):
        _lib.call("nnmg_sub", a.numel(), ptr(a), ptr(b), ptr(out), stream_ptr(self.device))
        return out

    def mul(self, a, b, out):
        _lib.call("nnmg_mul", a.numel(), ptr(a), ptr(b), ptr(out), stream_ptr(self.device))
        return out

    def cg_update(self, alpha, p, ap, x, r):
        _lib.call("nnmg_cg_update", p.numel(), float(alpha), ptr(p), ptr(ap), ptr(x), ptr(r),
                  stream_ptr(self.device))


_OPS = {}


def vector_ops(device):
    key = str(device)
    if key not in _OPS:
        _OPS[key] = DeviceVectorOps(device)
    return _OPS[key]
