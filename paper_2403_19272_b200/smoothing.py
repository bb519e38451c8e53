"""Module-level smoother drop-ins (reference smoothing.py:23-78) on the device.

``ajacobi_smooth`` runs the step's own rank-2 A-Jacobi kernels (k_jacobi_a / _b,
captured as one CUDA graph) over a device copy of ``system.H`` (SELL-32), bitwise
the reference's CSR order; ``jacobi_step`` is one damped Jacobi update.  Both take
and return numpy arrays with the reference's signatures and errors.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import SmootherDivergence  # noqa: F401  (reference export)
from . import context


def _dev(a):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def _as3(v):
    v = np.asarray(v, dtype=np.float64)
    return (v[:, None] if v.ndim == 1 else v), v.ndim == 1


def _check_diag(system, diag_delta):
    diag = system.diag if diag_delta is None else system.diag + diag_delta
    if (diag <= 0).any():
        raise ValueError("nonpositive diagonal entry")


def ajacobi_smooth(system, b, x0, iterations: int, omega: float = 0.0, diag_delta=None) -> np.ndarray:
    """ceil(iterations/2) rank-2 aggregated Jacobi steps (smoothing.py:23-66)."""
    _check_diag(system, diag_delta)
    ctx = context.get(system=system)
    b3, flat = _as3(b)
    x3, _ = _as3(x0)
    cols = b3.shape[1]
    out = np.empty_like(x3)
    # the kernels run 3 right-hand sides per row; narrower / wider blocks go 3 at a time
    for c0 in range(0, cols, 3):
        sl = slice(c0, min(cols, c0 + 3))
        bb = np.zeros((len(b3), 3))
        xx = np.zeros((len(x3), 3))
        bb[:, :sl.stop - sl.start] = b3[:, sl]
        xx[:, :sl.stop - sl.start] = x3[:, sl]
        bd, xd = _dev(bb), _dev(xx)
        dd = _dev(diag_delta) if diag_delta is not None else None
        _lib.check(ctx.lib.cs_ajacobi_smooth(ctx.ptr, bd.data_ptr(), xd.data_ptr(), int(iterations), float(omega),
                                             dd.data_ptr() if dd is not None else None, _lib.stream_handle()),
                   "cs_ajacobi_smooth")
        out[:, sl] = xd.cpu().numpy()[:, :sl.stop - sl.start]
    return out[:, 0] if flat else out


def jacobi_step(system, b, x, omega: float = 0.0, diag_delta=None) -> np.ndarray:
    """Single damped Jacobi update (smoothing.py:69-78)."""
    import torch

    ctx = context.get(system=system)
    b3, flat = _as3(b)
    x3, _ = _as3(x)
    cols = b3.shape[1]
    out = np.empty_like(x3)
    for c0 in range(0, cols, 3):
        sl = slice(c0, min(cols, c0 + 3))
        bb = np.zeros((len(b3), 3))
        xx = np.zeros((len(x3), 3))
        bb[:, :sl.stop - sl.start] = b3[:, sl]
        xx[:, :sl.stop - sl.start] = x3[:, sl]
        bd, xd = _dev(bb), _dev(xx)
        od = torch.empty_like(xd)
        dd = _dev(diag_delta) if diag_delta is not None else None
        _lib.check(ctx.lib.cs_jacobi_step(ctx.ptr, bd.data_ptr(), xd.data_ptr(), float(omega),
                                          dd.data_ptr() if dd is not None else None, od.data_ptr(),
                                          _lib.stream_handle()), "cs_jacobi_step")
        out[:, sl] = od.cpu().numpy()[:, :sl.stop - sl.start]
    return out[:, 0] if flat else out
