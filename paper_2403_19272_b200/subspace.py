"""Rest-shape eigenbasis (setup) for the two-level global solve.

``build_subspace`` mirrors reference ``pkg/src/clothsim/subspace.py:49-84``:
the smallest r_bar eigenpairs of the free-vertex elastic matrix H, computed by
shift-invert Lanczos (scipy ``eigsh``, sigma=0, fixed start vector from
``default_rng(0)``) so the basis is bit-identical to the reference's on the
same host, with a dense ``eigh`` for tiny systems.  This is A17 setup (done
once per scene); the per-iteration uses of the basis (U^T r reductions, the
r x r reduced solve, U q prolongation) are device kernels in
``csrc/solver.cu``.

For paper-scale garments the host ``eigsh`` is minutes long; ``method="device"``
selects the GPU Chebyshev-filtered subspace iteration (``eigen.py`` driving the
``csrc/eigen.cu`` block kernels through the C ABI).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse.linalg as spla

from .constraints import GlobalSystem


class EigensolverError(RuntimeError):
    """Eigensolver failure or non-SPD H (reference subspace.py:20-22)."""


@dataclass
class Subspace:
    """U (nf, r_bar) orthonormal with U^T H U = diag(eigenvalues); V = U[:, :r]."""

    U: np.ndarray
    eigenvalues: np.ndarray
    r: int
    UHX: np.ndarray
    VHX: np.ndarray
    rest: np.ndarray

    @property
    def V(self) -> np.ndarray:
        return self.U[:, : self.r]

    @property
    def eigenvalues_r(self) -> np.ndarray:
        return self.eigenvalues[: self.r]


def _finish(system: GlobalSystem, rest: np.ndarray, w: np.ndarray, vecs: np.ndarray, r: int) -> Subspace:
    if (w <= 0).any():
        raise EigensolverError(f"nonpositive eigenvalue {w.min():g}: H is not SPD")
    hx = system.H @ rest
    return Subspace(U=vecs, eigenvalues=w, r=r, UHX=vecs.T @ hx, VHX=vecs[:, :r].T @ hx, rest=rest.copy())


def build_subspace(system: GlobalSystem, rest: np.ndarray, r_bar: int, r: int, method: str = "host") -> Subspace:
    """Smallest-r_bar eigenpairs of H (reference subspace.py:49-84).

    method="host": scipy shift-invert Lanczos, identical to the reference.
    method="device": GPU Chebyshev-filtered subspace iteration for large meshes
    (eigen.py over the csrc/eigen.cu block kernels; the basis spans the same
    invariant subspace to solver tolerance; not bit-identical).
    """
    H = system.H
    n = H.shape[0]
    if not (0 < r <= r_bar <= n):
        raise ValueError("need 0 < r <= r_bar <= n")
    if method == "device":
        from .eigen import device_lowest_eigenpairs

        w, vecs = device_lowest_eigenpairs(system, r_bar)
        return _finish(system, rest, w, vecs, r)
    if r_bar >= n - 1:
        evals, evecs = np.linalg.eigh(H.toarray())
        w, vecs = evals[:r_bar], evecs[:, :r_bar]
    else:
        start = np.random.default_rng(0).standard_normal(n)
        try:
            w, vecs = spla.eigsh(H, k=r_bar, sigma=0.0, which="LM", v0=start)
        except (spla.ArpackNoConvergence, RuntimeError) as err:
            raise EigensolverError(f"shift-invert eigensolver failed: {err}") from err
        perm = np.argsort(w)
        w, vecs = w[perm], vecs[:, perm]
    return _finish(system, rest, w, vecs, r)


# ------------------------------------------------------------------ stage drop-ins (device)
# reference subspace.py:97-192 with the same signatures; the arithmetic runs in the
# step's own kernels (k_project_partial / k_gram_partial / k_reduced_solve / k_prolong)
# on a device context holding H (SELL-32) and the basis (context.py).

def _dev(a, dtype=np.float64):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a, dtype=dtype), device="cuda")


@dataclass
class ReducedSystem:
    """r x r collision-corrected system with its scaled approximate inverse (subspace.py:109-119)."""

    A: np.ndarray
    inverse: np.ndarray             # X with A X = (1/beta) Id
    beta: float
    used_fallback: bool = False
    _ctx: object = None             # device context holding it as its current reduced system
    _gen: int = -1

    def solve(self, rhs: np.ndarray) -> np.ndarray:
        return self.beta * (self.inverse @ rhs)


def _read_reduced(ctx, A: np.ndarray) -> ReducedSystem:
    import ctypes

    import torch

    from . import _lib

    r = A.shape[0]
    inv = torch.empty((r, r), dtype=torch.float64, device="cuda")
    beta = ctypes.c_double(0.0)
    fb = ctypes.c_int(0)
    _lib.check(ctx.lib.cs_reduced_get(ctx.ptr, inv.data_ptr(), ctypes.byref(beta), ctypes.byref(fb),
                                      _lib.stream_handle()), "cs_reduced_get")
    ctx.generation += 1
    return ReducedSystem(A=A, inverse=inv.cpu().numpy(), beta=float(beta.value), used_fallback=bool(fb.value),
                         _ctx=ctx, _gen=ctx.generation)


def _gram(ctx, rows: np.ndarray, weights: np.ndarray, r: int) -> np.ndarray:
    import torch

    from . import _lib

    G = torch.empty((r, r), dtype=torch.float64, device="cuda")
    rd = _dev(rows, np.int32) if len(rows) else _dev(np.zeros(1), np.int32)
    wd = _dev(weights) if len(rows) else _dev(np.zeros(1))
    _lib.check(ctx.lib.cs_reduced_update(ctx.ptr, rd.data_ptr(), wd.data_ptr(), int(len(rows)), G.data_ptr(),
                                         _lib.stream_handle()), "cs_reduced_update")
    return G.cpu().numpy()


def reduced_update(sub: Subspace, active_vertices, weights) -> np.ndarray:
    """sum_j w_j V_j V_j^T over the active rows (subspace.py:97-106)."""
    from . import context

    active = np.asarray(active_vertices, dtype=np.int64)
    w = np.asarray(weights, dtype=np.float64)
    if len(active) == 0:
        return np.zeros((sub.r, sub.r))
    if (w < 0).any():
        raise ValueError("collision weights must be nonnegative")
    return _gram(context.get(subspace=sub), active, w, sub.r)


def build_reduced(sub: Subspace, delta_reduced: np.ndarray, rhs_scale: float) -> ReducedSystem:
    """A = diag(lambda_r) + delta_reduced, beta-scaled inverse with the pinv fallback
    (subspace.py:122-140), factored in one CTA on the device."""
    from . import _lib, context

    ctx = context.get(subspace=sub)
    G = _dev(delta_reduced)
    import ctypes

    _lib.check(ctx.lib.cs_build_reduced(ctx.ptr, G.data_ptr(), float(rhs_scale), None, None, None,
                                        _lib.stream_handle()), "cs_build_reduced")
    A = np.diag(sub.eigenvalues_r) + np.asarray(delta_reduced, dtype=np.float64)
    return _read_reduced(ctx, A)


def reduced_correction(sub: Subspace, system: GlobalSystem, b: np.ndarray, x: np.ndarray, diag_delta: np.ndarray,
                       reduced: ReducedSystem | None = None):
    """Galerkin step in the reuse basis around x (subspace.py:165-186); returns
    (corrected x, reduced system for reuse within an iteration)."""
    from . import _lib, context

    ctx = context.get(system=system, subspace=sub)
    delta = np.asarray(diag_delta, dtype=np.float64)
    reuse = 0
    if reduced is not None:
        if reduced._ctx is ctx and reduced._gen == ctx.generation:
            reuse = 1
        else:  # a system from elsewhere: make it the context's current one
            import ctypes

            G = _dev(np.asarray(reduced.A) - np.diag(sub.eigenvalues_r))
            _lib.check(ctx.lib.cs_build_reduced(ctx.ptr, G.data_ptr(), float(reduced.beta), None, None, None,
                                                _lib.stream_handle()), "cs_build_reduced")
            reuse = 1
    bd, xd, dd = _dev(b), _dev(x), _dev(delta)
    _lib.check(ctx.lib.cs_reduced_correction(ctx.ptr, bd.data_ptr(), xd.data_ptr(), dd.data_ptr(), reuse,
                                             _lib.stream_handle()), "cs_reduced_correction")
    x_new = xd.cpu().numpy()
    if reduced is None:
        active = np.flatnonzero(delta)
        G = _gram(ctx, active, delta[active], sub.r) if len(active) else np.zeros((sub.r, sub.r))
        reduced = _read_reduced(ctx, np.diag(sub.eigenvalues_r) + G)
    return x_new, reduced


def warmstart_correction(sub: Subspace, system: GlobalSystem, b: np.ndarray, x: np.ndarray) -> np.ndarray:
    """x + U (U^T (b - H x) / lambda) in the full warm-start basis (subspace.py:189-192)."""
    from . import _lib, context

    ctx = context.get(system=system, subspace=sub)
    bd, xd = _dev(b), _dev(x)
    _lib.check(ctx.lib.cs_warmstart_correction(ctx.ptr, bd.data_ptr(), xd.data_ptr(), _lib.stream_handle()),
               "cs_warmstart_correction")
    return xd.cpu().numpy()
