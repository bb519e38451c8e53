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
selects the GPU block eigensolver (``csrc/eigen.cu``).
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
    method="device": GPU LOBPCG-style block solver for large meshes (basis
    spans the same invariant subspace to solver tolerance; not bit-identical).
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
