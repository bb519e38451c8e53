"""GPU rest-shape eigenbasis for paper-scale meshes.

Chebyshev-filtered subspace iteration (ChFSI) on H: a degree-d Chebyshev
polynomial damps the unwanted interval [lambda_cut, lambda_max] while
amplifying the lowest modes; each outer iteration orthonormalises the block
and Rayleigh-Ritz-projects it, so the returned basis satisfies U^T U = I and
U^T H U = diag(eigenvalues) to round-off - the two properties the two-level
solve relies on (reference subspace.py:28-31).  Converges the lowest r_bar Ritz
pairs to a relative residual ``tol`` using a guard block.

Replaces scipy's shift-invert ``eigsh`` (343 s at 341K vertices on the build
host) for setup only; parity tests use the host solver, whose basis is
bit-identical to the reference's.  Every n-sized operation runs in the
library's own kernels behind the C ABI (csrc/eigen.cu: the fused Chebyshev
SpMM recurrence over the block, the tall-skinny Gram A^T B, the block update
X S, the Ritz residual norms); only p x p algebra (p = r_bar + guard <= 256:
Cholesky, triangular inverse, symmetric eigensolve) runs here in numpy.
Orthonormalisation is repeated SVQB (eigen-decomposition of the scaled Gram),
robust to the numerically rank-deficient blocks a high-degree filter produces.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

# block slots in the device context
_X, _HX, _W1, _W2 = 0, 1, 2, 3


class _Ctx:
    def __init__(self, H, p):
        self.lib = _lib.load()
        self.stream = _lib.stream_handle()
        self.n = H.shape[0]
        self.p = p
        self.indptr = np.ascontiguousarray(H.indptr, dtype=np.int32)
        self.indices = np.ascontiguousarray(H.indices, dtype=np.int32)
        self.data = np.ascontiguousarray(H.data, dtype=np.float64)
        st = ctypes.c_int(0)
        self.h = self.lib.cs_eig_create(self.n, self.indptr.ctypes.data, self.indices.ctypes.data,
                                        self.data.ctypes.data, p, 4, ctypes.byref(st))
        if not self.h:
            _lib.check(st.value or _lib.CS_INTERNAL, "cs_eig_create")

    def close(self):
        if self.h:
            self.lib.cs_eig_destroy(self.h)
            self.h = None

    def set(self, blk, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        _lib.check(self.lib.cs_eig_set(self.h, blk, a.ctypes.data, self.stream), "cs_eig_set")

    def get(self, blk, cols):
        out = np.empty((self.n, cols))
        _lib.check(self.lib.cs_eig_get(self.h, blk, cols, out.ctypes.data, self.stream), "cs_eig_get")
        return out

    def spmm(self, src, dst):
        _lib.check(self.lib.cs_eig_spmm(self.h, src, dst, self.stream), "cs_eig_spmm")

    def filter(self, degree, a, lam_max, a0):
        _lib.check(self.lib.cs_eig_filter(self.h, _X, _W1, _W2, degree, a, lam_max, a0, self.stream),
                   "cs_eig_filter")

    def gram(self, a, b):
        out = np.empty((self.p, self.p))
        _lib.check(self.lib.cs_eig_gram(self.h, a, b, out.ctypes.data, self.stream), "cs_eig_gram")
        return out

    def mul(self, src, S, dst):
        S = np.ascontiguousarray(S, dtype=np.float64)
        _lib.check(self.lib.cs_eig_mul(self.h, src, S.ctypes.data, dst, self.stream), "cs_eig_mul")

    def swap(self, a, b):
        _lib.check(self.lib.cs_eig_swap(self.h, a, b), "cs_eig_swap")

    def residuals(self, w, cols):
        w = np.ascontiguousarray(w, dtype=np.float64)
        out = np.empty(cols)
        _lib.check(self.lib.cs_eig_residuals(self.h, _HX, _X, w.ctypes.data, cols, out.ctypes.data, self.stream),
                   "cs_eig_residuals")
        return out


def _orthonormalise(ctx: _Ctx, passes: int = 3) -> None:
    """Block X <- an orthonormal basis of its span: SVQB (Stathopoulos & Wu 2002) repeated,
    all n-sized work on the device (Gram X^T X, update X T), T from the host eigensolve of
    the column-scaled p x p Gram; eigenvalues below eps * max are lifted (a filtered block
    is numerically rank deficient: those columns become noise, orthogonalised by the next
    pass and refreshed by the next filter)."""
    p = ctx.p
    eps = np.finfo(np.float64).eps
    for _ in range(passes):
        G = ctx.gram(_X, _X)
        G = 0.5 * (G + G.T)
        dg = np.diag(G).copy()
        d = 1.0 / np.sqrt(np.where(dg > 0.0, dg, 1.0))
        lam, V = np.linalg.eigh(d[:, None] * G * d[None, :])
        lam = np.maximum(lam, eps * max(float(lam.max()), 1e-300))
        T = (d[:, None] * V) / np.sqrt(lam)[None, :]
        ctx.mul(_X, T, _W1)
        ctx.swap(_X, _W1)
        if lam.min() > 0.5 * lam.max():  # already orthonormal to round-off (a second pass)
            break


def _rayleigh_ritz(ctx: _Ctx):
    """X <- X S, HX <- H X S with S the eigenvectors of X^T H X (ascending)."""
    ctx.spmm(_X, _HX)
    G = ctx.gram(_X, _HX)
    G = 0.5 * (G + G.T)
    w, S = np.linalg.eigh(G)
    ctx.mul(_X, S, _W1)
    ctx.mul(_HX, S, _W2)
    ctx.swap(_X, _W1)
    ctx.swap(_HX, _W2)
    return w


def device_lowest_eigenpairs(system, k: int, guard: int | None = None, degree: int = 60, tol: float = 1e-7,
                             max_outer: int = 60, seed: int = 0):
    H = system.H.tocsr()
    H.sort_indices()
    n = H.shape[0]
    p = min(n, k + (guard if guard is not None else max(16, k // 3)))
    if p > 256:
        raise ValueError("device eigensolver supports r_bar + guard <= 256")
    # Gershgorin upper bound of the spectrum
    absrow = np.add.reduceat(np.abs(H.data), H.indptr[:-1]) if H.nnz else np.zeros(n)
    lam_max = float(absrow.max()) * 1.01
    ctx = _Ctx(H, p)
    try:
        ctx.set(_X, np.random.default_rng(seed).standard_normal((n, p)))
        _orthonormalise(ctx)
        w = _rayleigh_ritz(ctx)
        for _ in range(max_outer):
            res = np.sqrt(ctx.residuals(w, k)) / np.maximum(np.abs(w[:k]), 1e-300)
            if float(res.max()) <= tol:
                break
            ctx.filter(degree, float(w[-1]), lam_max, float(w[0]))   # damp [w_p, lam_max]
            _orthonormalise(ctx)
            w = _rayleigh_ritz(ctx)
        vals = w[:k].copy()
        vecs = ctx.get(_X, k)
    finally:
        ctx.close()
    # deterministic sign convention: largest-magnitude entry positive
    flip = np.sign(vecs[np.argmax(np.abs(vecs), axis=0), np.arange(k)])
    flip[flip == 0] = 1.0
    return vals, np.ascontiguousarray(vecs * flip)
