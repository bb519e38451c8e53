"""ORACLE (test infrastructure only): local/global solver stages.

numpy/scipy restatement of reference
  constraints.py:212-256  (edge projection rhs, pinned columns, collision stamps)
  smoothing.py:23-66      (rank-2 aggregated Jacobi with divergence guard)
  subspace.py:97-192      (reuse-basis reduced correction, warm-start correction)
  stepper.py:309-380      (variational energy + gradient, quadratic collision form)
using the same numpy/scipy/BLAS calls so results are bit-identical to the
reference on the host that generated tests/golden.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg as sla


class SmootherDivergence(RuntimeError):
    pass


# ------------------------------------------------------------ constraints.py
def edge_targets(xa, xb, rest):
    """Projected edge vector y = target_b - target_a (constraints.py:19-39, 219-221)."""
    d = xb - xa
    length = np.linalg.norm(d, axis=1)
    unit = np.zeros_like(d)
    nz = length > 0
    unit[nz] = d[nz] / length[nz, None]
    unit[~nz] = (1.0, 0.0, 0.0)
    mid = 0.5 * (xa + xb)
    half = 0.5 * rest[:, None] * unit
    return (mid + half) - (mid - half)


def assemble_rhs(system, mesh, elastic, z, x, pins, c_ids=None, c_w=None, c_t=None):
    """b over free vertices and the collision diagonal delta (constraints.py:229-256)."""
    n = mesh.vertex_count
    acc = np.zeros((n, 3))
    if len(elastic.edges):
        e0, e1 = elastic.edges[:, 0], elastic.edges[:, 1]
        y = edge_targets(x[e0], x[e1], elastic.edge_rest)
        w = elastic.stretch_w[:, None]
        np.add.at(acc, e0, -w * y)
        np.add.at(acc, e1, w * y)
    b = acc[mesh.free] + system.mass_over_h2[:, None] * z[mesh.free]
    if mesh.pinned.size:
        b -= system.H_fp @ pins
    delta = np.zeros(system.H.shape[0])
    if c_ids is not None and len(c_ids):
        rows = mesh.free_index[c_ids]
        ok = rows >= 0
        np.add.at(delta, rows[ok], c_w[ok])
        np.add.at(b, rows[ok], c_w[ok, None] * c_t[ok])
    return b, delta


# ------------------------------------------------------------ smoothing.py
def ajacobi_smooth(system, b, x0, iterations, omega=0.0, delta=None):
    """ceil(iterations/2) rank-2 steps x += c(2t - c D^-1 A t) (smoothing.py:23-66)."""
    H = system.H
    d = system.diag if delta is None else system.diag + delta
    if (d <= 0).any():
        raise ValueError("nonpositive diagonal entry")
    c = 1.0 - omega
    inv_d = 1.0 / d
    if x0.ndim == 2:
        inv_d = inv_d[:, None]
    dcol = None if delta is None else (delta[:, None] if x0.ndim == 2 else delta)

    def apply(v):
        out = H @ v
        return out if dcol is None else out + dcol * v

    x = x0.astype(np.float64, copy=True)
    last = None
    for k in range((iterations + 1) // 2):
        r = b - apply(x)
        if (2 * k) % 20 == 0:
            nr = float(np.linalg.norm(r))
            if last is not None and nr > 10.0 * last:
                raise SmootherDivergence(f"residual grew from {last:g} to {nr:g}; raise omega")
            last = nr
        t = inv_d * r
        x += c * (2.0 * t - c * (inv_d * apply(t)))
    return x


# ------------------------------------------------------------ subspace.py
class Reduced:
    """r x r collision-corrected system and scaled inverse (subspace.py:109-140)."""

    def __init__(self, sub, gram, rhs_scale):
        A = np.diag(sub.eigenvalues_r) + gram
        beta = rhs_scale if rhs_scale > 0 else 1.0
        self.A, self.beta, self.fallback = A, beta, False
        try:
            lu = sla.lu_factor(A)
            inv = sla.lu_solve(lu, np.eye(sub.r) / beta)
        except sla.LinAlgError:
            self.inverse, self.fallback = np.linalg.pinv(A) / beta, True
            return
        err = np.abs(A @ (beta * inv) - np.eye(sub.r)).max()
        if not np.isfinite(err) or err > 1e-4:
            inv, self.fallback = np.linalg.pinv(A) / beta, True
        self.inverse = inv

    def solve(self, rhs):
        return self.beta * (self.inverse @ rhs)


def reduced_gram(sub, rows, w):
    """sum_j w_j V_j V_j^T over active rows (subspace.py:97-106)."""
    if len(rows) == 0:
        return np.zeros((sub.r, sub.r))
    if (np.asarray(w) < 0).any():
        raise ValueError("collision weights must be nonnegative")
    Vr = sub.V[rows]
    return Vr.T @ (np.asarray(w, dtype=np.float64)[:, None] * Vr)


def reduced_correction(sub, system, b, x, delta, reduced=None):
    """Galerkin correction in the reuse basis around x (subspace.py:165-186)."""
    res = b - system.H @ x - delta[:, None] * x
    rhs = sub.V.T @ res
    if reduced is None:
        act = np.flatnonzero(delta)
        reduced = Reduced(sub, reduced_gram(sub, act, delta[act]), float(np.abs(rhs).mean()))
    return x + sub.V @ reduced.solve(rhs), reduced


def warmstart_correction(sub, system, b, x):
    """Elastic-only Galerkin correction in the wide basis (subspace.py:189-192)."""
    rhs = sub.U.T @ (b - system.H @ x)
    return x + sub.U @ (rhs / sub.eigenvalues[:, None])


# ------------------------------------------------------------ stepper.py energy
def energy(mesh, el, h, x, z, quad=None):
    """Energy and gradient with pinned rows zeroed (stepper.py:309-380, 'quad' form)."""
    grad = np.zeros_like(x)
    s = mesh.vertex_mass[:, None] / (h * h)
    e_in = 0.5 * float(np.sum(s * (x - z) ** 2))
    grad += s * (x - z)
    ev = x[el.edges[:, 1]] - x[el.edges[:, 0]]
    ln = np.linalg.norm(ev, axis=1)
    e_st = 0.5 * float((el.stretch_w * (ln - el.edge_rest) ** 2).sum())
    unit = np.zeros_like(ev)
    ok = ln > 0
    unit[ok] = ev[ok] / ln[ok, None]
    g = (el.stretch_w * (ln - el.edge_rest))[:, None] * unit
    np.add.at(grad, el.edges[:, 1], g)
    np.add.at(grad, el.edges[:, 0], -g)
    e_b = 0.0
    if len(el.stencils):
        flat = np.einsum("sj,sjd->sd", el.bend_k, x[el.stencils])
        e_b = 0.5 * float(np.sum(el.bend_w * np.einsum("sd,sd->s", flat, flat)))
        gb = el.bend_w[:, None, None] * el.bend_k[:, :, None] * flat[:, None, :]
        np.add.at(grad, el.stencils.ravel(), gb.reshape(-1, 3))
    e_c = 0.0
    if quad is not None:
        ids, w, tg = quad
        diff = x[ids] - tg
        e_c = 0.5 * float(np.sum(w * np.einsum("mj,mj->m", diff, diff)))
        np.add.at(grad, ids, w[:, None] * diff)
    grad[mesh.pinned] = 0.0
    return e_in + e_st + e_b + e_c, grad, {"inertia": e_in, "stretch": e_st, "bend": e_b, "barrier": e_c}
