"""ORACLE (test infrastructure only): exhaustive triangle-triangle intersection
check - restates reference oracles.py:21-131 (separating-axis test over 17
axes, x-sorted chunked sweep, adjacent triangles skipped)."""

from __future__ import annotations

import numpy as np


def _axes(p, q):
    ep = np.stack([p[:, 1] - p[:, 0], p[:, 2] - p[:, 1], p[:, 0] - p[:, 2]], axis=1)
    eq = np.stack([q[:, 1] - q[:, 0], q[:, 2] - q[:, 1], q[:, 0] - q[:, 2]], axis=1)
    npn = np.cross(ep[:, 0], ep[:, 1])[:, None, :]
    nqn = np.cross(eq[:, 0], eq[:, 1])[:, None, :]
    mixed = np.cross(ep[:, :, None, :], eq[:, None, :, :]).reshape(len(p), 9, 3)
    return np.concatenate([npn, nqn, mixed, np.cross(npn, ep), np.cross(nqn, eq)], axis=1)


def tri_tri_intersect(p, q):
    """True per pair when closed triangles intersect (oracles.py:33-48)."""
    p = np.asarray(p, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    if p.ndim == 2:
        p, q = p[None], q[None]
    ax = _axes(p, q)
    scale = np.abs(np.concatenate([p, q], axis=1)).max(axis=(1, 2)) + 1.0
    usable = np.linalg.norm(ax, axis=2) > 1e-14 * scale[:, None] ** 2
    pp = np.einsum("maj,mvj->mav", ax, p)
    pq = np.einsum("maj,mvj->mav", ax, q)
    sep = (pp.max(axis=2) < pq.min(axis=2)) | (pq.max(axis=2) < pp.min(axis=2))
    return ~(sep & usable).any(axis=1)


def intersecting_pairs(x, triangles, chunk: int = 512):
    """All intersecting non-adjacent triangle pairs, (k,2) sorted rows (oracles.py:83-131)."""
    x = np.asarray(x, dtype=np.float64)
    tris = np.asarray(triangles, dtype=np.int64)
    pts = x[tris]
    lo, hi = pts.min(axis=1), pts.max(axis=1)
    order = np.argsort(lo[:, 0], kind="stable")
    lo, hi, pts, ts = lo[order], hi[order], pts[order], tris[order]
    found = []
    for s in range(0, len(tris), chunk):
        rows = np.arange(s, min(s + chunk, len(tris)))
        stop = int(np.searchsorted(lo[:, 0], hi[rows, 0].max(), side="right"))
        cols = np.arange(s, stop)
        if not len(cols):
            continue
        ov = ((lo[rows, None] <= hi[None, cols]) & (lo[None, cols] <= hi[rows, None])).all(axis=2)
        ii, jj = np.nonzero(ov)
        ii, jj = rows[ii], cols[jj]
        keep = jj > ii
        ii, jj = ii[keep], jj[keep]
        if not len(ii):
            continue
        shared = (ts[ii][:, :, None] == ts[jj][:, None, :]).any(axis=(1, 2))
        ii, jj = ii[~shared], jj[~shared]
        if not len(ii):
            continue
        hit = tri_tri_intersect(pts[ii], pts[jj])
        if hit.any():
            found.append(np.stack([order[ii[hit]], order[jj[hit]]], axis=1))
    if not found:
        return np.zeros((0, 2), dtype=np.int64)
    out = np.concatenate(found)
    out.sort(axis=1)
    return out


def tri_tri_intersect_exact(p, q) -> bool:
    """Rational-arithmetic separating-axis verdict for one pair (oracles.py:51-80)."""
    from fractions import Fraction

    P = [[Fraction(float(c)) for c in v] for v in p]
    Q = [[Fraction(float(c)) for c in v] for v in q]

    def sub(a, b):
        return [a[i] - b[i] for i in range(3)]

    def cross(a, b):
        return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]

    def dot(a, b):
        return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]

    ep = [sub(P[1], P[0]), sub(P[2], P[1]), sub(P[0], P[2])]
    eq = [sub(Q[1], Q[0]), sub(Q[2], Q[1]), sub(Q[0], Q[2])]
    n_p, n_q = cross(ep[0], ep[1]), cross(eq[0], eq[1])
    axes = [n_p, n_q] + [cross(a, b) for a in ep for b in eq] + [cross(n_p, e) for e in ep] + \
        [cross(n_q, e) for e in eq]
    for ax in axes:
        if ax == [0, 0, 0]:
            continue
        dp = [dot(ax, v) for v in P]
        dq = [dot(ax, v) for v in Q]
        if max(dp) < min(dq) or max(dq) < min(dp):
            return False
    return True


def exact_separation_margin(p, q) -> float:
    """Largest normalised separation over the 17 axes in exact arithmetic, 0 when the
    triangles intersect (reference tests/test_harness.py:127-163)."""
    from fractions import Fraction

    P = [[Fraction(float(c)) for c in v] for v in p]
    Q = [[Fraction(float(c)) for c in v] for v in q]

    def sub(a, b):
        return [a[i] - b[i] for i in range(3)]

    def cross(a, b):
        return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]

    def dot(a, b):
        return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]

    ep = [sub(P[1], P[0]), sub(P[2], P[1]), sub(P[0], P[2])]
    eq = [sub(Q[1], Q[0]), sub(Q[2], Q[1]), sub(Q[0], Q[2])]
    n_p, n_q = cross(ep[0], ep[1]), cross(eq[0], eq[1])
    axes = [n_p, n_q] + [cross(a, b) for a in ep for b in eq] + [cross(n_p, e) for e in ep] + \
        [cross(n_q, e) for e in eq]
    best = Fraction(0)
    for ax in axes:
        norm2 = dot(ax, ax)
        if norm2 == 0:
            continue
        dp = [dot(ax, v) for v in P]
        dq = [dot(ax, v) for v in Q]
        gap = max(min(dq) - max(dp), min(dp) - max(dq))
        if gap > 0:
            best = max(best, gap * gap / norm2)
    return float(best) ** 0.5
