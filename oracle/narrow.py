"""ORACLE (test infrastructure only): closest points, full CCD, distance march,
partial CCD.  numpy restatement of reference pkg/src/clothsim/collision/
{geometry,ccd,partial}.py with numpy's exact evaluation order.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

VT, EE = 0, 1
_TINY = 1e-14                     # geometry.py:7


def dot3(a, b):
    """Row dot products exactly as the reference's einsum calls evaluate them
    over 3 terms: (a0 b0 + a2 b2) + a1 b1 (geometry.py:21-28, partial.py:193)."""
    if a.ndim == 2:
        return np.einsum("ij,ij->i", a, b)
    return np.einsum("mkj,mkj->mk", a, b)


def norm3(a):
    return np.linalg.norm(a, axis=-1)


def _safe_div(num, den, mask):
    out = np.zeros(np.broadcast(num, den).shape)
    np.divide(num, den, out=out, where=mask)
    return out


# --------------------------------------------------------------- geometry.py
def closest_on_triangle(p, a, b, c):
    """Voronoi-region closest point (reference geometry.py:10-79).

    Returns (closest, (u, v) barycentric weights of b and c, distance).
    """
    p, a, b, c = (np.atleast_2d(np.asarray(z, dtype=np.float64)) for z in (p, a, b, c))
    ab, ac = b - a, c - a
    ap, bp, cp = p - a, p - b, p - c
    d1, d2 = dot3(ab, ap), dot3(ac, ap)
    d3, d4 = dot3(ab, bp), dot3(ac, bp)
    d5, d6 = dot3(ab, cp), dot3(ac, cp)
    m = len(p)
    u = np.zeros(m)
    v = np.zeros(m)
    settled = (d1 <= 0) & (d2 <= 0)                              # region A
    at_b = ~settled & (d3 >= 0) & (d4 <= d3)                     # region B
    u[at_b] = 1.0
    settled |= at_b
    at_c = ~settled & (d6 >= 0) & (d5 <= d6)                     # region C
    v[at_c] = 1.0
    settled |= at_c
    vc = d1 * d4 - d3 * d2                                       # edge AB
    on_ab = ~settled & (vc <= 0) & (d1 >= 0) & (d3 <= 0)
    den = d1 - d3
    u[on_ab] = _safe_div(d1, den, np.abs(den) > _TINY)[on_ab]
    settled |= on_ab
    vb = d5 * d2 - d1 * d6                                       # edge AC
    on_ac = ~settled & (vb <= 0) & (d2 >= 0) & (d6 <= 0)
    den = d2 - d6
    v[on_ac] = _safe_div(d2, den, np.abs(den) > _TINY)[on_ac]
    settled |= on_ac
    va = d3 * d6 - d5 * d4                                       # edge BC
    g1, g2 = d4 - d3, d5 - d6
    on_bc = ~settled & (va <= 0) & (g1 >= 0) & (g2 >= 0)
    den = g1 + g2
    s = _safe_div(g1, den, np.abs(den) > _TINY)
    u[on_bc] = 1.0 - s[on_bc]
    v[on_bc] = s[on_bc]
    settled |= on_bc
    face = ~settled                                              # interior
    den = va + vb + vc
    inv = _safe_div(1.0, den, np.abs(den) > _TINY)
    u[face] = (vb * inv)[face]
    v[face] = (vc * inv)[face]
    q = a + u[:, None] * ab + v[:, None] * ac
    return q, np.stack([u, v], axis=1), norm3(p - q)


def closest_between_segments(a0, a1, b0, b1):
    """Clamped segment-segment closest points (reference geometry.py:82-112)."""
    a0, a1, b0, b1 = (np.atleast_2d(np.asarray(z, dtype=np.float64)) for z in (a0, a1, b0, b1))
    da, db, r = a1 - a0, b1 - b0, a0 - b0
    aa, bb = dot3(da, da), dot3(db, db)
    f, c, ab = dot3(db, r), dot3(da, r), dot3(da, db)
    den = aa * bb - ab * ab
    s = np.clip(_safe_div(ab * f - c * bb, den, den > _TINY * np.maximum(aa * bb, 1.0)), 0.0, 1.0)
    t_raw = _safe_div(ab * s + f, bb, bb > _TINY)
    t = np.clip(t_raw, 0.0, 1.0)
    refit = np.clip(_safe_div(ab * t - c, aa, aa > _TINY), 0.0, 1.0)
    s = np.where(t_raw != t, refit, s)
    pa = a0 + s[:, None] * da
    pb = b0 + t[:, None] * db
    return pa, pb, np.stack([s, t], axis=1), norm3(pa - pb)


def witness(kind, idx, x):
    """Per-pair closest points, parameters, distance (reference geometry.py:115-148)."""
    kind = np.asarray(kind)
    idx = np.asarray(idx)
    m = len(kind)
    first, second = np.zeros((m, 3)), np.zeros((m, 3))
    params, dist = np.zeros((m, 2)), np.zeros(m)
    for k, solve in ((VT, None), (EE, None)):
        sel = np.flatnonzero(kind == k)
        if sel.size == 0:
            continue
        q = x[idx[sel]]
        if k == VT:
            cl, pr, dd = closest_on_triangle(q[:, 0], q[:, 1], q[:, 2], q[:, 3])
            first[sel], second[sel] = q[:, 0], cl
        else:
            pa, pb, pr, dd = closest_between_segments(q[:, 0], q[:, 1], q[:, 2], q[:, 3])
            first[sel], second[sel] = pa, pb
        params[sel], dist[sel] = pr, dd
    return first, second, params, dist


def _distance_of_points(kind, q):
    """Witness distance from gathered (m,4,3) corners (reference ccd.py:207-218)."""
    out = np.empty(len(kind))
    vt = kind == VT
    if vt.any():
        out[vt] = closest_on_triangle(q[vt, 0], q[vt, 1], q[vt, 2], q[vt, 3])[2]
    if (~vt).any():
        out[~vt] = closest_between_segments(q[~vt, 0], q[~vt, 1], q[~vt, 2], q[~vt, 3])[3]
    return out


# --------------------------------------------------------------- ccd.py
NODES = (0.0, 1.0 / 3.0, 2.0 / 3.0, 1.0)                          # ccd.py:21
FIT = np.linalg.inv(np.vander(np.array(NODES), 4, increasing=True))   # ccd.py:22
_BARY_SLACK = 1e-8
_BISECTIONS = 80

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "lib", "liboracle_ccd.so")
_lib = None


def build_c(force: bool = False) -> str:
    """Compile oracle/c/ccd_fit.c (gcc, no FP contraction)."""
    src = os.path.join(_HERE, "c", "ccd_fit.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", src,
                               "-o", _LIB_PATH, "-lm"])
    return _LIB_PATH


def _fit_lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_c())
        _lib.oracle_ccd_fit.argtypes = [ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p, ctypes.c_void_p]
        _lib.oracle_ccd_fit.restype = None
    return _lib


def cubic_fit(samples: np.ndarray) -> np.ndarray:
    """samples (m,4) at NODES -> monomial coefficients (m,4) (ccd.py:44)."""
    f = np.ascontiguousarray(samples, dtype=np.float64)
    out = np.empty_like(f)
    fit = np.ascontiguousarray(FIT)
    _fit_lib().oracle_ccd_fit(f.ctypes.data, len(f), fit.ctypes.data, out.ctypes.data)
    return out


def _triple_rows(kind, q):
    """Coplanarity triple (u x v) . w per pair (ccd.py:25-33)."""
    vt = (kind == VT)[:, None]
    u = np.where(vt, q[:, 2] - q[:, 1], q[:, 1] - q[:, 0])
    v = np.where(vt, q[:, 3] - q[:, 1], q[:, 3] - q[:, 2])
    w = np.where(vt, q[:, 0] - q[:, 1], q[:, 2] - q[:, 0])
    return dot3(np.cross(u, v), w)


def coplanarity_cubic(kind, idx, x0, x1):
    """Cubic coefficients, lowest order first (ccd.py:36-44)."""
    vals = [_triple_rows(kind, ((1.0 - t) * x0 + t * x1)[idx]) for t in NODES]
    return cubic_fit(np.stack(vals, axis=1))


def horner(c, t):
    """c0 + t (c1 + t (c2 + t c3)) broadcast over trailing dims (ccd.py:47-50)."""
    cs = [c[:, j].reshape((-1,) + (1,) * (t.ndim - 1)) for j in range(4)]
    return cs[0] + t * (cs[1] + t * (cs[2] + t * cs[3]))


def root_candidates(c):
    """Up to 5 root candidates per pair in (0,1], nan padded (ccd.py:53-108)."""
    m = len(c)
    qa, qb, ql = 3.0 * c[:, 3], 2.0 * c[:, 2], c[:, 1]
    has_quad = np.abs(qa) > 0
    disc = qb * qb - 4.0 * qa * ql
    real = has_quad & (disc >= 0)
    root = np.sqrt(np.where(real, disc, 0.0))
    with np.errstate(divide="ignore", invalid="ignore"):
        ra = np.where(real, (-qb - root) / (2.0 * qa), np.nan)
        rb = np.where(real, (-qb + root) / (2.0 * qa), np.nan)
        r_lin = np.where(~has_quad & (np.abs(qb) > 0), -ql / qb, np.nan)
    brk = np.stack([np.where(has_quad, np.minimum(ra, rb), r_lin),
                    np.where(has_quad, np.maximum(ra, rb), np.nan)], axis=1)
    brk[~((brk > 0.0) & (brk < 1.0))] = np.nan
    brk = np.sort(brk, axis=1)
    k1 = np.where(np.isnan(brk[:, 0]), 1.0, brk[:, 0])
    k2 = np.where(np.isnan(brk[:, 1]), k1, np.maximum(brk[:, 1], k1))
    lo = np.stack([np.zeros(m), k1, k2], axis=1)
    hi = np.stack([k1, k2, np.ones(m)], axis=1)
    f_lo, f_hi = horner(c, lo), horner(c, hi)
    bracket = (hi > lo) & (f_lo * f_hi < 0)
    at_end = (hi > lo) & (f_hi == 0)
    a_lo, a_hi = lo.copy(), hi.copy()
    for _ in range(_BISECTIONS):
        mid = 0.5 * (a_lo + a_hi)
        fm = horner(c, mid)
        right = bracket & (np.sign(fm) == np.sign(f_lo))
        a_lo = np.where(right, mid, a_lo)
        f_lo = np.where(right, fm, f_lo)
        a_hi = np.where(bracket & ~right, mid, a_hi)
    out = np.full((m, 5), np.nan)
    out[:, :3] = np.where(bracket, 0.5 * (a_lo + a_hi), np.where(at_end, hi, np.nan))
    mag = np.abs(c).sum(axis=1) + 1e-300
    for j in range(2):
        tb = brk[:, j]
        fv = np.abs(horner(c, np.where(np.isnan(tb), 0.0, tb)))
        out[:, 3 + j] = np.where(~np.isnan(tb) & (fv <= 1e-9 * mag), tb, np.nan)
    out[~((out > 0.0) & (out <= 1.0))] = np.nan
    return out


def _extent(idx, x0, x1):
    q0, q1 = x0[idx], x1[idx]
    lo = np.minimum(q0.min(axis=1), q1.min(axis=1))
    hi = np.maximum(q0.max(axis=1), q1.max(axis=1))
    return norm3(hi - lo)                                         # ccd.py:199-204


def _confirm(kind, idx, x0, x1, t, tol):
    """Inflated inside test at time t (ccd.py:111-135)."""
    ok = np.zeros(len(t), dtype=bool)
    sel = np.flatnonzero(~np.isnan(t))
    if sel.size == 0:
        return ok
    tt = t[sel, None, None]
    q = (1.0 - tt) * x0[idx[sel]] + tt * x1[idx[sel]]
    kk = kind[sel]
    res = np.zeros(sel.size, dtype=bool)
    vt = kk == VT
    if vt.any():
        g = q[vt]
        _, uv, d = closest_on_triangle(g[:, 0], g[:, 1], g[:, 2], g[:, 3])
        size = norm3(g[:, 2] - g[:, 1]) + norm3(g[:, 3] - g[:, 1])
        inside = (uv[:, 0] >= -_BARY_SLACK) & (uv[:, 1] >= -_BARY_SLACK) & (uv[:, 0] + uv[:, 1] <= 1.0 + _BARY_SLACK)
        res[vt] = inside & (d <= tol * np.maximum(size, 1.0))
    if (~vt).any():
        g = q[~vt]
        d = closest_between_segments(g[:, 0], g[:, 1], g[:, 2], g[:, 3])[3]
        size = norm3(g[:, 1] - g[:, 0]) + norm3(g[:, 3] - g[:, 2])
        res[~vt] = d <= tol * np.maximum(size, 1.0)
    ok[sel] = res
    return ok


def full_ccd(kind, idx, x0, x1, tol: float = 1e-6):
    """Earliest validated impact time in (0,1], nan = miss (ccd.py:138-196)."""
    kind = np.asarray(kind)
    idx = np.asarray(idx)
    m = len(kind)
    if m == 0:
        return np.full(0, np.nan)
    c = coplanarity_cubic(kind, idx, x0, x1)
    cand = root_candidates(c)
    flat = np.abs(c).sum(axis=1) <= 1e-12 * np.maximum(np.abs(_extent(idx, x0, x1)) ** 3, 1e-30)
    cand[flat] = np.nan
    cand = np.sort(cand, axis=1)                                  # ascending, nan last
    toi = np.full(m, np.nan)
    for j in range(5):
        tj = cand[:, j]
        todo = np.isnan(toi) & ~np.isnan(tj)
        if todo.any():
            hit = _confirm(kind, idx, x0, x1, np.where(todo, tj, np.nan), tol)
            toi[todo & hit] = tj[todo & hit]
    if flat.any():
        toi[flat] = _flat_fallback(kind[flat], idx[flat], x0, x1)
    return toi


def _flat_fallback(fk, fi, x0, x1):
    """Dense distance sampling for identically-coplanar motion (ccd.py:171-195)."""
    out = np.full(len(fk), np.nan)
    _, _, _, d0 = witness(fk, fi, x0)
    move = norm3(x1[fi] - x0[fi])                                 # (f,4)
    side_a = np.where(fk[:, None] == VT, [True, False, False, False], [True, True, False, False])
    reach = np.max(np.where(side_a, move, 0.0), axis=1) + np.max(np.where(side_a, 0.0, move), axis=1)
    ext = np.maximum(_extent(fi, x0, x1), 1.0)
    near = d0 <= reach + 1e-9 * ext
    if not near.any():
        return out
    nk, ni = fk[near], fi[near]
    base = x0[ni]
    step = x1[ni] - base
    loc = np.arange(4 * len(ni)).reshape(-1, 4)
    got = np.full(len(ni), np.nan)
    for t in np.linspace(0.0, 1.0, 65)[1:]:
        d = witness(nk, loc, (base + t * step).reshape(-1, 3))[3]
        fresh = np.isnan(got) & (d <= 1e-9 * ext[near])
        got[fresh] = t
    out[near] = got
    return out


def _side_lipschitz(kind, move):
    side_a = np.zeros(move.shape, dtype=bool)
    side_a[kind == VT, 0] = True
    side_a[kind != VT, :2] = True
    return np.where(side_a, move, 0.0).max(axis=1) + np.where(side_a, 0.0, move).max(axis=1)


def distance_toi(kind, idx, x0, x1, floor_frac: float = 0.2, max_iterations: int = 64):
    """Conservative-advancement time to floor_frac of the start gap (ccd.py:221-266)."""
    kind = np.asarray(kind)
    idx = np.asarray(idx)
    m = len(kind)
    toi = np.full(m, np.nan)
    if m == 0:
        return toi
    q0 = x0[idx]
    dq = x1[idx] - q0
    lip = _side_lipschitz(kind, norm3(dq))
    d = _distance_of_points(kind, q0)
    goal = floor_frac * d
    toi[d <= 0.0] = 0.0
    t = np.zeros(m)
    live = np.flatnonzero((d > 0.0) & (lip > 0.0))
    for _ in range(max_iterations):
        if live.size == 0:
            break
        t[live] += (d[live] - goal[live]) / lip[live]
        live = live[t[live] <= 1.0]
        if live.size == 0:
            break
        d[live] = _distance_of_points(kind[live], q0[live] + t[live, None, None] * dq[live])
        reached = d[live] <= goal[live] * (1.0 + 1e-9)
        toi[live[reached]] = t[live[reached]]
        live = live[~reached]
    toi[live] = t[live]
    return toi


# --------------------------------------------------------------- partial.py
TRI_PATTERNS = {                                                  # partial.py:23-36
    1: np.array([[1.0 / 3.0, 1.0 / 3.0]]),
    3: np.array([[1.0 / 6.0, 1.0 / 6.0], [2.0 / 3.0, 1.0 / 6.0], [1.0 / 6.0, 2.0 / 3.0]]),
    6: np.array([[1.0 / 6.0, 1.0 / 6.0], [2.0 / 3.0, 1.0 / 6.0], [1.0 / 6.0, 2.0 / 3.0],
                 [0.5, 0.25], [0.25, 0.5], [1.0 / 3.0, 1.0 / 3.0]]),
}
BOX_PATTERNS = {                                                  # partial.py:37-50
    1: np.array([[0.5, 0.5]]),
    3: np.array([[0.25, 0.25], [0.5, 0.5], [0.75, 0.75]]),
    6: np.array([[0.25, 0.25], [0.5, 0.5], [0.75, 0.75], [0.25, 0.75], [0.75, 0.25], [0.5, 0.25]]),
}


def partial_ccd(kind, idx, x0, x1, count: int = 3):
    """Boolean classifier: any sampled Q(lambda) <= 0 (partial.py:149-204)."""
    kind = np.asarray(kind)
    idx = np.asarray(idx)
    m = len(kind)
    if m == 0:
        return np.zeros(0, dtype=bool)
    tri_pts, box_pts = TRI_PATTERNS[count], BOX_PATTERNS[count]
    width = max(len(tri_pts), len(box_pts))
    lam = np.empty((m, width + 1, 2))
    vt = kind == VT
    lam[vt, :width] = np.resize(tri_pts, (width, 2))
    lam[~vt, :width] = np.resize(box_pts, (width, 2))
    qs, qe = x0[idx], x1[idx]
    if vt.any():
        g = qs[vt]
        lam[vt, -1] = closest_on_triangle(g[:, 0], g[:, 1], g[:, 2], g[:, 3])[1]
    if (~vt).any():
        g = qs[~vt]
        lam[~vt, -1] = closest_between_segments(g[:, 0], g[:, 1], g[:, 2], g[:, 3])[2]
    sel = vt[:, None]

    def affine_basis(q):
        return (np.where(sel, q[:, 1] - q[:, 0], q[:, 2] - q[:, 0]),
                np.where(sel, q[:, 2] - q[:, 1], q[:, 0] - q[:, 1]),
                np.where(sel, q[:, 3] - q[:, 1], q[:, 3] - q[:, 2]))

    be, bs = affine_basis(qe), affine_basis(qs)
    g = [[dot3(be[i], bs[j])[:, None] for j in range(3)] for i in range(3)]
    l1, l2 = lam[:, :, 0], lam[:, :, 1]
    q = (g[0][0] + (g[0][1] + g[1][0]) * l1 + (g[0][2] + g[2][0]) * l2
         + g[1][1] * (l1 * l1) + (g[1][2] + g[2][1]) * (l1 * l2) + g[2][2] * (l2 * l2))
    return (q <= 0.0).any(axis=1)
