"""Validation oracles (reference oracles.py): the penetration-free invariant.

``tri_tri_intersect`` and ``oracle_intersect`` run the device 17-axis separating-
axis test (csrc/intersect.cu, numpy's evaluation order); ``tri_tri_intersect_exact``
is the reference's rational-arithmetic check of one pair (Fractions on the host -
exact arithmetic is the point of it; nothing on the step path calls it).
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

from . import _lib


def tri_tri_intersect(p: np.ndarray, q: np.ndarray) -> np.ndarray:
    """Boolean per pair: closed triangles p, q (m,3,3) intersect (oracles.py:33-48)."""
    import torch

    lib = _lib.load()
    p = np.asarray(p, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    if p.ndim == 2:
        p, q = p[None], q[None]
    m = len(p)
    if m == 0:
        return np.zeros(0, dtype=bool)
    pd = torch.as_tensor(np.ascontiguousarray(p), device="cuda")
    qd = torch.as_tensor(np.ascontiguousarray(q), device="cuda")
    out = torch.empty(m, dtype=torch.uint8, device="cuda")
    _lib.check(lib.cs_tri_tri_intersect(pd.data_ptr(), qd.data_ptr(), m, out.data_ptr(), _lib.stream_handle()),
               "cs_tri_tri_intersect")
    return out.cpu().numpy().astype(bool)


def tri_tri_intersect_exact(p, q) -> bool:
    """Rational-arithmetic separating-axis test for one pair (oracles.py:51-80)."""
    P = [[Fraction(float(c)) for c in v] for v in p]
    Q = [[Fraction(float(c)) for c in v] for v in q]

    def sub(a, b):
        return [a[0] - b[0], a[1] - b[1], a[2] - b[2]]

    def cross(a, b):
        return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]

    def dot(a, b):
        return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]

    ep = [sub(P[1], P[0]), sub(P[2], P[1]), sub(P[0], P[2])]
    eq = [sub(Q[1], Q[0]), sub(Q[2], Q[1]), sub(Q[0], Q[2])]
    n_p, n_q = cross(ep[0], ep[1]), cross(eq[0], eq[1])
    axes = [n_p, n_q] + [cross(a, b) for a in ep for b in eq]
    axes += [cross(n_p, e) for e in ep] + [cross(n_q, e) for e in eq]
    for ax in axes:
        if ax[0] == 0 and ax[1] == 0 and ax[2] == 0:
            continue
        dp = [dot(ax, v) for v in P]
        dq = [dot(ax, v) for v in Q]
        if max(dp) < min(dq) or max(dq) < min(dp):
            return False
    return True


def oracle_intersect(x: np.ndarray, triangles: np.ndarray, chunk: int = 512) -> np.ndarray:
    """All intersecting non-adjacent triangle pairs at positions x as sorted (k,2) rows
    (oracles.py:83-131), from the device hash-grid + SAT check over this topology."""
    import ctypes

    import torch

    from . import context
    from .collision import CollisionWorld

    x = np.asarray(x, dtype=np.float64)
    tris = np.asarray(triangles, dtype=np.int64)
    if len(tris) == 0:
        return np.zeros((0, 2), dtype=np.int64)
    world = _worlds.get((id(triangles), len(x)))
    if world is None or world[0] is not triangles:
        world = (triangles, CollisionWorld.build(tris, x))
        _worlds[(id(triangles), len(x))] = world
    ctx = context.get(world=world[1])
    xd = torch.as_tensor(np.ascontiguousarray(x), device="cuda")
    cap = 4096
    while True:
        count = ctypes.c_longlong(0)
        pairs = np.zeros((cap, 2), np.int32)
        _lib.check(ctx.lib.cs_intersections(ctx.ptr, xd.data_ptr(), ctypes.byref(count), pairs.ctypes.data, cap,
                                            _lib.stream_handle()), "cs_intersections")
        if count.value <= cap:
            out = pairs[:count.value].astype(np.int64)
            return out[np.lexsort((out[:, 1], out[:, 0]))]
        cap = int(count.value)


_worlds: dict = {}
