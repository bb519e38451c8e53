"""ORACLE (test infrastructure only): broad-phase candidate set.

Restates what reference ``broad_phase`` (pkg/src/clothsim/collision/bvh.py:207-292)
returns, derived from its code rather than its tree walk:

* the SET: every vertex-triangle pair (v, f) with v not in f whose
  margin-inflated swept boxes overlap, and every vertex-disjoint edge pair
  whose swept boxes overlap, minus pairs whose primitives are both on static
  (obstacle) triangles (bvh.py:236, 253-281).  Swept boxes are fp64 min/max
  of start/end positions -/+ margin (bvh.py:140-143, 242-246).  Found here by a
  uniform-grid hash join with exact box tests.
* the ROW ORDER and edge-edge ORIENTATION: each row sits at the first position
  the reference's concatenated candidate list produces it (bvh.py:283-286).
  That position is a pure function of the static patch partition
  (build_patches, bvh.py:20-51, restated below): block (VT a->b, VT b->a, EE),
  then the triangle pair's place (cross-patch pairs (P<Q, slot i, slot j)
  before same-patch pairs (P, i<j), bvh.py:221-232), then the sub-slot (vertex
  of the triangle, or 3x3 edge slot).  Row order only changes rounding in the
  reference's np.add.at accumulations; it is reproduced so oracle trajectories
  are bit-identical to the reference's.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass

import numpy as np

VT, EE = 0, 1
PATCH_LIMIT = 8                                   # bvh.py:17


def patch_partition(triangles: np.ndarray):
    """Greedy BFS patches of <= 8 edge-connected triangles (bvh.py:20-51).

    Returns (patch_of_tri, slot_of_tri).
    """
    m = len(triangles)
    open_edge: dict = {}
    nbrs = [[] for _ in range(m)]
    for t in range(m):
        a, b, c = (int(z) for z in triangles[t])
        for u, w in ((a, b), (b, c), (c, a)):
            key = (u, w) if u < w else (w, u)
            other = open_edge.pop(key, None)
            if other is None:
                open_edge[key] = t
            else:
                nbrs[t].append(other)
                nbrs[other].append(t)
    patch = np.full(m, -1, dtype=np.int64)
    slot = np.zeros(m, dtype=np.int64)
    count = 0
    for seed in range(m):
        if patch[seed] >= 0:
            continue
        members = 1
        patch[seed] = count
        frontier = deque([seed])
        while frontier and members < PATCH_LIMIT:
            t = frontier.popleft()
            for u in nbrs[t]:
                if patch[u] < 0 and members < PATCH_LIMIT:
                    patch[u] = count
                    slot[u] = members
                    members += 1
                    frontier.append(u)
        count += 1
    return patch, slot


@dataclass
class WorldTopology:
    triangles: np.ndarray      # (m,3) world triangles (cloth first, then obstacles)
    tri_static: np.ndarray     # (m,) obstacle triangle
    edges: np.ndarray          # (E,2) sorted unique world edges
    tri_edges: np.ndarray      # (m,3) edge ids in slot order (v0v1, v1v2, v2v0)
    patch: np.ndarray
    slot: np.ndarray

    @classmethod
    def build(cls, triangles, tri_static):
        tris = np.asarray(triangles, dtype=np.int64)
        m = len(tris)
        stack = np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]])
        stack.sort(axis=1)
        edges, inv = np.unique(stack, axis=0, return_inverse=True)
        patch, slot = patch_partition(tris)
        return cls(tris, np.asarray(tri_static, dtype=bool), edges,
                   inv.reshape(-1).reshape(3, m).T.copy(), patch, slot)


def _cell_entries(lo, hi, origin, h, dims):
    """(owner, cell key) for every grid cell a box touches."""
    c0 = np.floor((lo - origin) / h).astype(np.int64)
    c1 = np.floor((hi - origin) / h).astype(np.int64)
    span = c1 - c0 + 1
    cnt = span.prod(axis=1)
    owner = np.repeat(np.arange(len(lo)), cnt)
    local = np.arange(int(cnt.sum())) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    sx, sy = span[owner, 0], span[owner, 1]
    cx = c0[owner, 0] + local % sx
    cy = c0[owner, 1] + (local // sx) % sy
    cz = c0[owner, 2] + local // (sx * sy)
    return owner, (cx * dims[1] + cy) * dims[2] + cz


def _box_pairs(lo_a, hi_a, lo_b, hi_b):
    """All (i, j) with closed boxes overlapping: uniform-grid hash join + exact fp64 test.

    Two boxes that overlap share at least one grid cell (cells are closed on
    the low side, and floor() is monotone), so the join is a superset and the
    exact test below makes it the exact set.
    """
    if len(lo_a) == 0 or len(lo_b) == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    ext = np.concatenate([hi_a - lo_a, hi_b - lo_b])
    h = max(float(np.percentile(ext.max(axis=1), 90)), 1e-12)
    origin = np.minimum(lo_a.min(axis=0), lo_b.min(axis=0)) - h
    top = np.maximum(hi_a.max(axis=0), hi_b.max(axis=0))
    dims = (np.floor((top - origin) / h).astype(np.int64) + 2)
    oa, ka = _cell_entries(lo_a, hi_a, origin, h, dims)
    ob, kb = _cell_entries(lo_b, hi_b, origin, h, dims)
    order = np.argsort(kb, kind="stable")
    kb, ob = kb[order], ob[order]
    left = np.searchsorted(kb, ka, side="left")
    right = np.searchsorted(kb, ka, side="right")
    cnt = right - left
    ia = np.repeat(oa, cnt)
    pos = np.arange(int(cnt.sum())) - np.repeat(np.cumsum(cnt) - cnt, cnt) + np.repeat(left, cnt)
    ib = ob[pos]
    hit = ((lo_a[ia] <= hi_b[ib]) & (lo_b[ib] <= hi_a[ia])).all(axis=1)
    code = np.unique(ia[hit] * np.int64(len(lo_b)) + ib[hit])
    return code // len(lo_b), code % len(lo_b)


def _pair_place(pa, sa, pb, sb):
    """Canonical triangle-pair position key and whether 'a' comes first."""
    a_first = (pa < pb) | ((pa == pb) & (sa < sb))
    p1 = np.where(a_first, pa, pb)
    p2 = np.where(a_first, pb, pa)
    s1 = np.where(a_first, sa, sb)
    s2 = np.where(a_first, sb, sa)
    same = (pa == pb).astype(np.int64)
    place = (((same << 24 | p1) << 24 | p2) << 3 | s1) << 3 | s2
    return place, a_first


def _row_key(block, place, sub, flip):
    """Position of a row in the reference's concatenated list:
    block (VT a->b = 0, VT b->a = 1, EE = 2) | pair place (55 bits) | sub-slot | EE flip."""
    return (np.int64(block) << 60) | (place << 5) | (np.asarray(sub, np.int64) << 1) | np.asarray(flip, np.int64)


def _first_key(owner, keys, n_rows):
    """Minimum candidate key per row (owner sorted ascending)."""
    out = np.full(n_rows, np.iinfo(np.int64).max, dtype=np.int64)
    np.minimum.at(out, owner, keys)
    return out


def broad_phase(x0, x1, topo: WorldTopology, margin: float):
    """Reference-identical candidate pairs: (kind (P,) int8, idx (P,4) int64)."""
    tris, edges = topo.triangles, topo.edges
    if len(topo.patch) and topo.patch.max() >= (1 << 24):
        raise ValueError("oracle broad phase supports < 2^24 patches")
    v_lo = np.minimum(x0, x1) - margin
    v_hi = np.maximum(x0, x1) + margin
    t_lo, t_hi = v_lo[tris].min(axis=1), v_hi[tris].max(axis=1)
    e_lo, e_hi = v_lo[edges].min(axis=1), v_hi[edges].max(axis=1)

    n_w = len(x0)
    used = np.zeros(n_w, dtype=bool)
    used[tris.ravel()] = True
    v_static = np.ones(n_w, dtype=bool)
    v_static[tris[~topo.tri_static].ravel()] = False
    e_static = np.zeros(len(edges), dtype=bool)
    e_static[topo.tri_edges[topo.tri_static].ravel()] = True

    # ---- vertex-triangle set
    vid = np.flatnonzero(used)
    i, f = _box_pairs(v_lo[vid], v_hi[vid], t_lo, t_hi)
    v = vid[i]
    keep = (tris[f] != v[:, None]).all(axis=1) & ~(v_static[v] & topo.tri_static[f])
    v, f = v[keep], f[keep]

    # candidate triangles t containing v: expand rows over the vertex's triangles
    flat_t = np.repeat(np.arange(len(tris)), 3)
    flat_v = tris.ravel()
    flat_k = np.tile(np.arange(3), len(tris))
    ordv = np.argsort(flat_v, kind="stable")
    deg = np.bincount(flat_v, minlength=n_w)
    start = np.concatenate([[0], np.cumsum(deg)[:-1]])
    rows = np.repeat(np.arange(len(v)), deg[v])
    offs = np.arange(len(rows)) - np.repeat(np.cumsum(deg[v]) - deg[v], deg[v])
    pick = ordv[start[v[rows]] + offs]
    ct, ck = flat_t[pick], flat_k[pick]
    cf = f[rows]
    ok = ~(topo.tri_static[ct] & topo.tri_static[cf])
    rows, ct, ck, cf = rows[ok], ct[ok], ck[ok], cf[ok]
    place, t_first = _pair_place(topo.patch[ct], topo.slot[ct], topo.patch[cf], topo.slot[cf])
    block = np.where(t_first, 0, 1).astype(np.int64)
    vt_key = _first_key(rows, _row_key(block, place, ck, 0), len(v))

    # ---- edge-edge set
    ia, ib = _box_pairs(e_lo, e_hi, e_lo, e_hi)
    keep = ia < ib
    ia, ib = ia[keep], ib[keep]
    ea, eb = edges[ia], edges[ib]
    disjoint = ~((ea[:, 0:1] == eb).any(axis=1) | (ea[:, 1:2] == eb).any(axis=1))
    keep = disjoint & ~(e_static[ia] & e_static[ib])
    ia, ib = ia[keep], ib[keep]
    # triangles owning each edge, with the edge's slot inside them
    flat_e = topo.tri_edges.ravel()
    flat_te = np.repeat(np.arange(len(tris)), 3)
    flat_se = np.tile(np.arange(3), len(tris))
    orde = np.argsort(flat_e, kind="stable")
    edeg = np.bincount(flat_e, minlength=len(edges))
    estart = np.concatenate([[0], np.cumsum(edeg)[:-1]])
    cand_rows, cand_keys = [], []
    for ka in range(2):
        for kb in range(2):
            ra = np.flatnonzero((edeg[ia] > ka) & (edeg[ib] > kb))
            ta = flat_te[orde[estart[ia[ra]] + ka]]
            sa = flat_se[orde[estart[ia[ra]] + ka]]
            tb = flat_te[orde[estart[ib[ra]] + kb]]
            sb = flat_se[orde[estart[ib[ra]] + kb]]
            good = ~(topo.tri_static[ta] & topo.tri_static[tb])
            ra, ta, sa, tb, sb = ra[good], ta[good], sa[good], tb[good], sb[good]
            place, a_first = _pair_place(topo.patch[ta], topo.slot[ta], topo.patch[tb], topo.slot[tb])
            sub = np.where(a_first, sa * 3 + sb, sb * 3 + sa)
            flip = (~a_first).astype(np.int64)
            cand_rows.append(ra)
            cand_keys.append(_row_key(2, place, sub, flip))
    ee_key = _first_key(np.concatenate(cand_rows), np.concatenate(cand_keys), len(ia))

    ee_flip = (ee_key & 1).astype(bool)
    first_e = np.where(ee_flip, ib, ia)
    second_e = np.where(ee_flip, ia, ib)

    kind = np.concatenate([np.full(len(v), VT, np.int8), np.full(len(ia), EE, np.int8)])
    idx = np.concatenate([
        np.concatenate([v[:, None], tris[f]], axis=1),
        np.concatenate([edges[first_e], edges[second_e]], axis=1),
    ]).astype(np.int64)
    order = np.argsort(np.concatenate([vt_key, ee_key]), kind="stable")
    return kind[order], idx[order]
