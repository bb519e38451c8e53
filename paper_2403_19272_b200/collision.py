"""Collision API surface of the drop-in (mirrors ``clothsim.collision``).

Per-pair narrow-phase stages run on the GPU through the C ABI
(``cs_full_ccd``, ``cs_distance_toi``, ``cs_partial_ccd``, ``cs_pair_witness``);
the numpy-signature wrappers below copy inputs to the device, launch, and copy
results back, so reference callers and tests can be re-pointed unchanged.

Static setup pieces live here too: the reference's patch partition
(``build_patches``, reference bvh.py:20-51 - needed to reproduce the
reference's edge-edge row orientation) and the static world topology the device
broad phase (a per-query hash grid, csrc/broad.cu) enumerates.
"""

from __future__ import annotations

import ctypes
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from . import _lib

VT = 0
EE = 1
LIFE_SPAN_CAP = 64                 # reference pairs.py:21
PATCH_TARGET = 8                   # reference bvh.py:17


# ------------------------------------------------------------------ pair records
@dataclass
class PairSet:
    """Batched pairs + life spans/weights/witness (reference pairs.py:24-62)."""

    kind: np.ndarray
    idx: np.ndarray
    life_span: np.ndarray
    weight: np.ndarray
    bary: np.ndarray = field(default=None)
    distance: np.ndarray = field(default=None)
    normal: np.ndarray = field(default=None)

    @classmethod
    def empty(cls) -> "PairSet":
        return cls(np.zeros(0, np.int8), np.zeros((0, 4), np.int64), np.zeros(0, np.int64), np.zeros(0),
                   np.zeros((0, 2)), np.zeros(0), np.zeros((0, 3)))

    def __len__(self) -> int:
        return len(self.kind)

    def keys(self) -> np.ndarray:
        """Canonical carry-over keys (reference pairs.py:51-62)."""
        c = self.idx.copy()
        vt = self.kind == VT
        ee = self.kind == EE
        c[vt, 1:] = np.sort(c[vt, 1:], axis=1)
        c[ee, :2] = np.sort(c[ee, :2], axis=1)
        c[ee, 2:] = np.sort(c[ee, 2:], axis=1)
        flip = ee & (c[:, 0] > c[:, 2])
        c[flip] = c[flip][:, [2, 3, 0, 1]]
        return np.concatenate([self.kind[:, None].astype(np.int64), c], axis=1)


def ndb_weights(life_span, k: float, base: float) -> np.ndarray:
    """k * base**min(span, 64) (reference pairs.py:65-70); device twin in narrow.cu."""
    if k <= 0 or base <= 1:
        raise ValueError("need k > 0 and base > 1")
    return k * np.power(base, np.minimum(life_span, LIFE_SPAN_CAP).astype(np.float64))


def update_ndb_weights(pairs: PairSet, active, k: float, base: float) -> PairSet:
    """reference pairs.py:73-80."""
    pairs.life_span = np.where(active, np.minimum(pairs.life_span + 1, LIFE_SPAN_CAP), 0)
    pairs.weight = ndb_weights(pairs.life_span, k, base)
    return pairs


# ------------------------------------------------------------------ sample patterns
_TRI = {1: [[1 / 3, 1 / 3]], 3: [[1 / 6, 1 / 6], [2 / 3, 1 / 6], [1 / 6, 2 / 3]],
        6: [[1 / 6, 1 / 6], [2 / 3, 1 / 6], [1 / 6, 2 / 3], [0.5, 0.25], [0.25, 0.5], [1 / 3, 1 / 3]]}
_BOX = {1: [[0.5, 0.5]], 3: [[0.25, 0.25], [0.5, 0.5], [0.75, 0.75]],
        6: [[0.25, 0.25], [0.5, 0.5], [0.75, 0.75], [0.25, 0.75], [0.75, 0.25], [0.5, 0.25]]}


@dataclass
class SampleSet:
    """Partial-CCD sample points (reference partial.py:53-65)."""

    vt_points: np.ndarray
    ee_points: np.ndarray
    interval: float
    includes_projection: bool = True

    @property
    def count(self) -> int:
        return len(self.vt_points)


def _covering(points: np.ndarray, tri: bool, grid: int = 64) -> float:
    g = np.linspace(0.0, 1.0, grid)
    gx, gy = np.meshgrid(g, g)
    probe = np.stack([gx.ravel(), gy.ravel()], axis=1)
    if tri:
        probe = probe[probe.sum(axis=1) <= 1.0]
    return float(np.linalg.norm(probe[:, None, :] - points[None], axis=2).min(axis=1).max())


def default_samples(count: int = 3) -> SampleSet:
    """Built-in patterns (reference partial.py:79-85)."""
    if count not in _TRI:
        raise ValueError(f"no built-in pattern with {count} samples (choose 1, 3 or 6)")
    vt = np.asarray(_TRI[count], dtype=np.float64)
    ee = np.asarray(_BOX[count], dtype=np.float64)
    return SampleSet(vt, ee, max(_covering(vt, True), _covering(ee, False)))


def sample_bound(h0: float, h1: float, edge_bound: float, alpha: float) -> float:
    """Eq. 14 sampling interval (reference partial.py:105-114)."""
    if not (h0 > 0 and h1 >= h0 and edge_bound > 0 and 0 < alpha < 1):
        raise ValueError("need h0 > 0, h1 >= h0, edge_bound > 0, 0 < alpha < 1")
    return (1.0 / alpha - 1.0) * h0 * h0 / (2.0 * np.sqrt(2.0) * edge_bound * (h1 + 2.0 * edge_bound))


# ------------------------------------------------------------------ GPU per-stage wrappers
def _dev(a, dtype):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def _pair_inputs(kind, idx, *xs):
    import torch

    k = _dev(np.asarray(kind, dtype=np.int8), torch.int8)
    i = _dev(np.asarray(idx, dtype=np.int32).reshape(-1, 4), torch.int32)
    return k, i, [_dev(np.asarray(x, dtype=np.float64), torch.float64) for x in xs]


def full_ccd(kind, idx, x_start, x_end, tol: float = 1e-6) -> np.ndarray:
    """GPU twin of reference full_ccd (ccd.py:138-196): TOI per pair, nan = miss."""
    import torch

    lib = _lib.load()
    m = len(kind)
    if m == 0:
        return np.full(0, np.nan)
    k, i, (a, b) = _pair_inputs(kind, idx, x_start, x_end)
    out = torch.empty(m, dtype=torch.float64, device="cuda")
    _lib.check(lib.cs_full_ccd(k.data_ptr(), i.data_ptr(), a.data_ptr(), b.data_ptr(), m, tol, out.data_ptr(),
                               _lib.stream_handle()), "cs_full_ccd")
    return out.cpu().numpy()


def distance_toi(kind, idx, x_start, x_end, floor_frac: float = 0.2, max_iterations: int = 64) -> np.ndarray:
    """GPU twin of reference distance_toi (ccd.py:221-266)."""
    import torch

    lib = _lib.load()
    m = len(kind)
    if m == 0:
        return np.full(0, np.nan)
    k, i, (a, b) = _pair_inputs(kind, idx, x_start, x_end)
    out = torch.empty(m, dtype=torch.float64, device="cuda")
    _lib.check(lib.cs_distance_toi(k.data_ptr(), i.data_ptr(), a.data_ptr(), b.data_ptr(), m, floor_frac,
                                   max_iterations, out.data_ptr(), _lib.stream_handle()), "cs_distance_toi")
    return out.cpu().numpy()


def global_toi(kind, idx, x_start, x_end, alpha: float = 0.8) -> float:
    """Step scale from the minimum impact time (reference ccd.py:269-285)."""
    toi = full_ccd(kind, idx, x_start, x_end)
    hits = toi[~np.isnan(toi)]
    if hits.size == 0:
        return 1.0
    t = float(hits.min())
    if t <= 0.0:
        raise RuntimeError(f"nonpositive impact time {t}: start state was not collision-free "
                           f"(pair {int(np.nanargmin(toi))})")
    return alpha * t


def partial_ccd(kind, idx, x_start, x_end, samples: SampleSet) -> np.ndarray:
    """GPU twin of reference partial_ccd (partial.py:149-204)."""
    import torch

    lib = _lib.load()
    m = len(kind)
    if m == 0:
        return np.zeros(0, dtype=bool)
    k, i, (a, b) = _pair_inputs(kind, idx, x_start, x_end)
    out = torch.empty(m, dtype=torch.uint8, device="cuda")
    _lib.check(lib.cs_partial_ccd(k.data_ptr(), i.data_ptr(), a.data_ptr(), b.data_ptr(), m, samples.count,
                                  out.data_ptr(), _lib.stream_handle()), "cs_partial_ccd")
    return out.cpu().numpy().astype(bool)


def pair_witness(kind, idx, x):
    """GPU twin of reference pair_witness (geometry.py:115-148): (p1, p2, bary, dist)."""
    import torch

    lib = _lib.load()
    m = len(kind)
    if m == 0:
        z = np.zeros((0, 3))
        return z, z.copy(), np.zeros((0, 2)), np.zeros(0)
    k, i, (xx,) = _pair_inputs(kind, idx, x)
    p1 = torch.empty((m, 3), dtype=torch.float64, device="cuda")
    p2 = torch.empty_like(p1)
    bary = torch.empty((m, 2), dtype=torch.float64, device="cuda")
    dist = torch.empty(m, dtype=torch.float64, device="cuda")
    _lib.check(lib.cs_pair_witness(k.data_ptr(), i.data_ptr(), xx.data_ptr(), m, p1.data_ptr(), p2.data_ptr(),
                                   bary.data_ptr(), dist.data_ptr(), None, _lib.stream_handle()), "cs_pair_witness")
    return p1.cpu().numpy(), p2.cpu().numpy(), bary.cpu().numpy(), dist.cpu().numpy()


def witness_normals(kind, idx, x):
    """bary, distance and separating normal as Simulation._witness sets them (stepper.py:194-216)."""
    import torch

    lib = _lib.load()
    m = len(kind)
    if m == 0:
        return np.zeros((0, 2)), np.zeros(0), np.zeros((0, 3))
    k, i, (xx,) = _pair_inputs(kind, idx, x)
    bary = torch.empty((m, 2), dtype=torch.float64, device="cuda")
    dist = torch.empty(m, dtype=torch.float64, device="cuda")
    nrm = torch.empty((m, 3), dtype=torch.float64, device="cuda")
    _lib.check(lib.cs_pair_witness(k.data_ptr(), i.data_ptr(), xx.data_ptr(), m, None, None, bary.data_ptr(),
                                   dist.data_ptr(), nrm.data_ptr(), _lib.stream_handle()), "cs_pair_witness")
    return bary.cpu().numpy(), dist.cpu().numpy(), nrm.cpu().numpy()


# ------------------------------------------------------------------ static world topology
def build_patches(triangles: np.ndarray, n_vertices: int = 0) -> list:
    """Greedy BFS grouping of edge-connected triangles into patches of <= 8.

    Same partition as reference bvh.py:20-51 (its order decides which edge of
    an edge-edge pair the reference lists first).
    """
    tris = np.asarray(triangles, dtype=np.int64)
    m = len(tris)
    pending: dict = {}
    adj = [[] for _ in range(m)]
    for t, (a, b, c) in enumerate(tris.tolist()):
        for u, w in ((a, b), (b, c), (c, a)):
            key = (u, w) if u < w else (w, u)
            o = pending.pop(key, None)
            if o is None:
                pending[key] = t
            else:
                adj[t].append(o)
                adj[o].append(t)
    owner = [-1] * m
    groups = []
    for seed in range(m):
        if owner[seed] >= 0:
            continue
        pid = len(groups)
        grp = [seed]
        owner[seed] = pid
        q = deque([seed])
        while q and len(grp) < PATCH_TARGET:
            t = q.popleft()
            for u in adj[t]:
                if owner[u] < 0 and len(grp) < PATCH_TARGET:
                    owner[u] = pid
                    grp.append(u)
                    q.append(u)
        groups.append(np.asarray(grp, dtype=np.int64))
    return groups


@dataclass
class CollisionWorld:
    """Static world topology (cloth first, then obstacles) for the device broad phase.

    Plays the role of the reference's PatchBVH (bvh.py:54-137): fixed topology
    from the rest pose (``rest_positions`` kept for signature parity); the
    device rebuilds its hash grid from the query boxes every call.  ``triangles``/``tri_static``
    keep the reference attribute names.
    """

    triangles: np.ndarray
    tri_static: np.ndarray
    edges: np.ndarray
    tri_edges: np.ndarray
    patches: list
    patch_of_tri: np.ndarray
    slot_of_tri: np.ndarray
    edge_tris: np.ndarray
    edge_slot: np.ndarray
    vert_static: np.ndarray
    vert_used: np.ndarray
    edge_static: np.ndarray
    n_world: int = 0

    @classmethod
    def build(cls, triangles, rest_positions, tri_static=None) -> "CollisionWorld":
        tris = np.asarray(triangles, dtype=np.int64)
        m = len(tris)
        nw = len(rest_positions)
        stat = np.zeros(m, bool) if tri_static is None else np.asarray(tri_static, dtype=bool)
        stack = np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]])
        stack.sort(axis=1)
        edges, inv = np.unique(stack, axis=0, return_inverse=True)
        inv = inv.reshape(-1)
        tri_edges = inv.reshape(3, m).T.copy()
        owner = np.tile(np.arange(m), 3)
        slot = np.repeat(np.arange(3), m)
        order = np.argsort(inv, kind="stable")
        cnt = np.bincount(inv, minlength=len(edges))
        start = np.concatenate([[0], np.cumsum(cnt)[:-1]])
        edge_tris = np.full((len(edges), 2), -1, np.int64)
        edge_slot = np.zeros((len(edges), 2), np.int64)
        edge_tris[:, 0] = owner[order[start]]
        edge_slot[:, 0] = slot[order[start]]
        two = cnt >= 2
        edge_tris[two, 1] = owner[order[start[two] + 1]]
        edge_slot[two, 1] = slot[order[start[two] + 1]]
        patches = build_patches(tris, nw)
        patch_of = np.zeros(m, np.int64)
        slot_of = np.zeros(m, np.int64)
        for p, g in enumerate(patches):
            patch_of[g] = p
            slot_of[g] = np.arange(len(g))
        used = np.zeros(nw, bool)
        used[tris.ravel()] = True
        vstat = np.ones(nw, bool)
        vstat[tris[~stat].ravel()] = False
        estat = np.zeros(len(edges), bool)
        estat[tri_edges[stat].ravel()] = True
        return cls(tris, stat, edges, tri_edges, patches, patch_of, slot_of, edge_tris, edge_slot, vstat, used,
                   estat, nw)


# ------------------------------------------------------------------ module-level drop-ins
# (reference collision/__init__.py:1-5): same names and signatures; the per-pair
# arithmetic runs in the device kernels of csrc/stages.cu / narrow.cu / broad.cu.

def coplanarity_coefficients(kind, idx, x_start, x_end) -> np.ndarray:
    """Monomial coefficients (m,4), lowest order first, of the coplanarity cubic (ccd.py:36-44)."""
    import torch

    lib = _lib.load()
    m = len(kind)
    if m == 0:
        return np.zeros((0, 4))
    k, i, (a, b) = _pair_inputs(kind, idx, x_start, x_end)
    out = torch.empty((m, 4), dtype=torch.float64, device="cuda")
    _lib.check(lib.cs_coplanarity_coefficients(k.data_ptr(), i.data_ptr(), a.data_ptr(), b.data_ptr(), m,
                                               out.data_ptr(), _lib.stream_handle()), "cs_coplanarity_coefficients")
    return out.cpu().numpy()


def query_q(kind, idx, x_start, x_end, lam) -> np.ndarray:
    """Dot product of the pair offset at interval end and start, per sample
    (partial.py:133-146); lam (m,k,2) or (k,2) shared across pairs -> (m,k)."""
    import torch

    lib = _lib.load()
    lam = np.asarray(lam, dtype=np.float64)
    m = len(kind)
    shared = lam.ndim == 2
    kk = lam.shape[-2]
    if m == 0 or kk == 0:
        return np.zeros((m, kk))
    k, i, (a, b) = _pair_inputs(kind, idx, x_start, x_end)
    ld = _dev(lam, torch.float64)
    out = torch.empty((m, kk), dtype=torch.float64, device="cuda")
    _lib.check(lib.cs_query_q(k.data_ptr(), i.data_ptr(), a.data_ptr(), b.data_ptr(), m, ld.data_ptr(), kk,
                              int(shared), out.data_ptr(), _lib.stream_handle()), "cs_query_q")
    return out.cpu().numpy()


def swept_boxes(points_start: np.ndarray, points_end: np.ndarray, margin: float):
    """(lo, hi) over both ends of each point group, -/+ margin (bvh.py:140-143)."""
    import torch

    lib = _lib.load()
    ps = np.asarray(points_start, dtype=np.float64)
    pe = np.asarray(points_end, dtype=np.float64)
    m, kk = ps.shape[0], ps.shape[1]
    if m == 0:
        return np.zeros((0, 3)), np.zeros((0, 3))
    a, b = _dev(ps, torch.float64), _dev(pe, torch.float64)
    lo = torch.empty((m, 3), dtype=torch.float64, device="cuda")
    hi = torch.empty_like(lo)
    _lib.check(lib.cs_swept_boxes(a.data_ptr(), b.data_ptr(), m, kk, float(margin), lo.data_ptr(), hi.data_ptr(),
                                  _lib.stream_handle()), "cs_swept_boxes")
    return lo.cpu().numpy(), hi.cpu().numpy()


def _dbb(d, d_hat, kappa, gradient):
    import torch

    lib = _lib.load()
    arr = np.asarray(d, dtype=np.float64)
    flat = arr.reshape(-1)
    out = torch.empty(max(flat.size, 1), dtype=torch.float64, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    dd = _dev(flat if flat.size else np.zeros(1), torch.float64)
    rc = lib.cs_dbb_weight(dd.data_ptr(), flat.size, float(d_hat), float(kappa), int(gradient), out.data_ptr(),
                           flag.data_ptr(), _lib.stream_handle())
    if rc == _lib.CS_NONFINITE:
        raise FloatingPointError("nonpositive pair distance: infeasible state")
    _lib.check(rc, "cs_dbb_weight")
    res = out[:flat.size].cpu().numpy().reshape(arr.shape)
    return res if res.ndim else float(res)


def dbb_weight(d, d_hat: float, kappa: float):
    """Log barrier -kappa (d - d_hat)^2 ln(d / d_hat), zero beyond d_hat (pairs.py:83-98)."""
    if d_hat <= 0 or kappa <= 0:
        raise ValueError("need d_hat > 0 and kappa > 0")
    return _dbb(d, d_hat, kappa, False)


def dbb_weight_gradient(d, d_hat: float, kappa: float):
    """d/dd of dbb_weight, zero at and beyond d_hat (pairs.py:101-108)."""
    return _dbb(d, d_hat, kappa, True)


def _closest(kind_value, *pts):
    m = len(np.atleast_2d(pts[0]))
    x = np.concatenate([np.atleast_2d(np.asarray(p, dtype=np.float64)) for p in pts])
    idx = (np.arange(m)[:, None] + m * np.arange(4)[None, :]).astype(np.int64)
    return pair_witness(np.full(m, kind_value, np.int8), idx, x)


def point_triangle_closest(p, t0, t1, t2):
    """Closest point on each triangle to each point (geometry.py:10-79):
    (closest (m,3), bary (m,2), distance (m,))."""
    _, closest, bary, dist = _closest(VT, p, t0, t1, t2)
    return closest, bary, dist


def segment_segment_closest(a0, a1, b0, b1):
    """Closest points between segments (geometry.py:82-112): (pa, pb, params (m,2), distance)."""
    return _closest(EE, a0, a1, b0, b1)


def lattice_samples(interval: float, domain: str) -> np.ndarray:
    """Square lattice over the parameter domain with covering radius <= interval
    (partial.py:88-102); a sample-pattern generator (setup), not per-pair work."""
    if interval <= 0:
        raise ValueError("sample interval must be positive")
    spacing = interval * np.sqrt(2.0)
    k = max(int(np.ceil(1.0 / spacing)), 1)
    u = (np.arange(k) + 0.5) / k
    gx, gy = np.meshgrid(u, u)
    pts = np.stack([gx.ravel(), gy.ravel()], axis=1)
    if domain == "triangle":
        over = pts.sum(axis=1) > 1.0
        pts[over] = 1.0 - pts[over][:, ::-1]
        pts = np.unique(pts, axis=0)
    return pts


PatchBVH = CollisionWorld   # the reference's static-topology structure (bvh.py:54-137)


def broad_phase(x_start: np.ndarray, x_end: np.ndarray, bvh: CollisionWorld, margin: float) -> PairSet:
    """Candidate VT / EE pairs whose margin-inflated swept boxes overlap (bvh.py:207-292):
    exactly the reference's set (row order is the device's, deterministic), on the
    device hash grid of a world context for this topology."""
    import torch

    from . import context

    ctx = context.get(world=bvh)
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")  # noqa: E731
    a, b = dev(x_start), dev(x_end)
    count = ctypes.c_longlong(0)
    _lib.check(ctx.lib.cs_broad_phase(ctx.ptr, a.data_ptr(), b.data_ptr(), float(margin), ctypes.byref(count),
                                      _lib.stream_handle()), "cs_broad_phase")
    P = count.value
    kind = torch.empty(max(P, 1), dtype=torch.int8, device="cuda")
    idx = torch.empty((max(P, 1), 4), dtype=torch.int32, device="cuda")
    _lib.check(ctx.lib.cs_scene_pairs(ctx.ptr, kind.data_ptr(), idx.data_ptr(), _lib.stream_handle()),
               "cs_scene_pairs")
    return PairSet(kind=kind[:P].cpu().numpy(), idx=idx[:P].cpu().numpy().astype(np.int64),
                   life_span=np.zeros(P, np.int64), weight=np.zeros(P))
