"""Scene generators: the reference's built-ins plus the BASELINE configs.

``grid_cloth``, ``strip_cloth``, ``icosphere``, ``box_mesh`` and
``build_scene`` produce the same arrays as reference
``pkg/src/clothsim/scenes.py:16-207`` (pinned by tests/test_setup_parity.py).
New generators for the BASELINE.json configs (none exist in the reference):

  config 1  "two_corner"     64x64 grid pinned at two corners, no obstacles
  config 2  "sphere_ground"  128x128 grid over an icosphere + ground box
  config 3  "stacked_twist"  S stacked 256x256 sheets on twist rails
  config 4  "skirt"          ~340K-vertex tube skirt on an animated cylinder body
  config 5  drape_batch()    independent 100K-vertex sphere drapes, varied materials
"""

from __future__ import annotations

import numpy as np

from .mesh import build_mesh
from .stepconfig import StepConfig


def grid_cloth(resolution: int, size: float = 1.0, height: float = 0.0):
    """Square grid in the xy plane; vertex i*res+j at (t_i, t_j, height) (reference scenes.py:16-34)."""
    if resolution < 2:
        raise ValueError("resolution must be at least 2")
    t = np.linspace(0.0, size, resolution)
    gx, gy = np.meshgrid(t, t, indexing="ij")
    verts = np.stack([gx.ravel(), gy.ravel(), np.full(resolution * resolution, float(height))], axis=1)
    i, j = np.meshgrid(np.arange(resolution - 1), np.arange(resolution - 1), indexing="ij")
    a = (i * resolution + j).ravel()
    b, c = a + 1, a + resolution
    d = c + 1
    even = ((i + j) % 2 == 0).ravel()
    first = np.where(even[:, None], np.stack([a, b, c], 1), np.stack([a, b, d], 1))
    second = np.where(even[:, None], np.stack([b, d, c], 1), np.stack([a, d, c], 1))
    tris = np.stack([first, second], axis=1).reshape(-1, 3)
    return verts, tris.astype(np.int64)


def strip_cloth(length_segments: int, width_segments: int, length: float, width: float):
    """Strip along +x (reference scenes.py:37-52)."""
    xs = np.linspace(0.0, length, length_segments + 1)
    ys = np.linspace(0.0, width, width_segments + 1)
    gx, gy = np.meshgrid(xs, ys, indexing="ij")
    verts = np.stack([gx.ravel(), gy.ravel(), np.zeros(gx.size)], axis=1)
    cols = width_segments + 1
    i, j = np.meshgrid(np.arange(length_segments), np.arange(width_segments), indexing="ij")
    a = (i * cols + j).ravel()
    b, c = a + 1, a + cols
    d = c + 1
    tris = np.stack([np.stack([a, c, b], 1), np.stack([b, c, d], 1)], axis=1).reshape(-1, 3)
    return verts, tris.astype(np.int64)


_ICO_FACES = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
              (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5), (2, 4, 11),
              (6, 2, 10), (8, 6, 7), (9, 8, 1)]


def icosphere(subdivisions: int = 2, radius: float = 1.0, center=(0.0, 0.0, 0.0)):
    """Geodesic sphere by 4-way subdivision (reference scenes.py:55-88; same vertex order)."""
    phi = (1.0 + np.sqrt(5.0)) / 2.0
    base = np.array([[-1, phi, 0], [1, phi, 0], [-1, -phi, 0], [1, -phi, 0], [0, -1, phi], [0, 1, phi],
                     [0, -1, -phi], [0, 1, -phi], [phi, 0, -1], [phi, 0, 1], [-phi, 0, -1], [-phi, 0, 1]],
                    dtype=np.float64)
    base /= np.linalg.norm(base, axis=1)[:, None]
    pts = list(base)
    faces = list(_ICO_FACES)
    for _ in range(subdivisions):
        memo: dict = {}

        def mid(u, w):
            key = (u, w) if u < w else (w, u)
            got = memo.get(key)
            if got is None:
                s = pts[u] + pts[w]
                pts.append(s / np.linalg.norm(s))
                got = memo[key] = len(pts) - 1
            return got

        refined = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            refined.extend([(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)])
        faces = refined
    return np.asarray(pts) * radius + np.asarray(center), np.asarray(faces, dtype=np.int64)


def box_mesh(center=(0.0, 0.0, 0.0), extents=(1.0, 1.0, 1.0), divisions: int = 4):
    """Axis-aligned box, divisions^2 quads per face, welded (reference scenes.py:91-133)."""
    hx, hy, hz = (e / 2.0 for e in extents)
    o = np.array(center, dtype=np.float64)
    corner = o - np.array([hx, hy, hz])
    ex, ey, ez = np.array([2 * hx, 0, 0]), np.array([0, 2 * hy, 0]), np.array([0, 0, 2 * hz])
    verts, tris = [], []
    for origin, du, dv in ((corner + ez, ex, ey), (corner, ey, ex), (corner, ex, ez), (corner + ey, ez, ex),
                           (corner, ez, ey), (corner + ex, ey, ez)):
        base = len(verts)
        for i in range(divisions + 1):
            for j in range(divisions + 1):
                verts.append(origin + du * (i / divisions) + dv * (j / divisions))
        cols = divisions + 1
        for i in range(divisions):
            for j in range(divisions):
                a = base + i * cols + j
                tris.append([a, a + 1, a + cols])
                tris.append([a + 1, a + cols + 1, a + cols])
    v = np.asarray(verts, dtype=np.float64)
    t = np.asarray(tris, dtype=np.int64)
    key = np.round(v / (1e-9 * max(hx, hy, hz))).astype(np.int64)
    _, first, inverse = np.unique(key, axis=0, return_index=True, return_inverse=True)
    order = np.argsort(first)
    rank = np.empty_like(order)
    rank[order] = np.arange(len(order))
    return v[first[order]], rank[inverse.reshape(-1)[t]]


def _rows(resolution: int, rows) -> np.ndarray:
    return np.concatenate([np.arange(r * resolution, (r + 1) * resolution) for r in rows]).astype(np.int64)


def _twist_motion(rest_pins: np.ndarray, center: np.ndarray, rate: float, half: int):
    """Two pinned rails rotating about the x axis in opposite senses (reference scenes.py:188-203)."""

    def pin_motion(t: float) -> np.ndarray:
        out = rest_pins.copy()
        for sign, rows in ((1.0, slice(0, half)), (-1.0, slice(half, None))):
            ang = sign * rate * t
            ca, sa = np.cos(ang), np.sin(ang)
            rel = rest_pins[rows] - center
            out[rows] = center + np.stack([rel[:, 0], rel[:, 1] * ca - rel[:, 2] * sa,
                                           rel[:, 1] * sa + rel[:, 2] * ca], axis=1)
        return out

    return pin_motion


def scene_parts(kind: str, resolution: int = 32, size: float = 1.0, density: float = 0.3,
                stretch_stiffness: float = 160.0, bend_stiffness: float = 3e-4, config: StepConfig | None = None,
                **kw) -> dict:
    """Host-side scene description (mesh, obstacles, prescribed motions, material).

    Reference kinds follow scenes.py:144-207; the rest are the BASELINE configs.
    """
    cfg = config if config is not None else StepConfig()
    out = {"stretch": stretch_stiffness, "bend": bend_stiffness, "obstacles": None, "pin_motion": None,
           "obstacle_motion": None}
    if kind == "free_fall":
        v, t = grid_cloth(resolution, size, height=1.0)
        out["mesh"] = build_mesh(v, t, density, pins=[])
    elif kind == "hanging":
        v, t = grid_cloth(resolution, size, height=0.0)
        out["mesh"] = build_mesh(v, t, density, pins=_rows(resolution, [0]))
    elif kind == "sphere_drape":
        radius = 0.25 * size
        v, t = grid_cloth(resolution, size, height=radius + 2.0 * cfg.d_hat + 0.01 * size)
        v[:, :2] -= size / 2.0
        out["mesh"] = build_mesh(v, t, density, pins=[])
        out["obstacles"] = [icosphere(3, radius, center=(0.0, 0.0, 0.0))]
    elif kind == "desk_fold":
        v, t = grid_cloth(resolution, size, height=0.25 * size)
        v[:, :2] -= size / 2.0
        out["mesh"] = build_mesh(v, t, density, pins=[])
        out["obstacles"] = [
            box_mesh(center=(0.0, 0.0, 0.1 * size), extents=(0.45 * size, 0.45 * size, 0.2 * size), divisions=6),
            box_mesh(center=(0.0, 0.0, -0.05 * size), extents=(2.0 * size, 2.0 * size, 0.02 * size), divisions=4)]
    elif kind == "twist":
        v, t = grid_cloth(resolution, size, height=0.0)
        pins = _rows(resolution, [0, resolution - 1])
        out["mesh"] = build_mesh(v, t, density, pins=pins)
        out["pin_motion"] = _twist_motion(v[pins], v.mean(axis=0), np.pi / 2.0, len(pins) // 2)
    # ---------------- BASELINE configs (new; no reference generator exists)
    elif kind == "two_corner":
        v, t = grid_cloth(resolution, size)
        out["mesh"] = build_mesh(v, t, density, pins=[0, resolution - 1])
    elif kind == "sphere_ground":
        radius = 0.25 * size
        v, t = grid_cloth(resolution, size, height=radius + 2.0 * cfg.d_hat + 0.01 * size)
        v[:, :2] -= size / 2.0
        out["mesh"] = build_mesh(v, t, density, pins=[])
        # ground slab top 5 mm below the sphere's south pole (a touching slab would count
        # as an obstacle-obstacle intersection in the penetration check)
        out["obstacles"] = [icosphere(3, radius),
                            box_mesh(center=(0.0, 0.0, -(radius + 0.005 + 0.01 * size)),
                                     extents=(2.0 * size, 2.0 * size, 0.02 * size), divisions=4)]
    elif kind == "stacked_twist":
        sheets = int(kw.pop("sheets", 2))
        gap = float(kw.pop("gap", 0.005))
        v1, t1 = grid_cloth(resolution, size)
        vs, ts, rails = [], [], []
        for sh in range(sheets):
            v = v1.copy()
            v[:, 2] += sh * gap
            vs.append(v)
            ts.append(t1 + sh * len(v1))
            rails.append(_rows(resolution, [0, resolution - 1]) + sh * len(v1))
        verts = np.concatenate(vs)
        mesh = build_mesh(verts, np.concatenate(ts), density, pins=np.concatenate(rails))
        # left rails of every sheet turn one way, right rails the other
        left = np.concatenate([r[:resolution] for r in rails])
        right = np.concatenate([r[resolution:] for r in rails])
        order = np.concatenate([left, right])
        pos = np.searchsorted(mesh.pinned, order)
        base = _twist_motion(verts[order], verts.mean(axis=0), np.pi / 2.0, len(left))

        def pin_motion(t: float) -> np.ndarray:
            res = np.empty((len(order), 3))
            res[pos] = base(t)
            return res

        out["mesh"] = mesh
        out["pin_motion"] = pin_motion
    elif kind == "skirt":
        geo = {k: kw.pop(k) for k in list(kw) if k in ("around", "down", "radius", "length", "body_radius", "spin",
                                                        "sway", "sway_hz")}
        out.update(skirt_parts(density=density, **geo))
    else:
        raise ValueError(f"unknown scene kind {kind!r}")
    out["extra"] = kw
    return out


def build_scene(kind: str, resolution: int = 32, size: float = 1.0, density: float = 0.3,
                stretch_stiffness: float = 160.0, bend_stiffness: float = 3e-4, config: StepConfig | None = None,
                **kw):
    """Reference scene kinds (scenes.py:144-207) + BASELINE configs, as a GPU Simulation."""
    from .stepper import Simulation

    cfg = config if config is not None else StepConfig()
    p = scene_parts(kind, resolution, size, density, stretch_stiffness, bend_stiffness, cfg, **kw)
    return Simulation(p["mesh"], cfg, p["stretch"], p["bend"], obstacles=p["obstacles"], pin_motion=p["pin_motion"],
                      obstacle_motion=p["obstacle_motion"], **p["extra"])


# ------------------------------------------------------------------ config 4
def tube(around: int, down: int, radius_top: float, radius_bottom: float, length: float, top_z: float):
    """Seam-welded tube: ring k (top->bottom) of `around` vertices, flaring linearly."""
    ang = 2.0 * np.pi * np.arange(around) / around
    k = np.arange(down)
    frac = k / max(down - 1, 1)
    rad = radius_top + (radius_bottom - radius_top) * frac
    z = top_z - length * frac
    verts = np.stack([np.outer(rad, np.cos(ang)).ravel(), np.outer(rad, np.sin(ang)).ravel(),
                      np.repeat(z, around)], axis=1)
    i, j = np.meshgrid(np.arange(down - 1), np.arange(around), indexing="ij")
    a = (i * around + j).ravel()
    b = (i * around + (j + 1) % around).ravel()
    c, d = a + around, b + around
    even = ((i + j) % 2 == 0).ravel()
    first = np.where(even[:, None], np.stack([a, b, c], 1), np.stack([a, b, d], 1))
    second = np.where(even[:, None], np.stack([b, d, c], 1), np.stack([a, d, c], 1))
    return verts, np.stack([first, second], axis=1).reshape(-1, 3).astype(np.int64)


def capped_cylinder(radius: float, z_lo: float, z_hi: float, around: int = 48, rings: int = 12):
    """Closed cylinder body (side tube + fan caps)."""
    v, t = tube(around, rings, radius, radius, z_hi - z_lo, z_hi)
    n = len(v)
    top, bot = n, n + 1
    v = np.concatenate([v, [[0.0, 0.0, z_hi], [0.0, 0.0, z_lo]]])
    j = np.arange(around)
    jn = (j + 1) % around
    caps_top = np.stack([np.full(around, top), jn, j], 1)
    last = (rings - 1) * around
    caps_bot = np.stack([np.full(around, bot), last + j, last + jn], 1)
    return v, np.concatenate([t, caps_top, caps_bot]).astype(np.int64)


def skirt_parts(around: int = 584, down: int = 584, radius: float = 0.22, length: float = 0.6,
                body_radius: float = 0.20, spin: float = np.pi, sway: float = 0.03, sway_hz: float = 1.0,
                density: float = 0.3):
    """BASELINE config 4 geometry: procedural tube skirt (around x down vertices, ~341K
    at 584^2) on a capped-cylinder body that spins about z at `spin` rad/s and sways
    along x.  The waist ring is pinned and follows the body's rigid motion."""
    top = 0.0
    verts, tris = tube(around, down, radius, radius * 1.35, length, top)
    pins = np.arange(around)
    # waist ring hugs the body a little outside the barrier band
    verts[pins, :2] *= (body_radius + 0.004) / radius
    mesh = build_mesh(verts, tris, density, pins=pins)
    body_v, body_t = capped_cylinder(body_radius, top - 0.8 * length, top + 0.05)
    rest_pins = verts[pins].copy()

    def rigid(points: np.ndarray, t: float) -> np.ndarray:
        a = spin * t
        ca, sa = np.cos(a), np.sin(a)
        out = np.empty_like(points)
        out[:, 0] = ca * points[:, 0] - sa * points[:, 1] + sway * np.sin(2.0 * np.pi * sway_hz * t)
        out[:, 1] = sa * points[:, 0] + ca * points[:, 1]
        out[:, 2] = points[:, 2]
        return out

    return {"mesh": mesh, "obstacles": [(body_v, body_t)], "pin_motion": lambda t: rigid(rest_pins, t),
            "obstacle_motion": lambda t: rigid(body_v, t)}


def skirt_scene(cfg: StepConfig, density: float = 0.3, stretch_stiffness: float = 160.0,
                bend_stiffness: float = 3e-4, **kw):
    """BASELINE config 4 as a GPU Simulation (geometry: skirt_parts)."""
    return build_scene("skirt", density=density, stretch_stiffness=stretch_stiffness, bend_stiffness=bend_stiffness,
                       config=cfg, **kw)


# ------------------------------------------------------------------ config 5
def drape_materials(count: int = 64):
    """Per-scene materials from default_rng(seed=i): rho U[0.2,0.5], k_s U[80,320], k_b logU[1e-4,1e-3]."""
    out = []
    for i in range(count):
        g = np.random.default_rng(i)
        out.append((float(g.uniform(0.2, 0.5)), float(g.uniform(80.0, 320.0)),
                    float(10 ** g.uniform(-4.0, -3.0))))
    return out


def drape_scene(index: int, resolution: int = 317, config: StepConfig | None = None, **kw):
    """One scene of BASELINE config 5 (sphere drape with material `index`)."""
    rho, ks, kb = drape_materials(index + 1)[index]
    return build_scene("sphere_drape", resolution=resolution, density=rho, stretch_stiffness=ks, bend_stiffness=kb,
                       config=config, **kw)
