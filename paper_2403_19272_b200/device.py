"""Device layout of one scene: converts the reference-compatible setup objects
into the flat arrays of ``cs_scene_desc`` (include/clothsim_b200.h).

HBM layout (all fp64 unless noted, AoS xyz rows):
  * state x, v, x_prev, delta_f: (n, 3); candidate/anchor/start world arrays (n_w, 3)
  * H (free x free): SELL-32 - slices of 32 rows, column-major inside a slice,
    width = longest row in the slice, int32 cols (-1 padding), CSR column order
    preserved so row sums are evaluated in scipy's order
  * basis U (n_f, r_bar) row-major + a contiguous copy of V = U[:, :r] (n_f, r)
  * vertex->edge incidence lists (owner-computes rhs / gradient, no atomics)
  * pairs: kind int8, idx int4 (16 B), key u64, toi/filter/dist/weight fp64,
    bary (2) / normal (3) fp64, life int32, engaged u8
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def sell32(H):
    """CSR (scipy) -> SELL-32 arrays (slice_ptr, col, val); keeps stored column order."""
    n = H.shape[0]
    indptr = np.asarray(H.indptr, dtype=np.int64)
    lens = np.diff(indptr)
    nsl = (n + 31) // 32
    padded = np.zeros(nsl * 32, np.int64)
    padded[:n] = lens
    width = padded.reshape(nsl, 32).max(axis=1)
    slice_ptr = np.concatenate([[0], np.cumsum(width * 32)]).astype(np.int64)
    if slice_ptr[-1] >= 2**31:
        raise ValueError("matrix too large for int32 SELL offsets")
    col = np.full(int(slice_ptr[-1]), -1, np.int32)
    val = np.zeros(int(slice_ptr[-1]), np.float64)
    rows = np.repeat(np.arange(n), lens)
    k = np.arange(len(rows)) - np.repeat(indptr[:-1], lens)
    dest = slice_ptr[rows // 32] + k * 32 + rows % 32
    col[dest] = H.indices
    val[dest] = H.data
    return nsl, slice_ptr.astype(np.int32), col, val


def incidence(n: int, vertex: np.ndarray, code: np.ndarray):
    """CSR of codes grouped by vertex, stable in the given order."""
    order = np.argsort(vertex, kind="stable")
    ptr = np.zeros(n + 1, np.int64)
    np.add.at(ptr, vertex + 1, 1)
    return np.cumsum(ptr).astype(np.int32), code[order].astype(np.int32)


class _Keep:
    """Holds numpy buffers alive while the C struct points at them."""

    def __init__(self):
        self.arrays = []

    def ptr(self, a, ctype):
        a = np.ascontiguousarray(a)
        self.arrays.append(a)
        return a.ctypes.data_as(ctypes.POINTER(ctype))


def step_config_c(cfg, k: float, kappa: float = 0.0) -> _lib.StepConfigC:
    c = _lib.StepConfigC()
    for name in ("h", "eps_initial", "eps_inner", "eps_outer", "eps_toi", "alpha", "ndb_base", "d_hat", "omega",
                 "rf_tolerance", "delta_f_cap"):
        setattr(c, name, float(getattr(cfg, name)))
    c.ndb_k = float(k)
    for name in ("iteration_cap", "samples", "smoothing_iterations", "warm_start_cap", "inner_cap", "outer_cap",
                 "rf_iterations"):
        setattr(c, name, int(getattr(cfg, name)))
    c.dbb_kappa = float(kappa)
    c.barrier_mode = 1 if cfg.barrier_mode == "dbb" else 0
    c.smoother = 1 if getattr(cfg, "smoother", "ajacobi") == "chebyshev" else 0
    return c


def _fill_system(d, keep, system):
    I, D = ctypes.c_int, ctypes.c_double
    d.n_free = system.H.shape[0]
    nsl, sptr, scol, sval = sell32(system.H)
    d.sell_nslices = nsl
    d.sell_slice_ptr, d.sell_col, d.sell_val = keep.ptr(sptr, I), keep.ptr(scol, I), keep.ptr(sval, D)
    d.diag = keep.ptr(system.diag, D)


def _fill_cloth(d, keep, mesh, elastic, system, gravity_force):
    I, D = ctypes.c_int, ctypes.c_double
    n = mesh.vertex_count
    d.n_cloth, d.n_pinned = n, mesh.pinned.size
    d.n_edges = len(elastic.edges)
    d.n_stencils = len(elastic.stencils)
    d.free_ids = keep.ptr(mesh.free.astype(np.int32), I)
    d.free_index = keep.ptr(mesh.free_index.astype(np.int32), I)
    d.pin_ids = keep.ptr(np.concatenate([mesh.pinned, [0]]).astype(np.int32), I)
    d.mass = keep.ptr(mesh.vertex_mass.astype(np.float64), D)
    d.fext = keep.ptr(np.asarray(gravity_force, dtype=np.float64), D)
    d.mass_over_h2 = keep.ptr(system.mass_over_h2, D)
    e = elastic.edges.astype(np.int64)
    ne = len(e)
    d.edge_v = keep.ptr(e.astype(np.int32), I)
    d.edge_rest = keep.ptr(elastic.edge_rest, D)
    d.edge_w = keep.ptr(elastic.stretch_w, D)
    eid = np.arange(ne, dtype=np.int64)
    # rhs: np.add.at(b, e0, -w y) then np.add.at(b, e1, w y)  (constraints.py:223-224)
    ptr, codes = incidence(n, np.concatenate([e[:, 0], e[:, 1]]), np.concatenate([2 * eid, 2 * eid + 1]))
    d.rhs_inc_ptr, d.rhs_inc = keep.ptr(ptr, I), keep.ptr(codes, I)
    # gradient: np.add.at(grad, e1, g) then np.add.at(grad, e0, -g)  (stepper.py:331-332)
    ptr, codes = incidence(n, np.concatenate([e[:, 1], e[:, 0]]), np.concatenate([2 * eid + 1, 2 * eid]))
    d.grad_inc_ptr, d.grad_inc = keep.ptr(ptr, I), keep.ptr(codes, I)
    st = elastic.stencils.astype(np.int64).reshape(-1, 4)
    d.stencils = keep.ptr(np.concatenate([st.ravel(), [0]]).astype(np.int32), I)
    d.bend_k = keep.ptr(np.concatenate([elastic.bend_k.ravel(), [0.0]]), D)
    d.bend_w = keep.ptr(np.concatenate([elastic.bend_w, [0.0]]), D)
    ptr, codes = incidence(n, st.ravel(), np.arange(st.size, dtype=np.int64))
    d.bend_inc_ptr, d.bend_inc = keep.ptr(ptr, I), keep.ptr(np.concatenate([codes, [0]]).astype(np.int32), I)
    hfp = system.H_fp
    d.hfp_ptr = keep.ptr(np.asarray(hfp.indptr, dtype=np.int32), I)
    fp_cols = mesh.pinned[hfp.indices] if mesh.pinned.size else np.zeros(0, np.int64)
    d.hfp_col = keep.ptr(np.concatenate([fp_cols, [0]]).astype(np.int32), I)
    d.hfp_val = keep.ptr(np.concatenate([hfp.data, [0.0]]), D)


def _fill_basis(d, keep, subspace):
    D = ctypes.c_double
    d.r_bar = subspace.U.shape[1]
    d.r = subspace.r
    d.U = keep.ptr(np.ascontiguousarray(subspace.U, dtype=np.float64), D)
    d.eigenvalues = keep.ptr(subspace.eigenvalues, D)


def _fill_world(d, keep, world, n_world):
    I, U8 = ctypes.c_int, ctypes.c_uint8
    d.n_world = n_world
    d.n_world_tris = len(world.triangles)
    d.n_world_edges = len(world.edges)
    d.world_tris = keep.ptr(world.triangles.astype(np.int32), I)
    d.world_edges = keep.ptr(world.edges.astype(np.int32), I)
    d.tri_static = keep.ptr(world.tri_static.astype(np.uint8), U8)
    d.vert_static = keep.ptr(world.vert_static.astype(np.uint8), U8)
    d.vert_used = keep.ptr(world.vert_used.astype(np.uint8), U8)
    d.edge_static = keep.ptr(world.edge_static.astype(np.uint8), U8)
    d.edge_tris = keep.ptr(world.edge_tris.astype(np.int32), I)
    d.edge_slot = keep.ptr(world.edge_slot.astype(np.int32), I)
    d.patch = keep.ptr(world.patch_of_tri.astype(np.int32), I)
    d.patch_slot = keep.ptr(world.slot_of_tri.astype(np.int32), I)


def parts_desc(system=None, mesh=None, elastic=None, subspace=None, world=None, n_world=0, gravity_force=None):
    """(SceneDesc, keepalive, parts) of a partial context (cs_scene_create_parts) from
    whichever reference setup objects are given."""
    keep = _Keep()
    d = _lib.SceneDesc()
    parts = 0
    if system is not None:
        _fill_system(d, keep, system)
        parts |= _lib.CS_PART_SYSTEM
        if mesh is not None and elastic is not None:
            g = gravity_force if gravity_force is not None else np.zeros((mesh.vertex_count, 3))
            _fill_cloth(d, keep, mesh, elastic, system, g)
            parts |= _lib.CS_PART_CLOTH
    if subspace is not None:
        _fill_basis(d, keep, subspace)
        if system is None:
            d.n_free = subspace.U.shape[0]
        parts |= _lib.CS_PART_BASIS
    if world is not None:
        _fill_world(d, keep, world, n_world or getattr(world, "n_world", 0) or int(world.triangles.max()) + 1)
        parts |= _lib.CS_PART_WORLD
    return d, keep, parts


def scene_desc(mesh, elastic, system, subspace, world, obstacle_x, gravity_force, x0):
    """Build (SceneDesc, keepalive) for cs_scene_create (every part + the state)."""
    keep = _Keep()
    D = ctypes.c_double
    d = _lib.SceneDesc()
    nobs = len(obstacle_x)
    _fill_system(d, keep, system)
    _fill_cloth(d, keep, mesh, elastic, system, gravity_force)
    _fill_basis(d, keep, subspace)
    _fill_world(d, keep, world, mesh.vertex_count + nobs)
    d.n_obstacle = nobs
    d.x0 = keep.ptr(np.asarray(x0, dtype=np.float64), D)
    d.obstacle_x0 = keep.ptr(np.concatenate([np.asarray(obstacle_x, dtype=np.float64).ravel(), [0.0]]), D)
    return d, keep
