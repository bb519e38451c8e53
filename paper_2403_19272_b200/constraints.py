"""Projective-dynamics constraint set and global-matrix assembly (setup, host).

Mirrors the setup half of ``clothsim.constraints`` (reference
``pkg/src/clothsim/constraints.py``): per-edge stretch springs, quadratic
cotangent hinge bending (linear, so it lives only in H: reference
constraints.py:225), and H = M/h^2 + sum_i w_i S_i^T A_i^T A_i S_i with pinned
columns split into H_fp (reference constraints.py:161-209).

The per-iteration half (edge projection + rhs assembly, reference
constraints.py:212-256) runs on the device: ``csrc/solver.cu`` (k_assemble_rhs);
``project_stretch``/``assemble_rhs`` here are the numpy-signature entry points
of the drop-in surface and dispatch to the CUDA library.

The device copy of H is an ELL slab built by ``device.build_ell``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .mesh import ClothMesh, triangle_areas


def _cot(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """cot of the angle between rows of a and b (reference constraints.py:55-59)."""
    sin_part = np.maximum(np.linalg.norm(np.cross(a, b), axis=-1), 1e-300)
    return np.einsum("ij,ij->i", a, b) / sin_part


def bend_coefficients(rest_quad: np.ndarray) -> np.ndarray:
    """Cotangent hinge coefficients k (s,4) (reference constraints.py:42-66)."""
    q = np.asarray(rest_quad, dtype=np.float64)
    one = q.ndim == 2
    if one:
        q = q[None]
    p0, p1, p2, p3 = (q[:, j] for j in range(4))
    e01 = p1 - p0
    e10 = p0 - p1
    c_a = _cot(e01, p2 - p0)
    c_b = _cot(e01, p3 - p0)
    c_c = _cot(e10, p2 - p1)
    c_d = _cot(e10, p3 - p1)
    k = np.stack([c_c + c_d, c_a + c_b, -c_a - c_c, -c_b - c_d], axis=1)
    return k[0] if one else k


@dataclass
class ElasticConstraints:
    """Stretch springs and hinge stencils with fixed weights (reference constraints.py:101-115)."""

    edges: np.ndarray
    edge_rest: np.ndarray
    stretch_w: np.ndarray
    stencils: np.ndarray
    bend_k: np.ndarray
    bend_w: np.ndarray

    @property
    def mean_weight(self) -> float:
        allw = np.concatenate([self.stretch_w, self.bend_w])
        return float(allw.mean()) if allw.size else 1.0


def build_elastic(mesh: ClothMesh, stretch_stiffness: float, bend_stiffness: float) -> ElasticConstraints:
    """Weights scaled by rest measure (reference constraints.py:118-139)."""
    w_s = stretch_stiffness * mesh.edge_rest_lengths
    st = mesh.bend_stencils
    if len(st):
        k = bend_coefficients(mesh.rest_positions[st])
        area = triangle_areas(mesh.rest_positions, st[:, [0, 1, 2]]) + triangle_areas(mesh.rest_positions, st[:, [0, 1, 3]])
        w_b = bend_stiffness * area / 3.0
    else:
        k = np.zeros((0, 4))
        w_b = np.zeros(0)
    return ElasticConstraints(edges=mesh.edges, edge_rest=mesh.edge_rest_lengths, stretch_w=w_s,
                              stencils=st, bend_k=k, bend_w=w_b)


@dataclass
class GlobalSystem:
    """H over free vertices, pinned columns H_fp, diag, M/h^2 (reference constraints.py:142-158)."""

    H: sp.csr_matrix
    H_fp: sp.csr_matrix
    diag: np.ndarray
    mass_over_h2: np.ndarray
    collision_diag_delta: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def matvec(self, x: np.ndarray) -> np.ndarray:
        return self.H @ x


def assemble_global(mesh: ClothMesh, elastic: ElasticConstraints, h: float) -> GlobalSystem:
    """COO stamps -> CSR, then free/pinned split (reference constraints.py:161-209).

    The stamp order (stretch block, 16 bend blocks, mass diagonal) is kept so
    scipy's duplicate summation yields bit-identical values.
    """
    if h <= 0:
        raise ValueError("time step must be positive")
    if not (np.isfinite(elastic.stretch_w).all() and np.isfinite(elastic.bend_w).all()):
        raise ValueError("non-finite constraint weight")
    n = mesh.vertex_count
    e0, e1 = elastic.edges[:, 0], elastic.edges[:, 1]
    w = elastic.stretch_w
    rows = [np.concatenate([e0, e1, e0, e1])]
    cols = [np.concatenate([e0, e1, e1, e0])]
    vals = [np.concatenate([w, w, -w, -w])]
    st, kb, wb = elastic.stencils, elastic.bend_k, elastic.bend_w
    if len(st):
        for a in range(4):
            for b in range(4):
                rows.append(st[:, a])
                cols.append(st[:, b])
                vals.append(wb * kb[:, a] * kb[:, b])
    diag_ids = np.arange(n)
    rows.append(diag_ids)
    cols.append(diag_ids)
    vals.append(mesh.vertex_mass / (h * h))
    full = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
    free_rows = full[mesh.free]
    H = free_rows[:, mesh.free].tocsr()
    H_fp = free_rows[:, mesh.pinned].tocsr()
    return GlobalSystem(H=H, H_fp=H_fp, diag=H.diagonal().copy(),
                        mass_over_h2=mesh.vertex_mass[mesh.free] / (h * h),
                        collision_diag_delta=np.zeros(mesh.free.size))


def project_stretch(x_pair: np.ndarray, rest_length) -> np.ndarray:
    """Endpoint pair moved to rest length about its midpoint (reference constraints.py:19-39).

    Host helper of the drop-in surface (used by tests and harnesses); the
    stepper's projection is fused into the device rhs kernel.
    """
    x = np.asarray(x_pair, dtype=np.float64)
    one = x.ndim == 2
    if one:
        x = x[None]
    rest = np.atleast_1d(np.asarray(rest_length, dtype=np.float64))
    d = x[:, 1] - x[:, 0]
    length = np.linalg.norm(d, axis=1)
    unit = np.tile(np.array([1.0, 0.0, 0.0]), (len(d), 1))
    nz = length > 0
    unit[nz] = d[nz] / length[nz, None]
    mid = 0.5 * (x[:, 0] + x[:, 1])
    half = 0.5 * rest[:, None] * unit
    out = np.stack([mid - half, mid + half], axis=1)
    return out[0] if one else out


def assemble_rhs(system: GlobalSystem, mesh: ClothMesh, elastic: ElasticConstraints, z: np.ndarray, x: np.ndarray,
                 pinned_positions: np.ndarray, collision_vertices=None, collision_weights=None,
                 collision_targets=None):
    """Right-hand side over free vertices plus the collision diagonal delta
    (constraints.py:229-256), on the device: owner-computes per free vertex over its
    edge incidence in np.add.at order, M/h^2 z, -H_fp pins, then the collision stamps
    (stable by row, as np.add.at).  Returns numpy (b (n_free, 3), delta (n_free,))."""
    import torch

    from . import _lib, context

    ctx = context.get(system=system, mesh=mesh, elastic=elastic)
    dev = lambda a, t=np.float64: torch.as_tensor(np.ascontiguousarray(a, dtype=t), device="cuda")  # noqa: E731
    n = mesh.vertex_count
    pins = None
    if mesh.pinned.size:
        full = np.zeros((n, 3))
        full[mesh.pinned] = np.asarray(pinned_positions, dtype=np.float64).reshape(-1, 3)
        pins = dev(full)
    coll = collision_vertices is not None and len(collision_vertices) > 0
    if coll:
        ids = dev(np.asarray(collision_vertices), np.int32)
        w = dev(collision_weights)
        t = dev(np.asarray(collision_targets, dtype=np.float64).reshape(-1, 3))
    nf = mesh.free.size
    b = torch.empty((nf, 3), dtype=torch.float64, device="cuda")
    delta = torch.empty(nf, dtype=torch.float64, device="cuda")
    zd, xd = dev(z), dev(x)   # keep the device copies alive across the call
    _lib.check(ctx.lib.cs_assemble_rhs(ctx.ptr, zd.data_ptr(), xd.data_ptr(),
                                       pins.data_ptr() if pins is not None else None,
                                       ids.data_ptr() if coll else None, w.data_ptr() if coll else None,
                                       t.data_ptr() if coll else None, int(len(collision_vertices)) if coll else 0,
                                       b.data_ptr(), delta.data_ptr(), _lib.stream_handle()), "cs_assemble_rhs")
    return b.cpu().numpy(), delta.cpu().numpy()
