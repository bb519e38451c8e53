"""CPU: the product's host setup (mesh topology, weights, H, eigenbasis, scenes)
reproduces the reference's arrays bit-for-bit (tests/golden/setup_*.npz)."""

import numpy as np
import pytest

from conftest import golden
import paper_2403_19272_b200 as P
from paper_2403_19272_b200.scenes import scene_parts


def _setup(kind, cfg, **kw):
    parts = scene_parts(kind, config=cfg, **kw)
    mesh = parts["mesh"]
    el = P.build_elastic(mesh, parts["stretch"], parts["bend"])
    sy = P.assemble_global(mesh, el, cfg.h)
    r_bar = min(cfg.r_bar, mesh.free.size)
    sub = P.build_subspace(sy, mesh.rest_positions[mesh.free], r_bar, min(cfg.r, r_bar))
    return parts, mesh, el, sy, sub


@pytest.mark.parametrize("tag,kind,cfg_kw,scene_kw", [
    ("hanging10", "hanging", dict(h=1.0 / 200.0), dict(resolution=10)),
    ("sphere14", "sphere_drape", {}, dict(resolution=14, size=0.2)),
    ("twist16", "twist", dict(h=1.0 / 200.0), dict(resolution=16, size=0.5)),
])
def test_setup_matches_reference(tag, kind, cfg_kw, scene_kw):
    g = golden(f"setup_{tag}.npz")
    cfg = P.StepConfig(**cfg_kw)
    parts, mesh, el, sy, sub = _setup(kind, cfg, **scene_kw)
    assert np.array_equal(mesh.rest_positions, g["rest"])
    assert np.array_equal(mesh.triangles, g["tris"])
    assert np.array_equal(mesh.edges, g["edges"])
    assert np.array_equal(mesh.edge_rest_lengths, g["rest_len"])
    assert np.array_equal(mesh.bend_stencils, g["stencils"])
    assert np.array_equal(mesh.vertex_mass, g["mass"])
    assert np.array_equal(mesh.pinned, g["pinned"])
    assert np.array_equal(el.stretch_w, g["stretch_w"])
    assert np.array_equal(el.bend_k, g["bend_k"])
    assert np.array_equal(el.bend_w, g["bend_w"])
    assert np.array_equal(sy.H.data, g["H_data"]) and np.array_equal(sy.H.indices, g["H_indices"])
    assert np.array_equal(sy.H.indptr, g["H_indptr"])
    assert np.array_equal(sy.H_fp.data, g["Hfp_data"]) and np.array_equal(sy.H_fp.indices, g["Hfp_indices"])
    assert np.allclose(sub.eigenvalues, g["eigenvalues"], rtol=1e-12)
    # eigenvectors: same span (signs may flip only if ARPACK differs across hosts)
    cos = np.linalg.svd(sub.U.T @ g["U"], compute_uv=False)
    assert cos.min() > 1 - 1e-8
    assert np.isclose(el.mean_weight, float(g["k"]), rtol=0, atol=0)
    obs = [np.asarray(o[0]) for o in (parts["obstacles"] or [])]
    assert np.array_equal(np.concatenate(obs) if obs else np.zeros((0, 3)), g["obstacle_x"].reshape(-1, 3))


def test_mesh_validation_errors():
    """reference tests/test_mesh.py error classes."""
    with pytest.raises(P.MeshError):
        P.build_mesh(np.zeros((2, 3)), np.array([[0, 1, 1]]), 0.3)
    v = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]])
    with pytest.raises(P.MeshError):
        P.build_mesh(v, np.array([[0, 1, 3]]), 0.3)
    with pytest.raises(P.MeshError):
        P.build_mesh(v, np.array([[0, 1, 1]]), 0.3)
    with pytest.raises(P.MeshError):
        P.build_mesh(v, np.array([[0, 1, 2]]), 0.0)
    with pytest.raises(P.MeshError):
        P.build_mesh(v, np.array([[0, 1, 2]]), 0.3, pins=[5])
    m = P.build_mesh(v, np.array([[0, 1, 2]]), 2.0)
    assert np.isclose(m.total_mass, 1.0)


def test_step_config_validation():
    """reference tests/test_stepper.py:18-26."""
    for kw in (dict(h=0.0), dict(alpha=1.0), dict(eps_outer=0.0), dict(barrier_mode="ipc")):
        with pytest.raises(ValueError):
            P.StepConfig(**kw)


def test_patches_partition_triangles():
    v, t = P.grid_cloth(8, 1.0)
    seen = np.concatenate(P.build_patches(t, len(v)))
    assert np.array_equal(np.sort(seen), np.arange(len(t)))
    assert max(len(g) for g in P.build_patches(t, len(v))) <= 8


def test_sell32_roundtrip():
    from paper_2403_19272_b200.device import sell32

    parts, mesh, el, sy, sub = _setup("twist", P.StepConfig(), resolution=9, size=0.5)
    nsl, ptr, col, val = sell32(sy.H)
    x = np.random.default_rng(1).normal(size=(sy.H.shape[0], 3))
    y = np.zeros_like(x)
    for s in range(nsl):
        width = (ptr[s + 1] - ptr[s]) // 32
        for lane in range(32):
            row = 32 * s + lane
            if row >= sy.H.shape[0]:
                continue
            for k in range(width):
                c = col[ptr[s] + 32 * k + lane]
                if c < 0:
                    break
                y[row] = y[row] + val[ptr[s] + 32 * k + lane] * x[c]
    assert np.array_equal(y, sy.H @ x)


def test_skirt_config4_geometry():
    from paper_2403_19272_b200.scenes import skirt_parts

    parts = skirt_parts(around=64, down=32)
    m = parts["mesh"]
    assert m.vertex_count == 64 * 32 and m.pinned.size == 64
    # seam welded: every interior edge has two triangles -> 2*(down-1)*around triangles
    assert len(m.triangles) == 2 * 31 * 64
    x = parts["pin_motion"](0.25)
    assert x.shape == (64, 3)
    body = parts["obstacle_motion"](0.0)
    assert np.abs(np.linalg.norm(body[:, :2], axis=1)).max() <= 0.2 + 0.03 + 1e-12


def test_drape_materials_deterministic():
    from paper_2403_19272_b200.scenes import drape_materials

    a, b = drape_materials(64), drape_materials(64)
    assert a == b
    rho, ks, kb = zip(*a)
    assert 0.2 <= min(rho) and max(rho) <= 0.5 and 80 <= min(ks) and max(ks) <= 320
    assert 1e-4 <= min(kb) and max(kb) <= 1e-3
