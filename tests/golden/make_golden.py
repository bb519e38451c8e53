"""Generate golden fixtures by running the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference is imported read-only from /root/reference/pkg/src; its outputs
are stored as compressed .npz next to this script.  Nothing at test time
reads /root/reference.  Fixtures:

  setup_<scene>.npz      mesh topology, masses, weights, H / H_fp, eigenbasis
  narrow.npz             full_ccd / distance_toi / partial_ccd / pair_witness on
                         random and near-contact pairs (+ single-pair batches)
  broad_<k>.npz          broad_phase rows (kind, idx) in the reference's order
  solver.npz             assemble_rhs / ajacobi_smooth / reduced_correction /
                         warmstart_correction on a pinned system
  traj_<scene>.npz       positions + report counters after every step
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("CLOTHSIM_REF", "/root/reference/pkg/src"))

import clothsim  # noqa: E402
from clothsim.collision import (broad_phase, default_samples, distance_toi, full_ccd, pair_witness,  # noqa: E402
                                partial_ccd, PatchBVH)
from clothsim.constraints import assemble_rhs  # noqa: E402
from clothsim.scenes import build_scene, grid_cloth, icosphere  # noqa: E402
from clothsim.smoothing import ajacobi_smooth  # noqa: E402
from clothsim.subspace import reduced_correction, warmstart_correction  # noqa: E402


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)
    print("wrote", name, sum(a.nbytes for a in arrays.values()) // 1024, "KiB raw")


def setup_fixture(tag, sim):
    m, el, sy, sub = sim.mesh, sim.elastic, sim.system, sim.subspace
    save(f"setup_{tag}.npz", rest=m.rest_positions, tris=m.triangles, edges=m.edges, rest_len=m.edge_rest_lengths,
         stencils=m.bend_stencils, mass=m.vertex_mass, pinned=m.pinned, stretch_w=el.stretch_w, bend_k=el.bend_k,
         bend_w=el.bend_w, H_data=sy.H.data, H_indices=sy.H.indices, H_indptr=sy.H.indptr, Hfp_data=sy.H_fp.data,
         Hfp_indices=sy.H_fp.indices, Hfp_indptr=sy.H_fp.indptr, eigenvalues=sub.eigenvalues, U=sub.U,
         k=np.array(sim.k), world_tris=sim.bvh.triangles, tri_static=sim.bvh.tri_static,
         obstacle_x=sim.obstacle_x)


def narrow_fixture():
    rng = np.random.default_rng(7)
    n = 3000
    kind = np.zeros(n, dtype=np.int8)
    kind[n // 2:] = 1
    x0 = rng.uniform(-1.0, 1.0, size=(4 * n, 3))
    x1 = x0 + rng.uniform(-1.0, 1.0, size=(4 * n, 3))
    idx = np.arange(4 * n).reshape(n, 4)
    # near-contact population: almost coplanar, slow, some static / in-plane
    kn = (rng.random(n) < 0.5).astype(np.int8)
    base = rng.normal(size=(n, 4, 3)) * 0.2
    base[:, :, 2] *= 1e-3 * rng.random((n, 1))
    move = rng.normal(size=(n, 4, 3)) * 0.01
    move[rng.random(n) < 0.2] = 0.0
    move[rng.random(n) < 0.2, :, 2] = 0.0
    y0 = base.reshape(-1, 3)
    y1 = (base + move).reshape(-1, 3)
    out = dict(kind=kind, idx=idx, x0=x0, x1=x1, kind_n=kn, y0=y0, y1=y1)
    out["toi"] = full_ccd(kind, idx, x0, x1)
    out["toi_n"] = full_ccd(kn, idx, y0, y1)
    for f in (0.2, 1.0 - 0.8):
        out[f"dist_{f!r}"] = distance_toi(kind, idx, x0, x1, floor_frac=f)
        out[f"dist_n_{f!r}"] = distance_toi(kn, idx, y0, y1, floor_frac=f)
    for c in (1, 3, 6):
        out[f"partial_{c}"] = partial_ccd(kind, idx, x0, x0 + 0.4 * (x1 - x0), default_samples(c))
        out[f"partial_n_{c}"] = partial_ccd(kn, idx, y0, y1, default_samples(c))
    p1, p2, bary, dist = pair_witness(kn, idx, y0)
    out.update(w_p1=p1, w_p2=p2, w_bary=bary, w_dist=dist)
    single = np.full(200, np.nan)
    for i in range(200):
        single[i] = full_ccd(kind[i:i + 1], np.array([[0, 1, 2, 3]]), x0[4 * i:4 * i + 4], x1[4 * i:4 * i + 4])[0]
    out["toi_single"] = single
    save("narrow.npz", **out)


def broad_fixtures():
    rng = np.random.default_rng(11)
    cases = [(6, False, 0.08, 0.15, 0.01), (12, True, 0.02, 0.05, 0.01), (20, True, 0.004, 0.01, 1e-3),
             (33, False, 0.002, 0.004, 1e-3)]
    for k, (res, obst, jit, mv, margin) in enumerate(cases):
        v, t = grid_cloth(res, 1.0)
        if obst:
            sv, st = icosphere(2, 0.3, center=(0.5, 0.5, -0.05))
            wt = np.concatenate([t, st + len(v)])
            wr = np.concatenate([v, sv])
            stat = np.zeros(len(wt), bool)
            stat[len(t):] = True
        else:
            wt, wr, stat = t, v, np.zeros(len(t), bool)
        x0 = wr + jit * rng.normal(size=wr.shape)
        x1 = x0 + mv * rng.normal(size=wr.shape)
        ps = broad_phase(x0, x1, PatchBVH.build(wt, wr, stat), margin)
        save(f"broad_{k}.npz", tris=wt, tri_static=stat, x0=x0, x1=x1, margin=np.array(margin), kind=ps.kind,
             idx=ps.idx)


def solver_fixture():
    rng = np.random.default_rng(13)
    sim = build_scene("twist", resolution=16, size=0.5, config=clothsim.StepConfig(h=1.0 / 200.0))
    m, el, sy, sub = sim.mesh, sim.elastic, sim.system, sim.subspace
    n, nf = m.vertex_count, m.free.size
    x = m.rest_positions + 0.01 * rng.normal(size=(n, 3))
    z = m.rest_positions + 0.01 * rng.normal(size=(n, 3))
    pins = x[m.pinned]
    ids = rng.integers(0, n, size=300)
    w = rng.uniform(1.0, 1e4, size=300)
    tg = rng.normal(size=(300, 3))
    b0, d0 = assemble_rhs(sy, m, el, z, x, pins)
    b1, d1 = assemble_rhs(sy, m, el, z, x, pins, collision_vertices=ids, collision_weights=w, collision_targets=tg)
    bb = rng.normal(size=(nf, 3))
    xx = rng.normal(size=(nf, 3))
    dl = np.where(rng.random(nf) < 0.1, rng.uniform(0, 50, nf), 0.0)
    sm = ajacobi_smooth(sy, bb, xx, 32, 0.0, dl)
    rc0, _ = reduced_correction(sub, sy, bb, xx, np.zeros(nf))
    rc1, _ = reduced_correction(sub, sy, bb, xx, dl)
    big = np.zeros(nf)
    big[rng.choice(nf, 20, replace=False)] = 2.0 ** 60
    rc2, red2 = reduced_correction(sub, sy, bb, xx, big)
    ws = warmstart_correction(sub, sy, bb, xx)
    save("solver.npz", x=x, z=z, pins=pins, ids=ids, w=w, tg=tg, b0=b0, d0=d0, b1=b1, d1=d1, bb=bb, xx=xx, dl=dl,
         smooth=sm, rc0=rc0, rc1=rc1, big=big, rc2=rc2, rc2_fallback=np.array(red2.used_fallback), ws=ws)
    setup_fixture("twist16", sim)


def traj_fixture(tag, kind, steps, cfg_kw, **scene_kw):
    sim = build_scene(kind, config=clothsim.StepConfig(**cfg_kw), **scene_kw)
    if tag in ("hanging10", "sphere14"):
        setup_fixture(tag, sim)
    xs, lg, rf, outer, toi = [], [], [], [], []
    for _ in range(steps):
        r = sim.step()
        xs.append(sim.state.x.copy())
        lg.append(r.lg_iterations)
        rf.append(r.rf_triggered)
        outer.append(r.outer_loops)
        toi.append(r.toi_exit)
    save(f"traj_{tag}.npz", x=np.stack(xs), lg=np.array(lg), rf=np.array(rf), outer=np.array(outer),
         toi=np.array(toi), obstacle_x=sim.obstacle_x)


def contact_state_fixture(steps=25):
    """sphere_drape res 14 over the whole settling sequence, full SimState after every
    step (for teacher-forced GPU steps) + the reference's own intersection count."""
    from clothsim.oracles import oracle_intersect

    sim = build_scene("sphere_drape", resolution=14, size=0.2, config=clothsim.StepConfig())
    keys = ("x", "x_dot", "x_prev", "delta_f")
    out = {k: [sim.state.__dict__[k].copy()] for k in keys}
    out["obstacle_x"] = [sim.obstacle_x.copy()]
    lg, toi, rf, bad = [], [], [], []
    for _ in range(steps):
        r = sim.step()
        for k in keys:
            out[k].append(getattr(sim.state, k).copy())
        out["obstacle_x"].append(sim.obstacle_x.copy())
        lg.append(r.lg_iterations)
        toi.append(r.toi_exit)
        rf.append(r.rf_triggered)
        bad.append(len(oracle_intersect(sim.world(sim.state.x), sim.bvh.triangles)))
    save("contact_sphere14.npz", **{k: np.stack(v) for k, v in out.items()}, lg=np.array(lg), toi=np.array(toi),
         rf=np.array(rf), intersections=np.array(bad))


def dbb_fixture(steps=18):
    """sphere_drape res 14 in the DBB baseline mode (barrier_mode="dbb")."""
    traj_fixture("sphere14_dbb", "sphere_drape", steps, {"barrier_mode": "dbb"}, resolution=14, size=0.2)


def stages_fixture():
    """Module-level stage helpers the drop-in re-exports (collision/__init__.py,
    oracles.py): coplanarity coefficients (batched and single-pair BLAS paths), query_q
    (shared and per-pair samples), closest points, swept boxes, DBB weights, the float
    SAT on near-degenerate pairs (+ the exact rational verdict), lattice samples."""
    from clothsim.collision import (coplanarity_coefficients, dbb_weight, dbb_weight_gradient,
                                    lattice_samples, point_triangle_closest, query_q,
                                    segment_segment_closest, swept_boxes)
    from clothsim.oracles import tri_tri_intersect, tri_tri_intersect_exact

    rng = np.random.default_rng(11)
    n = 2000
    kind = (rng.random(n) < 0.5).astype(np.int8)
    x0 = rng.uniform(-1.0, 1.0, size=(4 * n, 3))
    x1 = x0 + 0.3 * rng.normal(size=(4 * n, 3))
    idx = np.arange(4 * n).reshape(n, 4)
    out = dict(kind=kind, idx=idx, x0=x0, x1=x1)
    out["coef"] = coplanarity_coefficients(kind, idx, x0, x1)
    out["coef_single"] = np.stack([coplanarity_coefficients(kind[i:i + 1], idx[:1], x0[4 * i:4 * i + 4],
                                                            x1[4 * i:4 * i + 4])[0] for i in range(50)])
    lam_shared = np.array([[0.25, 0.25], [0.5, 0.1], [0.1, 0.7]])
    lam_pair = rng.uniform(0.0, 0.5, size=(n, 4, 2))
    out.update(lam_shared=lam_shared, lam_pair=lam_pair, q_shared=query_q(kind, idx, x0, x1, lam_shared),
               q_pair=query_q(kind, idx, x0, x1, lam_pair))
    q = x0[idx]
    out["ptc"] = np.concatenate([np.asarray(a).reshape(n, -1) for a in point_triangle_closest(q[:, 0], q[:, 1],
                                                                                            q[:, 2], q[:, 3])], 1)
    out["ssc"] = np.concatenate([np.asarray(a).reshape(n, -1) for a in segment_segment_closest(q[:, 0], q[:, 1],
                                                                                             q[:, 2], q[:, 3])], 1)
    lo, hi = swept_boxes(x0[idx], x1[idx], 1e-3)
    out.update(sb_lo=lo, sb_hi=hi)
    d = np.concatenate([10.0 ** rng.uniform(-9, -2, 500), [1e-3, 2e-3]])
    out.update(dbb_d=d, dbb_w=dbb_weight(d, 1e-3, 3.0), dbb_g=dbb_weight_gradient(d, 1e-3, 3.0))
    # near-degenerate SAT pairs (the reference's tests/test_harness.py:_near_degenerate_pairs
    # mix: coplanar-offset, shared edge, vertex on plane, generic small separation)
    m = 1500
    p = rng.uniform(-1.0, 1.0, size=(m, 3, 3))
    qq = np.empty_like(p)
    mode = rng.integers(0, 4, size=m)
    for i in range(m):
        if mode[i] == 0:
            qq[i] = p[i][[1, 2, 0]] + rng.normal(scale=1e-9, size=(3, 3))
        elif mode[i] == 1:
            qq[i, 0], qq[i, 1], qq[i, 2] = p[i, 0], p[i, 1], rng.uniform(-1.0, 1.0, size=3)
        elif mode[i] == 2:
            nrm = np.cross(p[i, 1] - p[i, 0], p[i, 2] - p[i, 0])
            nrm /= np.linalg.norm(nrm)
            base = p[i, 0] + 0.3 * (p[i, 1] - p[i, 0]) + 0.3 * (p[i, 2] - p[i, 0])
            qq[i, 0] = base
            qq[i, 1] = base + rng.uniform(-0.5, 0.5, size=3)
            qq[i, 2] = base + rng.uniform(-0.5, 0.5, size=3)
        else:
            qq[i] = p[i] + rng.normal(scale=1e-3, size=(3, 3))
    p, qq = np.round(p, 6), np.round(qq, 6)
    out.update(sat_p=p, sat_q=qq, sat=tri_tri_intersect(p, qq),
               sat_exact=np.array([tri_tri_intersect_exact(p[i], qq[i]) for i in range(m)]))
    for dom in ("triangle", "box"):
        for iv in (0.3, 0.1):
            out[f"lattice_{dom}_{iv}"] = lattice_samples(iv, dom)
    save("stages.npz", **out)


def two_corner_fixture(steps=20):
    """BASELINE config 1: 64x64 grid pinned at two corners, h = 1/200."""
    v, t = grid_cloth(64, 1.0)
    mesh = clothsim.build_mesh(v, t, 0.3, pins=[0, 63])
    sim = clothsim.Simulation(mesh, clothsim.StepConfig(h=1.0 / 200.0))
    xs, lg, outer, sites = [], [], [], []
    for _ in range(steps):
        r = sim.step()
        xs.append(sim.state.x.copy())
        lg.append(r.lg_iterations)
        outer.append(r.outer_loops)
        sites.append(r.full_ccd_calls)
    save("traj_two_corner64.npz", x=np.stack(xs), lg=np.array(lg), outer=np.array(outer), sites=np.array(sites),
         x_dot=sim.state.x_dot)


def sphere_ground_fixture(steps=14, keep=6):
    """BASELINE config 2: 128x128 cloth dropped onto a sphere (r 0.25) above a ground slab,
    h = 1/200, run by the reference.  Positions of the last `keep` steps (the first
    contact steps) + counters of every step: a test rebuilds the full state before step s
    from them (x_prev = x[s-1], x_dot = (x[s] - x[s-1]) / h, delta_f stored when nonzero)
    and teacher-forces the GPU step against x[s+1]."""
    from clothsim.scenes import box_mesh

    cfg = clothsim.StepConfig(h=1.0 / 200.0)
    v, t = grid_cloth(128, 1.0, height=0.25 + 2.0 * cfg.d_hat + 0.01)
    v[:, :2] -= 0.5
    mesh = clothsim.build_mesh(v, t, 0.3, pins=[])
    obstacles = [icosphere(3, 0.25), box_mesh(center=(0.0, 0.0, -(0.25 + 0.005 + 0.01)), extents=(2.0, 2.0, 0.02),
                                              divisions=4)]
    sim = clothsim.Simulation(mesh, cfg, obstacles=obstacles)
    xs, dfs, lg, outer, rf, toi, act = [], [], [], [], [], [], []
    for _ in range(steps):
        r = sim.step()
        xs.append(sim.state.x.copy())
        dfs.append(sim.state.delta_f.copy())
        lg.append(r.lg_iterations)
        outer.append(r.outer_loops)
        rf.append(r.rf_triggered)
        toi.append(r.toi_exit)
        act.append(r.active_pairs)
        print("step", len(xs), r.lg_iterations, r.outer_loops, r.rf_triggered, r.toi_exit, r.active_pairs, flush=True)
    first = steps - keep
    df = np.stack(dfs[first:])
    save("traj_sphere_ground128.npz", x=np.stack(xs[first:]), first=np.array(first), h=np.array(cfg.h),
         df_nonzero=np.array([bool(np.any(d)) for d in df]), delta_f=df[[bool(np.any(d)) for d in df]],
         lg=np.array(lg), outer=np.array(outer), rf=np.array(rf), toi=np.array(toi), active=np.array(act),
         obstacle_x=sim.obstacle_x)


def io_fixture():
    """Frame/metrics I/O (cli.py:64-98, config.py): the reference CLI's `simulate` on a
    small hanging cloth - config text as written, OBJ frames, metrics CSV - plus
    parse/serialize of a non-default config and save_obj of a fixed array."""
    import tempfile
    from pathlib import Path

    from clothsim.cli import main
    from clothsim.config import parse_config, serialize_config
    from clothsim.mesh import save_obj

    text = ('name = "io"\nsteps = 4\nseed = 3\n\n[scene]\nkind = "hanging"\nresolution = 10\nsize = 1.0\n\n'
            '[solver]\nh = 0.005\ngravity = [0.0, -9.8, 0.0]\nsamples = 6\n\n[output]\nframe_stride = 2\n')
    with tempfile.TemporaryDirectory() as d:
        out = Path(d) / "out"
        cfg_path = Path(d) / "io.toml"
        cfg_path.write_text(text.replace("[output]\n", f'[output]\ndirectory = "{out}"\n'))
        assert main(["simulate", str(cfg_path)]) == 0
        frames = sorted(p.name for p in out.glob("frame_*.obj"))
        objs = [(out / f).read_text() for f in frames]
        metrics = (out / "metrics.csv").read_text()
        written = (out / "config.toml").read_text()
        obj_path = Path(d) / "fixed.obj"
        rng = np.random.default_rng(5)
        verts = rng.uniform(-2.0, 2.0, (17, 3))
        verts[0] = [-0.0, 1e-12, 123.456789012345]
        tris = rng.integers(0, 17, (9, 3))
        save_obj(obj_path, verts, tris)
        fixed_obj = obj_path.read_text()
    roundtrip = serialize_config(parse_config(text))
    save("io.npz", config_in=np.array(text), config_roundtrip=np.array(roundtrip), frames=np.array(frames),
         objs=np.array(objs), metrics=np.array(metrics), config_written=np.array(written),
         fixed_verts=verts, fixed_tris=tris, fixed_obj=np.array(fixed_obj))


if __name__ == "__main__":
    if len(sys.argv) > 1:          # regenerate selected fixtures only
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    narrow_fixture()
    broad_fixtures()
    solver_fixture()
    traj_fixture("hanging10", "hanging", 6, dict(h=1.0 / 200.0), resolution=10)
    traj_fixture("sphere14", "sphere_drape", 12, {}, resolution=14, size=0.2)
    traj_fixture("twist10", "twist", 6, {}, resolution=10, size=0.3)
    two_corner_fixture()
    sphere_ground_fixture()
    stages_fixture()
    contact_state_fixture()
    dbb_fixture()
    io_fixture()
