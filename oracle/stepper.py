"""ORACLE (test infrastructure only): one time step of the pipeline.

Restates reference ``Simulation.step`` (pkg/src/clothsim/stepper.py:454-624),
its helpers (:177-305, :384-452) and residual forwarding (:626-672) in the
non-distance-barrier (NDB) mode, the mode the north star builds.  Scene setup
(mesh, elastic weights, H, eigenbasis) is taken from the product's host setup
modules, which tests pin separately against the reference's arrays.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import narrow, solver
from .broad import WorldTopology, broad_phase

VT, EE = 0, 1
LIFE_CAP = 64                                     # pairs.py:21


class PenetrationError(RuntimeError):
    def __init__(self, message, state_dump=None):
        super().__init__(message)
        self.state_dump = state_dump


@dataclass
class Pairs:
    """Pair rows plus witness/NDB fields (pairs.py:24-62)."""

    kind: np.ndarray
    idx: np.ndarray
    life: np.ndarray = None
    weight: np.ndarray = None
    bary: np.ndarray = None
    dist: np.ndarray = None
    normal: np.ndarray = None

    def __len__(self):
        return len(self.kind)

    def keys(self):
        """Canonical carry-over keys (pairs.py:51-62)."""
        k = self.idx.copy()
        vt = self.kind == VT
        ee = ~vt
        k[vt, 1:] = np.sort(k[vt, 1:], axis=1)
        k[ee, :2] = np.sort(k[ee, :2], axis=1)
        k[ee, 2:] = np.sort(k[ee, 2:], axis=1)
        swap = ee & (k[:, 0] > k[:, 2])
        k[swap] = k[swap][:, [2, 3, 0, 1]]
        return np.concatenate([self.kind[:, None].astype(np.int64), k], axis=1)


def rms(v) -> float:
    return float(np.linalg.norm(v)) / max(np.sqrt(v.size), 1.0)   # stepper.py:96-98


def dbb_weight(d, d_hat, kappa):
    """Log barrier -kappa (d - d_hat)^2 ln(d / d_hat) below d_hat, else 0 (pairs.py:83-99)."""
    d = np.asarray(d, dtype=np.float64)
    if (d <= 0).any():
        raise FloatingPointError("nonpositive pair distance: infeasible state")
    out = np.zeros_like(d)
    near = d < d_hat
    dn = d[near]
    out[near] = -kappa * (dn - d_hat) ** 2 * np.log(dn / d_hat)
    return out


def ndb_weight(life, k, base):
    return k * np.power(base, np.minimum(life, LIFE_CAP).astype(np.float64))   # pairs.py:65-70


def shares(kind, bary):
    """Endpoint participation gamma (m,4) (stepper.py:107-121)."""
    g = np.empty((len(kind), 4))
    vt = kind == VT
    g[vt, 0] = 1.0
    g[vt, 1] = 1.0 - bary[vt, 0] - bary[vt, 1]
    g[vt, 2] = bary[vt, 0]
    g[vt, 3] = bary[vt, 1]
    ee = ~vt
    g[ee, 0] = 1.0 - bary[ee, 0]
    g[ee, 1] = bary[ee, 0]
    g[ee, 2] = 1.0 - bary[ee, 1]
    g[ee, 3] = bary[ee, 1]
    return np.clip(g, 0.0, 1.0)


def _sides_at(kind, idx, bary, xw):
    """Witness points p1 (first primitive) and p2 (second) at frozen params."""
    p = xw[idx]
    vt = (kind == VT)[:, None]
    l1, l2 = bary[:, 0:1], bary[:, 1:2]
    p1 = np.where(vt, p[:, 0], p[:, 0] + l1 * (p[:, 1] - p[:, 0]))
    p2 = np.where(vt, p[:, 1] + l1 * (p[:, 2] - p[:, 1]) + l2 * (p[:, 3] - p[:, 1]),
                  p[:, 2] + l2 * (p[:, 3] - p[:, 2]))
    return p, p1, p2


class OracleSimulation:
    """CPU replica of one scene; mirrors the reference constructor's state."""

    def __init__(self, mesh, config, elastic, system, subspace, k, obstacles_x, world_tris, tri_static,
                 pin_motion=None, obstacle_motion=None):
        self.mesh, self.cfg = mesh, config
        self.el, self.sys, self.sub = elastic, system, subspace
        self.k = k
        # stepper.py:165-169: kappa matched to the NDB mode's initial weight at d_hat / 2
        self.kappa = config.dbb_kappa if config.dbb_kappa > 0 else k / ((config.d_hat / 2.0) ** 2 * np.log(2.0))
        self.obstacle_x = np.asarray(obstacles_x, dtype=np.float64).reshape(-1, 3)
        self.topo = WorldTopology.build(world_tris, tri_static)
        self.pin_motion, self.obstacle_motion = pin_motion, obstacle_motion
        from paper_2403_19272_b200.mesh import SimState

        self.state = SimState.rest(mesh)
        self.gravity_force = mesh.vertex_mass[:, None] * np.asarray(config.gravity)
        self.last_outer_deltas = []

    @classmethod
    def from_parts(cls, parts: dict, config):
        """Build the scene on the host only (no GPU): mirrors the reference
        constructor (stepper.py:127-173) using the product's setup modules."""
        from paper_2403_19272_b200.constraints import assemble_global, build_elastic
        from paper_2403_19272_b200.subspace import build_subspace

        mesh = parts["mesh"]
        el = build_elastic(mesh, parts["stretch"], parts["bend"])
        sy = assemble_global(mesh, el, config.h)
        r_bar = min(config.r_bar, mesh.free.size)
        sub = build_subspace(sy, mesh.rest_positions[mesh.free], r_bar, min(config.r, r_bar))
        n = mesh.vertex_count
        verts, tris = [], [mesh.triangles]
        off = n
        for v, t in (parts.get("obstacles") or []):
            verts.append(np.asarray(v, dtype=np.float64))
            tris.append(np.asarray(t, dtype=np.int64) + off)
            off += len(v)
        wt = np.concatenate(tris)
        stat = np.zeros(len(wt), dtype=bool)
        stat[len(mesh.triangles):] = True
        obs = np.concatenate(verts) if verts else np.zeros((0, 3))
        k = config.ndb_k if config.ndb_k > 0 else el.mean_weight
        return cls(mesh, config, el, sy, sub, k, obs, wt, stat, parts.get("pin_motion"), parts.get("obstacle_motion"))

    @classmethod
    def from_simulation(cls, sim):
        """Clone the setup of a product Simulation (same arrays, host copies)."""
        o = cls(sim.mesh, sim.config, sim.elastic, sim.system, sim.subspace, sim.k, sim.obstacle_x,
                sim.world_triangles, sim.tri_static, sim.pin_motion, sim.obstacle_motion)
        o.state = sim.host_state()
        return o

    # ------------------------------------------------------------ helpers
    def world(self, cx, ox=None):
        ox = self.obstacle_x if ox is None else ox
        return np.concatenate([cx, ox]) if len(ox) else cx.copy()

    def _pins_at(self, t):
        if self.pin_motion is None or self.mesh.pinned.size == 0:
            return self.state.x[self.mesh.pinned]
        return np.asarray(self.pin_motion(t))

    def _obstacles_at(self, t):
        if self.obstacle_motion is None or not len(self.obstacle_x):
            return self.obstacle_x
        return np.asarray(self.obstacle_motion(t))

    def witness_into(self, pr: Pairs, xw):
        """stepper.py:194-216."""
        p1, p2, bary, dist = narrow.witness(pr.kind, pr.idx, xw)
        nrm = p1 - p2
        ln = np.linalg.norm(nrm, axis=1)
        good = ln > 1e-12
        nrm[good] /= ln[good, None]
        if (~good).any():
            bad = np.flatnonzero(~good)
            p = xw[pr.idx[bad]]
            alt = np.where((pr.kind[bad] == VT)[:, None],
                           np.cross(p[:, 2] - p[:, 1], p[:, 3] - p[:, 1]),
                           np.cross(p[:, 1] - p[:, 0], p[:, 3] - p[:, 2]))
            an = np.linalg.norm(alt, axis=1)
            alt[an > 0] /= an[an > 0, None]
            alt[an == 0] = (1.0, 0.0, 0.0)
            nrm[bad] = alt
        pr.bary, pr.dist, pr.normal = bary, dist, nrm

    def gaps(self, pr: Pairs, xw):
        """stepper.py:218-236."""
        if len(pr) == 0:
            return np.zeros(0)
        _, p1, p2 = _sides_at(pr.kind, pr.idx, pr.bary, xw)
        return np.einsum("mj,mj->m", p1 - p2, pr.normal)

    def collision_terms(self, pr: Pairs, engaged, xw):
        """stepper.py:238-285 -> (ids, weights, targets) or None."""
        sel = np.flatnonzero(engaged & (pr.weight > 0))
        if sel.size == 0:
            return None
        kind, idx, nrm, bary = pr.kind[sel], pr.idx[sel], pr.normal[sel], pr.bary[sel]
        gam = shares(kind, bary)
        p, p1, p2 = _sides_at(kind, idx, bary, xw)
        deficit = np.maximum(self.cfg.d_hat - np.einsum("mj,mj->m", p1 - p2, nrm), 0.0)
        nc = self.mesh.vertex_count
        movable = (idx < nc) & (self.mesh.free_index[np.minimum(idx, nc - 1)] >= 0)
        first = np.zeros((len(sel), 4), dtype=bool)
        first[kind == VT, 0] = True
        first[kind == EE, :2] = True
        m1 = (movable & first).any(axis=1)
        m2 = (movable & ~first).any(axis=1)
        both = m1 & m2
        s1 = np.where(both, 0.5, np.where(m1, 1.0, 0.0)) * deficit
        s2 = np.where(both, 0.5, np.where(m2, 1.0, 0.0)) * deficit
        move = np.where(first, s1[:, None], -s2[:, None])[:, :, None] * nrm[:, None, :]
        tg = (p + move).reshape(-1, 3)
        w = (pr.weight[sel][:, None] * gam).ravel()
        keep = movable.ravel() & (w > 0)
        return idx.ravel()[keep], w[keep], tg[keep]

    def carry_life(self, old: Pairs, new: Pairs):
        """stepper.py:300-305."""
        if len(old) == 0 or len(new) == 0:
            return
        table = {r.tobytes(): int(s) for r, s in zip(old.keys(), old.life)}
        new.life = np.array([table.get(r.tobytes(), 0) for r in new.keys()], dtype=np.int64)

    def ccd_site(self, xa, xb, rep):
        """broad -> full CCD -> distance march (stepper.py:426-443)."""
        t0 = time.perf_counter()
        kind, idx = broad_phase(xa, xb, self.topo, self.cfg.d_hat)
        rep["timings"]["broad"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        toi = narrow.full_ccd(kind, idx, xa, xb)
        filt = narrow.distance_toi(kind, idx, xa, xb, floor_frac=1.0 - self.cfg.alpha)
        rep["timings"]["narrow_full"] += time.perf_counter() - t0
        rep["full_ccd_calls"] += 1
        pr = Pairs(kind, idx, np.zeros(len(kind), np.int64), np.zeros(len(kind)))
        return pr, toi, filt

    def clamp(self, toi):
        """stepper.py:445-452."""
        fin = toi[~np.isnan(toi)]
        if fin.size == 0:
            return 1.0
        t = float(fin.min())
        if t <= 0.0:
            raise PenetrationError("impact at t<=0: step began in contact")
        return self.cfg.alpha * t

    def warm_start(self, z, pins):
        """stepper.py:384-400."""
        x = z.copy()
        fr = self.mesh.free
        if self.mesh.pinned.size:
            x[self.mesh.pinned] = pins
        its = 0
        for _ in range(self.cfg.warm_start_cap):
            b, _ = solver.assemble_rhs(self.sys, self.mesh, self.el, z, x, pins)
            xn = solver.warmstart_correction(self.sub, self.sys, b, x[fr])
            dx = rms(xn - x[fr])
            x[fr] = xn
            its += 1
            if dx < self.cfg.eps_initial:
                break
        return x, its

    def inner_solve(self, z, xc, pins, coll, rep):
        """stepper.py:402-424."""
        fr = self.mesh.free
        t0 = time.perf_counter()
        if coll is None:
            b, delta = solver.assemble_rhs(self.sys, self.mesh, self.el, z, xc, pins)
        else:
            b, delta = solver.assemble_rhs(self.sys, self.mesh, self.el, z, xc, pins, *coll)
        rep["timings"]["local"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        xf, _ = solver.reduced_correction(self.sub, self.sys, b, xc[fr], delta)
        rep["timings"]["global"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        xf = solver.ajacobi_smooth(self.sys, b, xf, self.cfg.smoothing_iterations, self.cfg.omega, delta)
        rep["timings"]["smoothing"] += time.perf_counter() - t0
        out = xc.copy()
        out[fr] = xf
        return out

    def energy(self, x, z, quad=None):
        return solver.energy(self.mesh, self.el, self.cfg.h, x, z, quad)

    # ------------------------------------------------------------ step
    def step(self):
        cfg, mesh, st = self.cfg, self.mesh, self.state
        dbb = cfg.barrier_mode == "dbb"
        rep = {"timings": {k: 0.0 for k in ("warm_start", "local", "global", "smoothing", "broad",
                                             "narrow_partial", "narrow_full")},
               "lg_iterations": 0, "outer_loops": 0, "full_ccd_calls": 0, "partial_ccd_calls": 0,
               "toi_exit": 1.0, "rf_triggered": False, "cap_hit": False, "active_pairs": 0}
        nc = mesh.vertex_count
        fr = mesh.free
        t_now = st.step_index * cfg.h
        pins = self._pins_at(t_now + cfg.h)
        obs_next = self._obstacles_at(t_now + cfg.h)
        # inertia target (mesh.py:174-196)
        z = st.x + cfg.h * st.x_dot + (cfg.h * cfg.h) * (self.gravity_force + st.delta_f) / mesh.vertex_mass[:, None]
        if mesh.pinned.size:
            z[mesh.pinned] = pins
        if not np.isfinite(z).all():
            raise FloatingPointError("non-finite inertia target")

        t0 = time.perf_counter()
        xc, _ = self.warm_start(z, pins)
        rep["timings"]["warm_start"] += time.perf_counter() - t0

        x_start_w = self.world(st.x)
        xc_w = self.world(xc, obs_next)
        pr, toi, filt = self.ccd_site(x_start_w, xc_w, rep)
        tc = self.clamp(filt)
        x_acc_w = x_start_w + tc * (xc_w - x_start_w) if tc < 1.0 else xc_w.copy()
        anchor_w = x_acc_w.copy()
        self.witness_into(pr, anchor_w)
        engaged = ~np.isnan(toi) | (pr.dist < 2.0 * cfg.d_hat)
        pr.life = np.zeros(len(pr), np.int64)
        if dbb:                                          # stepper.py:489-491
            pr.weight = dbb_weight(np.maximum(pr.dist, 1e-12), 2.0 * cfg.d_hat, self.kappa)
            engaged = pr.weight > 0
        else:
            pr.weight = np.where(engaged, ndb_weight(pr.life, self.k, cfg.ndb_base), 0.0)

        xc = x_acc_w[:nc].copy()
        obs_c = x_acc_w[nc:]
        pins_c = xc[mesh.pinned] if mesh.pinned.size else pins
        prev_outer = xc.copy()
        self.last_outer_deltas = []
        dx_last = np.inf
        cap_hit = False
        toi_exit = 1.0

        for _outer in range(cfg.outer_cap):
            for _inner in range(cfg.inner_cap):
                coll = self.collision_terms(pr, engaged, self.world(xc, obs_c))
                xn = self.inner_solve(z, xc, pins_c, coll, rep)
                dx_last = rms(xn[fr] - xc[fr])
                xc = xn
                rep["lg_iterations"] += 1
                xc_w = self.world(xc, obs_c)
                rep["partial_ccd_calls"] += 1
                if dbb:
                    # baseline: the partial-CCD classes are unused (stepper.py:513, 524-538);
                    # distances refreshed with the full distance march + clamp
                    toi_in = narrow.distance_toi(pr.kind, pr.idx, anchor_w, xc_w, floor_frac=1.0 - cfg.alpha)
                    t_in = self.clamp(toi_in)
                    if t_in < 1.0:
                        cw = anchor_w + t_in * (xc_w - anchor_w)
                        xc = cw[:nc].copy()
                        obs_c = cw[nc:]
                        pins_c = xc[mesh.pinned] if mesh.pinned.size else pins_c
                    self.witness_into(pr, self.world(xc, obs_c))
                    pr.weight = dbb_weight(np.maximum(pr.dist, 1e-12), 2.0 * cfg.d_hat, self.kappa)
                    engaged = pr.weight > 0
                else:
                    t0 = time.perf_counter()
                    active = narrow.partial_ccd(pr.kind, pr.idx, anchor_w, xc_w, cfg.samples)
                    rep["timings"]["narrow_partial"] += time.perf_counter() - t0
                    gap = self.gaps(pr, xc_w)
                    active = active | (gap < cfg.d_hat)
                    pr.life = np.where(active, np.minimum(pr.life + 1, LIFE_CAP), 0)
                    engaged = active | (gap < 2.0 * cfg.d_hat)
                    pr.weight = np.where(engaged, ndb_weight(pr.life, self.k, cfg.ndb_base), 0.0)
                if cfg.iteration_cap and rep["lg_iterations"] >= cfg.iteration_cap:
                    cap_hit = True
                    break
                if dx_last <= cfg.eps_inner:
                    break
            rep["outer_loops"] += 1
            xc_w = self.world(xc, obs_c)
            npr, toi, filt = self.ccd_site(anchor_w, xc_w, rep)
            tout = self.clamp(filt)
            if tout < 1.0:
                xc_w = anchor_w + tout * (xc_w - anchor_w)
                xc = xc_w[:nc].copy()
                obs_c = xc_w[nc:]
                pins_c = xc[mesh.pinned] if mesh.pinned.size else pins_c
                toi_exit = min(toi_exit, tout)
            anchor_w = xc_w.copy()
            self.witness_into(npr, anchor_w)
            if dbb:
                npr.weight = dbb_weight(np.maximum(npr.dist, 1e-12), 2.0 * cfg.d_hat, self.kappa)
                engaged = npr.weight > 0
            else:
                self.carry_life(pr, npr)
                engaged = ~np.isnan(toi) | (npr.dist < 2.0 * cfg.d_hat)
                npr.weight = np.where(engaged, ndb_weight(npr.life, self.k, cfg.ndb_base), 0.0)
            pr = npr
            d_out = rms(xc[fr] - prev_outer[fr])
            self.last_outer_deltas.append(d_out)
            prev_outer = xc.copy()
            if cap_hit or d_out <= cfg.eps_outer:
                break

        xc_w = self.world(xc, obs_c)
        exit_pr, toi, filt = self.ccd_site(anchor_w, xc_w, rep)
        tfin = self.clamp(filt)
        x_final_w = anchor_w + tfin * (xc_w - anchor_w) if tfin < 1.0 else xc_w
        toi_exit = min(toi_exit, tfin)
        rep["toi_exit"] = toi_exit
        rep["cap_hit"] = cap_hit
        rep["active_pairs"] = int(np.count_nonzero(engaged)) if len(pr) else 0

        from paper_2403_19272_b200.mesh import SimState

        x_final = x_final_w[:nc].copy()
        new = SimState(x=x_final, x_dot=(x_final - st.x) / cfg.h, x_prev=st.x.copy(),
                       delta_f=np.zeros_like(st.x), step_index=st.step_index + 1)
        self.obstacle_x = x_final_w[nc:].copy()
        if toi_exit < cfg.eps_toi or (cap_hit and dx_last > cfg.eps_outer):
            if len(exit_pr):
                self.witness_into(exit_pr, x_final_w)
            new.delta_f = self.residual_forward(x_final, z, exit_pr, x_final_w)
            rep["rf_triggered"] = True
        rep["timings"] = {k: v * 1e3 for k, v in rep["timings"].items()}
        self.state = new
        return rep

    def residual_forward(self, x, z, pr: Pairs, xw):
        """stepper.py:626-672."""
        mesh, cfg = self.mesh, self.cfg
        nc = mesh.vertex_count
        engaged = pr.dist < 2.0 * cfg.d_hat if len(pr) else np.zeros(0, dtype=bool)
        frozen = Pairs(pr.kind, pr.idx, np.zeros(len(pr), np.int64), np.where(engaged, self.k, 0.0),
                       pr.bary, pr.dist, pr.normal)
        coll = self.collision_terms(frozen, engaged, xw) if len(pr) else None
        quad = None
        if coll is not None:
            ids, w, tg = coll
            c = ids < nc
            quad = (ids[c], w[c], tg[c])
        _, grad, _ = self.energy(x, z, quad)
        f_r = -grad[mesh.free]
        delta = np.zeros(mesh.free.size)
        if quad is not None:
            rows = mesh.free_index[quad[0]]
            ok = rows >= 0
            np.add.at(delta, rows[ok], quad[1][ok])
        dx = np.zeros((mesh.free.size, 3))
        red = None
        for _ in range(cfg.rf_iterations):
            dx, red = solver.reduced_correction(self.sub, self.sys, f_r, dx, delta, red)
            dx = solver.ajacobi_smooth(self.sys, f_r, dx, cfg.smoothing_iterations, cfg.omega, delta)
            res = f_r - self.sys.H @ dx - delta[:, None] * dx
            if float(np.linalg.norm(res)) <= cfg.rf_tolerance * max(float(np.linalg.norm(f_r)), 1e-30):
                break
        out = np.zeros_like(x)
        out[mesh.free] = 2.0 * mesh.vertex_mass[mesh.free, None] * dx / (cfg.h * cfg.h)
        nrm = float(np.linalg.norm(out))
        if nrm > cfg.delta_f_cap:
            out *= cfg.delta_f_cap / nrm
        return out
