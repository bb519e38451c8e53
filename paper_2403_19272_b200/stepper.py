"""Drop-in ``Simulation`` (reference pkg/src/clothsim/stepper.py:124-681).

Same constructor, attributes and ``step()/run()`` contract as the reference.
Scene setup (elastic weights, H, eigenbasis, static collision topology) runs
once on the host; every step runs on the GPU inside ``cs_step`` (the native
driver in csrc/abi.cu), so Python crosses the C ABI once per frame.  Prescribed
pin/obstacle motion callbacks stay in Python (as in the reference) and their
values are uploaded each step.

``state`` is the device-resident ``SimState``: reading it downloads a host
mirror; in-place edits of that mirror (reference tests do
``sim.state.x_dot[:] = ...``) are written back before the next device call.
"""

from __future__ import annotations

import contextlib
import ctypes
import time

import numpy as np

from . import _lib
from .collision import CollisionWorld, PairSet, VT, EE, default_samples
from .constraints import assemble_global, build_elastic
from .device import scene_desc, step_config_c
from .mesh import ClothMesh, SimState
from .stepconfig import StepConfig, StepReport
from .subspace import build_subspace

PenetrationError = _lib.PenetrationError

_TIMING_KEYS = ("warm_start", "local", "global", "smoothing", "broad", "narrow_partial", "narrow_full")


def _rms(v: np.ndarray) -> float:
    return float(np.linalg.norm(v)) / max(np.sqrt(v.size), 1.0)


class _Tracked(np.ndarray):
    """ndarray view of a downloaded state field that records writes, so only modified
    fields are written back to the device.

    The field is handed out READ-ONLY at the numpy level; the writers numpy routes
    through the subclass (item assignment, in-place / ``out=`` ufuncs incl.
    ``np.add.at``, ``np.copyto`` / ``np.put`` / ``np.place`` / ``np.putmask``,
    ``.fill`` / ``.put`` / ``.sort``) open it for the write and mark the field
    dirty.  Any other write path (e.g. through ``np.asarray(field)``) raises
    "assignment destination is read-only" instead of being silently lost."""

    _WRITERS = ("copyto", "put", "place", "putmask", "fill_diagonal")

    # views keep a reference to the root array (never to themselves: a self-cycle would
    # leave the array to the cyclic GC and delay recycling its pinned buffer)
    def __array_finalize__(self, obj):
        if isinstance(obj, _Tracked):
            self._root = obj._root if obj._root is not None else obj
        else:
            self._root = None
        self._dirty = False

    @classmethod
    def wrap(cls, a: np.ndarray) -> "_Tracked":
        t = a.view(cls)
        t._dirty = False
        t.flags.writeable = False
        return t

    def _mark(self):
        (self._root if self._root is not None else self)._dirty = True

    @contextlib.contextmanager
    def _open(self):
        """Root and this view writeable for one write; yields a plain ndarray view."""
        root = self._root if self._root is not None else self
        self._mark()
        prev = root.flags.writeable
        root.flags.writeable = True
        own = self is not root and not self.flags.writeable
        if own:
            self.flags.writeable = True
        try:
            yield self.view(np.ndarray)
        finally:
            if own:
                self.flags.writeable = False
            root.flags.writeable = prev

    def __setitem__(self, key, value):
        with self._open() as w:
            w[key] = value

    def fill(self, value):
        with self._open() as w:
            w.fill(value)

    def put(self, *args, **kw):
        with self._open() as w:
            w.put(*args, **kw)

    def sort(self, *args, **kw):
        with self._open() as w:
            w.sort(*args, **kw)

    def __array_ufunc__(self, ufunc, method, *inputs, out=None, **kw):
        # arithmetic yields plain arrays; in-place ufuncs (out= / ufunc.at on a state
        # field) write through an opened view and mark the field dirty
        plain = tuple(a.view(np.ndarray) if isinstance(a, _Tracked) else a for a in inputs)
        with contextlib.ExitStack() as stack:
            if method == "at" and isinstance(inputs[0], _Tracked):
                plain = (stack.enter_context(inputs[0]._open()),) + plain[1:]
            if out is not None:
                kw["out"] = tuple(stack.enter_context(o._open()) if isinstance(o, _Tracked) else o for o in out)
            return getattr(ufunc, method)(*plain, **kw)

    def __array_function__(self, func, types, args, kwargs):
        if func.__name__ in self._WRITERS and args and isinstance(args[0], _Tracked):
            with args[0]._open() as w:
                return func(w, *args[1:], **kwargs)
        return super().__array_function__(func, types, args, kwargs)


class DeviceSimState:
    """SimState (reference mesh.py:55-73) backed by the device state: fields download
    lazily and are cached; in-place edits of a cached field (the reference tests do
    ``sim.state.x_dot[:] = ...``) are written back before the next device call."""

    FIELDS = ("x", "x_dot", "x_prev", "delta_f")

    def __init__(self, sim, step_index=None):
        self._sim = sim
        self._cache = {}
        self.step_index = sim._step_index if step_index is None else step_index

    def _field(name):
        def get(self):
            a = self._cache.get(name)
            if a is None:
                a = self._cache[name] = _Tracked.wrap(self._sim._download(name))
            return a

        def put(self, value):
            a = np.array(value, dtype=np.float64).view(_Tracked)
            a._dirty = True
            self._cache[name] = a

        return property(get, put)

    def dirty(self, name) -> bool:
        a = self._cache.get(name)
        return a is not None and bool(a._dirty)

    x = _field("x")
    x_dot = _field("x_dot")
    x_prev = _field("x_prev")
    delta_f = _field("delta_f")
    del _field


class Simulation:
    """One cloth plus optional obstacle meshes, stepped on the GPU under a StepConfig."""

    def __init__(self, mesh: ClothMesh, config: StepConfig, stretch_stiffness: float = 160.0,
                 bend_stiffness: float = 3e-4, obstacles=None, pin_motion=None, obstacle_motion=None,
                 eigensolver: str = "host"):
        self.mesh = mesh
        self.config = config
        self.elastic = build_elastic(mesh, stretch_stiffness, bend_stiffness)
        self.system = assemble_global(mesh, self.elastic, config.h)
        r_bar = min(config.r_bar, mesh.free.size)
        r = min(config.r, r_bar)
        self.subspace = build_subspace(self.system, mesh.rest_positions[mesh.free], r_bar, r, method=eigensolver)
        self.samples = default_samples(config.samples)
        self.pin_motion = pin_motion
        self.obstacle_motion = obstacle_motion

        n = mesh.vertex_count
        verts, tris = [], []
        offset = n
        for ov, ot in (obstacles or []):
            verts.append(np.asarray(ov, dtype=np.float64))
            tris.append(np.asarray(ot, dtype=np.int64) + offset)
            offset += len(ov)
        obstacle_x = np.concatenate(verts) if verts else np.zeros((0, 3))
        self.world_triangles = np.concatenate([mesh.triangles] + tris) if tris else mesh.triangles
        self.tri_static = np.zeros(len(self.world_triangles), dtype=bool)
        self.tri_static[len(mesh.triangles):] = True
        world_rest = np.concatenate([mesh.rest_positions, obstacle_x])
        self.bvh = CollisionWorld.build(self.world_triangles, world_rest, self.tri_static)

        self.k = config.ndb_k if config.ndb_k > 0 else self.elastic.mean_weight
        self.kappa = config.dbb_kappa if config.dbb_kappa > 0 else self.k / ((config.d_hat / 2.0) ** 2 * np.log(2.0))
        self.gravity_force = mesh.vertex_mass[:, None] * np.asarray(config.gravity)
        self._verify_oracle = None
        self._device_verify = False
        self.last_outer_deltas = []
        self.last_report_c = None

        self._lib = _lib.load()
        desc, keep = scene_desc(mesh, self.elastic, self.system, self.subspace, self.bvh, obstacle_x,
                                self.gravity_force, mesh.rest_positions)
        self._cfg_c = step_config_c(config, self.k, self.kappa)
        status = ctypes.c_int(0)
        self._scene = self._lib.cs_scene_create(ctypes.byref(desc), ctypes.byref(self._cfg_c), ctypes.byref(status))
        del keep
        if not self._scene:
            _lib.check(status.value or _lib.CS_BAD_ARGUMENT, "cs_scene_create")
        self._n_obs = len(obstacle_x)
        self._host_state = None
        self._host_obstacles = None
        self._obs_dirty = False
        self._pin_pool = {}
        self._step_index = 0
        # page-locked download buffers are allocated once, here (a cudaHostAlloc of a
        # large array costs milliseconds): two, so a result still referenced by the
        # caller does not force an allocation in the step loop
        self._prealloc_pinned(self.mesh.vertex_count, 2)

    def _prealloc_pinned(self, rows: int, count: int) -> None:
        import torch

        pool = self._pin_pool.setdefault(rows, [])
        for _ in range(count - len(pool)):
            pool.append(torch.empty((rows, 3), dtype=torch.float64, pin_memory=True))

    def __del__(self):
        scene = getattr(self, "_scene", None)
        if scene:
            self._lib.cs_scene_destroy(scene)
            self._scene = None

    @property
    def config(self) -> StepConfig:
        return self._config

    @config.setter
    def config(self, cfg: StepConfig) -> None:
        """Replacing the config takes effect at the next step, as in the reference (which
        reads self.config inside step()); k / kappa stay as resolved at construction
        (stepper.py:164-169)."""
        self._config = cfg
        if getattr(self, "_scene", None):
            self._cfg_c = step_config_c(cfg, self.k, self.kappa)
            _lib.check(self._lib.cs_scene_set_config(self._scene, ctypes.byref(self._cfg_c)), "cs_scene_set_config")

    # ------------------------------------------------------------ state mirror
    def _stream(self):
        return _lib.stream_handle()

    def _flush(self):
        """Write back host-mirror edits (fields that were read or assigned) before
        the device uses the state."""
        st = self._host_state
        obs = self._host_obstacles
        if st is None and obs is None:
            return
        ptrs = []
        keep = []
        for name in DeviceSimState.FIELDS:
            if st is None or not st.dirty(name):
                ptrs.append(None)
                continue
            a = np.ascontiguousarray(np.asarray(st._cache[name]), dtype=np.float64)
            keep.append(a)
            ptrs.append(a.ctypes.data)
        obs_dirty = self._obs_dirty or (isinstance(obs, _Tracked) and obs._dirty)
        o = np.ascontiguousarray(obs, dtype=np.float64) if (obs is not None and self._n_obs and obs_dirty) else None
        step = int(st.step_index) if st is not None else -1
        _lib.check(self._lib.cs_set_state(self._scene, *ptrs, o.ctypes.data if o is not None else None, step,
                                          self._stream()), "cs_set_state")
        self._obs_dirty = False
        if isinstance(obs, _Tracked):
            obs._dirty = False
        if st is not None:
            self._step_index = step
            for name in DeviceSimState.FIELDS:
                if st.dirty(name):
                    st._cache[name]._dirty = False

    def _pinned(self, rows: int) -> np.ndarray:
        """A (rows, 3) fp64 array in page-locked memory from a recycling pool: the device
        copies into it at full DMA rate (no staging memcpy), and the buffer returns to
        the pool once the last view of the array is garbage collected."""
        import weakref

        import torch

        pool = self._pin_pool.setdefault(rows, [])
        buf = pool.pop() if pool else torch.empty((rows, 3), dtype=torch.float64, pin_memory=True)
        arr = buf.numpy()
        weakref.finalize(arr, pool.append, buf)
        return arr

    def _download(self, name: str) -> np.ndarray:
        """One state field (n, 3) from the device (cs_get_state with only that pointer)."""
        rows = self.mesh.vertex_count if name != "obstacle_x" else self._n_obs
        out = self._pinned(rows) if rows else np.empty((0, 3))
        ptrs = [None] * 5
        ptrs[(*DeviceSimState.FIELDS, "obstacle_x").index(name)] = out.ctypes.data if out.size else None
        idx = ctypes.c_int(0)
        _lib.check(self._lib.cs_get_state(self._scene, *ptrs, ctypes.byref(idx), self._stream()), "cs_get_state")
        return out

    def host_state(self) -> SimState:
        """Full host copy of the device state (all fields)."""
        return SimState(**{k: self._download(k) for k in DeviceSimState.FIELDS}, step_index=self._step_index)

    @property
    def state(self):
        """``SimState`` view of the device state; each field downloads on first access,
        so reading ``sim.state.x`` moves only the positions."""
        if self._host_state is None:
            self._host_state = DeviceSimState(self)
        return self._host_state

    @state.setter
    def state(self, st):
        ds = DeviceSimState(self, step_index=int(st.step_index))
        for k in DeviceSimState.FIELDS:
            setattr(ds, k, getattr(st, k))
        self._host_state = ds

    @property
    def obstacle_x(self) -> np.ndarray:
        if self._host_obstacles is None:
            self._host_obstacles = _Tracked.wrap(self._download("obstacle_x"))
        return self._host_obstacles

    @obstacle_x.setter
    def obstacle_x(self, value):
        self._host_obstacles = np.array(value, dtype=np.float64).reshape(-1, 3)
        self._obs_dirty = True

    # ------------------------------------------------------------ reference helpers
    def world(self, cloth_x: np.ndarray, obstacle_x: np.ndarray | None = None) -> np.ndarray:
        """stepper.py:177-180."""
        if obstacle_x is None:
            obstacle_x = self.obstacle_x
        return np.concatenate([cloth_x, obstacle_x]) if len(obstacle_x) else cloth_x.copy()

    def _pin_targets(self, t: float):
        if self.pin_motion is None or self.mesh.pinned.size == 0:
            return None
        return np.ascontiguousarray(self.pin_motion(t), dtype=np.float64).reshape(-1, 3)

    def _obstacle_targets(self, t: float):
        if self.obstacle_motion is None or not self._n_obs:
            return None
        return np.ascontiguousarray(self.obstacle_motion(t), dtype=np.float64).reshape(-1, 3)

    # ------------------------------------------------------------ stepping
    def step(self) -> StepReport:
        """One Delta-t step on the GPU (reference stepper.py:454-624)."""
        cfg = self.config
        self._flush()
        t_now = self._step_index * cfg.h
        pins = self._pin_targets(t_now + cfg.h)
        obs = self._obstacle_targets(t_now + cfg.h)
        rep = _lib.StepReportC()
        # host-oracle verify mode checks after the device step: keep the state to roll
        # back to (the reference raises before `self.state = new_state`)
        host_verify = bool(cfg.verify and self._verify_oracle is not None)
        if host_verify:
            saved = (self.host_state(), np.array(self.obstacle_x, copy=True), self._step_index)
        # verify mode without an injected host oracle: the device intersection check
        # (csrc/intersect.cu, reference oracles.py:83-131) runs inside cs_step on x_final
        device_verify = bool(cfg.verify and self._verify_oracle is None)
        if device_verify != self._device_verify:
            _lib.check(self._lib.cs_scene_set_verify(self._scene, int(device_verify)), "cs_scene_set_verify")
            self._device_verify = device_verify
        rc = self._lib.cs_step(self._scene, pins.ctypes.data if pins is not None else None,
                               obs.ctypes.data if obs is not None else None, ctypes.byref(rep), self._stream())
        # a failed step leaves the state untouched (the reference raises before assigning)
        self._host_state = None
        self._host_obstacles = None
        if rc == _lib.CS_PENETRATION and device_verify:
            count = ctypes.c_longlong(0)
            self._lib.cs_last_intersections(self._scene, ctypes.byref(count), None, 0, None)
            if count.value:
                k = min(count.value, 1024)
                pairs = np.zeros((k, 2), np.int32)
                x_final = np.empty((self.mesh.vertex_count, 3))
                self._lib.cs_last_intersections(self._scene, None, pairs.ctypes.data, k, x_final.ctypes.data)
                pairs = pairs.astype(np.int64)
                pairs = pairs[np.lexsort((pairs[:, 1], pairs[:, 0]))]
                raise PenetrationError(f"step {self._step_index}: {count.value} intersecting triangle pairs",
                                       state_dump={"x": x_final, "pairs": pairs})
        _lib.check(rc, "cs_step")
        self._step_index += 1
        self.last_report_c = rep
        self.last_outer_deltas = [rep.outer_deltas[i] for i in range(rep.n_outer_deltas)]
        report = StepReport(
            lg_iterations=rep.lg_iterations, outer_loops=rep.outer_loops, toi_exit=rep.toi_exit,
            rf_triggered=bool(rep.rf_triggered), active_pairs=rep.active_pairs, full_ccd_calls=rep.full_ccd_calls,
            partial_ccd_calls=rep.partial_ccd_calls, cap_hit=bool(rep.cap_hit),
            timings={"warm_start": rep.t_warm_start, "local": rep.t_local, "global": rep.t_global,
                     "smoothing": rep.t_smoothing, "broad": rep.t_broad, "narrow_partial": rep.t_narrow_partial,
                     "narrow_full": rep.t_narrow_full, "rf": rep.t_rf})
        if device_verify:
            report.penetration_free = True
        elif host_verify:
            x_final = np.array(self.state.x, copy=True)
            xw = self.world(x_final)
            bad = self._verify_oracle(xw, self.bvh.triangles)
            report.penetration_free = len(bad) == 0
            if not report.penetration_free:
                st, obs, idx = saved
                self.state = st
                self.obstacle_x = obs
                self._flush()
                self._step_index = idx
                raise PenetrationError(f"step {idx}: {len(bad)} intersecting triangle pairs",
                                       state_dump={"x": x_final, "pairs": bad})
        return report

    def run(self, steps: int, on_step=None) -> list:
        """reference stepper.py:674-681."""
        out = []
        for _ in range(steps):
            rep = self.step()
            out.append(rep)
            if on_step is not None:
                on_step(self, rep)
        return out

    # ------------------------------------------------------------ stage-level API (device)
    def _dbuf(self, a):
        import torch

        return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")

    def warm_start(self, z: np.ndarray, pin_next: np.ndarray):
        """Collision-free LG iterations in the wide basis (stepper.py:384-400), device stages."""
        import torch

        cfg, mesh = self.config, self.mesh
        self._flush()
        x = np.array(z, dtype=np.float64)
        if mesh.pinned.size:
            x[mesh.pinned] = pin_next
        # device buffers are plumbing; the arithmetic is cs_assemble_rhs /
        # cs_warmstart_correction, the gathers and the exit norm are host glue
        zd = self._dbuf(z)
        b = torch.empty((mesh.free.size, 3), dtype=torch.float64, device="cuda")
        delta = torch.empty(mesh.free.size, dtype=torch.float64, device="cuda")
        its = 0
        for _ in range(cfg.warm_start_cap):
            xd = self._dbuf(x)
            _lib.check(self._lib.cs_assemble_rhs(self._scene, zd.data_ptr(), xd.data_ptr(), None, None, None, None, 0,
                                                 b.data_ptr(), delta.data_ptr(), self._stream()), "cs_assemble_rhs")
            x0 = np.ascontiguousarray(x[mesh.free])
            xf = self._dbuf(x0)
            _lib.check(self._lib.cs_warmstart_correction(self._scene, b.data_ptr(), xf.data_ptr(), self._stream()),
                       "cs_warmstart_correction")
            xn = xf.cpu().numpy()
            dx = float(np.linalg.norm(xn - x0)) / max(np.sqrt(xn.size), 1.0)
            x[mesh.free] = xn
            its += 1
            if dx < cfg.eps_initial:
                break
        return x, its

    def energy(self, x: np.ndarray, z: np.ndarray, collision=None):
        """Energy and gradient (stepper.py:309-380, 'quad' form).

        The gradient comes from the device kernel the residual forwarding uses;
        the scalar energy terms are a host diagnostic (not on the step path).
        """
        import torch

        mesh, el, h = self.mesh, self.elastic, self.config.h
        x = np.asarray(x, dtype=np.float64)
        z = np.asarray(z, dtype=np.float64)
        s = mesh.vertex_mass[:, None] / (h * h)
        e_in = 0.5 * float(np.sum(s * (x - z) ** 2))
        ln = np.linalg.norm(x[el.edges[:, 1]] - x[el.edges[:, 0]], axis=1)
        e_st = 0.5 * float((el.stretch_w * (ln - el.edge_rest) ** 2).sum())
        e_b = 0.0
        if len(el.stencils):
            flat = np.einsum("sj,sjd->sd", el.bend_k, x[el.stencils])
            e_b = 0.5 * float(np.sum(el.bend_w * np.einsum("sd,sd->s", flat, flat)))
        e_c = 0.0
        ids = w = tg = None
        nq = 0
        if collision is not None:
            if collision[0] != "quad":
                raise ValueError(f"unknown collision energy form {collision[0]!r}")
            _, ids_h, w_h, tg_h = collision
            diff = x[ids_h] - tg_h
            e_c = 0.5 * float(np.sum(w_h * np.einsum("mj,mj->m", diff, diff)))
            ids = torch.as_tensor(np.asarray(ids_h, dtype=np.int32), device="cuda")
            w = self._dbuf(w_h)
            tg = self._dbuf(tg_h)
            nq = len(ids_h)
        grad = torch.empty((mesh.vertex_count, 3), dtype=torch.float64, device="cuda")
        xd, zd = self._dbuf(x), self._dbuf(z)
        _lib.check(self._lib.cs_energy_gradient(self._scene, xd.data_ptr(), zd.data_ptr(),
                                                ids.data_ptr() if nq else None, w.data_ptr() if nq else None,
                                                tg.data_ptr() if nq else None, nq, grad.data_ptr(), self._stream()),
                   "cs_energy_gradient")
        total = e_in + e_st + e_b + e_c
        return total, grad.cpu().numpy(), {"inertia": e_in, "stretch": e_st, "bend": e_b, "barrier": e_c}

    def broad_phase(self, x_start_w, x_end_w, margin: float | None = None) -> PairSet:
        """Device broad phase over this scene's world (reference bvh.py:207-292)."""
        import torch

        margin = self.config.d_hat if margin is None else margin
        a, b = self._dbuf(x_start_w), self._dbuf(x_end_w)
        count = ctypes.c_longlong(0)
        _lib.check(self._lib.cs_broad_phase(self._scene, a.data_ptr(), b.data_ptr(), margin, ctypes.byref(count),
                                            self._stream()), "cs_broad_phase")
        P = count.value
        kind = torch.empty(max(P, 1), dtype=torch.int8, device="cuda")
        idx = torch.empty((max(P, 1), 4), dtype=torch.int32, device="cuda")
        _lib.check(self._lib.cs_scene_pairs(self._scene, kind.data_ptr(), idx.data_ptr(), self._stream()),
                   "cs_scene_pairs")
        kind = kind[:P].cpu().numpy()
        idx = idx[:P].cpu().numpy().astype(np.int64)
        return PairSet(kind=kind, idx=idx, life_span=np.zeros(P, np.int64), weight=np.zeros(P))

    def _full_ccd_site(self, x_from_w, x_to_w, report=None):
        """Broad phase + full CCD + distance march of one CCD site on the device
        (reference stepper.py:426-443); returns (pairs, toi, toi_filter) as numpy.
        The clamp of stepper.py:445-452 is applied by ``_clamp``."""
        import torch

        a, b = self._dbuf(x_from_w), self._dbuf(x_to_w)
        count = ctypes.c_longlong(0)
        clamp = ctypes.c_double(1.0)
        rc = self._lib.cs_ccd_site(self._scene, a.data_ptr(), b.data_ptr(), ctypes.byref(count), ctypes.byref(clamp),
                                   self._stream())
        if rc not in (_lib.CS_OK, _lib.CS_PENETRATION):
            _lib.check(rc, "cs_ccd_site")
        P = count.value
        n = max(P, 1)
        kind = torch.empty(n, dtype=torch.int8, device="cuda")
        idx = torch.empty((n, 4), dtype=torch.int32, device="cuda")
        toi = torch.empty(n, dtype=torch.float64, device="cuda")
        filt = torch.empty(n, dtype=torch.float64, device="cuda")
        _lib.check(self._lib.cs_scene_pairs(self._scene, kind.data_ptr(), idx.data_ptr(), self._stream()),
                   "cs_scene_pairs")
        _lib.check(self._lib.cs_scene_pair_results(self._scene, toi.data_ptr(), filt.data_ptr(), self._stream()),
                   "cs_scene_pair_results")
        if report is not None:
            report.full_ccd_calls += 1
        pairs = PairSet(kind=kind[:P].cpu().numpy(), idx=idx[:P].cpu().numpy().astype(np.int64),
                        life_span=np.zeros(P, np.int64), weight=np.zeros(P))
        return pairs, toi[:P].cpu().numpy(), filt[:P].cpu().numpy()

    def _clamp(self, toi: np.ndarray) -> float:
        """stepper.py:445-452."""
        finite = toi[~np.isnan(toi)]
        if finite.size == 0:
            return 1.0
        t = float(finite.min())
        if t <= 0.0:
            raise PenetrationError("impact at t<=0: step began in contact")
        return self.config.alpha * t

    def intersecting_pairs(self, x_world=None) -> np.ndarray:
        """All intersecting non-adjacent world-triangle pairs as sorted (k, 2) rows,
        computed on the device (reference oracles.py:83-131); x_world None = current state."""
        cap = 4096
        while True:
            count = ctypes.c_longlong(0)
            pairs = np.zeros((cap, 2), np.int32)
            xd = self._dbuf(x_world) if x_world is not None else None
            _lib.check(self._lib.cs_intersections(self._scene, xd.data_ptr() if xd is not None else None,
                                                  ctypes.byref(count), pairs.ctypes.data, cap, self._stream()),
                       "cs_intersections")
            if count.value <= cap:
                out = pairs[:count.value].astype(np.int64)
                return out[np.lexsort((out[:, 1], out[:, 0]))]
            cap = int(count.value)

    # ------------------------------------------------------------ contact helpers (device)
    def _witness(self, pairs: PairSet, x_ref) -> None:
        """Refresh bary / distance / separating normal at x_ref (reference stepper.py:194-216)."""
        from .collision import witness_normals

        pairs.bary, pairs.distance, pairs.normal = witness_normals(pairs.kind, pairs.idx, x_ref)

    def _collision_terms(self, pairs: PairSet, engaged, x_cand):
        """(ids, weights, targets) of the engaged pairs at x_cand, computed by the device
        kernel the step uses (reference stepper.py:238-285); None when nothing engages."""
        import torch

        P = len(pairs)
        if P == 0:
            return None
        dev = lambda a, t: torch.as_tensor(np.ascontiguousarray(a, dtype=t), device="cuda")  # noqa: E731
        k, i = dev(pairs.kind, np.int8), dev(pairs.idx, np.int32)
        bary, nrm = dev(pairs.bary, np.float64), dev(pairs.normal, np.float64)
        w, eng = dev(pairs.weight, np.float64), dev(np.asarray(engaged, dtype=bool), np.uint8)
        xw = dev(x_cand, np.float64)
        ids = torch.empty(4 * P, dtype=torch.int32, device="cuda")
        wo = torch.empty(4 * P, dtype=torch.float64, device="cuda")
        to = torch.empty((4 * P, 3), dtype=torch.float64, device="cuda")
        count = ctypes.c_longlong(0)
        _lib.check(self._lib.cs_collision_terms(self._scene, k.data_ptr(), i.data_ptr(), bary.data_ptr(),
                                                nrm.data_ptr(), w.data_ptr(), eng.data_ptr(), P, xw.data_ptr(),
                                                ids.data_ptr(), wo.data_ptr(), to.data_ptr(), ctypes.byref(count),
                                                self._stream()), "cs_collision_terms")
        m = count.value
        if m == 0:
            return None
        return ids[:m].cpu().numpy().astype(np.int64), wo[:m].cpu().numpy(), to[:m].cpu().numpy()

    def residual_forward(self, x, z, pairs: PairSet, x_world) -> np.ndarray:
        """Forwarded force from the exit residual (reference stepper.py:626-672), run with
        the device stages: frozen-weight collision terms, energy gradient, reduced
        corrections + A-Jacobi smoothing with the residual check on device."""
        import torch

        mesh, cfg = self.mesh, self.config
        self._flush()
        quad = None
        if len(pairs):
            engaged = pairs.distance < 2.0 * cfg.d_hat
            frozen = PairSet(kind=pairs.kind, idx=pairs.idx, life_span=np.zeros(len(pairs), np.int64),
                             weight=np.where(engaged, self.k, 0.0), bary=pairs.bary, distance=pairs.distance,
                             normal=pairs.normal)
            coll = self._collision_terms(frozen, engaged, x_world)
            if coll is not None:
                ids, w, tg = coll
                cl = ids < mesh.vertex_count
                quad = ("quad", ids[cl], w[cl], tg[cl])
        _, grad, _ = self.energy(x, z, collision=quad)
        nf = mesh.free.size
        f_r = self._dbuf(-grad[mesh.free])
        delta = torch.zeros(nf, dtype=torch.float64, device="cuda")
        if quad is not None:
            ids_d = torch.as_tensor(quad[1].astype(np.int32), device="cuda")
            w_d, t_d = self._dbuf(quad[2]), self._dbuf(quad[3])
            b = torch.empty((nf, 3), dtype=torch.float64, device="cuda")
            zz = self._dbuf(z)
            _lib.check(self._lib.cs_assemble_rhs(self._scene, zz.data_ptr(), zz.data_ptr(), None, ids_d.data_ptr(),
                                                 w_d.data_ptr(), t_d.data_ptr(), len(quad[1]), b.data_ptr(),
                                                 delta.data_ptr(), self._stream()), "cs_assemble_rhs")
        dx = torch.zeros((nf, 3), dtype=torch.float64, device="cuda")
        r = torch.empty_like(dx)
        fnorm = float(np.linalg.norm(grad[mesh.free]))
        for it in range(cfg.rf_iterations):
            _lib.check(self._lib.cs_reduced_correction(self._scene, f_r.data_ptr(), dx.data_ptr(), delta.data_ptr(),
                                                       int(it > 0), self._stream()), "cs_reduced_correction")
            _lib.check(self._lib.cs_ajacobi_smooth(self._scene, f_r.data_ptr(), dx.data_ptr(),
                                                   cfg.smoothing_iterations, cfg.omega, delta.data_ptr(),
                                                   self._stream()), "cs_ajacobi_smooth")
            _lib.check(self._lib.cs_residual(self._scene, f_r.data_ptr(), dx.data_ptr(), delta.data_ptr(),
                                             r.data_ptr(), self._stream()), "cs_residual")
            if float(np.linalg.norm(r.cpu().numpy())) <= cfg.rf_tolerance * max(fnorm, 1e-30):
                break
        delta_f = np.zeros_like(np.asarray(x, dtype=np.float64))
        delta_f[mesh.free] = 2.0 * mesh.vertex_mass[mesh.free, None] * dx.cpu().numpy() / (cfg.h * cfg.h)
        norm = float(np.linalg.norm(delta_f))
        if norm > cfg.delta_f_cap:
            delta_f *= cfg.delta_f_cap / norm
        return delta_f
