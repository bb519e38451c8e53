"""Command-line harness mirroring the reference's (pkg/src/clothsim/cli.py:1-216):

  simulate <config>   run a scene, write OBJ frames and a metrics CSV
  verify <config>     simulate with the per-step intersection check on (device SAT)
  bench-ccd           full CCD vs partial-CCD classifier on random pairs (device)

Same config files (``sceneconfig``), metrics columns and number formats
(cli.py:31-36, 84-91) and frame names.  Frames leave the device without stalling
the step loop: every ``frame_stride`` steps the positions are snapshotted on the
stepping stream and copied to page-locked memory on a copy stream
(``cs_frame_async``); a writer thread waits for the copy and formats the OBJ while
the GPU keeps stepping."""

from __future__ import annotations

import argparse
import csv
import ctypes
import queue
import sys
import threading
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

from . import _lib
from .sceneconfig import SceneConfig, load_config, save_config

METRIC_FIELDS = [  # cli.py:31-36
    "step", "lg_iterations", "outer_loops", "toi_exit", "active_pairs",
    "rf_triggered", "penetration_free",
    "t_warm_start", "t_local", "t_global", "t_smoothing",
    "t_broad", "t_narrow_partial", "t_narrow_full",
]
TIMING_KEYS = ("warm_start", "local", "global", "smoothing", "broad", "narrow_partial", "narrow_full")


def metrics_row(step: int, rep) -> list:
    """One metrics.csv row in the reference's formatting (cli.py:84-91)."""
    return [step, rep.lg_iterations, rep.outer_loops, f"{rep.toi_exit:.6f}", rep.active_pairs,
            int(rep.rf_triggered), int(rep.penetration_free)] + [f"{rep.timings[k]:.3f}" for k in TIMING_KEYS]


class ObjFormatter:
    """OBJ text identical to the reference's save_obj (mesh.py:220-226): 9-decimal
    vertices, 1-based faces.  The face block is formatted once per topology."""

    def __init__(self, triangles: np.ndarray):
        self.faces = "".join(f"f {a + 1} {b + 1} {c + 1}\n" for a, b, c in np.asarray(triangles).tolist())

    def write(self, path, vertices: np.ndarray) -> None:
        v = np.ascontiguousarray(vertices, dtype=np.float64)
        with open(path, "w") as fh:
            fh.write(self.vertex_text(v))
            fh.write(self.faces)

    @staticmethod
    def vertex_text(v: np.ndarray) -> str:
        """The vertex block, formatted by the native library (multi-threaded)."""
        lib = _lib.load()
        if len(v) == 0:
            return ""
        cap = 160 * len(v)
        buf = ctypes.create_string_buffer(cap)
        k = lib.cs_format_obj_vertices(v.ctypes.data, len(v), buf, cap)
        if k < 0:
            raise RuntimeError("cs_format_obj_vertices: buffer too small")
        return buf.raw[:k].decode("ascii")


class FrameWriter:
    """Asynchronous frame output for one Simulation: ``submit(path)`` snapshots the
    current positions (device-side copy, returns at once); a worker thread waits for
    the device-to-host copy of that snapshot and writes the OBJ.  At most ``depth``
    frames are in flight (each holds one page-locked host buffer)."""

    def __init__(self, sim, depth: int = 2):
        import torch

        self.sim = sim
        self.fmt = ObjFormatter(sim.mesh.triangles)
        n = sim.mesh.vertex_count
        self._free = queue.Queue()
        for _ in range(max(depth, 1)):
            self._free.put(torch.empty((n, 3), dtype=torch.float64, pin_memory=True))
        self._jobs = queue.Queue()
        self._err = None
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()

    def submit(self, path) -> None:
        if self._err is not None:
            raise self._err
        sim = self.sim
        sim._flush()  # host edits of the state reach the device first
        buf = self._free.get()
        ticket = ctypes.c_int(0)
        _lib.check(sim._lib.cs_frame_async(sim._scene, buf.data_ptr(), ctypes.byref(ticket), sim._stream()),
                   "cs_frame_async")
        self._jobs.put((Path(path), buf, ticket.value))

    def _run(self):
        while True:
            job = self._jobs.get()
            if job is None:
                return
            path, buf, ticket = job
            try:
                _lib.check(self.sim._lib.cs_frame_wait(self.sim._scene, ticket), "cs_frame_wait")
                self.fmt.write(path, buf.numpy())
            except BaseException as exc:  # surfaced on the next submit / close
                self._err = exc
            finally:
                self._free.put(buf)

    def close(self) -> None:
        self._jobs.put(None)
        self._thread.join()
        if self._err is not None:
            raise self._err


def build_from_config(cfg: SceneConfig, steps=None, verify=False, barrier=None, iteration_cap=None,
                      eigensolver: str = "host"):
    """cli.py:39-61: overrides applied to the solver section, then build_scene
    (eigensolver "device" = the GPU subspace precompute, for large meshes)."""
    from .scenes import build_scene

    solver = cfg.solver
    if steps:
        cfg.steps = steps
    if barrier:
        solver = replace(solver, barrier_mode=barrier)
    if iteration_cap is not None:
        solver = replace(solver, iteration_cap=iteration_cap)
    if verify:
        solver = replace(solver, verify=True)  # device intersection check inside every step
    cfg.solver = solver
    return build_scene(cfg.scene.kind, resolution=cfg.scene.resolution, size=cfg.scene.size,
                       density=cfg.material.density, stretch_stiffness=cfg.material.stretch_stiffness,
                       bend_stiffness=cfg.material.bend_stiffness, config=solver, eigensolver=eigensolver)


def simulate(cfg: SceneConfig, steps=None, verify=False, barrier=None, iteration_cap=None, log=sys.stdout,
             eigensolver: str = "host") -> int:
    """cli.py:64-98: frame_000000.obj, metrics.csv (one row per step), a frame every
    frame_stride steps and at the last step; exit code 2 with a state-dump OBJ on a
    penetration-invariant breach."""
    from ._lib import PenetrationError

    sim = build_from_config(cfg, steps, verify, barrier, iteration_cap, eigensolver)
    out = Path(cfg.output.directory)
    out.mkdir(parents=True, exist_ok=True)
    save_config(cfg, out / "config.toml")
    stride = max(cfg.output.frame_stride, 1)
    frames = FrameWriter(sim)
    frames.submit(out / "frame_000000.obj")
    t0 = time.perf_counter()
    try:
        with open(out / "metrics.csv", "w", newline="") as fh:
            writer = csv.writer(fh)
            writer.writerow(METRIC_FIELDS)
            for step in range(1, cfg.steps + 1):
                try:
                    rep = sim.step()
                except PenetrationError as exc:
                    dump = out / f"state_dump_{step:06d}.obj"
                    # the last good state, as the reference CLI dumps it (cli.py:81-86); the
                    # failing candidate stays in exc.state_dump["x"]
                    frames.fmt.write(dump, sim.state.x)
                    print(f"invariant breach at step {step}: {exc}; state dump: {dump}", file=sys.stderr)
                    return 2
                writer.writerow(metrics_row(step, rep))
                if step % stride == 0 or step == cfg.steps:
                    frames.submit(out / f"frame_{step:06d}.obj")
    finally:
        frames.close()
    print(f"{cfg.name}: {cfg.steps} steps in {time.perf_counter() - t0:.1f}s -> {out}", file=log)
    return 0


def bench_ccd(pairs: int, seed: int = 0, log=sys.stdout) -> int:
    """cli.py:147-181 on the device kernels: full CCD vs the partial-CCD classifier."""
    from .collision import default_samples, full_ccd, partial_ccd

    rng = np.random.default_rng(seed)
    kind = (np.arange(pairs) % 2).astype(np.int8)
    idx = np.arange(4 * pairs, dtype=np.int64).reshape(pairs, 4)
    x0 = rng.uniform(0.0, 1.0, (4 * pairs, 3))
    x1 = x0 + rng.uniform(-0.3, 0.3, (4 * pairs, 3))
    samples = default_samples(3)
    t = time.perf_counter()
    toi = full_ccd(kind, idx, x0, x1)
    t_full = time.perf_counter() - t
    t = time.perf_counter()
    active = partial_ccd(kind, idx, x0, x1, samples)
    t_partial = time.perf_counter() - t
    print(f"pairs: {pairs}", file=log)
    print(f"full ccd:     {t_full:.3f}s  ({1e9 * t_full / pairs:.0f} ns/pair), "
          f"{int(np.count_nonzero(~np.isnan(toi)))} impacts", file=log)
    print(f"partial ccd:  {t_partial:.3f}s  ({1e9 * t_partial / pairs:.0f} ns/pair), "
          f"{int(np.count_nonzero(active))} active", file=log)
    print(f"speedup:      {t_full / max(t_partial, 1e-12):.1f}x", file=log)
    return 0


def main(argv=None) -> int:
    parser = argparse.ArgumentParser(prog="paper_2403_19272_b200", description=__doc__)
    sub = parser.add_subparsers(dest="command", required=True)
    common = argparse.ArgumentParser(add_help=False)
    common.add_argument("--steps", type=int, default=None, help="override step count")
    common.add_argument("--verify", action="store_true", help="check the intersection invariant every step")
    common.add_argument("--barrier", choices=("ndb", "dbb"), default=None)
    common.add_argument("--iteration-cap", type=int, default=None, dest="iteration_cap")
    common.add_argument("--seed", type=int, default=0)
    common.add_argument("--eigensolver", choices=("host", "device"), default="host",
                        help="subspace precompute: scipy eigsh (reference) or the device solver")
    for name, verify in (("simulate", False), ("verify", True)):
        p = sub.add_parser(name, parents=[common])
        p.add_argument("config")
        p.set_defaults(verify_default=verify)
    p = sub.add_parser("bench-ccd", parents=[common])
    p.add_argument("--pairs", type=int, default=1_000_000)
    args = parser.parse_args(argv)
    if args.command == "bench-ccd":
        return bench_ccd(args.pairs, args.seed)
    cfg = load_config(args.config)
    return simulate(cfg, args.steps, args.verify or args.verify_default, args.barrier, args.iteration_cap,
                    eigensolver=args.eigensolver)


if __name__ == "__main__":
    sys.exit(main())
