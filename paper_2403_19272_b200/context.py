"""Device contexts behind the module-level stage functions.

The reference's stage functions take its setup objects (``ajacobi_smooth(system,
...)``, ``reduced_correction(sub, system, ...)``, ``assemble_rhs(system, mesh,
elastic, ...)``, ``broad_phase(x0, x1, bvh, margin)``; smoothing.py:23-78,
subspace.py:97-192, constraints.py:229-256, collision/bvh.py:207-292).  Their
drop-ins here run on the device: each (set of) setup object(s) gets one
``cs_scene_create_parts`` context holding just the parts it needs (SELL H, basis,
cloth arrays, world topology), created on first use and cached until one of the
objects is garbage collected.  Setup objects are treated as immutable, as in the
reference.
"""

from __future__ import annotations

import ctypes
import weakref

from . import _lib
from .device import parts_desc, step_config_c
from .stepconfig import StepConfig


class Context:
    """One partial scene on the device (cs_scene_create_parts)."""

    def __init__(self, config: StepConfig | None = None, **objs):
        self.lib = _lib.load()
        d, keep, parts = parts_desc(**objs)
        cfg = config if config is not None else StepConfig()
        self._cfg = step_config_c(cfg, cfg.ndb_k if cfg.ndb_k > 0 else 1.0)
        status = ctypes.c_int(0)
        self.ptr = self.lib.cs_scene_create_parts(ctypes.byref(d), ctypes.byref(self._cfg), parts,
                                                  ctypes.byref(status))
        del keep
        if not self.ptr:
            _lib.check(status.value or _lib.CS_BAD_ARGUMENT, "cs_scene_create_parts")
        self.parts = parts
        self.generation = 0      # bumped by every call that replaces the reduced system

    def __del__(self):
        ptr = getattr(self, "ptr", None)
        if ptr:
            self.lib.cs_scene_destroy(ptr)
            self.ptr = None


_cache: dict = {}


def get(**objs) -> Context:
    """Cached context for these setup objects (keyword names as parts_desc takes them)."""
    live = {k: v for k, v in objs.items() if v is not None and not isinstance(v, int)}
    key = tuple(sorted((k, id(v)) for k, v in live.items()))
    hit = _cache.get(key)
    if hit is not None:
        return hit
    ctx = Context(**objs)
    _cache[key] = ctx
    for v in live.values():
        try:
            weakref.finalize(v, _cache.pop, key, None)
        except TypeError:  # not weak-referenceable: the context lives for the process
            pass
    return ctx
