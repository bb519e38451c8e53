"""ctypes binding of the C ABI declared in include/clothsim_b200.h.

The shared library is built in-tree (``paper_2403_19272_b200/lib/
libclothsim_b200.so``, see ``build.py``).  There is no CPU fallback: importing a
GPU entry point without the library, or calling it without a CUDA device,
raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libclothsim_b200.so")

c_int_p = ctypes.POINTER(ctypes.c_int)
c_dbl_p = ctypes.POINTER(ctypes.c_double)
c_u8_p = ctypes.POINTER(ctypes.c_uint8)


class SceneDesc(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int) for name in (
        "n_cloth", "n_free", "n_pinned", "n_obstacle", "n_world", "n_edges", "n_stencils",
        "n_world_tris", "n_world_edges", "r_bar", "r")] + [
        ("free_ids", c_int_p), ("free_index", c_int_p), ("pin_ids", c_int_p),
        ("mass", c_dbl_p), ("fext", c_dbl_p), ("mass_over_h2", c_dbl_p),
        ("edge_v", c_int_p), ("edge_rest", c_dbl_p), ("edge_w", c_dbl_p),
        ("rhs_inc_ptr", c_int_p), ("rhs_inc", c_int_p), ("grad_inc_ptr", c_int_p), ("grad_inc", c_int_p),
        ("stencils", c_int_p), ("bend_k", c_dbl_p), ("bend_w", c_dbl_p),
        ("bend_inc_ptr", c_int_p), ("bend_inc", c_int_p),
        ("sell_nslices", ctypes.c_int), ("sell_slice_ptr", c_int_p), ("sell_col", c_int_p),
        ("sell_val", c_dbl_p), ("diag", c_dbl_p),
        ("hfp_ptr", c_int_p), ("hfp_col", c_int_p), ("hfp_val", c_dbl_p),
        ("U", c_dbl_p), ("eigenvalues", c_dbl_p),
        ("world_tris", c_int_p), ("world_edges", c_int_p),
        ("tri_static", c_u8_p), ("vert_static", c_u8_p), ("vert_used", c_u8_p), ("edge_static", c_u8_p),
        ("edge_tris", c_int_p), ("edge_slot", c_int_p), ("patch", c_int_p), ("patch_slot", c_int_p),
        ("x0", c_dbl_p), ("obstacle_x0", c_dbl_p),
    ]


class StepConfigC(ctypes.Structure):
    _fields_ = [(name, ctypes.c_double) for name in (
        "h", "eps_initial", "eps_inner", "eps_outer", "eps_toi", "alpha",
        "ndb_k", "ndb_base", "d_hat", "omega", "rf_tolerance", "delta_f_cap")] + [
        (name, ctypes.c_int) for name in (
            "iteration_cap", "samples", "smoothing_iterations", "warm_start_cap", "inner_cap", "outer_cap",
            "rf_iterations")] + [("dbb_kappa", ctypes.c_double), ("barrier_mode", ctypes.c_int),
                                 ("smoother", ctypes.c_int)]


class StepReportC(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int) for name in (
        "lg_iterations", "outer_loops", "full_ccd_calls", "partial_ccd_calls", "active_pairs",
        "rf_triggered", "cap_hit", "warm_start_iterations")] + [
        ("toi_exit", ctypes.c_double)] + [
        (name, ctypes.c_double) for name in (
            "t_warm_start", "t_local", "t_global", "t_smoothing", "t_broad", "t_narrow_partial",
            "t_narrow_full", "t_rf")] + [
        ("n_outer_deltas", ctypes.c_int), ("outer_deltas", ctypes.c_double * 64),
        ("pairs_last_site", ctypes.c_longlong), ("pairs_max_site", ctypes.c_longlong),
        ("reduced_fallbacks", ctypes.c_int), ("gpu_launches", ctypes.c_longlong), ("static_sites", ctypes.c_int),
        ("subset_sites", ctypes.c_int), ("verified_sites", ctypes.c_int), ("host_syncs", ctypes.c_int),
        ("stamp_plan_reuses", ctypes.c_int), ("lazy_exit_sites", ctypes.c_int)]


CS_OK, CS_PENETRATION, CS_NONFINITE, CS_DIVERGENCE, CS_BAD_DIAGONAL, CS_BAD_ARGUMENT, CS_INTERNAL = range(7)
CS_PART_SYSTEM, CS_PART_CLOTH, CS_PART_BASIS, CS_PART_WORLD, CS_PART_ALL = 1, 2, 4, 8, 15

# every symbol include/clothsim_b200.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "cs_scene_create", "cs_scene_destroy", "cs_scene_set_config", "cs_step", "cs_get_state", "cs_set_state",
    "cs_state_device", "cs_full_ccd", "cs_distance_toi", "cs_partial_ccd", "cs_pair_witness", "cs_broad_phase",
    "cs_scene_pairs", "cs_ccd_site", "cs_scene_pair_results", "cs_assemble_rhs", "cs_ajacobi_smooth", "cs_reduced_correction", "cs_warmstart_correction",
    "cs_energy_gradient", "cs_collision_terms", "cs_residual", "cs_intersections", "cs_scene_set_verify", "cs_last_intersections", "cs_version",
    "cs_frame_async", "cs_frame_wait", "cs_format_obj_vertices", "cs_scene_create_parts", "cs_tri_tri_intersect",
    "cs_coplanarity_coefficients", "cs_query_q", "cs_swept_boxes", "cs_dbb_weight", "cs_jacobi_step",
    "cs_reduced_update", "cs_build_reduced", "cs_reduced_get",
    "cs_eig_create", "cs_eig_destroy", "cs_eig_set", "cs_eig_get", "cs_eig_spmm", "cs_eig_filter", "cs_eig_gram",
    "cs_eig_mul", "cs_eig_residuals", "cs_eig_swap",
)

_lib = None


def load(path: str = LIB_PATH):
    """Load the CUDA library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"clothsim_b200 CUDA library missing at {path}; run "
                           "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    lib = ctypes.CDLL(path)
    vp = ctypes.c_void_p
    ll = ctypes.c_longlong
    sig = {
        "cs_scene_create": (vp, [ctypes.POINTER(SceneDesc), ctypes.POINTER(StepConfigC), c_int_p]),
        "cs_scene_destroy": (None, [vp]),
        "cs_scene_set_config": (ctypes.c_int, [vp, ctypes.POINTER(StepConfigC)]),
        "cs_step": (ctypes.c_int, [vp, vp, vp, ctypes.POINTER(StepReportC), vp]),
        "cs_get_state": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, c_int_p, vp]),
        "cs_set_state": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, ctypes.c_int, vp]),
        "cs_state_device": (ctypes.c_int, [vp, vp, vp, vp, vp]),
        "cs_frame_async": (ctypes.c_int, [vp, vp, c_int_p, vp]),
        "cs_frame_wait": (ctypes.c_int, [vp, ctypes.c_int]),
        "cs_format_obj_vertices": (ctypes.c_longlong, [vp, ll, vp, ll]),
        "cs_full_ccd": (ctypes.c_int, [vp, vp, vp, vp, ll, ctypes.c_double, vp, vp]),
        "cs_distance_toi": (ctypes.c_int, [vp, vp, vp, vp, ll, ctypes.c_double, ctypes.c_int, vp, vp]),
        "cs_partial_ccd": (ctypes.c_int, [vp, vp, vp, vp, ll, ctypes.c_int, vp, vp]),
        "cs_pair_witness": (ctypes.c_int, [vp, vp, vp, ll, vp, vp, vp, vp, vp, vp]),
        "cs_broad_phase": (ctypes.c_int, [vp, vp, vp, ctypes.c_double, ctypes.POINTER(ll), vp]),
        "cs_scene_pairs": (ctypes.c_int, [vp, vp, vp, vp]),
        "cs_ccd_site": (ctypes.c_int, [vp, vp, vp, ctypes.POINTER(ll), ctypes.POINTER(ctypes.c_double), vp]),
        "cs_scene_pair_results": (ctypes.c_int, [vp, vp, vp, vp]),
        "cs_assemble_rhs": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, vp, vp]),
        "cs_ajacobi_smooth": (ctypes.c_int, [vp, vp, vp, ctypes.c_int, ctypes.c_double, vp, vp]),
        "cs_reduced_correction": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_int, vp]),
        "cs_warmstart_correction": (ctypes.c_int, [vp, vp, vp, vp]),
        "cs_energy_gradient": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, vp]),
        "cs_collision_terms": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, vp, ll, vp, vp, vp, vp, ctypes.POINTER(ll), vp]),
        "cs_residual": (ctypes.c_int, [vp, vp, vp, vp, vp, vp]),
        "cs_intersections": (ctypes.c_int, [vp, vp, ctypes.POINTER(ll), vp, ctypes.c_int, vp]),
        "cs_scene_set_verify": (ctypes.c_int, [vp, ctypes.c_int]),
        "cs_last_intersections": (ctypes.c_int, [vp, ctypes.POINTER(ll), vp, ctypes.c_int, vp]),
        "cs_version": (ctypes.c_char_p, []),
        "cs_scene_create_parts": (vp, [ctypes.POINTER(SceneDesc), ctypes.POINTER(StepConfigC), ctypes.c_int,
                                       c_int_p]),
        "cs_tri_tri_intersect": (ctypes.c_int, [vp, vp, ll, vp, vp]),
        "cs_coplanarity_coefficients": (ctypes.c_int, [vp, vp, vp, vp, ll, vp, vp]),
        "cs_query_q": (ctypes.c_int, [vp, vp, vp, vp, ll, vp, ctypes.c_int, ctypes.c_int, vp, vp]),
        "cs_swept_boxes": (ctypes.c_int, [vp, vp, ll, ctypes.c_int, ctypes.c_double, vp, vp, vp]),
        "cs_dbb_weight": (ctypes.c_int, [vp, ll, ctypes.c_double, ctypes.c_double, ctypes.c_int, vp, vp, vp]),
        "cs_jacobi_step": (ctypes.c_int, [vp, vp, vp, ctypes.c_double, vp, vp, vp]),
        "cs_reduced_update": (ctypes.c_int, [vp, vp, vp, ctypes.c_int, vp, vp]),
        "cs_build_reduced": (ctypes.c_int, [vp, vp, ctypes.c_double, vp, ctypes.POINTER(ctypes.c_double), c_int_p,
                                            vp]),
        "cs_reduced_get": (ctypes.c_int, [vp, vp, ctypes.POINTER(ctypes.c_double), c_int_p, vp]),
        "cs_eig_create": (vp, [ctypes.c_int, vp, vp, vp, ctypes.c_int, ctypes.c_int, c_int_p]),
        "cs_eig_destroy": (ctypes.c_int, [vp]),
        "cs_eig_set": (ctypes.c_int, [vp, ctypes.c_int, vp, vp]),
        "cs_eig_get": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, vp, vp]),
        "cs_eig_spmm": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, vp]),
        "cs_eig_filter": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_double, vp]),
        "cs_eig_gram": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, vp, vp]),
        "cs_eig_mul": (ctypes.c_int, [vp, ctypes.c_int, vp, ctypes.c_int, vp]),
        "cs_eig_residuals": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int, vp, vp]),
        "cs_eig_swap": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class PenetrationError(RuntimeError):
    """Impact at t <= 0 or an intersecting state (reference stepper.py:101-104)."""

    def __init__(self, message, state_dump=None):
        super().__init__(message)
        self.state_dump = state_dump


class SmootherDivergence(RuntimeError):
    """Residual grew tenfold inside the smoother (reference smoothing.py:19-20)."""


def check(rc: int, what: str = "clothsim_b200") -> None:
    """Map a C status code to the reference's exception classes."""
    if rc == CS_OK:
        return
    if rc == CS_PENETRATION:
        raise PenetrationError("impact at t<=0: step began in contact")
    if rc == CS_NONFINITE:
        raise FloatingPointError("non-finite inertia target")
    if rc == CS_DIVERGENCE:
        raise SmootherDivergence("residual grew tenfold; raise omega")
    if rc == CS_BAD_DIAGONAL:
        raise ValueError("nonpositive diagonal entry")
    if rc == CS_BAD_ARGUMENT:
        raise ValueError(f"{what}: invalid argument")
    if rc == CS_INTERNAL:
        raise RuntimeError(f"{what}: internal consistency check failed")
    raise RuntimeError(f"{what}: CUDA error {rc - 1000}")


def stream_handle():
    """Current torch CUDA stream as a raw cudaStream_t (plumbing only)."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("clothsim_b200 needs a CUDA device (there is no CPU fallback)")
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
