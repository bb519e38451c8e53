"""paper_2403_19272_b200 - B200-native (sm_100a) penetration-free cloth pipeline.

Drop-in for the reference package ``clothsim``'s hot path
(``Simulation.step()``, pkg/src/clothsim/stepper.py:454-624): same names,
signatures and error classes; the per-frame pipeline runs in hand-written
CUDA kernels behind the C ABI in include/clothsim_b200.h.
"""

from .mesh import ClothMesh, MeshError, SimState, build_mesh, inertia_target, load_obj, save_obj, triangle_areas
from .constraints import (ElasticConstraints, GlobalSystem, assemble_global, assemble_rhs, bend_coefficients,
                          build_elastic, project_stretch)
from .subspace import (EigensolverError, ReducedSystem, Subspace, build_reduced, build_subspace, reduced_correction,
                       reduced_update, warmstart_correction)
from .smoothing import ajacobi_smooth, jacobi_step
from .stepconfig import StepConfig, StepReport
from ._lib import PenetrationError, SmootherDivergence
from .collision import (EE, VT, LIFE_SPAN_CAP, CollisionWorld, PairSet, PatchBVH, SampleSet, broad_phase,
                        build_patches, coplanarity_coefficients, dbb_weight, dbb_weight_gradient, default_samples,
                        distance_toi, full_ccd, global_toi, lattice_samples, ndb_weights, pair_witness, partial_ccd,
                        point_triangle_closest, query_q, sample_bound, segment_segment_closest, swept_boxes,
                        update_ndb_weights)
from .oracles import oracle_intersect, tri_tri_intersect, tri_tri_intersect_exact
from .sceneconfig import ConfigError, SceneConfig, load_config, parse_config, save_config, serialize_config
from .scenes import box_mesh, build_scene, grid_cloth, icosphere, strip_cloth


def __getattr__(name):
    # Simulation imports the CUDA library lazily so CPU-only setup/tests work
    if name == "Simulation":
        from .stepper import Simulation

        return Simulation
    raise AttributeError(name)


__version__ = "0.1.0"
