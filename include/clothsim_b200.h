/* clothsim_b200 - C ABI of the sm_100a cloth pipeline.
 *
 * Drop-in boundary for the reference's hot path, Simulation.step()
 * (pkg/src/clothsim/stepper.py:454-624) and the stage functions it calls.
 * Plain pointers and sizes only (no torch types).  "device" pointers are CUDA
 * device memory; "host" pointers are ordinary CPU memory.  Every entry point
 * returns 0 on success or a status code:
 *
 *   CS_PENETRATION  (1)  impact at t <= 0      -> clothsim.PenetrationError   (stepper.py:450-451)
 *   CS_NONFINITE    (2)  non-finite target     -> FloatingPointError          (mesh.py:194-195)
 *   CS_DIVERGENCE   (3)  smoother blew up      -> clothsim.SmootherDivergence (smoothing.py:55-62)
 *   CS_BAD_DIAGONAL (4)  nonpositive diagonal  -> ValueError                  (smoothing.py:39-40)
 *   CS_BAD_ARGUMENT (5)  invalid size/argument -> ValueError
 *   CS_INTERNAL     (6)  internal consistency check failed (test hooks) -> RuntimeError
 *   >= 1000              CUDA runtime error (1000 + cudaError_t)
 *
 * Which reference interface each entry point replaces is cited per function;
 * INTEGRATION.md shows the ctypes binding.
 */
#ifndef CLOTHSIM_B200_H
#define CLOTHSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CS_OK 0
#define CS_PENETRATION 1
#define CS_NONFINITE 2
#define CS_DIVERGENCE 3
#define CS_BAD_DIAGONAL 4
#define CS_BAD_ARGUMENT 5
#define CS_INTERNAL 6

typedef struct cs_scene cs_scene;

/* Static scene description; all pointers are HOST memory, copied at creation.
 * Produced by paper_2403_19272_b200/device.py from the reference-compatible
 * setup objects (ClothMesh, ElasticConstraints, GlobalSystem, Subspace). */
typedef struct {
    int n_cloth, n_free, n_pinned, n_obstacle, n_world;
    int n_edges, n_stencils;
    int n_world_tris, n_world_edges;
    int r_bar, r;
    /* cloth */
    const int *free_ids;        /* (n_free) */
    const int *free_index;      /* (n_cloth) -1 if pinned */
    const int *pin_ids;         /* (n_pinned) */
    const double *mass;         /* (n_cloth) */
    const double *fext;         /* (n_cloth*3) gravity force m g */
    const double *mass_over_h2; /* (n_free) */
    const int *edge_v;          /* (n_edges*2) */
    const double *edge_rest, *edge_w;
    const int *rhs_inc_ptr, *rhs_inc;   /* (n_cloth+1), (2 n_edges) codes e*2+endpoint, np.add.at order */
    const int *grad_inc_ptr, *grad_inc; /* same, endpoint-1 block first (energy gradient order) */
    const int *stencils;        /* (n_stencils*4) */
    const double *bend_k, *bend_w;
    const int *bend_inc_ptr, *bend_inc; /* codes s*4+j */
    /* global matrix H (free x free), SELL-32 */
    int sell_nslices;
    const int *sell_slice_ptr, *sell_col;
    const double *sell_val, *diag;
    const int *hfp_ptr, *hfp_col;       /* pinned columns, hfp_col = cloth vertex id */
    const double *hfp_val;
    /* rest-shape eigenbasis */
    const double *U;            /* (n_free*r_bar) row-major */
    const double *eigenvalues;  /* (r_bar) */
    /* collision world (cloth vertices first, then obstacles) */
    const int *world_tris, *world_edges;
    const uint8_t *tri_static, *vert_static, *vert_used, *edge_static;
    const int *edge_tris, *edge_slot;   /* (n_world_edges*2) */
    const int *patch, *patch_slot;      /* (n_world_tris) reference build_patches partition */
    /* initial state */
    const double *x0;           /* (n_cloth*3) */
    const double *obstacle_x0;  /* (n_obstacle*3) */
} cs_scene_desc;

#define CS_BARRIER_NDB 0
#define CS_BARRIER_DBB 1

/* Mirrors reference StepConfig (stepper.py:43-79).  barrier_mode: CS_BARRIER_NDB
 * (non-distance barrier, the paper's method) or CS_BARRIER_DBB (log-barrier baseline,
 * stepper.py:524-538); dbb_kappa is the resolved kappa (stepper.py:165-169). */
typedef struct {
    double h, eps_initial, eps_inner, eps_outer, eps_toi, alpha;
    double ndb_k, ndb_base, d_hat, omega, rf_tolerance, delta_f_cap;
    int iteration_cap, samples, smoothing_iterations;
    int warm_start_cap, inner_cap, outer_cap, rf_iterations;
    double dbb_kappa;
    int barrier_mode;
    int smoother;  /* CS_SMOOTHER_AJACOBI (reference) or CS_SMOOTHER_CHEBYSHEV (opt-in) */
} cs_step_config;
#define CS_SMOOTHER_AJACOBI 0
#define CS_SMOOTHER_CHEBYSHEV 1

/* Mirrors reference StepReport (stepper.py:81-92) + device-side diagnostics. */
typedef struct {
    int lg_iterations, outer_loops, full_ccd_calls, partial_ccd_calls;
    int active_pairs, rf_triggered, cap_hit, warm_start_iterations;
    double toi_exit;
    /* stage times in ms (CUDA events), reference timing keys */
    double t_warm_start, t_local, t_global, t_smoothing, t_broad, t_narrow_partial, t_narrow_full, t_rf;
    int n_outer_deltas;
    double outer_deltas[64];
    long long pairs_last_site, pairs_max_site;
    int reduced_fallbacks;
    long long gpu_launches;
    int static_sites;           /* motion-free CCD sites served from the previous site's pairs */
    int subset_sites;           /* moving CCD sites served from the step's base site (+ violator queries) */
    int verified_sites;         /* subset / motion-free sites re-checked against a full broad phase (CS_VERIFY_STATIC_SITE) */
    int host_syncs;             /* host<->device synchronisations inside this cs_step */
    int stamp_plan_reuses;      /* LG iterations whose collision stamps reused the cached row order
                                   (stamp plan of the pair set, abi.cu) */
    int lazy_exit_sites;        /* motion-free exit sites settled from the last site's witness
                                   distances without materialising their pair set */
} cs_step_report;

/* ---- scene lifetime ---------------------------------------------------- */
/* replaces Simulation.__init__'s device-side state (stepper.py:127-173) */
cs_scene *cs_scene_create(const cs_scene_desc *desc, const cs_step_config *cfg, int *status);
/* A context holding only some parts of a scene, for the module-level stage functions
 * that take the reference's setup objects rather than a Simulation
 * (ajacobi_smooth(system, ...), reduced_correction(sub, system, ...),
 * assemble_rhs(system, mesh, elastic, ...), broad_phase(x0, x1, bvh, margin);
 * smoothing.py:23-78, subspace.py:165-192, constraints.py:229-256, bvh.py:207-292).
 * Only the desc fields of the requested parts are read; stage entry points return
 * CS_BAD_ARGUMENT on a context missing a part they need; cs_step needs CS_PART_ALL. */
#define CS_PART_SYSTEM 1  /* H (SELL-32), diag: smoothing, residual */
#define CS_PART_CLOTH 2   /* mesh + elastic + H_fp: rhs, collision terms, energy gradient (with SYSTEM) */
#define CS_PART_BASIS 4   /* U, eigenvalues: reduced update / build (alone), corrections (with SYSTEM) */
#define CS_PART_WORLD 8   /* world topology: broad phase, CCD site, intersections */
#define CS_PART_ALL 15    /* every part + the state: a full scene */
cs_scene *cs_scene_create_parts(const cs_scene_desc *desc, const cs_step_config *cfg, int parts, int *status);
void cs_scene_destroy(cs_scene *scene);
int cs_scene_set_config(cs_scene *scene, const cs_step_config *cfg);

/* ---- the hot path ------------------------------------------------------- */
/* Simulation.step() (stepper.py:454-624): pin_next (n_pinned*3) and obstacle_next
 * (n_obstacle*3) are HOST arrays (prescribed positions at t+h; may be NULL =
 * stay put).  stream: cudaStream_t (NULL = legacy default stream). */
int cs_step(cs_scene *scene, const double *pin_next, const double *obstacle_next, cs_step_report *report,
            void *stream);

/* SimState access (mesh.py:55-73), HOST arrays (n_cloth*3 each; obstacle n_obstacle*3). */
int cs_get_state(cs_scene *scene, double *x, double *x_dot, double *x_prev, double *delta_f, double *obstacle_x,
                 int *step_index, void *stream);
int cs_set_state(cs_scene *scene, const double *x, const double *x_dot, const double *x_prev, const double *delta_f,
                 const double *obstacle_x, int step_index, void *stream);
/* device pointers of the resident state (n_cloth*3 doubles each) */
int cs_state_device(cs_scene *scene, double **x, double **x_dot, double **delta_f, double **obstacle_x);
/* Frame output (reference cli.py:64-98, frame_stride): snapshot x on `stream` and
 * copy it to the PAGE-LOCKED host array host_x (n_cloth*3) on an internal copy
 * stream; returns at once with a ticket (two slots, reused alternately).
 * cs_frame_wait blocks until that frame has landed in host_x. */
int cs_frame_async(cs_scene *scene, double *host_x, int *ticket, void *stream);
int cs_frame_wait(cs_scene *scene, int ticket);

/* ---- per-stage entry points (DEVICE pointers) ---------------------------- */
/* full_ccd (collision/ccd.py:138-196): toi (P) nan = miss */
int cs_full_ccd(const int8_t *kind, const int *idx4, const double *x_start, const double *x_end, long long P,
                double tol, double *toi, void *stream);
/* distance_toi (collision/ccd.py:221-266) */
int cs_distance_toi(const int8_t *kind, const int *idx4, const double *x_start, const double *x_end, long long P,
                    double floor_frac, int max_iterations, double *toi, void *stream);
/* partial_ccd (collision/partial.py:149-204): active (P) 0/1; samples in {1,3,6} */
int cs_partial_ccd(const int8_t *kind, const int *idx4, const double *x_start, const double *x_end, long long P,
                   int samples, uint8_t *active, void *stream);
/* pair_witness (collision/geometry.py:115-148) + Simulation._witness normal (stepper.py:194-216);
 * p1/p2 may be NULL */
int cs_pair_witness(const int8_t *kind, const int *idx4, const double *x, long long P, double *p1, double *p2,
                    double *bary, double *dist, double *normal, void *stream);
/* broad_phase (collision/bvh.py:207-292) over the scene's world topology.  Runs the
 * query into the scene's pair buffer and returns the pair count; cs_scene_pairs
 * copies kind/idx (DEVICE pointers, capacity >= count) out. */
int cs_broad_phase(cs_scene *scene, const double *x_start_w, const double *x_end_w, double margin,
                   long long *count, void *stream);
int cs_scene_pairs(cs_scene *scene, int8_t *kind, int *idx4, void *stream);
/* Simulation._full_ccd_site + _clamp (stepper.py:426-452): broad phase, full CCD (hit
 * TOIs) and the distance-march line-search filter over the scene's pair buffer, with
 * the device's filter/worklist narrow phase.  clamp = alpha * min filter TOI (1 if
 * none); returns CS_PENETRATION when the minimum is <= 0.  cs_scene_pairs /
 * cs_scene_pair_results copy the site's rows and (P) TOIs (DEVICE pointers). */
int cs_ccd_site(cs_scene *scene, const double *x_start_w, const double *x_end_w, long long *count, double *clamp,
                void *stream);
int cs_scene_pair_results(cs_scene *scene, double *toi, double *toi_filter, void *stream);
/* assemble_rhs (constraints.py:229-256); pins (n_cloth*3, only the pinned rows are read)
 * carries pinned_positions (NULL: the pinned rows of x); coll_* (n_coll) are the flat
 * (ids, weights, targets) of Simulation._collision_terms in order; ids are cloth ids. */
int cs_assemble_rhs(cs_scene *scene, const double *z, const double *x, const double *pins, const int *coll_ids,
                    const double *coll_w, const double *coll_t, int n_coll, double *b, double *delta, void *stream);
/* Simulation._collision_terms (stepper.py:238-285): per engaged pair with weight > 0, its
 * movable cloth vertices' (ids, weights, targets) in pair-then-slot order; DEVICE arrays
 * (ids/w capacity 4P, targets 4P*3); count = entries written */
int cs_collision_terms(cs_scene *scene, const int8_t *kind, const int *idx4, const double *bary, const double *normal,
                       const double *weight, const uint8_t *engaged, long long P, const double *x_world, int *ids,
                       double *w, double *targets, long long *count, void *stream);
/* r = b - H x - delta x over the free rows (the residual of reduced_correction /
 * residual_forward, subspace.py:179, stepper.py:663) */
int cs_residual(cs_scene *scene, const double *b, const double *x, const double *delta, double *r, void *stream);
/* ajacobi_smooth (smoothing.py:23-66), x (n_free*3) updated in place; delta may be NULL */
int cs_ajacobi_smooth(cs_scene *scene, const double *b, double *x, int iterations, double omega,
                      const double *delta, void *stream);
/* reduced_correction (subspace.py:165-186); reuse != 0 keeps the last reduced system */
int cs_reduced_correction(cs_scene *scene, const double *b, double *x, const double *delta, int reuse,
                          void *stream);
/* jacobi_step (smoothing.py:69-78): out = x + (1 - omega) D^-1 (b - (H + delta) x); delta may be NULL */
int cs_jacobi_step(cs_scene *scene, const double *b, const double *x, double omega, const double *delta,
                   double *out, void *stream);
/* reduced_update (subspace.py:97-106): G (r*r) = sum_j weights[j] V_rows[j] V_rows[j]^T */
int cs_reduced_update(cs_scene *scene, const int *rows, const double *weights, int m, double *G, void *stream);
/* build_reduced (subspace.py:122-140): A = diag(lambda_r) + G (G may be NULL), beta = rhs_scale
 * (1 if <= 0), inverse (r*r, DEVICE) with A inverse = I / beta, LU with the pinv fallback;
 * beta / fallback HOST.  Becomes the context's current reduced system (reuse != 0 in
 * cs_reduced_correction applies it). */
int cs_build_reduced(cs_scene *scene, const double *G, double rhs_scale, double *inverse, double *beta,
                     int *fallback, void *stream);
/* the context's current reduced system: inverse (r*r, DEVICE), beta / fallback (HOST); any may be NULL */
int cs_reduced_get(cs_scene *scene, double *inverse, double *beta, int *fallback, void *stream);
/* warmstart_correction (subspace.py:189-192) */
int cs_warmstart_correction(cs_scene *scene, const double *b, double *x, void *stream);
/* Simulation.energy gradient (stepper.py:309-380, "quad" form); grad (n_cloth*3) */
int cs_energy_gradient(cs_scene *scene, const double *x, const double *z, const int *q_ids, const double *q_w,
                       const double *q_t, int n_q, double *grad, void *stream);

/* ---- scene-free module-level helpers (DEVICE pointers) -------------------- */
/* tri_tri_intersect (oracles.py:33-48): p, q (m,3,3); out (m) 1 = closed triangles intersect */
int cs_tri_tri_intersect(const double *p, const double *q, long long m, uint8_t *out, void *stream);
/* coplanarity_coefficients (collision/ccd.py:36-44): coef (P,4), lowest order first */
int cs_coplanarity_coefficients(const int8_t *kind, const int *idx4, const double *x_start, const double *x_end,
                                long long P, double *coef, void *stream);
/* query_q (collision/partial.py:133-146): lam (P,k,2), or (k,2) when shared != 0; out (P,k) */
int cs_query_q(const int8_t *kind, const int *idx4, const double *x_start, const double *x_end, long long P,
               const double *lam, int k, int shared, double *out, void *stream);
/* swept_boxes (collision/bvh.py:140-143): points (m,k,3) at both ends -> lo, hi (m,3) */
int cs_swept_boxes(const double *points_start, const double *points_end, long long m, int k, double margin,
                   double *lo, double *hi, void *stream);
/* dbb_weight / dbb_weight_gradient (collision/pairs.py:83-108); flag: DEVICE int scratch;
 * returns CS_NONFINITE when a distance is <= 0 (weight only; FloatingPointError) */
int cs_dbb_weight(const double *d, long long m, double d_hat, double kappa, int gradient, double *out, int *flag,
                  void *stream);

/* ---- penetration-free invariant ----------------------------------------- */
/* oracle_intersect (oracles.py:83-131): intersecting non-adjacent world-triangle pairs at
 * x_world (DEVICE, n_world*3; NULL = current state).  count = all pairs; the first
 * min(count, cap) are written to `pairs` (HOST, (cap,2) rows (lo, hi), unordered). */
int cs_intersections(cs_scene *scene, const double *x_world, long long *count, int *pairs, int cap, void *stream);
/* verify mode (stepper.py:614-621): with on != 0, cs_step checks x_final before committing
 * the state and returns CS_PENETRATION (state untouched) when triangles intersect;
 * cs_last_intersections reports that check (pairs HOST (cap,2), x_final HOST n_cloth*3). */
int cs_scene_set_verify(cs_scene *scene, int on);
int cs_last_intersections(cs_scene *scene, long long *count, int *pairs, int cap, double *x_final);

/* ---- device eigensolver (setup; subspace.py:49-84 for paper-scale meshes) --- */
/* Opaque context: H (CSR, HOST arrays copied at creation, n x n) and nblocks row-major
 * n x p device blocks.  The block operations of a Chebyshev-filtered subspace iteration;
 * the p x p algebra stays with the caller (eigen.py).  HOST pointers throughout. */
typedef struct cs_eig cs_eig;
cs_eig *cs_eig_create(int n, const int *indptr, const int *indices, const double *data, int p, int nblocks,
                      int *status);
int cs_eig_destroy(cs_eig *eig);
int cs_eig_set(cs_eig *eig, int block, const double *host, void *stream);            /* block <- host (n,p) */
int cs_eig_get(cs_eig *eig, int block, int cols, double *host, void *stream);        /* host (n,cols) <- block */
int cs_eig_spmm(cs_eig *eig, int src, int dst, void *stream);                        /* dst = H src */
int cs_eig_filter(cs_eig *eig, int x, int w1, int w2, int degree, double a, double lam_max, double a0,
                  void *stream);                                                      /* Chebyshev filter of x */
int cs_eig_gram(cs_eig *eig, int a, int b, double *out, void *stream);               /* out (p,p) = A^T B */
int cs_eig_mul(cs_eig *eig, int src, const double *S, int dst, void *stream);        /* dst = src S, S (p,p) */
int cs_eig_swap(cs_eig *eig, int a, int b);                                          /* exchange block slots */
int cs_eig_residuals(cs_eig *eig, int hx, int x, const double *w, int cols, double *out,
                     void *stream);                                                  /* |HX_j - w_j X_j|^2 */

const char *cs_version(void);

/* Host helper for frame output: the OBJ vertex block "v %.9f %.9f %.9f\n" of n
 * vertices (reference mesh.py:220-226) into out; returns bytes, -1 if cap is short. */
long long cs_format_obj_vertices(const double *v, long long n, char *out, long long cap);

#ifdef __cplusplus
}
#endif

#endif /* CLOTHSIM_B200_H */
