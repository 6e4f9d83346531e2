/*
 * vrod C-ABI — the drop-in boundary for the VIPER rod-solver substep hot path.
 *
 * The reference (`/root/reference/proj`) has no FFI: its boundary is the C++ header API in
 * `proj/core/include/vrod/` headers. This header restates exactly that API as
 * plain C (pointers + sizes, no C++/torch types) so one binding drives three libraries:
 *
 *   paper_1906_05260_b200/lib/libvrod_b200.so   the product: host C++ + sm_100a CUDA
 *   oracle/lib/libvrod_oracle.so                CPU restatement (test infrastructure)
 *   oracle/_ref/libvrod_ref.so                  the reference's own sources + adapter (tests)
 *
 * Every entry point names the reference interface it replaces. Conventions:
 *   - return value: VROD_OK or an error code mirroring the reference exception type
 *     (std::invalid_argument via require, types.h:67-69; std::out_of_range via
 *     require_index, types.h:71-77; vrod::SimulationError, types.h:25-28); the message
 *     (identical to the reference's what()) is available from vrod_last_error().
 *   - vectors are packed doubles: Vec3 = 3 doubles (x,y,z); Quat = 4 doubles (w,x,y,z).
 *   - "global slot" order is DofLayout's (layout.h:17-41): rods in order, vertices /
 *     elements in order within a rod.
 *   - a solver handle is single-caller; handles are independent.
 */
#ifndef VROD_CAPI_H
#define VROD_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VROD_CAPI_VERSION 1

enum vrod_status {
  VROD_OK = 0,
  VROD_INVALID_ARGUMENT = 1, /* std::invalid_argument (require, types.h:67-69) */
  VROD_OUT_OF_RANGE = 2,     /* std::out_of_range (require_index, types.h:71-77) */
  VROD_SIMULATION_ERROR = 3, /* vrod::SimulationError (types.h:25-28) */
  VROD_RUNTIME_ERROR = 4,    /* any other std::exception */
  VROD_DEVICE_ERROR = 5      /* CUDA failure (product only) */
};

/* Message of the last failing call on this thread (what() of the reference exception). */
const char* vrod_last_error(void);
/* "b200-cuda", "oracle-cpu" or "reference-cpu". */
const char* vrod_backend_name(void);
int32_t vrod_capi_version(void);

/* ---- plain data (reference structs) -------------------------------------------------- */

/* MaterialParams, rod.h:13-24 (defaults :14-21). */
typedef struct vrod_material {
  double stretch_x, stretch_y, stretch_z;
  double bend_x, bend_y, bend_z;
  double volume, density;
} vrod_material;

/* SolverSettings, scene.h:25-39 (scale_mode: 0 kSimulated, 1 kPostStepLengthRatio). */
typedef struct vrod_settings {
  double dt;
  int32_t iterations;
  int32_t substeps;
  double beta;
  double gravity[3];
  int32_t dichotomous_iterations;
  int32_t shape_match_period;
  double contact_stiffness;
  double velocity_damping;
  int32_t deterministic;
  int32_t scale_mode;
} vrod_settings;

/* Pill, collision.h:16-25. rod == -1 for kinematic pills. */
typedef struct vrod_pill {
  double c0[3];
  double c1[3];
  double r0, r1;
  int32_t rod, element, group, self_collide;
} vrod_pill;

/* StepReport, solver.h:23-33 (+ PhaseTimings :14-21). residuals are indexed by
 * ConstraintKind (constraints.h:14-26) for the 8 elastic kinds. */
typedef struct vrod_step_report {
  int32_t step;
  int32_t contact_count;
  int32_t broad_pairs;
  int32_t skipped_singular;
  int32_t dof_count;
  int32_t pad_;
  double time;
  double residuals[8];
  double max_penetration;
  double predict_ms, broad_ms, narrow_ms, solve_ms, finalize_ms, total_ms;
} vrod_step_report;

/* One rod: RodRestPose (rod.h:30-46) + RodState (:50-60) + Rod (:64-74). n = vertex_count,
 * m = n - 1. All rest/state arrays are required; pinned may be NULL (nothing pinned). */
typedef struct vrod_rod_desc {
  int32_t vertex_count;
  int32_t material;
  int32_t collision_group;
  int32_t self_collide;
  const double* rest_centers;     /* 3n */
  const double* rest_scales;      /* n */
  const double* radii;            /* n */
  const double* lengths;          /* m  (strain targets) */
  const double* initial_lengths;  /* m  (as-built) */
  const double* rest_frames;      /* 4m */
  const double* darboux;          /* 3(m-1) */
  const double* tangent_dots;     /* m */
  const double* scale_grads;      /* m */
  const double* scale_laplacians; /* m-1 */
  const double* centers;          /* 3n */
  const double* scales;           /* n */
  const double* frames;           /* 4m */
  const double* center_vel;       /* 3n */
  const double* scale_vel;        /* n */
  const double* angular_vel;      /* 3m, body frame */
  const uint8_t* pinned;          /* n, 0/1, or NULL */
  int32_t bone_count;             /* optional two-bone rig (rod.h:71-73) */
  int32_t pad_;
  const int32_t* bones;           /* bone_count */
  const double* bone_weights;     /* n * bone_count, row per vertex */
} vrod_rod_desc;

/* Output of make_rest_pose (caller-allocated, sizes as in vrod_rod_desc). */
typedef struct vrod_rest_pose_out {
  double* rest_scales;      /* n */
  double* radii;            /* n */
  double* lengths;          /* m */
  double* initial_lengths;  /* m */
  double* rest_frames;      /* 4m */
  double* darboux;          /* 3(m-1) */
  double* tangent_dots;     /* m */
  double* scale_grads;      /* m */
  double* scale_laplacians; /* m-1 */
} vrod_rest_pose_out;

void vrod_default_material(vrod_material* out); /* rod.h:14-21 */
void vrod_default_settings(vrod_settings* out); /* scene.h:26-37 */

/* make_rest_pose(centers, radii, scales), rod.h:88-90 / rod.cpp:60-112. radii_count is 1 or
 * n; scales_count is 0 (unit), 1 or n. */
int vrod_make_rest_pose(int32_t n, const double* centers, int32_t radii_count, const double* radii,
                        int32_t scales_count, const double* scales, vrod_rest_pose_out* out);

/* ---- scene builder (Scene, scene.h:109-126) ------------------------------------------- */

typedef struct vrod_scene vrod_scene;
int vrod_scene_create(vrod_scene** out);
void vrod_scene_destroy(vrod_scene* scene);
int vrod_scene_set_settings(vrod_scene* scene, const vrod_settings* settings);
int vrod_scene_add_material(vrod_scene* scene, const vrod_material* material);
int vrod_scene_add_rod(vrod_scene* scene, const vrod_rod_desc* rod);
int vrod_scene_add_plane(vrod_scene* scene, const double normal[3], double offset);     /* HalfPlane */
/* Bone (scene.h:49-53): key_count keyframes (t, position xyz, rotation wxyz). */
int vrod_scene_add_bone(vrod_scene* scene, int32_t key_count, const double* times,
                        const double* positions, const double* rotations);
int vrod_scene_add_kinematic_pill(vrod_scene* scene, const vrod_pill* pill, int32_t bone); /* KinematicPill */
int vrod_scene_add_bundle(vrod_scene* scene, int32_t member_count, const int32_t* rods,
                          const int32_t* vertices);                                     /* BundleMember list */
int vrod_scene_add_pin_motion(vrod_scene* scene, int32_t rod, int32_t vertex, const double start[3],
                              const double target[3], double t0, double t1);            /* PinMotion */
int vrod_scene_add_soft_pin(vrod_scene* scene, int32_t rod, int32_t vertex, const double target[3],
                            double stiffness);                                          /* SoftPin */
int vrod_scene_add_activation(vrod_scene* scene, int32_t rod, double factor, double t_start,
                              double t_end, int32_t first_element, int32_t last_element); /* Activation */
/* Scene::validate, scene.cpp:63-157 — same checks, same messages. */
int vrod_scene_validate(const vrod_scene* scene);

/* ---- solver (class Solver, solver.h:54-115) ------------------------------------------- */

typedef struct vrod_solver vrod_solver;

typedef struct vrod_solver_info {
  int32_t rod_count;
  int32_t total_vertices;
  int32_t total_elements;
  int32_t dof_count;     /* Solver::dof_count, 4V + 3E */
  int32_t step_index;    /* Solver::step_index */
  int32_t bundle_count;
  int32_t elastic_blocks;
  int32_t pad_;
  double time;           /* Solver::time */
} vrod_solver_info;

/* Solver::Solver(Scene), solver.cpp:102-136. The scene is copied; it may be destroyed after. */
int vrod_solver_create(const vrod_scene* scene, vrod_solver** out);
void vrod_solver_destroy(vrod_solver* solver);
/* Solver::step(), solver.cpp:363-388. */
int vrod_solver_step(vrod_solver* solver, vrod_step_report* report);
/* Solver::probe_convergence(iterations), solver.cpp:390-398: writes iterations x 8 residuals. */
int vrod_solver_probe_convergence(vrod_solver* solver, int32_t iterations, double* residual_log);
int vrod_solver_get_info(const vrod_solver* solver, vrod_solver_info* info);
/* Per-rod vertex counts (rod_count entries). */
int vrod_solver_get_rod_sizes(const vrod_solver* solver, int32_t* vertex_counts);

/* Solver::scene() state access, global slot order; any pointer may be NULL. get = read the
 * live state; set = the mutable scene() write-back between steps (SURVEY.md §7 hard part 5). */
int vrod_solver_get_state(vrod_solver* solver, double* centers, double* scales, double* frames,
                          double* center_vel, double* scale_vel, double* angular_vel);
int vrod_solver_set_state(vrod_solver* solver, const double* centers, const double* scales,
                          const double* frames, const double* center_vel, const double* scale_vel,
                          const double* angular_vel);
/* Product options, no reference counterpart (the reference has no GPU); name -> value:
 *   "state_prefetch"        1: each step also copies the state to pinned host memory inside the
 *                           step's own synchronisation (get_state after a step is a memcpy);
 *                           0 (default): get_state copies on demand.
 *   "exact_shape_matching"  1: shape matching in the reference's exact operation order (states
 *                           bit-identical to the reference); 0: the latency-tuned path (within
 *                           BASELINE.md §5's tolerance). Default: environment VROD_SHAPE_EXACT.
 *   "phase_timing"          1: fill vrod_step_report's predict/broad/narrow/solve/finalize_ms
 *                           (device time per phase, solver.h:14-21) at the cost of direct kernel
 *                           launches instead of one CUDA graph per step; 0 (default): zeros.
 * Unknown name: VROD_INVALID_ARGUMENT. */
int vrod_solver_set_option(vrod_solver* solver, const char* name, int64_t value);

/* Live rest quantities (activation rewrites lengths & derived data, rod.cpp:164-176). */
int vrod_solver_get_rest(vrod_solver* solver, double* lengths, double* darboux_per_element,
                         double* scale_grads, double* scale_laplacians_per_element);
/* ExternalLoads (solver.h:35-41) via Solver::loads(). Arrays are global-slot sized; the
 * per-rod flag arrays say which rods carry that load (an empty vector in the reference).
 * Passing NULL for an array clears that load. */
int vrod_solver_set_loads(vrod_solver* solver, const double* force_density, const uint8_t* fd_rods,
                          const double* torque, const uint8_t* torque_rods, const double* scale_load,
                          const uint8_t* scale_load_rods);
/* Solver::kinetic_energy / total_volume / total_rest_volume, solver.cpp:400-430. */
int vrod_solver_energy(vrod_solver* solver, double* kinetic, double* volume, double* rest_volume);
/* DofLayout weights (layout.h:25-34): per vertex center/scale inverse weights, per element
 * theta inverse weights (3 each). Any may be NULL. */
int vrod_solver_get_inverse_weights(vrod_solver* solver, double* inv_center, double* inv_scale,
                                    double* inv_theta);
/* DofLayout lumped weights (layout.h:25-27, build_layout layout.cpp:43-72): per vertex center and
 * scale weights (+inf when pinned), per element theta weights (3 each, body-frame diagonal, as of the
 * last refresh_orientation_inertia, layout.cpp:76-93). Any may be NULL. */
int vrod_solver_get_weights(vrod_solver* solver, double* center_weight, double* scale_weight,
                            double* theta_weight);
/* Contacts of the last substep (contact blocks, solver.cpp:210-224): pill ids in the pill
 * array of that substep, frozen alpha/beta. */
int vrod_solver_get_contacts(vrod_solver* solver, int64_t capacity, int64_t* count,
                             int32_t* pill_a, int32_t* pill_b, double* alpha, double* beta);
/* Solver::current_pills(), solver.cpp:432-436 (rod pills then kinematic pills). */
int vrod_solver_current_pills(vrod_solver* solver, int64_t capacity, int64_t* count, vrod_pill* pills);

/* One apply_shape_match pass over the solver's bundle groups in group order (bundling.cpp:116-133
 * — the pass Solver::substep runs every shape_match_period sweeps, solver.cpp:336-338) on the live
 * state, warm rotations updated. fits: 14 doubles per group (SimilarityFit, bundling.h:18-23:
 * scale, translation xyz, rotation row-major 3x3, degenerate 0/1); at most `capacity` groups
 * written, *count = the group count. */
int vrod_solver_shape_match(vrod_solver* solver, int32_t capacity, int32_t* count, double* fits);

/* jacobi_sweep (constraints.h:124-126 / constraints.cpp:491-556) of the solver's elastic blocks
 * and soft pins — in the order of Solver::substep's block list (solver.cpp:324-328), multipliers
 * zero — on the live state, with step h and relaxation beta; contacts and half-planes are not part
 * of it (and the last substep's contact list is consumed). State updated in place. active /
 * skipped_singular: the SweepOutcome (either may be NULL). VROD_SIMULATION_ERROR on a non-finite
 * update, naming the constraint like the reference. */
int vrod_solver_jacobi_sweep(vrod_solver* solver, double h, double beta, int32_t* active, int32_t* skipped_singular);
/* eval_constraint(block, ctx).W (constraints.h:82 / constraints.cpp:101-214) of every elastic block
 * in block order on the live state: 3 doubles per block (unused components 0); at most
 * `capacity` blocks written, *count = the elastic block count. */
int vrod_solver_elastic_residuals(vrod_solver* solver, int64_t capacity, int64_t* count, double* W);

/* ---- batches of independent scenes (BASELINE config C5) --------------------------------
 * The reference has no batch API: a batch is N independent vrod::Solver(Scene) objects
 * stepped in lockstep (solver.h:54-115, once per scene). Here one solver handle steps them
 * all in one device world: pairs never cross scenes, pair_key ids stay scene-local, every
 * scene's results equal that scene solved alone. All scenes must share one SolverSettings
 * (dt, substeps, iterations, ...). State / rod-size queries see the scenes concatenated in
 * order (global slot order of scene 0, then scene 1, ...). vrod_solver_step on a batch
 * returns the batch total: contact_count, broad_pairs, skipped_singular summed (saturating
 * at INT32_MAX), max_penetration and each residual the maximum over scenes. */
int vrod_batch_create(int32_t scene_count, const vrod_scene* const* scenes, vrod_solver** out);
/* Number of scenes of a solver (1 for vrod_solver_create). */
int vrod_solver_scene_count(const vrod_solver* solver, int32_t* count);
/* Per-scene StepReports of the last step (the same report Solver::step() of that scene alone
 * returns). capacity >= scene count. */
int vrod_solver_scene_reports(const vrod_solver* solver, int32_t capacity, vrod_step_report* reports);

/* ---- skinning (skinning.h / skinning.cpp): the consumer of the step's output, SURVEY.md §8(f)
 * rows 2-3. The CLI flow (vrod_main.cpp:52-73) is: rest pills + rest transforms of the rods ->
 * bind_skin -> smooth_binding, then every frame deform_mesh(binding, solver.pill_transforms()). */

/* PillTransform (skinning.h:19-25): element midpoint center, midpoint scale, element frame. */
typedef struct vrod_pill_transform {
  double center[3];
  double scale;
  double rotation[4]; /* w, x, y, z */
} vrod_pill_transform;

/* Solver::pill_transforms() = rod_pill_transforms(rods) of the live state (solver.cpp:438-440,
 * skinning.cpp:9-22): rod pills in rod-major, element-major order. */
int vrod_solver_pill_transforms(vrod_solver* solver, int64_t capacity, int64_t* count,
                                vrod_pill_transform* out);
/* rod_rest_pill_transforms / rod_rest_pills of the solver's rods (skinning.cpp:24-57): the
 * bind-time inputs (rest centers, rest scales x radii). */
int vrod_solver_rest_pill_transforms(vrod_solver* solver, int64_t capacity, int64_t* count,
                                     vrod_pill_transform* out);
int vrod_solver_rest_pills(vrod_solver* solver, int64_t capacity, int64_t* count, vrod_pill* out);

/* SkinBinding (skinning.h:31-40) together with the TriMesh it was bound to. */
typedef struct vrod_skin vrod_skin;
/* bind_skin(mesh, rest_pills, rest_transforms, max_influences, epsilon), skinning.cpp:59-105:
 * inverse-square surface-distance weights (pill_project), top max_influences per vertex with
 * ties by pill index, renormalized, listed by pill index. vertices: 3 per vertex; triangles:
 * 3 vertex ids each (used by smoothing; may be 0 triangles). */
int vrod_skin_bind(int32_t vertex_count, const double* vertices, int32_t triangle_count, const int32_t* triangles,
                   int32_t pill_count, const vrod_pill* rest_pills, const vrod_pill_transform* rest_transforms,
                   int32_t max_influences, double epsilon, vrod_skin** out);
void vrod_skin_destroy(vrod_skin* skin);
/* smooth_binding(binding, mesh, iterations), skinning.cpp:107-163. */
int vrod_skin_smooth(vrod_skin* skin, int32_t iterations);
/* The binding's CSR: offsets (vertex_count + 1), pills and weights (nnz each); any pointer may
 * be NULL; *nnz and *clamped_vertices always written. */
int vrod_skin_get_binding(const vrod_skin* skin, int32_t* offsets, int32_t* pills, double* weights, int32_t* nnz,
                          int32_t* clamped_vertices);
/* deform_mesh(binding, current, rest_mesh, out), skinning.cpp:165-185: out = 3 per vertex. */
int vrod_skin_deform(vrod_skin* skin, int32_t pill_count, const vrod_pill_transform* current, double* out_vertices);
/* The per-frame path on one device: pill transforms of the solver's live state, then the
 * deformation, without a host round trip of the transforms. out_vertices may be NULL (result
 * stays on the device, for timing). */
int vrod_skin_deform_solver(vrod_skin* skin, vrod_solver* solver, double* out_vertices);

/* ---- fine-grained (kernel-level) boundary, on host arrays ------------------------------ */

/* pill_project(x, pill), collision.h:64 / collision.cpp:15-49 — n independent queries. */
int vrod_pill_project(int64_t n, const double* points, const vrod_pill* pills, double* t,
                      double* distance, uint8_t* degenerate);
/* deepest_penetration(a, b, iterations, warm_alpha), collision.h:74-75 / :78-135. warm may be
 * NULL (= -1 for all). */
int vrod_deepest_penetration(int64_t n, const vrod_pill* a, const vrod_pill* b, int32_t iterations,
                             const double* warm_alpha, double* alpha, double* beta, double* distance);
/* broad_phase(pills), collision.h:87 / collision.cpp:184-238. Pairs (i<j) ascending; writes at
 * most `capacity` pairs but always reports the full count. */
int vrod_broad_phase(int64_t n, const vrod_pill* pills, int64_t capacity, int64_t* pair_count,
                     int32_t* pairs);
/* find_contacts(pills, pairs, iterations, warm), collision.h:92-95 / collision.cpp:251-273.
 * warm_keys/warm_alpha may be NULL (no warm list). */
int vrod_find_contacts(int64_t n, const vrod_pill* pills, int64_t pair_count, const int32_t* pairs,
                       int32_t iterations, int64_t warm_count, const uint64_t* warm_keys,
                       const double* warm_alpha, int64_t capacity, int64_t* count, int32_t* pill_a,
                       int32_t* pill_b, double* alpha, double* beta, double* distance);
/* extract_rotation(covariance, guess, max_iterations, tolerance), bundling.h:42-43 /
 * bundling.cpp:50-67: n independent problems; covariance row-major (9 each), guess and out
 * quaternions (w, x, y, z). */
int vrod_extract_rotation(int64_t n, const double* covariance, const double* guess, int32_t max_iterations,
                          double tolerance, double* out);
/* pair_key(a, b), collision.h:90 / collision.cpp:240-249. */
uint64_t vrod_pair_key(const vrod_pill* a, const vrod_pill* b);

#ifdef __cplusplus
}
#endif

#endif /* VROD_CAPI_H */
