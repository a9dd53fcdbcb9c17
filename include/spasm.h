/*
 * spasm.h — C-ABI of libspasm.so, the B200-native (sm_100a) replacement for the
 * SPaSM two-stage particle optimizer's hot path.
 *
 * The reference (arxiv 2510.07674, package `seqplace`) is pure Python/numpy; its
 * plugin surface is the CostModel ABC + particle_opt.solve (stage 1) and
 * trajopt.solve_al / lift_placements / validate (stage 2). Each entry point below
 * names the reference function it replaces (path:line into /root/reference/pkg/src/seqplace).
 * The Python host package `paper_2510_07674_b200` binds these with ctypes and keeps the
 * reference's Python API; INTEGRATION.md shows the binding stub.
 *
 * Conventions
 *   - plain pointers + sizes only; device pointers are caller-owned CUDA memory,
 *     `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *   - every call returns an int status: 0 ok, 1 no solution, 2 lift failure,
 *     3 AL failure, >= 100 usage / CUDA error; spasm_last_error() describes the last
 *     failure of the calling thread. No C++ exception crosses this boundary;
 *   - dtype selects the arithmetic: SPASM_F32 (perf) or SPASM_F64 (parity);
 *     value/cost/gradient buffers are float* or double* accordingly;
 *   - values are row-major (P, D) matrices, exactly the reference's layout
 *     (block-major (x, y, z[, yaw]) rows, tetris.py:189-203 / tower.py:171-179).
 */
#ifndef SPASM_H_
#define SPASM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPASM_OK 0
#define SPASM_NO_SOLUTION 1
#define SPASM_LIFT_FAILURE 2
#define SPASM_AL_FAILURE 3
#define SPASM_ERR_USAGE 100
#define SPASM_ERR_CUDA 101

#define SPASM_F32 0
#define SPASM_F64 1

#define SPASM_LINEAR 0    /* geometry.LINEAR    (geometry.py:23) */
#define SPASM_QUADRATIC 1 /* geometry.QUADRATIC (geometry.py:24) */

#define SPASM_SAMPLER_PCG64 0  /* bit-exact numpy PCG64 restart streams (parity) */
#define SPASM_SAMPLER_PHILOX 1 /* Philox4x32-10 counter stream (perf mode)      */

typedef struct spasm_model spasm_model; /* opaque placement cost model (scene tables) */

const char* spasm_last_error(void);
int spasm_version(void);
/* sizeof() of an ABI struct by its type name ("spasm_solve_config", "spasm_solve_report",
 * "spasm_chain", "spasm_traj_desc", "spasm_al_config", "spasm_al_result"); -1 if unknown.
 * Lets a foreign binder (ctypes / cffi) check its struct mirrors against the library. */
int64_t spasm_abi_sizeof(const char* type_name);
/* Release the process-wide cache of pinned result-staging buffers (kept across model /
 * trajectory handles, capped at 32 buffers and 64 MB). Always SPASM_OK. */
int spasm_trim(void);
/* Measured FP32 CUDA-core peak (TFLOP/s) of the current device at its current clock: the
 * larger of a saturating scalar-FFMA and a packed-FFMA2 kernel on every SM (2 flops per FMA
 * lane). The bench's roofline denominator for the FP32 kernels. ffma / ffma2 optional. */
int spasm_fp32_peak(double* tflops, double* ffma_tflops, double* ffma2_tflops, void* stream);
/* Process-wide tuning switches (not in the reference; results stay within the parity
 * tolerances under every setting). "stage1_tile": -1 auto (default: on), 0 = generic
 * stage-1 kernels only, 1..4 = on (the fp32 tetris tile kernels, 4 lanes per particle;
 * stage1_tile.cuh). "graphs": 1 (default) runs each spasm_solve restart as a cached CUDA
 * graph, 0 launches its kernels one by one (same results). */
int spasm_set_option(const char* key, int value);

/* ---- model construction ------------------------------------------------------
 * Tetris packing model: replaces TetrisCostModel.__init__ + SphereInteractions.__init__
 * (problems/tetris.py:168-195, problems/_interactions.py:23-93).
 *   spheres_per_body[n_bodies]; local_centers[S_mov*3]; radii[S_mov] (body-major C order)
 *   static_*: wall spheres (tetris.py:54-70); static_normals[n_static*3] is the unit
 *   direction from each static centre towards the packing region (used by the fp32
 *   cancellation-free wall form; any unit vector is exact).
 *   lower/upper[D] clamp box (tetris.py:174-187). */
int spasm_tetris_model_create(spasm_model** out, int n_bodies, const int32_t* spheres_per_body,
                              const double* local_centers, const double* radii, int n_static,
                              const double* static_centers, const double* static_radii,
                              const double* static_normals, double w_block_block, double w_block_wall,
                              double w_height, double z_star, int free_yaw, const double* lower,
                              const double* upper);

/* Tower stacking model: replaces TowerCostModel.__init__ (problems/tower.py:150-169). */
int spasm_tower_model_create(spasm_model** out, int n_blocks, double side, double footprint_halfwidth,
                             const double* height_targets, int n_obstacles, const double* obstacle_centers,
                             const double* obstacle_radii, double w_stability, double w_height,
                             double w_collision, int free_yaw, const double* lower, const double* upper);

void spasm_model_destroy(spasm_model* model);
int spasm_model_dimension(const spasm_model* model);

/* ---- CostModel plugin surface ------------------------------------------------- */
/* CostModel.evaluate(values (P,D), mode) -> (P,)   (particle_opt.py:52; tetris.py:222; tower.py:234) */
int spasm_evaluate(const spasm_model* model, int dtype, const void* values, int64_t P, int mode, void* costs,
                   void* stream);
/* CostModel.gradient(values (P,D), mode) -> (P,D)  (particle_opt.py:55; tetris.py:230; tower.py:261) */
int spasm_gradient(const spasm_model* model, int dtype, const void* values, int64_t P, int mode, void* grad,
                   void* stream);

/* ---- engine pieces ----------------------------------------------------------- */
/* restart_stream(seed, restart) (particle_opt.py:176-178): the PCG64 state numpy derives
 * from SeedSequence(entropy=seed, spawn_key=(restart,)). out = {state_hi, state_lo, inc_hi, inc_lo}. */
int spasm_pcg64_state(uint64_t seed, uint64_t restart, uint64_t out[4]);

/* sample_uniform (+ inject_warm_start) for rows [row_offset, row_offset+N) of the restart's
 * (N_total, D) draw (particle_opt.py:181-192, 250-263). warm_dev: n_warm*D doubles (device). */
int spasm_sample(int dtype, int D, const double* lower, const double* upper, uint64_t seed, uint64_t restart,
                 int sampler, int64_t row_offset, int64_t N, const double* warm_dev, int64_t n_warm, void* values,
                 void* stream);

/* Fused sample + LINEAR evaluate + ranking keys (particle_opt.py:326-330): writes values,
 * order-preserving keys (uint32 for F32, uint64 for F64) and global row indices. */
int spasm_sample_eval(const spasm_model* model, int dtype, uint64_t seed, uint64_t restart, int sampler,
                      int64_t row_offset, int64_t N, const double* warm_dev, int64_t n_warm, void* values,
                      void* keys, uint32_t* idx, void* stream);

/* _step_values (particle_opt.py:214-228) for a caller-supplied gradient. lower/upper are
 * device arrays of the value dtype. flagged may be NULL. */
int spasm_step(int dtype, void* values, const void* grad, int64_t P, int D, double rate, const void* lower,
               const void* upper, uint8_t* flagged, void* stream);

/* run_descent_schedule (particle_opt.py:266-300) fused into one launch, plus the final
 * QUADRATIC cost (particle_opt.py:359). rows (optional) gathers src rows (the top-M
 * selection). trace_* optional (n_traced rows x (k_lin+k_quad) steps). */
int spasm_descent_schedule(const spasm_model* model, int dtype, const void* src, const uint32_t* rows, int64_t M,
                           int k_lin, int k_quad, double eta_init, double alpha, double epsilon, void* out_values,
                           void* out_cost, uint8_t* flagged, uint32_t* flagged_count, void* trace_cost,
                           uint8_t* trace_sat, int n_traced, void* stream);

/* Stable key sort (np.argsort(kind="stable"), particle_opt.py:199, 363). keys are uint32
 * (F32) or uint64 (F64); result left in (keys, vals). workspace >= spasm_sort_workspace_bytes. */
int64_t spasm_sort_workspace_bytes(int dtype, int64_t n);
int spasm_sort_pairs(int dtype, void* keys, uint32_t* vals, int64_t n, void* workspace, void* stream);

/* Order-preserving keys of costs (P,) for the stable sort. If threshold is finite, rows
 * with cost >= threshold get the maximal key and n_below counts the others. */
int spasm_cost_keys(int dtype, const void* costs, int64_t P, double threshold, void* keys, uint32_t* vals,
                    uint32_t* n_below, void* stream);

/* ---- whole stage-1 solve (particle_opt.solve, particle_opt.py:303-400) ---------- */
typedef struct {
  int64_t n, m;           /* sampling / optimization batch sizes */
  int32_t k_lin, k_quad;  /* phase lengths */
  double eta_init, alpha, epsilon;
  int32_t p_return, max_restarts;
  uint64_t seed;
  int32_t sampler;        /* SPASM_SAMPLER_* */
  int32_t n_traced;       /* 0 = no trace; else min(m, 4096) rows traced */
  /* perf-mode particle update (north_star item 4; not in the reference). All zero = the
   * reference's clamped gradient step (particle_opt.py:214-228), used by every parity path. */
  int32_t update;         /* 0 = gradient step (reference), 1 = Adam scaled by the lr schedule */
  float adam_beta1, adam_beta2, adam_eps;
  float noise_sigma;      /* initial Gaussian noise std / bound width, annealed to 0 over K_lin */
} spasm_solve_config;

typedef struct {
  int32_t success;        /* SolveResult.success */
  int32_t restarts;       /* SolveReport.restarts (0-based restart of success, or max_restarts) */
  int32_t steps;          /* SolveReport.steps */
  int32_t n_satisfying;   /* SolveReport.n_satisfying */
  int32_t flagged;        /* SolveReport.flagged */
  int32_t n_chosen;       /* rows written to the outputs (<= p_return) */
  int32_t launches;       /* libspasm kernels launched by this solve */
  int32_t reserved;
  double device_ms;       /* stream time of the solve (CUDA events) */
} spasm_solve_report;

/* spasm_solve in two halves, for callers that chain device work after stage 1 without a
 * host round trip (bench_api.solve_scene -> stage-2 lifting): spasm_solve_launch starts the
 * solve (with a repeated shape the whole restart loop is ONE CUDA graph launch -- a
 * conditional WHILE node, success test on the device -- and the call returns at once);
 * spasm_solve_device_rows gives device pointers to the compacted result rows (float64,
 * p_return x D) and their count (int32), valid in stream order after the launch;
 * spasm_solve_collect waits (the one host sync) and fills the same outputs as spasm_solve.
 * One pending solve per model. */
int spasm_solve_launch(const spasm_model* model, int dtype, const spasm_solve_config* cfg, const double* warm_host,
                       int64_t n_warm, void* workspace, int64_t workspace_bytes, void* stream);
int spasm_solve_device_rows(const spasm_model* model, const double** rows, const int32_t** n_rows);
int spasm_solve_collect(const spasm_model* model, double* particles, double* costs, int64_t* indices,
                        spasm_solve_report* report);

int64_t spasm_solve_workspace_bytes(const spasm_model* model, int dtype, const spasm_solve_config* cfg,
                                    int64_t n_warm);
/* Runs the restart loop on `stream`. Outputs (host): particles[p_return*D], costs[p_return],
 * indices[p_return] (row index in the restart's sampled batch), trace_* (device, optional,
 * steps x n_traced) and trace_ids (device int32[n_traced], the traced rows' batch indices).
 * Returns SPASM_OK (success) or SPASM_NO_SOLUTION (normal failure return). */
int spasm_solve(const spasm_model* model, int dtype, const spasm_solve_config* cfg, const double* warm_host,
                int64_t n_warm, void* workspace, int64_t workspace_bytes, double* particles, double* costs,
                int64_t* indices, spasm_solve_report* report, void* trace_cost, uint8_t* trace_sat,
                int32_t* trace_ids, void* stream);


/* ---- sharded stage-1 restart (multi-GPU, one process per GPU) -------
 * The two device halves of one restart of particle_opt.solve (particle_opt.py:325-384)
 * when the restart's N sampled rows are split into contiguous per-rank ranges (the
 * np.array_split analogue of _BatchOps, particle_opt.py:146-173). The host exchanges
 * between the halves (NCCL all-gather); results are identical to spasm_solve for any
 * world size. Workspace: spasm_shard_workspace_bytes(n_local_max, m_local_max).
 *
 * spasm_shard_select: sample + LINEAR-evaluate rows [row_lo, row_lo + n_local) of the
 *   restart's centralized draw (particle_opt.py:326-330), stable-sort them, and write the
 *   rank's elite run elite[m][2] = {order key, global row} (u64), ascending, padded with
 *   all-ones records when n_local < m.
 * spasm_shard_descend: merge the world*m gathered elite records into the global stable
 *   top-m (select_topk, particle_opt.py:195-200), re-draw the rows at positions
 *   [pos_lo, pos_hi) of it, run the fused descent schedule (particle_opt.py:266-300,
 *   359), order the satisfying rows (particle_opt.py:360-365) and re-check the first
 *   p_return (particle_opt.py:366). candidates (device float64) =
 *   [n_satisfying, flagged, k, p_return x (position, row, cost, recheck, values[D])]. */
int64_t spasm_shard_workspace_bytes(const spasm_model* model, int dtype, const spasm_solve_config* cfg,
                                    int64_t n_local, int64_t m_local);
int spasm_shard_select(const spasm_model* model, int dtype, const spasm_solve_config* cfg, int restart, int64_t row_lo,
                       int64_t n_local, const double* warm_dev, int64_t n_warm, void* workspace,
                       int64_t workspace_bytes, uint64_t* elite, int32_t* launches, void* stream);
int spasm_shard_descend(const spasm_model* model, int dtype, const spasm_solve_config* cfg, int restart,
                        const uint64_t* elite_all, int world, int64_t run_len, int64_t pos_lo, int64_t pos_hi,
                        const double* warm_dev, int64_t n_warm, void* workspace, int64_t workspace_bytes,
                        double* candidates, int32_t* launches, void* stream);
/* Exact distributed top-m selection (replaces the all-gather of m records per rank when that
 * gather is large): after spasm_shard_select (elite may then be NULL), per 8-bit key digit
 * (4 for F32, 8 for F64) spasm_shard_topm_hist counts the rank's keys per digit value under
 * the agreed prefix (256 int64), the caller all-reduces (sums) the counts over the ranks and
 * spasm_shard_topm_pick extends the prefix (state: spasm_shard_topm_state_bytes, set up by
 * spasm_shard_topm_init with m). spasm_shard_topm_local then gives the rank's
 * {records below K*, records at K*, K* records the top m takes}; the caller allots the ties
 * to the lowest ranks (lowest global rows) and spasm_shard_topm_contrib writes the rank's
 * first `take` sorted (key, row) records padded to `cap` (the largest take over the ranks);
 * the gathered contributions (m records in total) go to spasm_shard_descend with
 * run_len = cap. Same result as the all-gather protocol, bit for bit. */
int64_t spasm_shard_topm_state_bytes(void);
int spasm_shard_topm_init(int dtype, int64_t m, void* state, void* stream);
int spasm_shard_topm_hist(const spasm_model* model, int dtype, const spasm_solve_config* cfg, int64_t n_local,
                          void* workspace, const void* state, int64_t* hist, void* stream);
int spasm_shard_topm_pick(void* state, const int64_t* hist_sum, void* stream);
int spasm_shard_topm_local(const spasm_model* model, int dtype, const spasm_solve_config* cfg, int64_t n_local,
                           void* workspace, const void* state, int64_t* counts, void* stream);
int spasm_shard_topm_contrib(const spasm_model* model, int dtype, const spasm_solve_config* cfg, int64_t n_local,
                             void* workspace, int64_t take, int64_t cap, uint64_t* records, void* stream);

/* =====================================================================================
 * Stage 2: trajectory optimization (reference trajopt.py / robot.py)
 * ===================================================================================== */
typedef struct spasm_traj spasm_traj; /* opaque: one problem's _Geometry (trajopt.py:235-367) */

/* KinematicChain (robot.py:45-68) + its flattened link-sphere table (trajopt.py:311-321). */
typedef struct {
  int32_t dof, n_spheres;
  const double* axes;             /* dof*3 unit joint axes in the body frame */
  const double* offsets;          /* dof*3 translation applied before each joint */
  const double* lower;            /* dof joint limits */
  const double* upper;
  const double* tool_translation; /* 3 */
  const double* tool_rotation;    /* 9, row-major */
  const double* sphere_centers;   /* n_spheres*3 link-frame centres, sorted by link */
  const double* sphere_radii;     /* n_spheres */
  const int32_t* sphere_link;     /* n_spheres owning joint index (ascending) */
} spasm_chain;

/* Problem side of _build_geometry (trajopt.py:305-367). */
typedef struct {
  int32_t manipulation;           /* 0 = point-to-point MotionProblem (problems/motion.py) */
  int32_t n_blocks;               /* segments, skeleton order */
  const int32_t* spheres_per_block;
  const double* block_centers;    /* object-frame sphere centres (sum spheres_per_block)*3 */
  const double* block_radii;
  const double* staged_poses;     /* n_blocks*4 (x, y, z, yaw): problem.initial_poses */
  const double* grasp_offset;     /* GraspSpec.offset (3) */
  double grasp_yaw_offset;        /* GraspSpec.yaw_offset */
  int32_t n_static;
  const double* static_centers;   /* n_static*3 */
  const double* static_radii;
  const spasm_model* place_model; /* free-yaw placement twin (trajopt.py:281-302); NULL for motion */
  int32_t anchor_yaw;             /* problem.yaw_mode == fixed */
  int32_t rows_have_yaw;          /* stage-1 rows are (x, y, z, yaw) per block */
  const double* start;            /* motion endpoints (dof each) */
  const double* goal;
} spasm_traj_desc;

int spasm_traj_create(spasm_traj** out, const spasm_chain* chain, const spasm_traj_desc* desc);
void spasm_traj_destroy(spasm_traj* traj);
int spasm_traj_segments(const spasm_traj* traj);

/* TrajOptConfig (trajopt.py:118-177); waypoints = k_interp*(k_waypoint+1)+1. */
typedef struct {
  double w_start, w_arm, w_block, w_place, mu0, beta, lr_init, lr_final, validation_epsilon;
  int32_t outer_iters, inner_steps;
  int32_t place_mode;             /* placement-term mode used inside solve_al */
  int32_t waypoints;
} spasm_al_config;

typedef struct {
  int32_t status;                 /* SPASM_OK, SPASM_AL_FAILURE or SPASM_LIFT_FAILURE */
  int32_t accepted_outer;         /* outer iteration of the accepted particle (-1 on failure) */
  int32_t particle_index;         /* AlResult.particle_index */
  int32_t n_outers;               /* OuterRecords in the report */
  int32_t n_particles;            /* particles in the batch (after lifting) */
  int32_t lift_pick_fail;         /* first unreachable staged pose, -1 if none */
  double objective;               /* AlResult.objective */
  double least_violation;         /* TrajOptFailure.best_violation */
  double device_ms;
  /* float64 validate (trajopt.py:1071-1153) of the accepted trajectory, run on the device in
   * the same stream before the one host sync (the independent re-check of bench.py:249);
   * meaningful when status == SPASM_OK */
  double checked_violation;
  int32_t checked_feasible;
  int32_t reserved;
} spasm_al_result;

/* fk_batch (+ yaw_jacobian_batch) (robot.py:160-224). Q (n,dof) device; ee (n,3), rot (n,9);
 * origins/axes (n,dof,3) and yaw_jacobian (n,dof) optional (NULL). */
int spasm_fk(const spasm_traj* traj, int dtype, const void* Q, int64_t n, void* ee, void* rot, void* origins,
             void* axes, void* yaw_jacobian, void* stream);
/* ik_solve_batch (robot.py:227-302): per target, `restarts` seeds from
 * SeedSequence(seed, spawn_key=(target,)); targets are float64 device arrays. */
int spasm_ik_solve(const spasm_traj* traj, int dtype, const double* target_pos, const double* target_yaw,
                   int64_t n_targets, uint64_t seed, int restarts, int max_iters, double damping, void* solutions,
                   uint8_t* success, void* errors, void* stream);
/* _polish_tool_down (trajopt.py:726-776), in place on Q (n,dof). */
int spasm_polish_tool_down(const spasm_traj* traj, int dtype, void* Q, const double* target_pos,
                           const double* target_yaw, int64_t n, uint8_t* ok, void* stream);
/* _evaluate (trajopt.py:416-653): values (P,B,T,dof); lam (P,3), mu (P) may be NULL (zero).
 * Outputs objective (P), constraints (P,3), lagrangian (P), grad (P,B,T,dof) (each optional). */
int spasm_traj_evaluate(const spasm_traj* traj, int dtype, const spasm_al_config* cfg, const void* values,
                        int64_t P, int mode, int place_mode, const void* lam, const void* mu, int want_grad,
                        void* objective, void* constraints, void* lagrangian, void* grad, void* stream);
/* validate (trajopt.py:1071-1153) for P trajectories. */
int spasm_traj_validate(const spasm_traj* traj, int dtype, const spasm_al_config* cfg, const void* values,
                        int64_t P, uint8_t* feasible, void* violation, void* stream);
/* lift_placements (trajopt.py:795-876), asynchronous: placements (P,D) float64 device rows;
 * n_rows (device int32, optional): only the first min(P, *n_rows) rows exist (the stage-1
 * result read in place, spasm_solve_device_rows). Writes endpoints (kept,B,2,dof), kept[]
 * row indices and status[2] = {first unreachable staged pose or -1, kept count} on the
 * device. */
int64_t spasm_lift_workspace_bytes(const spasm_traj* traj, int dtype, int64_t P, int candidates);
int spasm_lift(const spasm_traj* traj, int dtype, const double* placements, int64_t P, const int32_t* n_rows, int D,
               uint64_t seed, int candidates, void* workspace, int64_t workspace_bytes, void* endpoints, int32_t* kept,
               int32_t* status, void* stream);
/* init_trajectories (trajopt.py:892-923) from a PCG64 state (the Generator the caller passes);
 * n_active (device, optional) bounds the live rows. spasm_trajectory_stream_state gives the
 * state of SeedSequence(seed, spawn_key=(1<<20,)) (bench.py:88-91). */
int spasm_trajectory_stream_state(uint64_t seed, uint64_t out[4]);
int spasm_init_trajectories(const spasm_traj* traj, int dtype, const void* endpoints, int64_t P, int n_segments,
                            const int32_t* n_active, int k_waypoint, int k_interp, const uint64_t pcg_state[4],
                            void* out, void* stream);
/* solve_al (trajopt.py:936-1063) as one persistent launch. Synchronous: returns
 * SPASM_OK / SPASM_AL_FAILURE / SPASM_LIFT_FAILURE (lift_status from spasm_lift, optional)
 * and fills result; best_values (B,T,dof) receives the accepted trajectory. The per-outer
 * records (OuterRecord) stay in the workspace: spasm_al_records gives their device
 * pointers {mu, lam, cons, upd, obj, viol, feas, first_feasible, n_outers, best_x}, each
 * [outer][P] (x3 for lam/cons/upd). */
int64_t spasm_al_workspace_bytes(const spasm_traj* traj, int dtype, int64_t P, const spasm_al_config* cfg);
int spasm_al_records(const spasm_traj* traj, int dtype, int64_t P, const spasm_al_config* cfg, void* workspace,
                     void* ptrs[10]);
int spasm_solve_al(const spasm_traj* traj, int dtype, const spasm_al_config* cfg, const void* values, int64_t P,
                   const int32_t* n_active, const int32_t* lift_status, void* workspace, int64_t workspace_bytes,
                   void* best_values, spasm_al_result* result, void* stream);
/* Host copy of the last SPASM_OK spasm_solve_al's accepted trajectory as float64 (B,T,dof),
 * n = B*T*dof values: staged in pinned memory by the solve's one D2H copy, so reading it
 * needs no CUDA call (AlResult.trajectory, trajopt.py:1056-1063; the values
 * _particle_trajectory turns into segments). SPASM_ERR_USAGE when nothing is staged. */
int spasm_al_best_host(const spasm_traj* traj, double* out, int64_t n);

/* Diagnostic: per-phase cycle counters of the fp32 AL kernel (marks 0-4: inner-step phases
 * P1-P5, 8: pick-waypoint polish, 9: re-evaluation + validate; 12-19 / 20-27: when thread
 * 0 / the aux warp reached each phase's barrier). enable 1/0; out (28 doubles, optional)
 * receives and resets the counters. */
int spasm_al_profile(int enable, double* out);
/* Diagnostic: per-warp own-work cycles per phase of the fp32 AL kernel (lane 0 of every
 * warp; out = 32 x 8 doubles [warp][phase], summed over CTAs) followed by 4 pick-polish
 * counters (iterations, calls, calls at the cap, max iterations); 260 doubles. Resets. */
int spasm_al_profile_warps(double* out);
/* Diagnostic: counters of the fp32 lift kernel k_ik_group, summed over CTAs (CTAs, cycles
 * to the last restart's IK, cycles to the end, max / winner IK iterations, winner polish
 * iterations after IK, speculatively completed polishes, all restarts' IK iterations), then
 * maxima over CTAs (cycles to the last restart's IK, cycles to the end, winner polish
 * iterations, IK iterations). enable 1/0; out (12 doubles, optional) receives and resets them. */
int spasm_ik_profile(int enable, double* out);

/* Self-test of the fp32 branch-free math on the device (n pseudo-random inputs from seed):
 * counts[0] = bit mismatches of the branch-free atan2 against atan2f, counts[1] / [2] = of
 * the normalize_yaw / np.mod fast-range folds against the scalar routines. All 0 expected. */
int spasm_selftest_math(int64_t n, uint64_t seed, int64_t counts[3]);

#ifdef __cplusplus
}
#endif
#endif /* SPASM_H_ */
