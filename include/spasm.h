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

#ifdef __cplusplus
}
#endif
#endif /* SPASM_H_ */
