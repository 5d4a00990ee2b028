/*
 * bilevel_b200.h — C ABI of the B200-native bi-level planner hot path.
 *
 * This is the drop-in boundary for the data-parallel path of the reference
 * package `bilevel-drive` (arXiv 2212.02224): the batch Frenet trajectory
 * optimizer (stage-1 QP + alternating-minimisation projection) and the CEM
 * upper level.  The reference is pure Python with no FFI; each entry point
 * below names the reference interface whose work it replaces
 * (`pkg/` = pkg/src/bilevel_drive/).  INTEGRATION.md shows the ctypes binding.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Every array argument may be a HOST
 *     pointer (pageable or pinned; the library copies it over) or a DEVICE
 *     pointer on the context's device (used in place, no copy).  Calls whose
 *     outputs include a host pointer synchronise before returning; calls on
 *     device pointers only are asynchronous on the context stream.
 *   - Layouts are row-major and SAMPLE-MAJOR: a batch of B coefficient vectors
 *     is B x 2n (the reference stores 2n x B column-per-sample; the Python shim
 *     transposes).  Several independent scenes ("fleet") are stacked scene-major:
 *     sample s of scene j lives at row j*B + s.
 *   - Return 0 on success or a negative BD_ERR_* code; bd_last_error() gives text.
 *   - One context per device; a context is not thread-safe.
 */
#ifndef BILEVEL_B200_H
#define BILEVEL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BD_ABI_VERSION 4

#define BD_OK 0
#define BD_ERR_VALUE (-1)      /* ValueError        pkg/batch_qp.py:99-106,223-227,265-269; pkg/projection.py:225-233 */
#define BD_ERR_STRUCTURE (-2)  /* StructureError    pkg/batch_qp.py:39-40,127-140 */
#define BD_ERR_NUMERICAL (-3)  /* NumericalFailure  pkg/batch_qp.py:43-44,272-279; pkg/projection.py:290-291 */
#define BD_ERR_CUDA (-4)       /* CUDA runtime error (RuntimeError) */
#define BD_ERR_STATE (-5)      /* constants not uploaded / call order */

typedef struct bd_ctx bd_ctx;

/* Scalars of ConstraintSpec (pkg/constraints.py:31-42). */
typedef struct bd_limits {
    double ellipse_a, ellipse_b, v_min, v_max, a_max, kappa_max, c_max, y_lb, y_ub;
} bd_limits;

/* BiLevelConfig (pkg/bilevel.py:72-97) plus the projection budget (pkg/projection.py:38-46). */
typedef struct bd_cem_config {
    int batch;          /* n-bar: samples per scene and CEM iteration          */
    int n_cons;         /* constraint_elites n                                 */
    int n_elite;        /* elites q                                            */
    int iterations;     /* CEM iterations N                                    */
    int am_iters;       /* ProjectionConfig.max_iters                          */
    double eta, gamma, residual_weight, tol;
    uint64_t seed;      /* Philox key when z == NULL (device RNG mode)         */
    int scene_offset;   /* global index of scene 0 (Philox counter; shard-invariant fleets) */
    int iter_begin;     /* run CEM iterations [iter_begin, iter_end) of the cycle (0, 0 = all);  */
    int iter_end;       /* a cycle may be split over calls on one context (state stays on the   */
                        /* device; no other solve in between), z then covering only this range */
    /* numpy stream mode (z == NULL and pcg64_state != NULL): the normals are numpy's
     * Generator(PCG64).standard_normal stream, drawn on the device from pcg64_state = {state lo,
     * state hi, increment lo, increment hi} (bit generator state before the first draw of this
     * call); needs bd_set_normal_tables.  pcg64_positions (host or device, draw-iterations + 1
     * entries) receives the raw 64-bit outputs consumed after each drawing CEM iteration, so the
     * caller can advance its Generator exactly (pkg/bilevel.py:51-57 consumption). */
    const uint64_t* pcg64_state;
    int64_t* pcg64_positions;
} bd_cem_config;

/* ------------------------------------------------------------------ lifecycle */
int bd_abi_version(void);
int bd_create(int device, bd_ctx** out);
void bd_destroy(bd_ctx* ctx);
const char* bd_last_error(const bd_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL restores the library stream. */
int bd_set_stream(bd_ctx* ctx, void* cuda_stream);
int bd_synchronize(bd_ctx* ctx);
/* Knobs: "lanes_per_sample" (0=auto, 4/8/16/32/64), "samples_per_cta" (0=auto), "timing" (0/1),
 * "latency_instance" (1=auto / 0=never pick the up-to-255-register one-warp AM instance for 5-8
 * samples per SM), "remainder_warp" (1=auto / 0=never add the remainder warp to that instance at
 * 3-8 samples per SM), "persistent_cycle" (1=auto / 0=never run a single-scene bd_cem_cycle as
 * the persistent cooperative kernel), "cvae_tensor_cores" (1/0), "cvae_fused" (1/0: the decoder
 * as one cooperative kernel), "sticky_errors" (1/0). */
int bd_set_option(bd_ctx* ctx, const char* key, int value);
/* Kernel launches issued by this context since creation (instrumentation). */
int64_t bd_launch_count(const bd_ctx* ctx);
/* Instrumentation (enable with bd_set_option(ctx, "timing", 1)): "am_ms" = summed CUDA-event
 * time of the AM kernel launches (recorded on the launching stream), "am_launches",
 * "am_sample_iters" = samples x iterations executed; "reset" clears them; "persistent_cycles" =
 * bd_cem_cycle calls run as the persistent cooperative kernel (any time). Synchronises. */
int bd_get_stat(bd_ctx* ctx, const char* key, double* value);
/* Measurement probes for roofline denominators: "fp32_tflops" = dense FFMA throughput of an
 * all-SM register-resident kernel (CUDA events, current clocks); "fp32x2_tflops" = the same with
 * packed fma.rn.f32x2 (FFMA2). */
int bd_probe(bd_ctx* ctx, const char* what, double* value);
/* Synchronise and return (in *bits) the OR of the device error words of the last
 * asynchronous call: 1 = non-finite iterate, 2 = stage-1 KKT residual above 1e-8. */
int bd_error_bits(bd_ctx* ctx, int* bits);

/* ------------------------------------------------------------------ constants
 * Uploaded once per LowerLevelSolver (pkg/bilevel.py:204-215); the host keeps
 * the LU factorizations (FACTORIZATION_COUNT, pkg/batch_qp.py:31-36).          */

/* Sampled basis W, Wdot, Wddot, m x n row-major fp64 (build_basis, pkg/basis.py:156-179). */
int bd_set_basis(bd_ctx* ctx, int m, int n, const double* W, const double* Wd, const double* Wdd);

/* Stage-1 tracking QP (build_qp_structure / build_rhs_batch / solve_batch,
 * pkg/batch_qp.py:152-280): set-point -> linear-cost maps q_map_x/q_map_y
 * (n x m_seg), the bordered KKT and its inverse ((2n+neq)^2, fp64).           */
int bd_set_stage1(bd_ctx* ctx, int m_seg, int with_goal, int neq, const double* q_map_x,
                  const double* q_map_y, const double* kkt, const double* kkt_inv);

/* Projection operator (ProjectionOperator.__init__, pkg/projection.py:189-214):
 * inverse of the penalty-augmented KKT ((2n+neq)^2) and A_eq (neq x 2n).
 * The x/y blocks must decouple (they do for every reference layout).         */
int bd_set_projection(bd_ctx* ctx, int n_obs, double rho, int neq, const double* kkt_inv_aug,
                      const double* a_eq);

/* Scenes (PlanningScene / ConstraintSpec, pkg/constraints.py:19-92):
 * obstacles S x n_obs x m, limits S, initial states S x 6, optional tabulated
 * road curvature S x n_curv (np.interp semantics; n_curv = 0 for straight roads). */
int bd_set_scenes(bd_ctx* ctx, int n_scenes, int n_obs, int m, const double* ox, const double* oy,
                  const bd_limits* limits, const double* b0, int n_curv, const double* curv_x,
                  const double* curv_k);

/* ------------------------------------------------------------------ lower level */

/* Stage-1 batch solve: solve_batch(build_rhs_batch(params)) (pkg/batch_qp.py:209-280),
 * including the 1e-8*(1+|rhs|) KKT residual check -> BD_ERR_NUMERICAL.
 * params (S*B) x dim; outputs xi_bar (S*B) x 2n, mu (S*B) x neq, b (S*B) x neq (each may be NULL). */
int bd_stage1(bd_ctx* ctx, int n_scenes, int batch, const double* params, double* xi_bar, double* mu,
              double* b_out);

/* AM projection: ProjectionOperator.project (pkg/projection.py:216-339), incl. the
 * residual evaluator (pkg/constraints.py:142-153) and the batch-global early exit
 * (pkg/projection.py:329), per scene.  b may be NULL (scene b0, zero goal rows).
 * Outputs: xi (S*B) x 2n, residuals S*B, optional upper cost S*B (pkg/bilevel.py:125-126),
 * optional history S x max_iters x B (fp32; rows >= iterations_used are undefined),
 * iterations_used S, clip_conflicts S.                                          */
int bd_project(bd_ctx* ctx, int n_scenes, int batch, const double* xi_bar, const double* b, int max_iters,
               double tol, double* xi, double* residuals, double* cost, float* history, int* iters_used,
               int64_t* conflicts);

/* LowerLevelSolver.solve + upper_cost_batch fused (pkg/bilevel.py:217-225,125-126). */
int bd_solve_lower(bd_ctx* ctx, int n_scenes, int batch, const double* params, int max_iters, double tol,
                   double* xi_bar, double* mu, double* xi, double* residuals, double* cost, float* history,
                   int* iters_used, int64_t* conflicts);

/* Trajectory evaluation on the basis grid: eval_trajectory / LowerLevelSolver.velocities
 * (pkg/basis.py:182-195, pkg/bilevel.py:223-225).  xi N x 2n -> each output N x m (may be NULL). */
int bd_eval(bd_ctx* ctx, int count, const double* xi, double* x, double* y, double* xd, double* yd,
            double* xdd, double* ydd);

/* Direct residual evaluator batch_residuals (pkg/constraints.py:142-153) on given coefficients,
 * scene-major (S*B) x 2n -> S*B. */
int bd_residuals(bd_ctx* ctx, int n_scenes, int batch, const double* xi, double* residuals);

/* Generic batched KKT solve: solve_batch(structure, rhs) (pkg/batch_qp.py:258-280) for any
 * bordered system with nvar + neq <= 32: sol = kkt_inv rhs per column, with the reference's
 * residual check.  rhs and sol are count x (nvar+neq) (one row per sample). */
int bd_kkt_solve(bd_ctx* ctx, int nvar, int neq, const double* kkt, const double* kkt_inv, int count,
                 const double* rhs, double* sol);

/* Sharded single-scene batch (multi-GPU, BASELINE config 4).  Stage 1 + AM projection of this
 * rank's contiguous shard WITHOUT the batch-global exit decision: iter_max (max_iters floats)
 * receives the shard's per-iteration maximum residual, which the caller all-reduces (MAX) over
 * ranks to apply pkg/projection.py:329 globally; bd_replay_shard then re-runs the shard for
 * exactly the global iteration count when the exit fired earlier.  One scene (S = 1). */
int bd_solve_lower_shard(bd_ctx* ctx, int batch, const double* params, int max_iters, double* xi_bar, double* xi,
                         double* residuals, double* cost, float* iter_max);
int bd_replay_shard(bd_ctx* ctx, int batch, const double* xi_bar, int iterations, double* xi, double* residuals,
                    double* cost);
/* Sharded batch over NVLink peer memory.  Each rank passes device arrays of the world's symmetric
 * buffers and signal pads (e.g. torch symmetric memory: buffer_ptrs_dev / signal_pad_ptrs_dev) and
 * the byte offsets of: gathered residuals (batch doubles), gathered costs (batch doubles), the
 * per-rank iteration maxima (world x iters_cap floats), one coefficient row per rank (world x 22
 * doubles).  bd_solve_lower_shard_p2p = bd_solve_lower_shard + the exchange: the AM epilogue
 * stores every (residual, cost) into every rank's buffer at row0 + i, the maxima are published and
 * awaited, the batch-global exit is decided on the device (iterations used -> *used) and the shard
 * replayed if it fired -- after it every rank holds the whole batch's residuals and costs.
 * bd_shard_p2p_best_row hands the coefficients of global row *best_index to every rank.  epoch:
 * strictly increasing per CEM iteration, identical on all ranks. */
int bd_shard_p2p_set(bd_ctx* ctx, int world, int rank, void* const* buffers, unsigned* const* signal_pads,
                     size_t res_offset, size_t cost_offset, size_t itmax_offset, size_t row_offset, int iters_cap);
int bd_solve_lower_shard_p2p(bd_ctx* ctx, int batch, const double* params, int max_iters, double* xi_bar, double* xi,
                             double* residuals, double* cost, long long row0, unsigned epoch, double tol, int* used);
int bd_shard_p2p_best_row(bd_ctx* ctx, const int64_t* best_index, long long row0, int batch, const double* xi_shard,
                          unsigned epoch, double* xi_out);
/* Same, with the iteration count read on the device (one int; <= 0: keep the first pass) so a
 * sharded CEM iteration needs no host round trip between the all-reduce and the ranking. */
int bd_replay_shard_dev(bd_ctx* ctx, int batch, const double* xi_bar, int max_iters, const int* iterations,
                        double* xi, double* residuals, double* cost);

/* ------------------------------------------------------------------ upper level */

/* Device-RNG sampling: p = mean + z chol(cov)^T with z = Philox4x32-10 normals keyed by
 * (seed, scene, iteration, first_index + i) -- the same stream bd_cem_cycle draws, so any
 * shard of a batch can be regenerated on any rank. */
int bd_sample_philox(bd_ctx* ctx, int dim, int count, const double* mean, const double* cov, uint64_t seed,
                     int scene, int iteration, int first_index, double* params);

/* SamplingDistribution.sample (pkg/bilevel.py:51-57): p = mean + z chol(cov)^T, with the
 * reference's 1e-5 I fallback; z count x dim (e.g. from the caller's numpy Generator). */
int bd_sample(bd_ctx* ctx, int dim, int count, const double* mean, const double* cov, const double* z,
              double* params);

/* rank_samples + update_distribution (pkg/bilevel.py:129-137,163-194) per scene.
 * mean (S x dim) and cov (S x dim x dim) are updated in place.  Outputs (may be NULL):
 * cons_idx S x n_cons, elite_idx S x n_elite, elite_aug S x n_elite,
 * stats S x 6 = IterationStats fields (pkg/bilevel.py:100-108) after the update. */
int bd_rank_refit(bd_ctx* ctx, int n_scenes, int batch, int dim, const double* residuals, const double* cost,
                  const double* params, int n_cons, int n_elite, double residual_weight, double eta,
                  double gamma, double* mean, double* cov, int64_t* cons_idx, int64_t* elite_idx,
                  double* elite_aug, double* stats);

/* One full CEM planning cycle per scene: solve_bilevel (pkg/bilevel.py:228-295).
 * Samples p = mean + z L^T (pkg/bilevel.py:51-57) with z supplied (iterations x S x B x dim,
 * e.g. from the caller's numpy Generator) or drawn on device with Philox (z == NULL).
 * warm (S x B x dim or NULL) replaces the first iteration's draw (pkg/bilevel.py:250-251).
 * Per-scene outputs (each may be NULL): best_index, best_params (dim), best_xi (2n),
 * best_cost, best_residual, best_aug, stats (iterations x 6), final mean/cov,
 * iterations_done (completed CEM iterations; < iterations means degraded, pkg/bilevel.py:254-261). */
int bd_cem_cycle(bd_ctx* ctx, int n_scenes, const bd_cem_config* cfg, const double* init_mean,
                 const double* init_cov, const double* z, const double* warm, int64_t* best_index,
                 double* best_params, double* best_xi, double* best_cost, double* best_residual,
                 double* best_aug, double* stats, double* final_mean, double* final_cov, int* iterations_done);

/* numpy's 256-layer ziggurat tables (ki: uint64, wi / fi: double, 256 each) for the numpy stream
 * mode of bd_cem_cycle and bd_numpy_normals.  Host pointers. */
int bd_set_normal_tables(bd_ctx* ctx, const uint64_t* ki, const double* wi, const double* fi);

/* numpy's Generator(PCG64).standard_normal stream on the device: `count` normals from the PCG64
 * state {state lo, state hi, increment lo, increment hi} into z (host or device), and the raw
 * outputs consumed after every block of block_len draws into positions (count / block_len + 1
 * entries, host or device).  Replaces rng.standard_normal in SamplingDistribution.sample
 * (pkg/bilevel.py:56). */
int bd_numpy_normals(bd_ctx* ctx, const uint64_t* pcg64_state, long long count, long long block_len, double* z,
                     int64_t* positions);

/* The last CEM iteration's batch of the preceding bd_cem_cycle on this context (the arguments of the
 * reference's trace_hook, pkg/bilevel.py:269-270): set-points S x B x dim, projected coefficients
 * S x B x 2n, residuals S x B, upper costs S x B (each may be NULL). */
int bd_cem_last_batch(bd_ctx* ctx, int n_scenes, int batch, double* params, double* xi, double* residuals,
                      double* cost);

/* ------------------------------------------------------------------ scene construction / control emission
 * the steps either side of the path, on the device.                          */

/* Planner-side constants of build_scene (PlannerEnvConfig, pkg/planners.py:40-87). */
typedef struct bd_env {
    int max_obstacles;          /* obstacle rows per scene (must equal the projection's n_obs)      */
    double obstacle_range;      /* longitudinal neighbour filter [m]                                */
    double wheelbase;           /* ego_flat_state yaw rate                                          */
    double v_max, a_max, kappa_max, c_max, v_min;
    double other_length, other_width;   /* neighbour footprint for combined_ellipse (5 x 2 m)      */
} bd_env;

/* build_scene + ego_flat_state (pkg/planners.py:99-160) and observe (pkg/highway.py:208-246) for S
 * worlds, writing the scenes straight into the context (replaces bd_set_scenes).
 * ego S x 8 (x, y, psi, v, accel, steer, length, width); veh S x n_veh_max x 5 (x, y, psi, v,
 * lateral_rate) in world.neighbors order; n_veh S; road S x 2 (lane_count, lane_width);
 * times m (basis.times).  Optional outputs: obstacles S x n_obs x m (x, y), initial states S x 6,
 * limits S x 9 (a b v_min v_max a_max kappa_max c_max y_lb y_ub), observations S x 55. */
int bd_build_scenes(bd_ctx* ctx, int n_scenes, int n_veh_max, const double* ego, const double* veh,
                    const int* n_veh, const double* road, const bd_env* env, const double* times, double* ox_out,
                    double* oy_out, double* b0_out, double* limits_out, double* observations);

/* Road curvature for the scenes currently in the context (e.g. after bd_build_scenes):
 * ConstraintSpec.road_curvature = world.road.curvature (pkg/planners.py:154, pkg/constraints.py:67-72),
 * S tables of n_curv strictly increasing abscissae cx and curvatures ck (row-major S x n_curv);
 * n_curv = 0 removes them. */
int bd_set_curvature(bd_ctx* ctx, int n_scenes, int n_curv, const double* cx, const double* ck);

/* controls_on_grid -> flat_to_controls (pkg/planners.py:209-216, pkg/basis.py:206-234): the basis
 * derivative rows at the n_ctrl control instants (matrices_at), then per trajectory the clipped
 * (accel, steer) sequence; singular[i] = 1 where the speed drops to eps_v (SpeedSingularity). */
int bd_set_control_grid(bd_ctx* ctx, int n_ctrl, const double* Wd_ctrl, const double* Wdd_ctrl, double wheelbase,
                        double a_max, double steer_limit, double eps_v);
int bd_controls(bd_ctx* ctx, int count, const double* xi, double* accel, double* steer, int* singular);

/* ------------------------------------------------------------------ closed-loop simulation
 * SURVEY §8f row 4.  Replaces the Python simulator tick step (pkg/highway.py:358-410: neighbour
 * IDM + MOBIL decisions on the frozen snapshot, ego RK4 bicycle, neighbour updates, SAT collision,
 * lane departure) and the open-loop inner loop of run_episode (pkg/highway.py:517-529) for S worlds.
 * Traffic constants: IDMParams / MOBILParams (pkg/highway.py:73-89), ScenarioConfig.dt, wheelbase. */
typedef struct bd_traffic {
    double idm_v0, idm_time_headway, idm_s0, idm_a_max, idm_b_comfort, idm_delta, idm_b_hard;
    double mobil_politeness, mobil_b_safe, mobil_a_threshold, mobil_cooldown;
    double dt, wheelbase;
} bd_traffic;

/* Run n_steps ticks of S worlds in place.  World state (device or host pointers; host arrays are
 * copied in and back): ego S x 8 (x, y, psi, v, accel, steer, length, width — the bd_build_scenes
 * layout), ego_target_speed S, veh S x n_veh_max x 5 (x, y, psi, v, lateral_rate), veh_ext
 * S x n_veh_max x 7 (length, width, target_speed, target_lane, cooldown, accel, lane_index),
 * n_veh S, road S x 2 (lane_count, lane_width), world S x 5 (time, step_count, collided,
 * collision_step or -1, lane_departed).  Tick j applies controls[s][min(ctrl_offset + j, n_ctrl-1)]
 * (accel, steer).  x_end NULL: plain ticks.  x_end S: run_episode semantics — a world stops after
 * the tick that collides or reaches ego.x >= x_end[s], and its active flag is cleared.  active S
 * (nullable, in/out): worlds with 0 are not stepped.  steps_done S (nullable): ticks executed.
 * snapshots (nullable): S x n_steps x (8 + 4 n_veh_max) doubles per tick: time, ego x y psi v
 * accel steer, collided, then each neighbour's x y psi v (the run_episode step record). */
int bd_sim_run(bd_ctx* ctx, int n_worlds, int n_veh_max, double* ego, double* ego_target_speed, double* veh,
               double* veh_ext, const int* n_veh, const double* road, double* world, const bd_traffic* traffic,
               int n_steps, const double* controls, int n_ctrl, int ctrl_offset, const double* x_end, int* active,
               int* steps_done, double* snapshots);

/* ------------------------------------------------------------------ CVAE warm start
 * Decoder MLP of the paper (not in the reference package):
 * (obs 55 + z 2) -> 1024 -> 1024 -> 1024 -> 1024 -> 256 -> dim, BatchNorm folded
 * into the Linear layers, ReLU between.  Weights fp32 row-major [out x in] + bias. */
int bd_cvae_set_weights(bd_ctx* ctx, int n_layers, const int* dims, const float* const* weights,
                        const float* const* biases);
int bd_cvae_decode(bd_ctx* ctx, int count, const float* obs /* 55 */, const float* z /* count x 2 */,
                   double* params /* count x dim */);
/* The decoder's samples as warm-start rows, kept on the device: rows = decode * scale + shift
 * (per column; either may be NULL; two float64 roundings, as numpy's p * scale + shift).
 * *rows_dev receives the device address of the count x dim rows, valid until the next call of
 * this function on the context; pass it as bd_cem_cycle's `warm` (device pointers are used in
 * place).  params (host or device, count x dim) may be NULL: then nothing is copied back and
 * the call does not synchronise. */
int bd_cvae_warm_start(bd_ctx* ctx, int count, const float* obs, const float* z, const double* scale,
                       const double* shift, double* params, const double** rows_dev);

#ifdef __cplusplus
}
#endif
#endif /* BILEVEL_B200_H */
