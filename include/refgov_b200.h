/*
 * refgov_b200.h -- C ABI of the B200-native robust Reference Governor hot path.
 *
 * Drop-in boundary for the reference package `refgov` (arxiv 2510.08288,
 * pkg/src/refgov).  The reference reaches its device through a subprocess
 * and temp-file protocol (backend_gpu.fill, backend_gpu.py:50-140) and runs
 * its CPU hot loop in numba (kernels.py:47-162); this library replaces both
 * with in-process calls into sm_100a kernels.  Plain C types only: host or
 * device pointers plus sizes; no torch or CUDA types in any signature.
 *
 * Return codes map onto the reference's error taxonomy (errors.py:8-32):
 *   RG_OK              0
 *   RG_E_NODEVICE     -1  -> BackendUnavailableError (no CUDA device)
 *   RG_E_UNSUPPORTED  -2  -> BackendUnavailableError (not sm_100, or a host
 *                            libm whose tanh neither port reproduces)
 *   RG_E_ARGS         -3  -> ConfigError (shapes, ranges)
 *   RG_E_CUDA         -4  -> RefgovError (device failure)
 * rg_last_error() returns a thread-local message for the last failure.
 *
 * Threading: one call at a time per context (the reference's governor is not
 * re-entrant either).  Calls are synchronous unless RG_ASYNC is
 * passed; results are on the host when a synchronous call returns.
 */
#ifndef REFGOV_B200_H
#define REFGOV_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define RG_API __attribute__((visibility("default")))
#else
#define RG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define RG_ABI_VERSION 1

#define RG_OK 0
#define RG_E_NODEVICE (-1)
#define RG_E_UNSUPPORTED (-2)
#define RG_E_ARGS (-3)
#define RG_E_CUDA (-4)

/* cell status codes: kernels.py:37-39 */
#define RG_CELL_VIOLATED 0
#define RG_CELL_OK 1
#define RG_CELL_OVERFLOW 2

/* which glibc expm1 build the device tanh reproduces */
#define RG_TANH_AUTO 0    /* probe the host libm once at rg_create */
#define RG_TANH_FMA 1     /* __expm1_fma (x86-64 hosts with FMA+AVX2) */
#define RG_TANH_GENERIC 2 /* generic SSE2 __expm1 */

/* flags */
#define RG_DEVICE_PTRS 0x1  /* array arguments are device pointers (x0[3] is always host) */
#define RG_ASYNC 0x2        /* enqueue only; no host readback, no sync */
#define RG_ABANDON 0x4      /* grid step: stop rows already known infeasible */
#define RG_NO_TIMING 0x8    /* no CUDA-event timing: kernel_ms is the device clock's span (globaltimer) */
#define RG_TANH_LOCKSTEP 0x10 /* rg_tanh: use the rollout's lockstep form */
#define RG_FUSED_RNG 0x20   /* RNG source: hash inside the rollout loop */
#define RG_STAGE_RNG 0x40   /* RNG source: generate the SoA tensor first */
/* With neither RG_FUSED_RNG nor RG_STAGE_RNG an RNG source is staged when the
 * SoA block (n_sim * j_star * 24 bytes) is at most 16 GB for the fill and the
 * grid step (all candidate rows share it), at most 96 MB for the bisections
 * (whose rollouts often stop after a few steps), and fused above.  The batched
 * grid step stages each episode's block, in chunks of episodes of at most 16 GB,
 * unless RG_FUSED_RNG is given. */
#define RG_JOINT_ITER 0x80  /* rg_bisect_joint: one kernel per iteration (the sharded form's
                               kernels) instead of the single persistent kernel */
#define RG_XCHG 0x100      /* rg_grid_step: the scenario-sharded step's all-reduce fused into the
                               kernel over NVLink (see rg_xchg_init) */

typedef struct rg_ctx rg_ctx;

/* Plant and constraint set for every call.
 * step_size:        SurrogateFuelCellPlant.step_size (dynamics.py:247-263)
 * y_lower, y_upper: ConstraintSet.lower/upper on y = x1 (constraints.py:37-70)
 * ss_v_lower/upper: the setpoints v whose steady state passes the tightened
 *                   set, tight.contains(np.tanh(v)) (governor.py:302, 401),
 *                   as an exact interval computed and verified on the host
 * j_star:           prediction horizon in steps */
typedef struct {
    double step_size;
    double y_lower, y_upper;
    double ss_v_lower, ss_v_upper;
    int32_t j_star;
    int32_t _pad;
} rg_problem;

/* Counter-RNG scenario set (disturbance.py:179-203): scenario k of the set is
 * k0 + k of the stream `seed`, entry (k, j, i) = lo[i] + span[i] * u.  The
 * surrogate plant uses components 0..2, a linear plant 0..n-1 (n <= 4). */
typedef struct {
    uint64_t seed;
    int64_t k0;
    int64_t n_sim;
    double lo[4];
    double span[4];
} rg_scenarios;

/* A LinearOraclePlant (dynamics.py:162-206): x+ = A x + B v, y = C x + D v,
 * n <= 4 states, A row-major; the steady-state gate is
 * ss_lower <= dc_gain * v <= ss_upper (governor.py:302 with the tightened set). */
typedef struct {
    int32_t n;
    int32_t _pad;
    double A[16];
    double B[4];
    double C[4];
    double D;
    double dc_gain;
    double ss_lower, ss_upper;
} rg_linear_plant;

/* Result of rg_grid_step (robust_rg_parallel, governor.py:520-579). */
typedef struct {
    int32_t row;            /* 0-based best all-feasible row, -1 when none */
    int32_t n_active;       /* rows simulated after the steady-state gate and dedup */
    int32_t ss_pruned_rows; /* governor.py:344 */
    int32_t dedup_rows;     /* governor.py:345 */
    int64_t sims_run;       /* n_active * n_sim (governor.py:341) */
    int64_t early_terms;    /* evaluated cells with steps < j_star (governor.py:342) */
    int64_t overflows;      /* cells ending in CELL_OVERFLOW (governor.py:343) */
    int64_t abandoned;      /* cells stopped by RG_ABANDON (0 without it) */
    float kernel_ms;        /* CUDA-event time of the step kernel */
    float reduce_us;        /* device time of the final reduction: the last block's row
                               extraction and result publication (globaltimer; 0 when the
                               kernel does not record it) */
} rg_grid_result;

/* Result of rg_bisect (robust_rg_sequential / bisection_rg). */
typedef struct {
    double kappa;           /* min over scenarios of the bisected kappa */
    int32_t found;          /* AND over scenarios */
    int32_t _pad;
    int64_t cells;          /* sims_run (governor.py:501) */
    int64_t early;          /* early_terms (governor.py:502) */
    float kernel_ms;
    int32_t _pad2;
} rg_bisect_result;

RG_API int32_t rg_abi_version(void);
RG_API const char *rg_last_error(void);
RG_API int32_t rg_device_count(int32_t *n);

/* Create a context on CUDA device `device` (sm_100 required). */
RG_API int32_t rg_create(int32_t device, int32_t tanh_variant, rg_ctx **out);
RG_API int32_t rg_destroy(rg_ctx *ctx);
RG_API int32_t rg_get_tanh_variant(rg_ctx *ctx, int32_t *variant);
/* Per-context tuning knobs (none changes a result bit): "force_tpb" (0/32/64/128),
 * "no_placement", "no_pdl", "no_step2", "fused_gen" (0/1), "batch_chunk" (episodes
 * per staged chunk, 0 = automatic), "xchg_timeout_ms" (fused exchange, default 10000),
 * "no_row_plan" (0/1: grid steps without P derive their rows on the device instead of
 * launching only the host-planned simulated rows), "no_ts" (0/1: never the time-split
 * grid kernel for host-planned steps with few cells), "ts_staged" (0/1: the time-split
 * kernel reads a staged scenario block instead of generating the disturbances itself),
 * "no_ts_probe" (0/1: rg_bisect and the persistent rg_bisect_joint roll their kappa = 1
 * probe out inside their own kernels instead of on the time-split kernel first),
 * "no_device_loop" (0/1: rg_closed_loop launches one grid step per closed-loop step instead
 * of running the whole trace in one kernel).  Defaults come from the RG_FORCE_TPB,
 * RG_NO_PLACEMENT, RG_NO_PDL, RG_NO_STEP2, RG_FUSED_GEN, RG_NO_ROW_PLAN, RG_NO_TS,
 * RG_TS_STAGED, RG_NO_TS_PROBE, RG_NO_DEVICE_LOOP and RG_BATCH_CHUNK environment variables,
 * read once at rg_create.  Unknown names give RG_E_ARGS. */
RG_API int32_t rg_set_option(rg_ctx *ctx, const char *name, int64_t value);
/* Read a knob of rg_set_option, or the read-only "last_grid_kernel": which kernel the
 * context's last grid step launched (0 = k_grid, one warp per 32 rollouts; 1 = k_grid_ts,
 * the time-split form), "grid_step_kernels": how many kernels the context's grid steps
 * have launched so far (the scenario staging kernel, when used, and the step kernel; a
 * device closed loop counts one), or "last_loop_device": 1 if the last rg_closed_loop ran
 * on the device as one kernel. */
RG_API int32_t rg_get_option(rg_ctx *ctx, const char *name, int64_t *value);
/* The cudaStream_t the context launches on, as an opaque pointer. */
RG_API int32_t rg_get_stream(rg_ctx *ctx, void **stream);
RG_API int32_t rg_synchronize(rg_ctx *ctx);

/* y[i] = tanh(x[i]) with the device port of glibc tanh (self-test hook). */
RG_API int32_t rg_tanh(rg_ctx *ctx, const double *x, double *y, int64_t n, int32_t flags);

/* sample_scenarios / _uniform_grid (disturbance.py:85-92, 179-203):
 * out[n_sim][horizon][width], width <= 16; scenario k is stream index k0 + k. */
RG_API int32_t rg_sample_scenarios(rg_ctx *ctx, uint64_t seed, int64_t k0, int64_t n_sim,
                            int64_t horizon, int32_t width, const double *lo,
                            const double *span, double *out, int32_t flags);

/* Parity fill: the kernels.run_cells seam (kernels.py:260-300) behind
 * backend_gpu.fill (backend_gpu.py:50).  For each active row rows[a] the
 * candidate v_rows[rows[a]] is rolled out against every scenario and
 * S[rows[a]][k] (RG_CELL_*) and steps[rows[a]][k] are written; other rows are
 * untouched.  Scenarios come from `dist` ([n_sim][horizon][3], horizon >=
 * j_star + 1) or, when dist is NULL, from the counter RNG `rng`. */
RG_API int32_t rg_fill(rg_ctx *ctx, const rg_problem *prob, const double *x0, const double *v_rows,
                int32_t m_rows, const int32_t *rows, int32_t n_rows, const double *dist,
                int64_t n_sim, int64_t horizon, const rg_scenarios *rng, uint8_t *S,
                int32_t *steps, int32_t flags);

/* Fused robust grid step (robust_rg_parallel): candidates kappa_i = i/(m-1),
 * v_i = update_setpoint(v_prev, r, kappa_i), steady-state gate and dedup on
 * the device, rollouts with fused RNG (dist NULL) or staged dist, per-row
 * feasibility reduction and extraction of the best row (prefix_mode as in
 * extract_kappa_opt, governor.py:351-377).  Optional outputs:
 *   row_viol[m]       per-row violating-scenario counts (UINT32_MAX = pruned)
 *   pbits[m][ceil(n_sim/32)]  P as a bitmask, bit k%32 of word k/32
 * With RG_ASYNC nothing is read back; the result lands in device memory and
 * rg_grid_fetch copies it out later.  A synchronous call with host outputs has
 * the kernel write its result straight into pinned host memory and returns once
 * the kernel has published it (no copy, no stream synchronisation); work that
 * only resets device counters may still be in flight on the context's stream,
 * ordered before any later call.  rg_grid_fetch after such a call returns the
 * same result again. */
RG_API int32_t rg_grid_step(rg_ctx *ctx, const rg_problem *prob, const double *x0, double v_prev,
                     double r, int32_t m_grid, int32_t prefix_mode, const double *dist,
                     int64_t n_sim, int64_t horizon, const rg_scenarios *rng,
                     uint32_t *row_viol, uint32_t *pbits, rg_grid_result *out, int32_t flags);
RG_API int32_t rg_grid_fetch(rg_ctx *ctx, uint32_t *row_viol, int32_t m_grid, rg_grid_result *out);

/* Exact Alg. 2 (robust_rg_sequential, governor.py:469-517): each scenario runs
 * _bisect_kappa (governor.py:380-430) on its own disturbance; reductions give
 * min kappa, AND found and the summed counters.  Scenario source: dist, rng,
 * or both NULL for the nominal (zero-disturbance) prediction of bisection_rg.
 * Per-scenario outputs and the tested path ([n_sim][n_kappa+1], unused slots
 * untouched) are optional. */
RG_API int32_t rg_bisect(rg_ctx *ctx, const rg_problem *prob, const double *x0, double v_prev,
                  double r, int32_t n_kappa, const double *dist, int64_t n_sim, int64_t horizon,
                  const rg_scenarios *rng, double *kappa_k, int32_t *found_k, int32_t *cells_k,
                  int32_t *early_k, double *path_kappa, uint8_t *path_ok,
                  rg_bisect_result *out, int32_t flags);

/* Batched robust grid step: n_episodes independent governor instances
 * (BASELINE configs C3/C5) in one launch, each with its own state x0[e][3],
 * v_prev[e], request r[e] and scenario stream seeds[e] (scenarios k0..k0+n_sim-1
 * of that stream, uniform lo/span shared).  Per episode: the best row (-1
 * none), kappa = row/(m_grid-1) (0 when none), v = update_setpoint(v_prev, r,
 * kappa) (v_prev when none), early terminations, and optionally the per-row
 * violation counts row_viol[e][m].  All arrays are host memory; the call is
 * synchronous.  RG_ABANDON lets rows already known infeasible stop early. */
RG_API int32_t rg_grid_step_batch(rg_ctx *ctx, const rg_problem *prob, int32_t n_episodes,
                                  const double *x0, const double *v_prev, const double *r,
                                  const uint64_t *seeds, int64_t k0, int64_t n_sim,
                                  const double *lo, const double *span, int32_t m_grid,
                                  int32_t prefix_mode, int32_t *row_out, double *kappa_out,
                                  double *v_out, int64_t *early_out, uint32_t *row_viol,
                                  int32_t flags);

/* Linear-plant counterparts of rg_fill and rg_bisect (kernels.py:90-118 behind
 * governor.py:245-348, 380-517).  `prob` supplies j_star and the output bounds
 * (its setpoint-interval fields are unused); dist is [n_sim][horizon][n]; x0 has n
 * entries.  The reference's GPU backend refuses linear plants
 * (backend_gpu.py:66-71); this library runs them. */
RG_API int32_t rg_fill_linear(rg_ctx *ctx, const rg_linear_plant *plant, const rg_problem *prob,
                              const double *x0, const double *v_rows, int32_t m_rows,
                              const int32_t *rows, int32_t n_rows, const double *dist,
                              int64_t n_sim, int64_t horizon, const rg_scenarios *rng,
                              uint8_t *S, int32_t *steps, int32_t flags);
RG_API int32_t rg_bisect_linear(rg_ctx *ctx, const rg_linear_plant *plant,
                                const rg_problem *prob, const double *x0, double v_prev,
                                double r, int32_t n_kappa, const double *dist, int64_t n_sim,
                                int64_t horizon, const rg_scenarios *rng, double *kappa_k,
                                int32_t *found_k, int32_t *cells_k, int32_t *early_k,
                                rg_bisect_result *out, int32_t flags);

/* FP64 roofline probe: independent DFMA chains; returns achieved FLOP/s. */
/* Joint bisection (the north-star form of Alg. 2): every
 * scenario tests the same kappa per iteration (kappa = 1 first, then
 * n_kappa midpoints of [0, 1], governor.py:407-431) and the violations are
 * OR-reduced into one device flag, with every scenario abandoning its rollout
 * as soon as the flag is raised.  kappa and found equal robust_rg_sequential's
 * whenever every scenario's feasible set is a down-set in kappa (SURVEY.md
 * §8(a) row A9); cells/early count like Alg. 2 summed over scenarios, except
 * that abandoned rollouts are not early terminations.
 *
 * rg_bisect_joint runs the whole search on one device in ONE persistent kernel
 * (cooperative launch, every block resident): per iteration the warps roll the
 * candidate out over 32-scenario tiles with early abandonment, meet at a grid
 * barrier and read the OR-reduced flag; every block applies the same decision, so
 * the search never returns to the host between iterations.  With RG_JOINT_ITER (or
 * n_kappa >= 64) it enqueues n_kappa + 1 kernels instead, the decision taken by each
 * kernel's last block.  One host synchronisation at the end either way.  The begin/iter/flag/decide/end calls
 * expose the same search one iteration at a time for a scenario-sharded run:
 * rg_joint_iter(ctx, it, 0) rolls the local shard out, the caller all-reduces
 * (MAX) the uint32 at rg_joint_flag on the context's stream, and
 * rg_joint_decide(ctx, it) applies the decision on every rank.  kernel_ms is
 * the event span from rg_joint_begin to rg_joint_end.
 * Replaces: robust_rg_sequential governor.py:469-517 (joint form). */
RG_API int32_t rg_bisect_joint(rg_ctx *ctx, const rg_problem *prob, const double *x0,
                               double v_prev, double r, int32_t n_kappa, const double *dist,
                               int64_t n_sim, int64_t horizon, const rg_scenarios *rng,
                               rg_bisect_result *out, int32_t flags);
RG_API int32_t rg_joint_begin(rg_ctx *ctx, const rg_problem *prob, const double *x0,
                              double v_prev, double r, int32_t n_kappa, const double *dist,
                              int64_t n_sim, int64_t horizon, const rg_scenarios *rng,
                              int32_t flags);
RG_API int32_t rg_joint_iter(rg_ctx *ctx, int32_t it, int32_t fold);
RG_API int32_t rg_joint_flag(rg_ctx *ctx, void **dev_flag);
RG_API int32_t rg_joint_decide(rg_ctx *ctx, int32_t it);
RG_API int32_t rg_joint_end(rg_ctx *ctx, rg_bisect_result *out);

/* Fused exchange of the scenario-sharded grid step (one process per GPU, same node).
 * Every rank calls rg_xchg_init(ctx, rank, world, handle[64]) -- it allocates the rank's
 * exchange window in device memory and returns its CUDA IPC handle -- gathers the world's
 * handles (rank-major, 64 bytes each) by any means (torch.distributed.all_gather_object),
 * and calls rg_xchg_connect(ctx, handles), which maps every peer's window.  From then on
 * rg_grid_step(..., RG_XCHG) does the step's all-reduce inside the kernel: the finalizing
 * block stores the shard's per-row words into every rank's window over NVLink, raises its
 * epoch flag there, waits for all ranks' flags and extracts the GLOBAL best row (row,
 * row_viol are global; the other counters stay the shard's).  Every rank must run the same
 * sequence of exchanged steps; a peer missing for "xchg_timeout_ms" (rg_set_option,
 * default 10 s) fails the step with RG_E_CUDA instead of hanging.  m_grid <= 64,
 * world <= 16.  Replaces: the NCCL all-reduce of the row counts (sharded.py). */
RG_API int32_t rg_xchg_init(rg_ctx *ctx, int32_t rank, int32_t world, void *handle_out);
RG_API int32_t rg_xchg_connect(rg_ctx *ctx, const void *handles);
RG_API int32_t rg_xchg_close(rg_ctx *ctx);
/* The joint search over this rank's scenario shard with the per-round exchange fused into
 * the persistent kernel (needs a connected exchange): after each round's local barrier the
 * shard's candidate verdicts go to every rank's window over NVLink and every block waits for
 * all ranks' and ORs them, so each rank walks the same global decisions without leaving the
 * kernel.  n_sim_max: the largest shard (the same on every rank, it fixes the speculation
 * depth); it must fit in one wave.  kappa / found are global, cells / early this shard's.
 * Replaces: robust_rg_joint_sharded's per-iteration NCCL all-reduce of the flag. */
RG_API int32_t rg_bisect_joint_sharded(rg_ctx *ctx, const rg_problem *prob, const double *x0,
                                       double v_prev, double r, int32_t n_kappa,
                                       const double *dist, int64_t n_sim, int64_t horizon,
                                       const rg_scenarios *rng, int64_t n_sim_max,
                                       rg_bisect_result *out, int32_t flags);

RG_API int32_t rg_fp64_peak(rg_ctx *ctx, double *flops_per_s);

/* ---- the closed loop in native code (harness.py:138-224) ----------------------------
 * run_closed_loop's governed loop without a Python round trip per step: per step t the
 * grid step (rg_grid_step on the scenario set seed scen_seed + t, k0 = 0, ranges lo/span:
 * derive_seed(seed, "scenarios") + t), kappa = row / (M - 1), v = update_setpoint, the
 * true plant's RK4 step with numpy's tanh (rg_np_tanh), then x += d_true[t].  Per-step
 * outputs (host arrays of `steps`, each may be NULL): v_t, kappa, y_t = x1 before the
 * plant step, feasible, sims_run, early_terms, wall time of the governor step.  The loop
 * stops early as the reference does (res->abort_kind): the plant's integration overflow
 * (|x_i| > 1e6 or non-finite after the RK4 step; dynamics.py:125-130), the state leaving
 * the box after the disturbance (harness.py:222-224), or -- with infeasible_error --
 * the first step without a feasible row (InfeasibleError).  res->steps_done rows were
 * written.  x_out (3 doubles, may be NULL): the final state.
 * With m_grid <= 64, every r[t] finite and one row's scenarios within one wave of the time-split
 * form (ceil(n_sim / 32) <= 3 x the SM count: 14,208 scenarios on a B200) the whole trace runs on
 * the device as one
 * cooperative kernel (k_loop_ts: the steps on the time-split form, and between them the
 * row, kappa, v_t, the true plant with numpy's tanh and the next step's row plan, all on
 * the device; wall_us_out then holds each governor step's device time); the "no_device_loop"
 * option (or no_ts / no_row_plan) keeps one grid-step launch per closed-loop step with the
 * plant on the host.  Both give the same rows bit for bit.  rg_get_option
 * "last_loop_device" tells which ran last. */
#define RG_LOOP_OVERFLOW 1
#define RG_LOOP_LEFT_BOX 2
#define RG_LOOP_INFEASIBLE 3
typedef struct {
    int32_t steps_done;
    int32_t abort_kind;  /* 0, or RG_LOOP_* */
    int32_t abort_step;  /* -1, or the step the loop stopped at */
    int32_t abort_index; /* the state component for RG_LOOP_OVERFLOW / LEFT_BOX */
    double abort_value;
} rg_loop_result;
RG_API int32_t rg_closed_loop(rg_ctx *ctx, const rg_problem *prob, int32_t m_grid,
                              int32_t prefix_mode, int32_t infeasible_error, const double *x0,
                              double v0, int32_t steps, const double *r, const double *d_true,
                              uint64_t scen_seed, int64_t n_sim, const double *lo,
                              const double *span, double *v_out, double *kappa_out,
                              double *y_out, uint8_t *feasible_out, int64_t *sims_out,
                              int64_t *early_out, int32_t *wall_us_out, double *x_out,
                              rg_loop_result *res);
/* The nominal bisection governor's closed loop (BASELINE C1: harness.py:138-224 with
 * bisection_rg, governor.py:433-466, at harness.py:200) on the device as one kernel: per
 * step t the kappa = 1 probe and n_kappa midpoint candidates of the one nominal cell (no
 * disturbance; governor.py:380-430), v = update_setpoint, then the true plant with numpy's
 * tanh and x += d_true[t].  Per-step outputs (host arrays of `steps`, each may be NULL):
 * kappa, v_t, y_t = x1 before the step, found, cells (rollouts incl. gated-out candidates),
 * early terminations, the step's device time.  Stops at the plant's integration overflow
 * (RG_LOOP_OVERFLOW, as plant.step raises); x_out: the final state of a completed run. */
RG_API int32_t rg_closed_loop_bisection(rg_ctx *ctx, const rg_problem *prob, int32_t n_kappa,
                                        const double *x0, double v0, int32_t steps,
                                        const double *r, const double *d_true,
                                        double *kappa_out, double *v_out, double *y_out,
                                        uint8_t *feasible_out, int64_t *cells_out,
                                        int64_t *early_out, int32_t *wall_us_out, double *x_out,
                                        rg_loop_result *res);
/* numpy's float64 tanh (numpy 2.3.5's SIMD kernel, rg_nptanh.h) on the host: y[i] =
 * np.tanh(x[i]) bit for bit for finite x.  And the surrogate true plant's step with it
 * (dynamics.py: SurrogateFuelCellPlant.step without the overflow check).  No device. */
RG_API int32_t rg_np_tanh(const double *x, double *y, int64_t n);
RG_API int32_t rg_plant_step(double step_size, const double *x, double v, double *out);

#ifdef __cplusplus
}
#endif
#endif /* REFGOV_B200_H */
