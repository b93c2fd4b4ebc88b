// rg_kernels.h -- argument blocks and launchers shared by rg_kernels.cu and
// the C-ABI layer (rg_capi.cu).  Internal to the library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "rg_cell.cuh"
#include "rg_rng.cuh"

namespace rg {

// Plant + constraints, pre-digested for the device.
struct ProblemDev {
    double h, hh, c;   // step size, 0.5*h, h/6
    double ylo, yhi;   // output bounds (cset.lower/upper)
    double vlo, vhi;   // admissible setpoints of the steady-state gate
    int32_t j_star;
};

struct SampleArgs {
    uint64_t hs;       // splitmix64(seed)
    int64_t k0, n_sim, horizon;
    int32_t width;
    double lo[16], span[16];
    double* out;       // [n_sim][horizon][width]
};

struct FillArgs {
    ProblemDev p;
    double x0[3];
    const double* v_rows;  // device [m_rows]
    const int32_t* rows;   // device [n_rows]
    int32_t n_rows;
    int64_t n_sim, k0;
    ScenarioStream stream;  // RNG source
    const double* soa;      // staged source, d[(j*3+i)*ld + k]
    int64_t ld;
    uint8_t* S;             // device [m_rows][n_sim]
    int32_t* steps;         // device [m_rows][n_sim]
    int tpb;
};

struct GridOut {
    int32_t row;            // best all-feasible row (0-based), -1 none
    int32_t n_active, ss_pruned_rows, dedup_rows;
    long long sims_run, early_terms, overflows, abandoned;
    unsigned long long seq;
    unsigned long long kernel_ns;  // device span of the step (globaltimer)
    unsigned long long reduce_ns;  // the last block's row extraction and publication
    int32_t xchg_failed;           // fused exchange: a peer's words never arrived (timeout)
};

// Cross-GPU exchange window of the fused grid step (RG_XCHG).  Every rank owns one in its
// device memory; peers write into it over NVLink (CUDA IPC mappings).  Parity-double-buffered
// by the step epoch: a rank can be at most one step ahead of a peer that still reads.
constexpr int kXMaxWorld = 16;
constexpr int kXMaxRows = 64;
struct XWin {
    unsigned long long flag[2][kXMaxWorld];    // [parity][sender] = epoch of the sender's words
    int words[2][kXMaxWorld][kXMaxRows];       // [parity][sender][row] per-row verdict words
};

constexpr int kListMax = 64;  // host-planned grid steps: at most this many candidate rows

// The time-split grid step (rg_ts.cu): per block kTsTanhWarps tanh warps and one x2-chain
// and one x1/x3-chain warp for each of up to kTsUnits units (32 scenarios of a row), chunks
// of kTsChunk steps through kTsSlots shared-memory slots.  The staged scenario block carries
// kTsPadSteps steps of padding past j* for the producer's look-ahead loads.
#ifndef RG_TS_CHUNK
#define RG_TS_CHUNK 8
#endif
#ifndef RG_TS_SLOTS
#define RG_TS_SLOTS 3
#endif
constexpr int kTsTanhWarps = 12, kTsUnits = 3, kTsChunk = RG_TS_CHUNK, kTsSlots = RG_TS_SLOTS;
constexpr int kTsThreads = (kTsTanhWarps + 2 * kTsUnits) * 32;
constexpr int kTsSmemDyn =
    kTsSlots * kTsChunk * 6 * kTsUnits * 32 * 8 + kTsSlots * kTsUnits * 32 * 4;
constexpr int kTsPadSteps = 32;

struct GridArgs {
    ProblemDev p;
    double x0[3];
    double v_prev, r;
    int32_t m_grid, prefix_mode;
    int64_t n_sim, k0;
    ScenarioStream stream;
    const double* soa;
    int64_t ld;
    // accumulators (zero between launches; the last block resets them)
    unsigned* viol;                 // [m]
    unsigned long long* early;      // [m]
    unsigned long long* ovf;        // [m]
    unsigned long long* abandoned;  // [m]
    int* row_src;                   // [m]
    unsigned* ticket;
    unsigned long long* t0;  // earliest block start (globaltimer), re-armed to ~0 by finalize
    unsigned* viol_out;             // [m] per-row violation count (0xffffffff = pruned)
    GridOut* out;
    unsigned* pbits;                // optional [m][pwords] feasibility bitmask
    unsigned* pbits_host;           // zero-copy: finalize copies pbits here (pinned)
    int64_t pwords;
    int tpb;
    // out/viol_out/pbits live in pinned host memory (zero-copy): system-scope
    // fences before the ticket, and out->seq = seq_token published last
    int host_out;
    unsigned long long seq_token;
    int pdl;  // launched behind k_gen_soa with programmatic stream serialization
    // shared memory per block (static + dynamic) of the launch: more than half an
    // SM's pins one block per SM (the single-wave placement, see rg_capi.cu:
    // grid_placement); 0: no pin
    int smem_dyn;
    int no_s2;  // single-wave step without the two-step rollout (A/B and tests)
    unsigned* ebits;  // optional [m][pwords]: cells that ended before j* (the time-split step)
    // single-wave staged step with the generator fused in (gen = 1): every block writes its
    // share of the SoA block to soa_w, then a grid barrier (bar[0] count, bar[1] generation;
    // cooperative launch, every block resident) before any rollout reads it
    int gen;
    double* soa_w;
    unsigned* bar;
    // fused cross-GPU exchange (xchg = 1): the finalizing block writes this shard's per-row
    // words into every rank's window (xpeers[r], rank xrank of xworld), raises its epoch
    // flag there, waits for every rank's flag in its own window (xlocal) and extracts the
    // row from the MAX over ranks -- the all-reduce done by the step kernel over NVLink
    int xchg, xrank, xworld;
    unsigned long long xepoch, xtimeout_ns;
    XWin* xlocal;
    XWin* const* xpeers;
    // host-planned rows (listed = 1, m_grid <= kListMax): the host evaluated every row's
    // setpoint, gate and dedup (the same arithmetic, governor.py:286-317) and launches one
    // grid row per simulated row only -- blockIdx.y indexes row_list; src_tab is every row's
    // status (-2 gated out, -1 simulated, >= 0 duplicate of that row) for the extraction
    int listed, list_n;
    int row_list[kListMax];
    int src_tab[kListMax];
};

// The closed loop on the device (k_loop_ts, rg_closed_loop): one persistent cooperative
// kernel runs every governor step of the trace on the time-split form, and between steps
// every block extracts the row, applies kappa, steps the true plant (numpy's tanh
// restated, rg_nptanh.h) and plans the next step's rows (the same bits everywhere; block 0
// writes the outputs).  LoopCtl carries step 0's inputs and plan in and the end state out.
struct LoopCtl {
    double x[3];                  // the plant state before the next step
    double v_prev, r;             // the next step's previous setpoint and reference
    unsigned long long hs;        // its scenario stream key splitmix64(seed + t)
    int32_t list_n, stop;         // simulated rows; 1 once the loop is over
    int32_t row_list[kListMax];
    int32_t src_tab[kListMax];
    int32_t steps_done, abort_kind, abort_step, abort_index;  // abort_kind: RG_LOOP_*
    double abort_value;
    double x_final[3];
};
struct LoopArgs {
    GridArgs g;             // the constant part of every step (listed, fused RNG, no P);
                            // viol / early / ovf: three zeroed sets of m_grid counters
    LoopCtl* ctl;
    unsigned* bar;          // grid barrier (count, generation), zeroed
    const double* r;        // [steps] references
    const double* d_true;   // [steps][3] true-plant disturbances
    uint64_t scen_seed;     // step t's scenarios: seed scen_seed + t
    int32_t steps, infeasible_error;
    double* v_out;          // [steps] outputs, as rg_closed_loop's
    double* kappa_out;
    double* y_out;
    unsigned char* feas_out;
    long long* sims_out;
    long long* early_out;
    long long* ns_out;      // device time of each governor step (globaltimer)
    unsigned spin_cap_ns;   // the barrier's longest poll interval
};

// The nominal bisection governor's closed loop on the device (k_loop_bisect, BASELINE C1:
// bisection_rg at harness.py:200): one block; per step the kappa = 1 probe and the
// n_kappa midpoint candidates (governor.py:380-430) each roll out the one nominal cell on
// the time-split passes, then kappa, v_t and the true plant (the driver checks only the
// plant's integration overflow).  g: n_sim 1, no disturbances, one counter of each kind.
struct LoopBisArgs {
    GridArgs g;
    LoopCtl* ctl;           // x / v_prev in (step 0); steps_done, abort_*, x_final out
    const double* r;        // [steps]
    const double* d_true;   // [steps][3]
    int32_t steps, n_kappa;
    double* kappa_out;
    double* v_out;
    double* y_out;
    unsigned char* feas_out;
    long long* cells_out;
    long long* early_out;
    long long* ns_out;
};

// Batch of independent governor instances (episodes).  The host evaluates every
// episode's candidate rows (setpoint, steady-state gate, dedup -- the reference's
// governor.py:286-317, same arithmetic as the device) and hands the kernel a compacted
// list of the (episode, row) pairs that need rollouts: in a closed loop about one row
// per episode is live, so a launch over E x M x blocks would be
// ~97% empty blocks.  One launch covers pairs [p0, p0 + gridDim.x / bpr).
struct BatchArgs {
    ProblemDev p;
    int32_t n_ep, m_grid, prefix_mode;
    int64_t n_sim, k0;
    double lo[3], span[3];
    const double* x0;       // [E][3]
    const double* v_prev;   // [E]
    const double* r;        // [E]
    const uint64_t* hs;     // [E] splitmix64(seed_e)
    const int* row_src;     // [E][M]: -2 gated out, -1 simulated, >= 0 duplicate of that row
    const int* pair_e;      // [P] episode of each simulated pair
    const int* pair_i;      // [P] row of each simulated pair
    const double* pair_v;   // [P] its setpoint
    const unsigned* expect; // [E] blocks that report to episode e (its pairs x bpr)
    int64_t p0;             // first pair of this launch
    int bpr;                // blocks per pair (ceil(n_sim / tpb))
    unsigned* viol;         // [E][M] accumulators (reset by the last block of e)
    unsigned long long* early;  // [E]
    unsigned* ticket;       // [E]
    int* row_out;           // [E]
    double* kappa_out;      // [E]
    double* v_out;          // [E]
    long long* early_out;   // [E]
    unsigned* viol_out;     // [E][M] or null
    int tpb;
    // staged source (k_gen_soa_batch): episode e's block at soa + (e - e0) * ep_stride,
    // d[(j*3+i)*ld + k]; null: fused RNG
    const double* soa;
    int64_t ld, ep_stride;
    int32_t e0;
};

// Linear-plant fill and bisection (kernels.py:90-118 behind governor.py).
struct LinArgs {
    LinPlant L;
    ProblemDev p;           // j_star, y bounds (the setpoint interval fields are unused)
    double x0[4];
    int64_t n_sim, k0;
    uint64_t hs;            // RNG source: splitmix64(seed), lo/span in L-independent arrays
    double lo[4], span[4];
    const double* soa;      // staged source d[(j*n+i)*ld + k], or null for the RNG
    int64_t ld;
    // fill
    const double* v_rows;
    const int32_t* rows;
    int32_t n_rows;
    uint8_t* S;
    int32_t* steps;
    // bisection
    double v_prev, r;
    int32_t n_kappa;
    double* kappa_k;
    int32_t *found_k, *cells_k, *early_k;
    struct BisectAcc* acc;
    struct BisectOut* out;
    int tpb;
};

struct BisectAcc {
    unsigned long long kappa_bits;  // min over scenarios (as bits; kappa >= 0)
    int found;                      // AND
    unsigned long long cells, early;
    unsigned ticket;
};

struct BisectOut {
    double kappa;
    int found;
    long long cells, early;
    unsigned long long seq;
};

struct BisectArgs {
    ProblemDev p;
    double x0[3];
    double v_prev, r;
    int32_t n_kappa;
    int64_t n_sim, k0;
    ScenarioStream stream;
    const double* soa;
    int64_t ld;
    double* kappa_k;   // optional per-scenario results
    int32_t* found_k;
    int32_t* cells_k;
    int32_t* early_k;
    double* path_kappa;  // optional [n_sim][n_kappa+1]
    uint8_t* path_ok;
    BisectAcc* acc;
    BisectOut* out;
    int tpb;
    int smem_dyn;  // shared memory per block, static + dynamic (single-wave placement pin)
    // the kappa = 1 probe already rolled out (by the time-split kernel, rg_capi.cu: rg_bisect):
    // bit k of word k/32 -- the probe's verdict and whether it ended before j*
    const unsigned* probe_ok;
    const unsigned* probe_early;
    // the result's publication: out->seq = seq_token after the fields; host_out: *out is
    // pinned host memory (zero copy), written behind a system-scope fence
    unsigned long long seq_token;
    int host_out;
};

// Joint bisection: one candidate kappa for every
// scenario per iteration, violations OR-reduced into one flag.
constexpr int kJointMaxRounds = 64;  // persistent search: at most n_kappa + 1 rounds
constexpr int kJointNodes = 7;       // speculation tree of depth <= 3 (heap order)

struct JointState {
    double lo, hi, kopt;
    int found, done;
    unsigned viol;    // OR of this iteration's violations (all-reduced across ranks when sharded)
    unsigned ticket;  // last-block election for the folded decision
    unsigned long long cells, early;
    unsigned long long seq;
    // persistent speculative search (k_joint_spec): per round and tree node the
    // violation word (a scenario of this candidate left the set), the abandon word the
    // rollouts poll (this candidate violated, or an ancestor whose feasible branch holds
    // it did), the early terminations, and per round the work-item counter.  Zero
    // between launches (the last block out resets what it used); the grid barrier's
    // count returns to 0 after every barrier and gen only grows.
    unsigned sviol[kJointMaxRounds * 8];
    unsigned sdead[kJointMaxRounds * 8];
    unsigned long long searly[kJointMaxRounds * 8];
    unsigned sitem[kJointMaxRounds];
    unsigned bar_count, bar_gen, exit_ticket;
    int rounds;  // rounds the last persistent search ran (diagnostics)
    int xfail;   // fused exchange: a peer's words did not arrive (timeout)
};

struct JointArgs {
    ProblemDev p;
    double x0[3];
    double v_prev, r;
    int32_t n_kappa;
    int64_t n_sim, k0;
    ScenarioStream stream;
    const double* soa;
    int64_t ld;
    JointState* st;
    int tpb;
    int smem_dyn;  // shared memory per block, static + dynamic (single-wave placement pin)
    int fold;  // 1: the last block decides (single GPU); 0: k_joint_decide after the all-reduce
    int depth;  // persistent search: speculation depth (1..3): 2^depth - 1 candidates per round
    // persistent search: the kappa = 1 probe already rolled out by the time-split kernel (its
    // result block and violation count), applied before the first round
    const GridOut* probe_out;
    const unsigned* probe_viol;
    // scenario-sharded persistent search with the per-round exchange fused in (xchg = 1): after
    // the local grid barrier block 0 writes this shard's candidate verdicts into every rank's
    // window over NVLink (epoch xepoch0 + round), every block waits for every rank's verdicts
    // and the walk uses their OR -- no collective launch, the search stays one kernel per GPU
    int xchg, xrank, xworld;
    unsigned long long xepoch0, xtimeout_ns;
    XWin* xlocal;
    XWin* const* xpeers;
    // persistent search: the result also into pinned host memory (zero copy), published by
    // hout->seq = seq_token behind a system-scope fence; null: device state only
    struct JointOut* hout;
    unsigned long long seq_token;
};

struct JointOut {
    double kopt;
    int found, rounds, xfail;
    unsigned long long cells, early;
    unsigned long long seq;
};

cudaError_t launch_joint_roll(const JointArgs& a, int it, bool fma, int src, cudaStream_t s);
// The whole joint search in one cooperative launch (every block co-resident), with
// speculative evaluation of the next bisection levels while the GPU would otherwise sit
// idle.  For searches of at most `max_tiles()` 32-scenario tiles; `sm_count` sizes the grid.
cudaError_t launch_joint_spec(const JointArgs& a, bool fma, int src, int sm_count,
                              cudaStream_t s);
// Largest speculation depth whose candidates' tiles all fit in one wave of two warps per
// SM sub-partition; 0 when even depth 1 does not fit (use the per-iteration launches).
int joint_spec_depth(int64_t n_sim, int sm_count);
cudaError_t launch_joint_decide(const JointArgs& a, int it, cudaStream_t s);

cudaError_t launch_sample(const SampleArgs& a, cudaStream_t s);
cudaError_t launch_to_soa(const double* src, double* dst, int64_t n_sim, int64_t horizon,
                          int32_t j_star, int64_t ld, cudaStream_t s, int64_t ncols = -1);
cudaError_t launch_fill(const FillArgs& a, bool fma, bool rng, cudaStream_t s);
cudaError_t launch_gen_soa_batch(const uint64_t* hs, const double* lo, const double* span,
                                 int64_t k0, int64_t n_sim, int32_t j_star, int64_t ld,
                                 int32_t n_ep, int64_t ep_stride, double* dst, cudaStream_t s);
cudaError_t launch_grid(const GridArgs& a, bool fma, bool rng, bool poll, cudaStream_t s);
// the time-split form (rg_ts.cu), no polling: src 1 the fused counter RNG, 2 the staged
// scenarios, 0 no disturbance (the nominal prediction); ts_blocks = its grid size
int ts_blocks(int64_t units, int sms);
cudaError_t launch_grid_ts(const GridArgs& a, bool fma, int src, int sms, cudaStream_t s);
// the device closed loop: one cooperative block per SM (kTsThreads threads)
cudaError_t launch_loop_ts(const LoopArgs& L, bool fma, int sms, cudaStream_t s);
cudaError_t launch_loop_bisect(const LoopBisArgs& B, bool fma, cudaStream_t s);
// Pairs [a.p0, a.p0 + n_pairs) of the compacted list, a.bpr blocks of a.tpb threads each.
cudaError_t launch_grid_batch(const BatchArgs& a, int64_t n_pairs, bool fma, bool poll,
                              cudaStream_t s);
cudaError_t launch_bisect(const BisectArgs& a, bool fma, int src, cudaStream_t s);
cudaError_t launch_fill_lin(const LinArgs& a, cudaStream_t s);
cudaError_t launch_bisect_lin(const LinArgs& a, cudaStream_t s);
cudaError_t launch_gen_soa_w(uint64_t hs, const double* lo, const double* span, int width,
                             int64_t k0, int64_t n_sim, int32_t j_star, int64_t ld, double* dst,
                             cudaStream_t s);
cudaError_t launch_tanh(const double* x, double* y, int64_t n, bool fma, bool lockstep,
                        cudaStream_t s);
cudaError_t launch_gen_soa(const ScenarioStream& st, int64_t k0, int64_t n_sim, int32_t j_star,
                           int64_t ld, double* dst, cudaStream_t s);
cudaError_t launch_dfma_peak(double* out, int blocks, int threads, int iters, cudaStream_t s);

}  // namespace rg
