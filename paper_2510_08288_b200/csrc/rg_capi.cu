// rg_capi.cu -- extern "C" boundary of the library (include/refgov_b200.h).
//
// Owns the per-context CUDA stream, the device scratch (grown on demand and
// reused across calls, so a steady-state governor loop allocates nothing) and
// the pinned host staging for results.  Every entry point validates its
// arguments the way the reference does (governor.py:81-108, 268-282) and maps
// failures onto the RG_E_* codes.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <string>
#include <vector>

#include "../../include/refgov_b200.h"
#include "rg_kernels.h"
#include "rg_math.cuh"
#include "rg_nptanh.h"

namespace {

thread_local std::string g_err;

int32_t fail(int32_t code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int32_t fail(int32_t code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define RG_CUDA(call)                                                                      \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(RG_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                               \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t n) {
        if (n <= bytes && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, std::max<size_t>(n, 256));
        if (e == cudaSuccess) bytes = std::max<size_t>(n, 256);
        return e;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
};

struct HostBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t n) {
        if (n <= bytes && p) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMallocHost(&p, std::max<size_t>(n, 256));
        if (e == cudaSuccess) bytes = std::max<size_t>(n, 256);
        return e;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
    }
};

// Inputs where glibc's two expm1 builds give different tanh bits.
const uint64_t kProbeBits[16] = {
    0xbfc3bab49ff59a00ull, 0xbfbf607d2a367f40ull, 0xbff1e04607439275ull, 0xbfc87c559853f610ull,
    0x3fc1bd2970c05a80ull, 0xbfc4df513e0c5a90ull, 0x3fc813eee33158a0ull, 0x3fc351feaea207e0ull,
    0xbfbf0d9c6d2f7d40ull, 0xbfc324032814df90ull, 0xbffe08c8d2bc0699ull, 0x3fc00ecbb330a320ull,
    0x3ff319e0623618f8ull, 0xbff949e37cad90c4ull, 0xbfb3d362eb61dac0ull, 0x3fc779d23c26eb20ull};

bool same_bits(double a, double b) { return memcmp(&a, &b, 8) == 0; }

// Which glibc expm1 build does this process's libm tanh use?  0 when neither.
int probe_host_tanh() {
    int fma_ok = 0, gen_ok = 0;
    for (uint64_t b : kProbeBits) {
        double x;
        memcpy(&x, &b, 8);
        const double ref = ::tanh(x);
        fma_ok += same_bits(ref, rg::tanh_glibc<true>(x));
        gen_ok += same_bits(ref, rg::tanh_glibc<false>(x));
    }
    int v = 0;
    if (fma_ok == 16 && gen_ok < 16) v = rg::kTanhFma;
    if (gen_ok == 16 && fma_ok < 16) v = rg::kTanhGeneric;
    if (!v) return 0;
    // confirm on a deterministic sweep of the branches the rollout uses
    uint64_t s = 0x243F6A8885A308D3ull;
    for (int i = 0; i < 8192; ++i) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        const double x = ((double)(s >> 11) * 0x1p-53 - 0.5) * (i & 1 ? 8.0 : 50.0);
        if (!same_bits(::tanh(x), rg::tanh_variant(x, v))) return 0;
    }
    return v;
}

}  // namespace

// Tuning knobs for experiments and tests.  Read from the environment once, at
// rg_create (RG_FORCE_TPB, RG_NO_PLACEMENT, RG_NO_PDL, RG_NO_STEP2,
// RG_BATCH_CHUNK), and settable per context with rg_set_option.  None changes a
// result bit; the defaults are the measured-best configuration.
struct Tuning {
    int force_tpb = 0;        // 32 / 64 / 128: fixed block size, no single-wave placement
    int no_placement = 0;     // single-wave placement off
    int no_pdl = 0;           // grid step not launched with programmatic dependent launch
    int no_step2 = 0;         // single-wave step with the one-step rollout
    int fused_gen = 0;        // single-wave staged step generates its block itself (grid barrier)
    int64_t xchg_timeout_ms = 10000;  // fused exchange: give up on a missing peer after this
    int no_row_plan = 0;      // grid step: rows always derived on the device
    int no_ts = 0;            // grid step: never the time-split form (rg_ts.cu)
    int ts_staged = 0;        // time-split step: staged scenario block instead of the fused RNG
    int no_ts_probe = 0;      // Alg. 2: the kappa = 1 probe inside k_bisect, not time-split
    int no_device_loop = 0;   // rg_closed_loop: one launch per step instead of k_loop_ts
    int64_t batch_chunk = 0;  // batched step: at most this many staged episodes per chunk
};

struct rg_ctx {
    int device = 0;
    Tuning tune;
    int variant = rg::kTanhFma;
    int sm_count = 0;
    int smem_per_sm = 0;  // bytes of shared memory per SM
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // grid-step accumulators and outputs
    int grid_cap = 0;
    int last_m = 0;
    int last_grid_kernel = 0;  // 0 k_grid, 1 k_grid_ts (rg_get_option)
    int64_t grid_step_kernels = 0;  // kernels launched by rg_grid_step (staging + step)
    DevBuf g_viol, g_early, g_ovf, g_aband, g_src, g_ticket, g_t0, g_out, g_bar;
    // bisection accumulators and outputs
    DevBuf b_acc, b_out;
    // batched grid step: inputs, accumulators (zeroed on growth, reset by the kernel), outputs
    int batch_cap = 0;
    int64_t batch_cap_m = 0;
    DevBuf e_in, e_viol, e_early, e_ticket, e_out, e_violout;
    std::vector<int> b_src;        // host: [E][M] row status of the batched step
    std::vector<double> b_v;       // host: one episode's candidate setpoints
    std::vector<int64_t> b_first;  // host: first pair of every episode (E + 1)
    // scratch
    DevBuf dist_raw, soa, S, steps, pbits, rows, vrows, tmp_a, tmp_b, kap_k, fnd_k, cel_k,
        erl_k, path_k, path_o;
    HostBuf h_stage;
    HostBuf h_out;                  // zero-copy grid result block (pinned, UVA-mapped)
    HostBuf h_bout;                 // zero-copy bisection result (pinned, UVA-mapped)
    HostBuf h_jout;                 // zero-copy persistent joint search result
    DevBuf j_state;                 // joint bisection state (rg::JointState)
    DevBuf probe;                   // the bisection's kappa = 1 probe bits (ok, early)
    DevBuf loop_buf;                // the device closed loop's inputs, outputs and state
    int last_loop_device = 0;       // the last rg_closed_loop ran as k_loop_ts
    rg::JointArgs j_args{};         // the joint search in progress (rg_joint_begin)
    int j_src = -1;                 // its scenario source; -1 = none begun
    unsigned long long seq_ctr = 0; // grid-step publication tokens
    bool last_zero_copy = false;    // the last grid step published into h_out
    // fused cross-GPU exchange (rg_xchg_*): this rank's window, the device table of every
    // rank's window, the peer mappings opened through CUDA IPC, the step epoch
    DevBuf x_win, x_peers;
    std::vector<void*> x_opened;
    int x_rank = -1, x_world = 0;
    unsigned long long x_epoch = 0;
    bool x_ready = false;
};

static void xchg_release(rg_ctx* ctx);  // the fused exchange's windows and mappings
static int32_t episode_rows(const rg::ProblemDev& p, double v_prev, double r, int32_t M,
                            int* src, double* v);

namespace {

int32_t enter(rg_ctx* ctx) {
    if (!ctx) return fail(RG_E_ARGS, "null context");
    RG_CUDA(cudaSetDevice(ctx->device));
    return RG_OK;
}

int32_t make_problem(const rg_problem* p, rg::ProblemDev* out) {
    if (!p) return fail(RG_E_ARGS, "null problem");
    if (!(p->step_size > 0.0) || !isfinite(p->step_size))
        return fail(RG_E_ARGS, "step_size must be positive, got %g", p->step_size);
    if (p->j_star < 1) return fail(RG_E_ARGS, "j_star must be >= 1, got %d", p->j_star);
    if (isnan(p->y_lower) || isnan(p->y_upper) || !(p->y_lower < p->y_upper))
        return fail(RG_E_ARGS, "constraint requires lower < upper, got [%g, %g]", p->y_lower,
                    p->y_upper);
    out->h = p->step_size;
    out->hh = 0.5 * p->step_size;  // kernels.py:59 evaluates 0.5 * h first
    out->c = p->step_size / 6.0;   // kernels.py:54
    out->ylo = p->y_lower;
    out->yhi = p->y_upper;
    out->vlo = p->ss_v_lower;
    out->vhi = p->ss_v_upper;
    out->j_star = p->j_star;
    return RG_OK;
}

rg::ScenarioStream make_stream(const rg_scenarios* s) {
    rg::ScenarioStream st{};
    st.hs = rg::splitmix64(s->seed);
    for (int i = 0; i < 3; ++i) {
        st.lo[i] = s->lo[i];
        st.span[i] = s->span[i];
    }
    return st;  // the surrogate's three components
}

cudaMemcpyKind kind_h2d(int32_t flags) {
    return (flags & RG_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
}

// Stage a [n_sim][horizon][3] tensor as SoA d[(j*3+i)*ld + k] (rows j < j_star).  From
// host memory: one pageable cudaMemcpyAsync (the driver pipelines its own pinned staging;
// measured faster than a chunked copy through our pinned buffer fed by a host thread pool:
// 0.55 vs 0.83 ms for C2's 6.2 MB), then the transpose.
int32_t stage_dist(rg_ctx* ctx, const double* dist, int64_t n_sim, int64_t horizon,
                   int32_t j_star, int32_t flags, const double** soa, int64_t* ld) {
    const size_t raw_bytes = (size_t)n_sim * horizon * 3 * sizeof(double);
    const double* dsrc = dist;
    if (!(flags & RG_DEVICE_PTRS)) {
        RG_CUDA(ctx->dist_raw.ensure(raw_bytes));
        RG_CUDA(cudaMemcpyAsync(ctx->dist_raw.p, dist, raw_bytes, cudaMemcpyHostToDevice,
                                ctx->stream));
        dsrc = ctx->dist_raw.as<double>();
    }
    *ld = (n_sim + 31) / 32 * 32;
    RG_CUDA(ctx->soa.ensure((size_t)(j_star + rg::kTsPadSteps) * 3 * (*ld) * sizeof(double)));
    RG_CUDA(rg::launch_to_soa(dsrc, ctx->soa.as<double>(), n_sim, horizon, j_star, *ld,
                              ctx->stream));
    *soa = ctx->soa.as<double>();
    return RG_OK;
}

// Small scenario sets: generate the RNG stream once into SoA scratch (L2
// resident) so the per-cell loop loads three doubles per step instead of
// re-hashing them for every candidate row.  Large sets keep the fused RNG.
// Staging the scenario block (k_gen_soa, then SoA reads) beats generating the
// disturbances inside every rollout at every measured size -- the block is
// shared by all M candidate rows, and its reads are a small fraction of HBM
// bandwidth even when it does not fit in L2 (1M scenarios: 6.4 GB, 116 vs 142
// ms per step).  Above 16 GB of SoA the rollout generates them (fused).
constexpr int64_t kStageMaxScenarioSteps = (16ll << 30) / 24;

int32_t stage_rng(rg_ctx* ctx, const rg_scenarios* rng, int64_t n_sim, int32_t j_star,
                  const double** soa, int64_t* ld) {
    *ld = (n_sim + 31) / 32 * 32;
    // kTsPadSteps steps of padding: the time-split step's look-ahead loads (rg_ts.cu)
    RG_CUDA(ctx->soa.ensure((size_t)(j_star + rg::kTsPadSteps) * 3 * (*ld) * sizeof(double)));
    RG_CUDA(rg::launch_gen_soa(make_stream(rng), rng->k0, n_sim, j_star, *ld,
                               ctx->soa.as<double>(), ctx->stream));
    *soa = ctx->soa.as<double>();
    return RG_OK;
}

// The bisections run each scenario only until it fails, often a few steps:
// generating the whole block up front pays off only while it is L2-sized.
constexpr int64_t kStageMaxScenarioStepsBisect = 4ll << 20;  // 96 MB of SoA
// internal rg_joint_begin flag (not in the public header): an RNG stream is not staged
constexpr int32_t kJointPreferFused = 0x40000000;

bool want_stage(int64_t n_sim, int32_t j_star, int32_t flags,
                int64_t max_steps = kStageMaxScenarioSteps) {
    if (flags & RG_FUSED_RNG) return false;
    if (flags & RG_STAGE_RNG) return true;
    return n_sim * (int64_t)j_star <= max_steps;
}

// The grid step's results live in one device block -- [GridOut | viol_out[m] |
// pbits[m][pwords] when requested] -- so a synchronous call reads everything
// back with a single copy.
constexpr size_t kOutHead = 128;  // >= sizeof(GridOut), keeps viol_out aligned
static_assert(sizeof(rg::GridOut) <= kOutHead, "result block header too small");
size_t viol_bytes(int64_t m) { return ((size_t)m * sizeof(unsigned) + 15) / 16 * 16; }

int32_t grow_grid(rg_ctx* ctx, int m) {
    if (m <= ctx->grid_cap) return RG_OK;
    const int cap = std::max(m, 64);
    RG_CUDA(ctx->g_viol.ensure(cap * sizeof(unsigned)));
    RG_CUDA(ctx->g_early.ensure(cap * sizeof(unsigned long long)));
    RG_CUDA(ctx->g_ovf.ensure(cap * sizeof(unsigned long long)));
    RG_CUDA(ctx->g_aband.ensure(cap * sizeof(unsigned long long)));
    RG_CUDA(ctx->g_src.ensure(cap * sizeof(int)));
    RG_CUDA(ctx->g_ticket.ensure(sizeof(unsigned)));
    RG_CUDA(ctx->g_t0.ensure(sizeof(unsigned long long)));
    RG_CUDA(ctx->g_bar.ensure(2 * sizeof(unsigned)));
    RG_CUDA(ctx->g_out.ensure(kOutHead + viol_bytes(cap)));
    RG_CUDA(cudaMemsetAsync(ctx->g_viol.p, 0, ctx->g_viol.bytes, ctx->stream));
    RG_CUDA(cudaMemsetAsync(ctx->g_early.p, 0, ctx->g_early.bytes, ctx->stream));
    RG_CUDA(cudaMemsetAsync(ctx->g_ovf.p, 0, ctx->g_ovf.bytes, ctx->stream));
    RG_CUDA(cudaMemsetAsync(ctx->g_aband.p, 0, ctx->g_aband.bytes, ctx->stream));
    RG_CUDA(cudaMemsetAsync(ctx->g_ticket.p, 0, ctx->g_ticket.bytes, ctx->stream));
    RG_CUDA(cudaMemsetAsync(ctx->g_t0.p, 0xff, ctx->g_t0.bytes, ctx->stream));
    RG_CUDA(cudaMemsetAsync(ctx->g_bar.p, 0, ctx->g_bar.bytes, ctx->stream));
    RG_CUDA(cudaMemsetAsync(ctx->g_out.p, 0, ctx->g_out.bytes, ctx->stream));
    ctx->grid_cap = cap;
    return RG_OK;
}

// One lane per (row, scenario) cell everywhere.  Round 1 measured two alternatives
// on the B200 and removed them: 2 or 4 lanes per cell sharing its four tanh (more
// total FP64 work: 0.322 / 0.417 ms at C2 against 0.255 then), and phase-decoupled
// or warp-specialised grid kernels (barrier and handoff overhead: 0.451 / 0.292 ms
// at C2).  DESIGN.md §4 keeps the table.

Tuning env_tuning() {
    Tuning t;
    if (const char* e = getenv("RG_FORCE_TPB")) t.force_tpb = atoi(e);
    if (getenv("RG_NO_PLACEMENT")) t.no_placement = 1;
    if (getenv("RG_NO_PDL")) t.no_pdl = 1;
    if (getenv("RG_NO_STEP2")) t.no_step2 = 1;
    if (getenv("RG_FUSED_GEN")) t.fused_gen = 1;
    if (const char* e = getenv("RG_XCHG_TIMEOUT_MS")) t.xchg_timeout_ms = atoll(e);
    if (getenv("RG_NO_ROW_PLAN")) t.no_row_plan = 1;
    if (getenv("RG_NO_TS")) t.no_ts = 1;
    if (getenv("RG_TS_STAGED")) t.ts_staged = 1;
    if (getenv("RG_NO_TS_PROBE")) t.no_ts_probe = 1;
    if (getenv("RG_NO_DEVICE_LOOP")) t.no_device_loop = 1;
    if (const char* e = getenv("RG_BATCH_CHUNK")) t.batch_chunk = atoll(e);
    if (!(t.force_tpb == 32 || t.force_tpb == 64 || t.force_tpb == 128)) t.force_tpb = 0;
    return t;
}

int tpb_for(const rg_ctx* ctx, int64_t n_sim, int64_t rows) {
    if (ctx->tune.force_tpb) return ctx->tune.force_tpb;
    // Small problems: single-warp blocks spread the warps over more SMs; above
    // one wave, 64-thread blocks (measured equal or better than 128 at 10k-1M).
    const int64_t warps = (n_sim + 31) / 32 * std::max<int64_t>(rows, 1);
    if (warps <= (int64_t)ctx->sm_count * 8) return 32;
    return 64;
}

// Single-wave placement of the grid step (and of the bisection kernels).  The step's time is set by the SM
// sub-partition (SMSP) holding the most warps: each SMSP has its own FP64 unit and
// issue slot, and one to three resident rollout warps share them.  With single-warp
// blocks the block scheduler decides how a wave's warps land on SMSPs, and at
// C2 (1024 warps over 592 SMSPs) about 40% of the steps put three warps on some
// SMSP: 226 us instead of 165 us (scripts/timing_dist.py).  When one wave holds
// the step, this picks blocks of 4L warps (L per SMSP, the smallest L that fits)
// and requests more than half an SM's shared memory, so the scheduler can place
// only one block per SM: no SMSP ever holds more than L warps.
void grid_placement(const rg_ctx* ctx, int64_t n_sim, int32_t rows, int* tpb, int* smem_dyn) {
    *smem_dyn = 0;
    if (ctx->tune.force_tpb || ctx->tune.no_placement) return;
    for (int L = 1; L <= 2; ++L) {
        const int t = 128 * L;
        const int64_t blocks = (n_sim + t - 1) / t * (int64_t)rows;
        if (blocks <= ctx->sm_count) {
            *tpb = t;
            *smem_dyn = ctx->smem_per_sm / 2 + 1024;
            return;
        }
    }
}

}  // namespace

extern "C" {

int32_t rg_abi_version(void) { return RG_ABI_VERSION; }

const char* rg_last_error(void) { return g_err.c_str(); }

int32_t rg_device_count(int32_t* n) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (n) *n = 0;
        return fail(RG_E_NODEVICE, "no CUDA device: %s", cudaGetErrorString(e));
    }
    if (n) *n = c;
    return RG_OK;
}

int32_t rg_create(int32_t device, int32_t tanh_variant, rg_ctx** out) {
    if (!out) return fail(RG_E_ARGS, "null output pointer");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(RG_E_NODEVICE, "no CUDA device available (%s)",
                    e == cudaSuccess ? "count 0" : cudaGetErrorString(e));
    }
    if (device < 0 || device >= n) return fail(RG_E_ARGS, "device %d out of range [0, %d)", device, n);
    cudaDeviceProp prop;
    RG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (!(prop.major == 10 && prop.minor == 0))
        return fail(RG_E_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a",
                    device, prop.major, prop.minor);
    int variant = tanh_variant;
    if (variant == RG_TANH_AUTO) {
        variant = probe_host_tanh();
        if (!variant)
            return fail(RG_E_UNSUPPORTED,
                        "host libm tanh matches neither glibc expm1 build; device results "
                        "would not be bit-identical to the reference");
    } else if (variant != RG_TANH_FMA && variant != RG_TANH_GENERIC) {
        return fail(RG_E_ARGS, "unknown tanh variant %d", variant);
    }
    rg_ctx* ctx = new rg_ctx();
    ctx->device = device;
    ctx->variant = variant;
    ctx->sm_count = prop.multiProcessorCount;
    ctx->smem_per_sm = (int)prop.sharedMemPerMultiprocessor;
    ctx->tune = env_tuning();
    int32_t rc = enter(ctx);
    if (rc) { delete ctx; return rc; }
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess) {
        delete ctx;
        return fail(RG_E_CUDA, "stream/event creation failed: %s",
                    cudaGetErrorString(cudaGetLastError()));
    }
    rc = grow_grid(ctx, 64);
    if (!rc) {
        if (ctx->b_acc.ensure(sizeof(rg::BisectAcc)) != cudaSuccess ||
            ctx->b_out.ensure(sizeof(rg::BisectOut)) != cudaSuccess ||
            ctx->h_stage.ensure(1 << 16) != cudaSuccess)
            rc = fail(RG_E_CUDA, "allocation failed");
    }
    if (!rc) {
        rg::BisectAcc acc{0x3ff0000000000000ull, 1, 0ull, 0ull, 0u};
        if (cudaMemcpy(ctx->b_acc.p, &acc, sizeof acc, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemset(ctx->b_out.p, 0, sizeof(rg::BisectOut)) != cudaSuccess ||
            cudaStreamSynchronize(ctx->stream) != cudaSuccess)
            rc = fail(RG_E_CUDA, "context init failed");
    }
    if (rc) {
        rg_destroy(ctx);
        return rc;
    }
    *out = ctx;
    return RG_OK;
}

int32_t rg_destroy(rg_ctx* ctx) {
    if (!ctx) return RG_OK;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    xchg_release(ctx);
    DevBuf* bufs[] = {&ctx->g_viol, &ctx->g_early, &ctx->g_ovf, &ctx->g_aband, &ctx->g_src,
                      &ctx->g_ticket, &ctx->g_t0, &ctx->g_out, &ctx->g_bar, &ctx->j_state, &ctx->b_acc, &ctx->b_out,
                      &ctx->dist_raw, &ctx->soa, &ctx->S, &ctx->steps, &ctx->pbits, &ctx->rows,
                      &ctx->vrows, &ctx->tmp_a, &ctx->tmp_b, &ctx->kap_k, &ctx->fnd_k,
                      &ctx->cel_k, &ctx->erl_k, &ctx->path_k, &ctx->path_o, &ctx->e_in,
                      &ctx->e_viol, &ctx->e_early, &ctx->e_ticket, &ctx->e_out,
                      &ctx->e_violout, &ctx->probe, &ctx->loop_buf};
    for (DevBuf* b : bufs) b->release();
    ctx->h_stage.release();
    ctx->h_out.release();
    ctx->h_bout.release();
    ctx->h_jout.release();
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return RG_OK;
}

int32_t rg_set_option(rg_ctx* ctx, const char* name, int64_t value) {
    if (!ctx || !name) return fail(RG_E_ARGS, "null argument");
    Tuning& t = ctx->tune;
    if (!strcmp(name, "force_tpb")) {
        if (value != 0 && value != 32 && value != 64 && value != 128)
            return fail(RG_E_ARGS, "force_tpb must be 0, 32, 64 or 128, got %lld", (long long)value);
        t.force_tpb = (int)value;
    } else if (!strcmp(name, "no_placement")) {
        t.no_placement = value != 0;
    } else if (!strcmp(name, "no_pdl")) {
        t.no_pdl = value != 0;
    } else if (!strcmp(name, "no_step2")) {
        t.no_step2 = value != 0;
    } else if (!strcmp(name, "fused_gen")) {
        t.fused_gen = value != 0;
    } else if (!strcmp(name, "no_row_plan")) {
        t.no_row_plan = value != 0;
    } else if (!strcmp(name, "no_ts")) {
        t.no_ts = value != 0;
    } else if (!strcmp(name, "ts_staged")) {
        t.ts_staged = value != 0;
    } else if (!strcmp(name, "no_ts_probe")) {
        t.no_ts_probe = value != 0;
    } else if (!strcmp(name, "no_device_loop")) {
        t.no_device_loop = value != 0;
    } else if (!strcmp(name, "xchg_timeout_ms")) {
        if (value < 1) return fail(RG_E_ARGS, "xchg_timeout_ms must be >= 1");
        t.xchg_timeout_ms = value;
    } else if (!strcmp(name, "batch_chunk")) {
        if (value < 0) return fail(RG_E_ARGS, "batch_chunk must be >= 0");
        t.batch_chunk = value;
    } else {
        return fail(RG_E_ARGS, "unknown option '%s'", name);
    }
    return RG_OK;
}

int32_t rg_get_option(rg_ctx* ctx, const char* name, int64_t* value) {
    if (!ctx || !name || !value) return fail(RG_E_ARGS, "null argument");
    const Tuning& t = ctx->tune;
    if (!strcmp(name, "force_tpb")) *value = t.force_tpb;
    else if (!strcmp(name, "no_placement")) *value = t.no_placement;
    else if (!strcmp(name, "no_pdl")) *value = t.no_pdl;
    else if (!strcmp(name, "no_step2")) *value = t.no_step2;
    else if (!strcmp(name, "fused_gen")) *value = t.fused_gen;
    else if (!strcmp(name, "no_row_plan")) *value = t.no_row_plan;
    else if (!strcmp(name, "no_ts")) *value = t.no_ts;
    else if (!strcmp(name, "ts_staged")) *value = t.ts_staged;
    else if (!strcmp(name, "no_ts_probe")) *value = t.no_ts_probe;
    else if (!strcmp(name, "no_device_loop")) *value = t.no_device_loop;
    else if (!strcmp(name, "xchg_timeout_ms")) *value = t.xchg_timeout_ms;
    else if (!strcmp(name, "batch_chunk")) *value = t.batch_chunk;
    else if (!strcmp(name, "last_grid_kernel")) *value = ctx->last_grid_kernel;
    else if (!strcmp(name, "grid_step_kernels")) *value = ctx->grid_step_kernels;
    else if (!strcmp(name, "last_loop_device")) *value = ctx->last_loop_device;
    else return fail(RG_E_ARGS, "unknown option '%s'", name);
    return RG_OK;
}

int32_t rg_get_tanh_variant(rg_ctx* ctx, int32_t* variant) {
    if (!ctx || !variant) return fail(RG_E_ARGS, "null argument");
    *variant = ctx->variant;
    return RG_OK;
}

int32_t rg_get_stream(rg_ctx* ctx, void** stream) {
    if (!ctx || !stream) return fail(RG_E_ARGS, "null argument");
    *stream = (void*)ctx->stream;
    return RG_OK;
}

int32_t rg_synchronize(rg_ctx* ctx) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    return RG_OK;
}

int32_t rg_tanh(rg_ctx* ctx, const double* x, double* y, int64_t n, int32_t flags) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    if (n < 0 || (n > 0 && (!x || !y))) return fail(RG_E_ARGS, "bad tanh arguments");
    if (n == 0) return RG_OK;
    const size_t bytes = (size_t)n * sizeof(double);
    const double* dx = x;
    double* dy = y;
    if (!(flags & RG_DEVICE_PTRS)) {
        RG_CUDA(ctx->tmp_a.ensure(bytes));
        RG_CUDA(ctx->tmp_b.ensure(bytes));
        RG_CUDA(cudaMemcpyAsync(ctx->tmp_a.p, x, bytes, cudaMemcpyHostToDevice, ctx->stream));
        dx = ctx->tmp_a.as<double>();
        dy = ctx->tmp_b.as<double>();
    }
    RG_CUDA(rg::launch_tanh(dx, dy, n, ctx->variant == rg::kTanhFma,
                            (flags & RG_TANH_LOCKSTEP) != 0, ctx->stream));
    if (!(flags & RG_DEVICE_PTRS))
        RG_CUDA(cudaMemcpyAsync(y, dy, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    return RG_OK;
}

int32_t rg_sample_scenarios(rg_ctx* ctx, uint64_t seed, int64_t k0, int64_t n_sim,
                            int64_t horizon, int32_t width, const double* lo,
                            const double* span, double* out, int32_t flags) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    if (n_sim < 1 || horizon < 1)
        return fail(RG_E_ARGS, "n_sim and horizon must be >= 1, got %lld, %lld",
                    (long long)n_sim, (long long)horizon);
    if (width < 1 || width > 16) return fail(RG_E_ARGS, "width must be in [1, 16], got %d", width);
    if (k0 < 0) return fail(RG_E_ARGS, "k0 must be >= 0");
    if (!lo || !span || !out) return fail(RG_E_ARGS, "null buffer");
    rg::SampleArgs a{};
    a.hs = rg::splitmix64(seed);
    a.k0 = k0;
    a.n_sim = n_sim;
    a.horizon = horizon;
    a.width = width;
    for (int i = 0; i < width; ++i) {
        a.lo[i] = lo[i];
        a.span[i] = span[i];
    }
    const size_t bytes = (size_t)n_sim * horizon * width * sizeof(double);
    if (flags & RG_DEVICE_PTRS) {
        a.out = out;
    } else {
        RG_CUDA(ctx->dist_raw.ensure(bytes));
        a.out = ctx->dist_raw.as<double>();
    }
    RG_CUDA(rg::launch_sample(a, ctx->stream));
    if (!(flags & RG_DEVICE_PTRS))
        RG_CUDA(cudaMemcpyAsync(out, a.out, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    if (!(flags & RG_ASYNC)) RG_CUDA(cudaStreamSynchronize(ctx->stream));
    return RG_OK;
}

int32_t rg_fill(rg_ctx* ctx, const rg_problem* prob, const double* x0, const double* v_rows,
                int32_t m_rows, const int32_t* rows, int32_t n_rows, const double* dist,
                int64_t n_sim, int64_t horizon, const rg_scenarios* rng, uint8_t* S,
                int32_t* steps, int32_t flags) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    rg::FillArgs a{};
    if ((rc = make_problem(prob, &a.p))) return rc;
    if (!x0 || !v_rows || (n_rows > 0 && !rows) || !S || !steps)
        return fail(RG_E_ARGS, "null buffer");
    if (m_rows < 1 || n_rows < 0 || n_rows > m_rows)
        return fail(RG_E_ARGS, "bad row counts m=%d n=%d", m_rows, n_rows);
    if (n_sim < 1) return fail(RG_E_ARGS, "n_sim must be >= 1");
    if (!dist && !rng) return fail(RG_E_ARGS, "need a scenario tensor or an RNG stream");
    if (dist && horizon < (int64_t)prob->j_star + 1)
        return fail(RG_E_ARGS, "scenario horizon %lld too short: need >= j_star+1 = %d",
                    (long long)horizon, prob->j_star + 1);
    if (!(flags & RG_DEVICE_PTRS)) {
        for (int32_t q = 0; q < n_rows; ++q)
            if (rows[q] < 0 || rows[q] >= m_rows)
                return fail(RG_E_ARGS, "row index %d out of range", rows[q]);
    }
    for (int i = 0; i < 3; ++i) a.x0[i] = x0[i];  // x0 is a kernel parameter: host memory
    if (n_rows == 0) return RG_OK;
    RG_CUDA(ctx->vrows.ensure(m_rows * sizeof(double)));
    RG_CUDA(ctx->rows.ensure(n_rows * sizeof(int32_t)));
    RG_CUDA(cudaMemcpyAsync(ctx->vrows.p, v_rows, m_rows * sizeof(double), kind_h2d(flags),
                            ctx->stream));
    RG_CUDA(cudaMemcpyAsync(ctx->rows.p, rows, n_rows * sizeof(int32_t), kind_h2d(flags),
                            ctx->stream));
    a.v_rows = ctx->vrows.as<double>();
    a.rows = ctx->rows.as<int32_t>();
    a.n_rows = n_rows;
    a.n_sim = n_sim;
    a.tpb = tpb_for(ctx, n_sim, n_rows);
    bool use_rng = dist == nullptr;
    if (use_rng && want_stage(n_sim, prob->j_star, flags)) {
        if ((rc = stage_rng(ctx, rng, n_sim, prob->j_star, &a.soa, &a.ld))) return rc;
        use_rng = false;
    } else if (use_rng) {
        a.stream = make_stream(rng);
        a.k0 = rng->k0;
    } else {
        if ((rc = stage_dist(ctx, dist, n_sim, horizon, prob->j_star, flags, &a.soa, &a.ld)))
            return rc;
    }
    const size_t cells = (size_t)m_rows * n_sim;
    if (flags & RG_DEVICE_PTRS) {
        a.S = S;
        a.steps = steps;
    } else {
        RG_CUDA(ctx->S.ensure(cells));
        RG_CUDA(ctx->steps.ensure(cells * sizeof(int32_t)));
        a.S = ctx->S.as<uint8_t>();
        a.steps = ctx->steps.as<int32_t>();
    }
    RG_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    RG_CUDA(rg::launch_fill(a, ctx->variant == rg::kTanhFma, use_rng, ctx->stream));
    RG_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    if (!(flags & RG_DEVICE_PTRS)) {
        // copy back only the active rows (the caller's other rows stay untouched), one copy
        // per run of consecutive rows: the reference's active rows are ascending and mostly
        // contiguous, so a 32-row fill is one or two copies instead of 64
        for (int32_t q = 0; q < n_rows;) {
            int32_t e = q + 1;
            while (e < n_rows && rows[e] == rows[e - 1] + 1) ++e;
            const int64_t off = (int64_t)rows[q] * n_sim, cnt = (int64_t)(e - q) * n_sim;
            RG_CUDA(cudaMemcpyAsync(S + off, a.S + off, cnt, cudaMemcpyDeviceToHost, ctx->stream));
            RG_CUDA(cudaMemcpyAsync(steps + off, a.steps + off, cnt * sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, ctx->stream));
            q = e;
        }
    }
    if (!(flags & RG_ASYNC)) RG_CUDA(cudaStreamSynchronize(ctx->stream));
    return RG_OK;
}

// Spin until the grid step publishes `token` in the pinned result block.  The
// stream is polled now and then so a failed launch surfaces as an error
// instead of a hang.
static cudaError_t wait_seq(rg_ctx* ctx, volatile unsigned long long* seq,
                            unsigned long long token) {
    for (unsigned long n = 1;; ++n) {
        if (*seq == token) break;
        if ((n & 1023u) == 0) {
            const cudaError_t q = cudaStreamQuery(ctx->stream);
            if (q == cudaSuccess) {  // stream drained: the token must be there now
                if (*seq == token) break;
                return cudaErrorUnknown;
            }
            if (q != cudaErrorNotReady) return q;
        }
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return cudaSuccess;
}

static cudaError_t wait_token(rg_ctx* ctx, volatile rg::GridOut* ho, unsigned long long token) {
    return wait_seq(ctx, &ho->seq, token);
}

static int32_t unpack_grid(rg_ctx* ctx, const char* h, uint32_t* row_viol, int32_t m_grid,
                           rg_grid_result* out, uint32_t* pbits_host, size_t pbits_bytes,
                           bool timed);

static int32_t read_grid(rg_ctx* ctx, uint32_t* row_viol, int32_t m_grid, rg_grid_result* out,
                         uint32_t* pbits_host, size_t pbits_bytes, bool timed) {
    const size_t bytes = kOutHead + viol_bytes(m_grid) + pbits_bytes;
    RG_CUDA(ctx->h_stage.ensure(bytes));
    char* h = ctx->h_stage.as<char>();
    RG_CUDA(cudaMemcpyAsync(h, ctx->g_out.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    return unpack_grid(ctx, h, row_viol, m_grid, out, pbits_host, pbits_bytes, timed);
}

static int32_t unpack_grid(rg_ctx* ctx, const char* h, uint32_t* row_viol, int32_t m_grid,
                           rg_grid_result* out, uint32_t* pbits_host, size_t pbits_bytes,
                           bool timed) {
    const rg::GridOut* ho = reinterpret_cast<const rg::GridOut*>(h);
    if (ho->xchg_failed)
        return fail(RG_E_CUDA, "fused exchange: a peer's words did not arrive within %lld ms "
                    "(every rank must run the same exchanged steps)",
                    (long long)ctx->tune.xchg_timeout_ms);
    if (row_viol) memcpy(row_viol, h + kOutHead, m_grid * sizeof(unsigned));
    if (pbits_host) memcpy(pbits_host, h + kOutHead + viol_bytes(m_grid), pbits_bytes);
    if (out) {
        out->row = ho->row;
        out->n_active = ho->n_active;
        out->ss_pruned_rows = ho->ss_pruned_rows;
        out->dedup_rows = ho->dedup_rows;
        out->sims_run = ho->sims_run;
        out->early_terms = ho->early_terms;
        out->overflows = ho->overflows;
        out->abandoned = ho->abandoned;
        out->kernel_ms = (float)((double)ho->kernel_ns * 1e-6);  // device globaltimer span
        out->reduce_us = (float)((double)ho->reduce_ns * 1e-3);
        if (timed) {
            float ms = 0.f;
            cudaEventSynchronize(ctx->ev1);
            if (cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1) == cudaSuccess) out->kernel_ms = ms;
            cudaGetLastError();
        }
    }
    return RG_OK;
}

int32_t rg_grid_step(rg_ctx* ctx, const rg_problem* prob, const double* x0, double v_prev,
                     double r, int32_t m_grid, int32_t prefix_mode, const double* dist,
                     int64_t n_sim, int64_t horizon, const rg_scenarios* rng,
                     uint32_t* row_viol, uint32_t* pbits, rg_grid_result* out, int32_t flags) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    rg::GridArgs a{};
    if ((rc = make_problem(prob, &a.p))) return rc;
    if (!x0) return fail(RG_E_ARGS, "null x0");
    if (m_grid < 2) return fail(RG_E_ARGS, "m_grid must be >= 2, got %d", m_grid);
    if (m_grid > 65535) return fail(RG_E_ARGS, "m_grid must be <= 65535, got %d", m_grid);
    if (n_sim < 1) return fail(RG_E_ARGS, "n_sim must be >= 1");
    if (!dist && !rng) return fail(RG_E_ARGS, "need a scenario tensor or an RNG stream");
    if (dist && horizon < (int64_t)prob->j_star + 1)
        return fail(RG_E_ARGS, "scenario horizon %lld too short: need >= j_star+1 = %d",
                    (long long)horizon, prob->j_star + 1);
    if (!isfinite(v_prev) || !isfinite(r)) return fail(RG_E_ARGS, "v_prev and r must be finite");
    for (int i = 0; i < 3; ++i) a.x0[i] = x0[i];  // x0 is a kernel parameter: host memory
    if (!(isfinite(a.x0[0]) && isfinite(a.x0[1]) && isfinite(a.x0[2])))
        return fail(RG_E_ARGS, "state entries must be finite");
    if ((rc = grow_grid(ctx, m_grid))) return rc;
    a.v_prev = v_prev;
    a.r = r;
    a.m_grid = m_grid;
    a.prefix_mode = prefix_mode ? 1 : 0;
    a.n_sim = n_sim;
    bool use_rng = dist == nullptr;
    // Host-planned rows: the host evaluates the candidates' setpoints, gate and dedup itself
    // and launches grid rows for the simulated ones only -- a closed-loop step has about one
    // (SURVEY.md §0 fact 6), and the placement below then sees the real work (with P the
    // kernels zero the other rows' words: zero_unlisted_pbits).  When every row is
    // simulated the kernel derives the rows on the device (row_source).
    int grid_rows = m_grid;
    if (m_grid <= rg::kListMax && !ctx->tune.no_row_plan) {
        int src[rg::kListMax];
        double vv[rg::kListMax];
        const int32_t n_act = episode_rows(a.p, v_prev, r, m_grid, src, vv);
        if (n_act > 0 && n_act < m_grid) {
            a.listed = 1;
            a.list_n = 0;
            for (int32_t q = 0; q < m_grid; ++q) {
                a.src_tab[q] = src[q];
                if (src[q] == -1) a.row_list[a.list_n++] = q;
            }
            grid_rows = a.list_n;
        }
    }
    a.tpb = tpb_for(ctx, n_sim, grid_rows);
    grid_placement(ctx, n_sim, grid_rows, &a.tpb, &a.smem_dyn);
    a.no_s2 = ctx->tune.no_step2;
    // Option: the single-wave staged step (the two-step rollout, rg_grid.cu: launch_grid)
    // generates its own scenario block -- every block is resident, so a grid barrier can
    // stand in for the separate generator kernel.  Measured slower at C2 (0.1618 vs 0.1583
    // ms: k_gen_soa behind programmatic dependent launch overlaps the step's prologue,
    // scripts/ab_fused_gen.py), so it is off by default.
    const bool single_wave_s2 = a.smem_dyn > 0 && a.tpb <= rg::kRing4Stride && !a.no_s2;
    // A host-planned step whose simulated cells fit one wave of the time-split form
    // (rg_ts.cu: the x2 chain, the tanh and the x1/x3 chain on separate warps) runs that
    // instead of one warp per 32 rollouts: a closed-loop step (about one row) is bound by
    // the rollout's per-step latency, not by FP64 throughput.  With an RNG stream its
    // producer warps generate the disturbances themselves (no generator kernel, no block).
    const int64_t ts_units = (int64_t)grid_rows * ((n_sim + 31) / 32);
    const bool ts_ok = a.listed && !((flags & RG_ABANDON) && !pbits) && !ctx->tune.no_ts &&
                       ts_units <= (int64_t)rg::kTsUnits * ctx->sm_count;
    if (ts_ok && use_rng && !ctx->tune.ts_staged && !(flags & RG_STAGE_RNG)) {
        a.stream = make_stream(rng);
        a.k0 = rng->k0;
    } else if (use_rng && want_stage(n_sim, prob->j_star, flags) && single_wave_s2 &&
        ctx->tune.fused_gen) {
        a.ld = (n_sim + 31) / 32 * 32;
        RG_CUDA(ctx->soa.ensure((size_t)prob->j_star * 3 * a.ld * sizeof(double)));
        a.soa = a.soa_w = ctx->soa.as<double>();
        a.stream = make_stream(rng);
        a.k0 = rng->k0;
        a.gen = 1;
        a.bar = ctx->g_bar.as<unsigned>();
        use_rng = false;
    } else if (use_rng && want_stage(n_sim, prob->j_star, flags)) {
        if ((rc = stage_rng(ctx, rng, n_sim, prob->j_star, &a.soa, &a.ld))) return rc;
        use_rng = false;
        a.pdl = ctx->tune.no_pdl ? 0 : 1;  // k_gen_soa is the kernel right before
    } else if (use_rng) {
        a.stream = make_stream(rng);
        a.k0 = rng->k0;
    } else if ((rc = stage_dist(ctx, dist, n_sim, horizon, prob->j_star, flags, &a.soa, &a.ld))) {
        return rc;
    }
    a.viol = ctx->g_viol.as<unsigned>();
    a.early = ctx->g_early.as<unsigned long long>();
    a.ovf = ctx->g_ovf.as<unsigned long long>();
    a.abandoned = ctx->g_aband.as<unsigned long long>();
    a.row_src = ctx->g_src.as<int>();
    a.ticket = ctx->g_ticket.as<unsigned>();
    a.t0 = ctx->g_t0.as<unsigned long long>();
    a.pwords = (n_sim + 31) / 32;
    if (flags & RG_XCHG) {
        if (!ctx->x_ready) return fail(RG_E_ARGS, "RG_XCHG without a connected exchange (rg_xchg_connect)");
        if (m_grid > rg::kXMaxRows)
            return fail(RG_E_ARGS, "RG_XCHG supports m_grid <= %d, got %d", rg::kXMaxRows, m_grid);
        a.xchg = 1;
        a.xrank = ctx->x_rank;
        a.xworld = ctx->x_world;
        a.xepoch = ++ctx->x_epoch;
        a.xtimeout_ns = (unsigned long long)ctx->tune.xchg_timeout_ms * 1000000ull;
        a.xlocal = ctx->x_win.as<rg::XWin>();
        a.xpeers = ctx->x_peers.as<rg::XWin* const>();
    }
    const size_t pbytes = pbits ? (size_t)m_grid * a.pwords * sizeof(unsigned) : 0;
    const bool pbits_in_block = pbits && !(flags & RG_DEVICE_PTRS);
    // synchronous host-pointer calls: results land in pinned host memory and the
    // call returns when the kernel publishes its token (no copy, no stream sync)
    const bool zero_copy = !(flags & (RG_ASYNC | RG_DEVICE_PTRS));
    const size_t blk_bytes = kOutHead + viol_bytes(m_grid) + (pbits_in_block ? pbytes : 0);
    RG_CUDA(ctx->g_out.ensure(blk_bytes));
    if (zero_copy) RG_CUDA(ctx->h_out.ensure(blk_bytes));
    char* blk = zero_copy ? ctx->h_out.as<char>() : ctx->g_out.as<char>();
    char* dblk = ctx->g_out.as<char>();  // device copy: the blocks' P bits land here
    a.host_out = zero_copy ? 1 : 0;
    a.seq_token = ++ctx->seq_ctr;
    if (zero_copy) reinterpret_cast<volatile rg::GridOut*>(blk)->seq = 0ull;
    a.out = reinterpret_cast<rg::GridOut*>(blk);
    a.viol_out = reinterpret_cast<unsigned*>(blk + kOutHead);
    const bool abandon = (flags & RG_ABANDON) && !pbits;
    if (pbits) {
        // blocks write P to device memory; in zero-copy mode the finalizing block
        // copies it into the pinned result block
        a.pbits = pbits_in_block ? reinterpret_cast<unsigned*>(dblk + kOutHead + viol_bytes(m_grid))
                                 : pbits;
        if (zero_copy && pbits_in_block)
            a.pbits_host = reinterpret_cast<unsigned*>(blk + kOutHead + viol_bytes(m_grid));
    }
    const bool use_ts = ts_ok && !a.gen;
    // the staging kernel (k_gen_soa / k_to_soa) when the step reads a block it did not write
    ctx->grid_step_kernels += 1 + ((a.soa != nullptr && !a.gen) ? 1 : 0);
    const bool timed = !(flags & RG_NO_TIMING);
    if (timed) RG_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    if (use_ts)
        RG_CUDA(rg::launch_grid_ts(a, ctx->variant == rg::kTanhFma, use_rng ? 1 : 2,
                                   ctx->sm_count, ctx->stream));
    else
        RG_CUDA(rg::launch_grid(a, ctx->variant == rg::kTanhFma, use_rng, abandon, ctx->stream));
    if (timed) RG_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    ctx->last_m = m_grid;
    ctx->last_grid_kernel = use_ts ? 1 : 0;
    // rg_grid_fetch reads the pinned block only after a synchronous zero-copy step
    ctx->last_zero_copy = zero_copy;
    if (flags & RG_ASYNC) {
        if (row_viol && (flags & RG_DEVICE_PTRS))
            RG_CUDA(cudaMemcpyAsync(row_viol, a.viol_out, m_grid * sizeof(unsigned),
                                    cudaMemcpyDeviceToDevice, ctx->stream));
        return RG_OK;
    }
    if (zero_copy) {
        RG_CUDA(wait_token(ctx, reinterpret_cast<volatile rg::GridOut*>(blk), a.seq_token));
        return unpack_grid(ctx, blk, row_viol, m_grid, out, pbits_in_block ? pbits : nullptr,
                           pbits_in_block ? pbytes : 0, timed);
    }
    if (row_viol && (flags & RG_DEVICE_PTRS)) {
        RG_CUDA(cudaMemcpyAsync(row_viol, a.viol_out, m_grid * sizeof(unsigned),
                                cudaMemcpyDeviceToDevice, ctx->stream));
        row_viol = nullptr;
    }
    return read_grid(ctx, row_viol, m_grid, out, pbits_in_block ? pbits : nullptr,
                     pbits_in_block ? pbytes : 0, timed);
}

// ---------------------------------------------------------------------------
// fused cross-GPU exchange of the grid step (RG_XCHG)
// ---------------------------------------------------------------------------

}  // extern "C"

static void xchg_release(rg_ctx* ctx) {
    for (void* p : ctx->x_opened)
        if (p) cudaIpcCloseMemHandle(p);
    ctx->x_opened.clear();
    ctx->x_win.release();
    ctx->x_peers.release();
    ctx->x_ready = false;
    ctx->x_rank = -1;
    ctx->x_world = 0;
    ctx->x_epoch = 0;
}

extern "C" {

int32_t rg_xchg_init(rg_ctx* ctx, int32_t rank, int32_t world, void* handle_out) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    if (world < 1 || world > rg::kXMaxWorld || rank < 0 || rank >= world)
        return fail(RG_E_ARGS, "rank %d / world %d outside [0, world), world <= %d", rank, world,
                    rg::kXMaxWorld);
    if (!handle_out) return fail(RG_E_ARGS, "null handle_out");
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    xchg_release(ctx);
    RG_CUDA(ctx->x_win.ensure(sizeof(rg::XWin)));
    RG_CUDA(cudaMemset(ctx->x_win.p, 0, sizeof(rg::XWin)));
    RG_CUDA(ctx->x_peers.ensure(rg::kXMaxWorld * sizeof(void*)));
    cudaIpcMemHandle_t h;
    RG_CUDA(cudaIpcGetMemHandle(&h, ctx->x_win.p));
    memcpy(handle_out, &h, sizeof h);
    ctx->x_rank = rank;
    ctx->x_world = world;
    return RG_OK;
}

int32_t rg_xchg_connect(rg_ctx* ctx, const void* handles) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    if (ctx->x_rank < 0) return fail(RG_E_ARGS, "rg_xchg_connect before rg_xchg_init");
    if (!handles) return fail(RG_E_ARGS, "null handles");
    cudaIpcMemHandle_t mine;
    RG_CUDA(cudaIpcGetMemHandle(&mine, ctx->x_win.p));
    void* table[rg::kXMaxWorld] = {};
    for (int r = 0; r < ctx->x_world; ++r) {
        const char* hr = static_cast<const char*>(handles) + (size_t)r * sizeof(cudaIpcMemHandle_t);
        if (r == ctx->x_rank || !memcmp(hr, &mine, sizeof mine)) {
            table[r] = ctx->x_win.p;  // our own window (or a test naming it twice)
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, hr, sizeof h);
        void* p = nullptr;
        const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            cudaGetLastError();
            xchg_release(ctx);
            return fail(RG_E_CUDA, "cudaIpcOpenMemHandle of rank %d's window failed: %s", r,
                        cudaGetErrorString(e));
        }
        ctx->x_opened.push_back(p);
        table[r] = p;
    }
    RG_CUDA(cudaMemcpy(ctx->x_peers.p, table, sizeof table, cudaMemcpyHostToDevice));
    ctx->x_epoch = 0;
    ctx->x_ready = true;
    return RG_OK;
}

int32_t rg_xchg_close(rg_ctx* ctx) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    xchg_release(ctx);
    return RG_OK;
}

int32_t rg_grid_fetch(rg_ctx* ctx, uint32_t* row_viol, int32_t m_grid, rg_grid_result* out) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    if (m_grid < 1 || m_grid > ctx->grid_cap || m_grid != ctx->last_m)
        return fail(RG_E_ARGS, "bad m_grid %d (last step used %d)", m_grid, ctx->last_m);
    if (ctx->last_zero_copy)  // the last step published into the pinned block
        return unpack_grid(ctx, ctx->h_out.as<char>(), row_viol, m_grid, out, nullptr, 0, false);
    return read_grid(ctx, row_viol, m_grid, out, nullptr, 0, false);
}

}  // extern "C"

// The kappa = 1 probe of the bisections (v = r for every scenario) on the time-split kernel:
// a one-row step (row 1 of two, row 0 gated out) writing each scenario's verdict (ok) and
// early bit, and the result block (the row's violation count, early terminations).  All
// outputs are device pointers valid until the next grid step or probe.
static int32_t ts_probe(rg_ctx* ctx, const rg::ProblemDev& p, const double* x0, double v_prev,
                        double r, int64_t n_sim, int src, const double* soa, int64_t ld,
                        const rg::ScenarioStream& stream, int64_t k0, const unsigned** ok,
                        const unsigned** early, const rg::GridOut** out,
                        const unsigned** viol) {
    int32_t rc;
    if ((rc = grow_grid(ctx, 2))) return rc;
    rg::GridArgs g{};
    g.p = p;
    for (int i = 0; i < 3; ++i) g.x0[i] = x0[i];
    g.v_prev = v_prev;
    g.r = r;  // row 1 of 2: kappa = 1, v = r
    g.m_grid = 2;
    g.n_sim = n_sim;
    g.listed = 1;
    g.list_n = 1;
    g.row_list[0] = 1;
    g.src_tab[0] = -2;
    g.src_tab[1] = -1;
    if (src == 2) {
        g.soa = soa;
        g.ld = ld;
    } else {
        g.stream = stream;
        g.k0 = k0;
    }
    g.viol = ctx->g_viol.as<unsigned>();
    g.early = ctx->g_early.as<unsigned long long>();
    g.ovf = ctx->g_ovf.as<unsigned long long>();
    g.abandoned = ctx->g_aband.as<unsigned long long>();
    g.row_src = ctx->g_src.as<int>();
    g.ticket = ctx->g_ticket.as<unsigned>();
    const int64_t pwords = (n_sim + 31) / 32;
    g.pwords = pwords;
    const size_t words = (size_t)2 * pwords;
    RG_CUDA(ctx->probe.ensure(2 * words * sizeof(unsigned)));
    g.pbits = ctx->probe.as<unsigned>();
    g.ebits = g.pbits + words;
    RG_CUDA(ctx->g_out.ensure(kOutHead + viol_bytes(2)));
    g.out = ctx->g_out.as<rg::GridOut>();
    g.viol_out = reinterpret_cast<unsigned*>(ctx->g_out.as<char>() + kOutHead);
    g.seq_token = ++ctx->seq_ctr;
    RG_CUDA(rg::launch_grid_ts(g, ctx->variant == rg::kTanhFma, src, ctx->sm_count,
                               ctx->stream));
    *ok = g.pbits + pwords;  // row 1
    *early = g.ebits + pwords;
    *out = g.out;
    *viol = g.viol_out + 1;
    return RG_OK;
}

extern "C" {

int32_t rg_bisect(rg_ctx* ctx, const rg_problem* prob, const double* x0, double v_prev,
                  double r, int32_t n_kappa, const double* dist, int64_t n_sim, int64_t horizon,
                  const rg_scenarios* rng, double* kappa_k, int32_t* found_k, int32_t* cells_k,
                  int32_t* early_k, double* path_kappa, uint8_t* path_ok,
                  rg_bisect_result* out, int32_t flags) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    rg::BisectArgs a{};
    if ((rc = make_problem(prob, &a.p))) return rc;
    if (!x0) return fail(RG_E_ARGS, "null x0");
    if (n_kappa < 1) return fail(RG_E_ARGS, "n_kappa must be >= 1, got %d", n_kappa);
    if (n_sim < 1) return fail(RG_E_ARGS, "n_sim must be >= 1");
    if (dist && horizon < (int64_t)prob->j_star + 1)
        return fail(RG_E_ARGS, "scenario horizon %lld too short: need >= j_star+1 = %d",
                    (long long)horizon, prob->j_star + 1);
    if (!isfinite(v_prev) || !isfinite(r)) return fail(RG_E_ARGS, "v_prev and r must be finite");
    if ((kappa_k || found_k || cells_k || early_k) && !(kappa_k && found_k && cells_k && early_k))
        return fail(RG_E_ARGS, "per-scenario outputs come as a set of four");
    if ((path_kappa != nullptr) != (path_ok != nullptr))
        return fail(RG_E_ARGS, "path outputs come as a pair");
    for (int i = 0; i < 3; ++i) a.x0[i] = x0[i];  // x0 is a kernel parameter: host memory
    a.v_prev = v_prev;
    a.r = r;
    a.n_kappa = n_kappa;
    a.n_sim = n_sim;
    // Every scenario's search starts with the kappa = 1 probe (v = r), one candidate over all
    // scenarios -- the time-split kernel's regime (rg_ts.cu).  When v = r passes the gate
    // and the scenarios fit one wave of it, the probe runs there first and k_bisect takes
    // each scenario's verdict and early bit from its output instead of rolling it out; a
    // closed loop's steady-state search is the probe alone.  With an RNG stream neither
    // stages a block: the probe's producers and k_bisect's rollouts hash their own.
    const int64_t probe_units = (n_sim + 31) / 32;
    const bool probe = !ctx->tune.no_ts && !ctx->tune.no_ts_probe &&
                       a.p.vlo <= r && r <= a.p.vhi &&
                       probe_units <= (int64_t)rg::kTsUnits * ctx->sm_count;
    int src = 0;
    if (dist) {
        src = 2;
        if ((rc = stage_dist(ctx, dist, n_sim, horizon, prob->j_star, flags, &a.soa, &a.ld)))
            return rc;
    } else if (rng && probe && !(flags & RG_STAGE_RNG)) {
        src = 1;
        a.stream = make_stream(rng);
        a.k0 = rng->k0;
    } else if (rng && want_stage(n_sim, prob->j_star, flags, kStageMaxScenarioStepsBisect)) {
        src = 2;
        if ((rc = stage_rng(ctx, rng, n_sim, prob->j_star, &a.soa, &a.ld))) return rc;
    } else if (rng) {
        src = 1;
        a.stream = make_stream(rng);
        a.k0 = rng->k0;
    }
    const bool dev = (flags & RG_DEVICE_PTRS) != 0;
    if (kappa_k) {
        if (dev) {
            a.kappa_k = kappa_k;
            a.found_k = found_k;
            a.cells_k = cells_k;
            a.early_k = early_k;
        } else {
            RG_CUDA(ctx->kap_k.ensure(n_sim * sizeof(double)));
            RG_CUDA(ctx->fnd_k.ensure(n_sim * sizeof(int32_t)));
            RG_CUDA(ctx->cel_k.ensure(n_sim * sizeof(int32_t)));
            RG_CUDA(ctx->erl_k.ensure(n_sim * sizeof(int32_t)));
            a.kappa_k = ctx->kap_k.as<double>();
            a.found_k = ctx->fnd_k.as<int32_t>();
            a.cells_k = ctx->cel_k.as<int32_t>();
            a.early_k = ctx->erl_k.as<int32_t>();
        }
    }
    const size_t npath = (size_t)n_sim * (n_kappa + 1);
    if (path_kappa) {
        if (dev) {
            a.path_kappa = path_kappa;
            a.path_ok = path_ok;
        } else {
            RG_CUDA(ctx->path_k.ensure(npath * sizeof(double)));
            RG_CUDA(ctx->path_o.ensure(npath));
            a.path_kappa = ctx->path_k.as<double>();
            a.path_ok = ctx->path_o.as<uint8_t>();
            // unused slots read back as NaN / 255
            RG_CUDA(cudaMemsetAsync(a.path_kappa, 0xff, npath * sizeof(double), ctx->stream));
            RG_CUDA(cudaMemsetAsync(a.path_ok, 0xff, npath, ctx->stream));
        }
    }
    a.acc = ctx->b_acc.as<rg::BisectAcc>();
    // a synchronous call without per-scenario outputs: the last block writes the result into
    // pinned host memory and the call spins on its token (no copy, no stream sync)
    const bool zero_copy = !(flags & RG_ASYNC) && !kappa_k && !path_kappa;
    if (zero_copy) {
        RG_CUDA(ctx->h_bout.ensure(sizeof(rg::BisectOut)));
        a.out = ctx->h_bout.as<rg::BisectOut>();
        a.host_out = 1;
    } else {
        a.out = ctx->b_out.as<rg::BisectOut>();
    }
    a.seq_token = ++ctx->seq_ctr;
    a.tpb = tpb_for(ctx, n_sim, 1);
    grid_placement(ctx, n_sim, 1, &a.tpb, &a.smem_dyn);
    const bool timed = !(flags & RG_NO_TIMING);
    if (timed) RG_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    if (probe) {  // the kappa = 1 probe on the time-split kernel
        const rg::GridOut* pout;
        const unsigned* pviol;
        if ((rc = ts_probe(ctx, a.p, a.x0, v_prev, r, n_sim, src, a.soa, a.ld, a.stream, a.k0,
                           &a.probe_ok, &a.probe_early, &pout, &pviol)))
            return rc;
    }
    RG_CUDA(rg::launch_bisect(a, ctx->variant == rg::kTanhFma, src, ctx->stream));
    if (timed) RG_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    if (!dev) {
        if (kappa_k) {
            RG_CUDA(cudaMemcpyAsync(kappa_k, a.kappa_k, n_sim * sizeof(double),
                                    cudaMemcpyDeviceToHost, ctx->stream));
            RG_CUDA(cudaMemcpyAsync(found_k, a.found_k, n_sim * sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, ctx->stream));
            RG_CUDA(cudaMemcpyAsync(cells_k, a.cells_k, n_sim * sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, ctx->stream));
            RG_CUDA(cudaMemcpyAsync(early_k, a.early_k, n_sim * sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, ctx->stream));
        }
        if (path_kappa) {
            RG_CUDA(cudaMemcpyAsync(path_kappa, a.path_kappa, npath * sizeof(double),
                                    cudaMemcpyDeviceToHost, ctx->stream));
            RG_CUDA(cudaMemcpyAsync(path_ok, a.path_ok, npath, cudaMemcpyDeviceToHost,
                                    ctx->stream));
        }
    }
    if (flags & RG_ASYNC) return RG_OK;
    rg::BisectOut* ho;
    if (zero_copy) {
        ho = ctx->h_bout.as<rg::BisectOut>();
        RG_CUDA(wait_seq(ctx, &ho->seq, a.seq_token));
        if (timed) RG_CUDA(cudaEventSynchronize(ctx->ev1));
    } else {
        RG_CUDA(ctx->h_stage.ensure(sizeof(rg::BisectOut)));
        ho = ctx->h_stage.as<rg::BisectOut>();
        RG_CUDA(cudaMemcpyAsync(ho, ctx->b_out.p, sizeof(rg::BisectOut), cudaMemcpyDeviceToHost,
                                ctx->stream));
        RG_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    if (out) {
        out->kappa = ho->kappa;
        out->found = ho->found;
        out->cells = ho->cells;
        out->early = ho->early;
        out->kernel_ms = 0.f;
        if (timed) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1) == cudaSuccess) out->kernel_ms = ms;
            cudaGetLastError();
        }
    }
    return RG_OK;
}

// ---------------------------------------------------------------------------
// joint bisection
// ---------------------------------------------------------------------------

int32_t rg_joint_begin(rg_ctx* ctx, const rg_problem* prob, const double* x0, double v_prev,
                       double r, int32_t n_kappa, const double* dist, int64_t n_sim,
                       int64_t horizon, const rg_scenarios* rng, int32_t flags) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    rg::JointArgs a{};
    if ((rc = make_problem(prob, &a.p))) return rc;
    if (!x0) return fail(RG_E_ARGS, "null x0");
    if (n_kappa < 1) return fail(RG_E_ARGS, "n_kappa must be >= 1, got %d", n_kappa);
    if (n_sim < 1) return fail(RG_E_ARGS, "n_sim must be >= 1");
    if (dist && horizon < (int64_t)prob->j_star + 1)
        return fail(RG_E_ARGS, "scenario horizon %lld too short: need >= j_star+1 = %d",
                    (long long)horizon, prob->j_star + 1);
    if (!isfinite(v_prev) || !isfinite(r)) return fail(RG_E_ARGS, "v_prev and r must be finite");
    for (int i = 0; i < 3; ++i) a.x0[i] = x0[i];
    a.v_prev = v_prev;
    a.r = r;
    a.n_kappa = n_kappa;
    a.n_sim = n_sim;
    int src = 0;
    if (dist) {
        src = 2;
        if ((rc = stage_dist(ctx, dist, n_sim, horizon, prob->j_star, flags, &a.soa, &a.ld)))
            return rc;
    } else if (rng && !(flags & kJointPreferFused) &&
               want_stage(n_sim, prob->j_star, flags, kStageMaxScenarioStepsBisect)) {
        src = 2;
        if ((rc = stage_rng(ctx, rng, n_sim, prob->j_star, &a.soa, &a.ld))) return rc;
    } else if (rng) {
        src = 1;
        a.stream = make_stream(rng);
        a.k0 = rng->k0;
    }
    RG_CUDA(ctx->j_state.ensure(sizeof(rg::JointState)));
    a.st = ctx->j_state.as<rg::JointState>();
    rg::JointState init{};
    init.lo = 0.0;
    init.hi = 1.0;
    init.kopt = 0.0;
    RG_CUDA(ctx->h_stage.ensure(sizeof(rg::JointState)));
    memcpy(ctx->h_stage.p, &init, sizeof(init));
    RG_CUDA(cudaMemcpyAsync(a.st, ctx->h_stage.p, sizeof(init), cudaMemcpyHostToDevice,
                            ctx->stream));
    a.tpb = tpb_for(ctx, n_sim, 1);
    grid_placement(ctx, n_sim, 1, &a.tpb, &a.smem_dyn);
    a.fold = 1;
    ctx->j_args = a;
    ctx->j_src = src;
    RG_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    return RG_OK;
}

int32_t rg_joint_iter(rg_ctx* ctx, int32_t it, int32_t fold) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    if (ctx->j_src < 0) return fail(RG_E_ARGS, "no joint search begun (rg_joint_begin)");
    if (it < -1 || it >= ctx->j_args.n_kappa)
        return fail(RG_E_ARGS, "iteration %d outside [-1, %d)", it, ctx->j_args.n_kappa);
    rg::JointArgs a = ctx->j_args;
    a.fold = fold ? 1 : 0;
    RG_CUDA(rg::launch_joint_roll(a, it, ctx->variant == rg::kTanhFma, ctx->j_src, ctx->stream));
    return RG_OK;
}

int32_t rg_joint_decide(rg_ctx* ctx, int32_t it) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    if (ctx->j_src < 0) return fail(RG_E_ARGS, "no joint search begun (rg_joint_begin)");
    RG_CUDA(rg::launch_joint_decide(ctx->j_args, it, ctx->stream));
    return RG_OK;
}

int32_t rg_joint_flag(rg_ctx* ctx, void** dev_flag) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    if (ctx->j_src < 0) return fail(RG_E_ARGS, "no joint search begun (rg_joint_begin)");
    if (!dev_flag) return fail(RG_E_ARGS, "null dev_flag");
    *dev_flag = &ctx->j_args.st->viol;
    return RG_OK;
}

int32_t rg_joint_end(rg_ctx* ctx, rg_bisect_result* out) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    if (ctx->j_src < 0) return fail(RG_E_ARGS, "no joint search begun (rg_joint_begin)");
    RG_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    RG_CUDA(ctx->h_stage.ensure(sizeof(rg::JointState)));
    rg::JointState* hs = ctx->h_stage.as<rg::JointState>();
    RG_CUDA(cudaMemcpyAsync(hs, ctx->j_args.st, sizeof(rg::JointState), cudaMemcpyDeviceToHost,
                            ctx->stream));
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    const bool xchg = ctx->j_args.xchg != 0;
    if (xchg) ctx->x_epoch += (unsigned long long)hs->rounds;  // one epoch per exchanged round
    ctx->j_src = -1;
    if (xchg && hs->xfail)
        return fail(RG_E_CUDA, "fused exchange: a peer's verdicts did not arrive within %lld ms "
                    "(every rank must run the same searches)", (long long)ctx->tune.xchg_timeout_ms);
    if (out) {
        out->kappa = hs->kopt;
        out->found = hs->found;
        out->cells = (int64_t)hs->cells;
        out->early = (int64_t)hs->early;
        float ms = 0.f;
        out->kernel_ms = cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1) == cudaSuccess ? ms : 0.f;
        cudaGetLastError();
    }
    return RG_OK;
}

int32_t rg_bisect_joint_sharded(rg_ctx* ctx, const rg_problem* prob, const double* x0,
                                double v_prev, double r, int32_t n_kappa, const double* dist,
                                int64_t n_sim, int64_t horizon, const rg_scenarios* rng,
                                int64_t n_sim_max, rg_bisect_result* out, int32_t flags) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    if (!ctx->x_ready) return fail(RG_E_ARGS, "no connected exchange (rg_xchg_connect)");
    if (n_sim_max < n_sim || n_sim_max < 1) return fail(RG_E_ARGS, "n_sim_max must be >= n_sim");
    const int depth = rg::joint_spec_depth(n_sim_max, ctx->sm_count);
    if (depth == 0 || n_kappa + 1 > rg::kJointMaxRounds)
        return fail(RG_E_ARGS, "the fused sharded search needs shards within one wave and "
                    "n_kappa < %d (use rg_joint_iter with an all-reduce)", rg::kJointMaxRounds);
    if ((rc = rg_joint_begin(ctx, prob, x0, v_prev, r, n_kappa, dist, n_sim, horizon, rng, flags)))
        return rc;
    rg::JointArgs& a = ctx->j_args;
    a.depth = depth;  // from the largest shard: every rank builds the same trees
    a.xchg = 1;
    a.xrank = ctx->x_rank;
    a.xworld = ctx->x_world;
    a.xepoch0 = ctx->x_epoch + 1;
    a.xtimeout_ns = (unsigned long long)ctx->tune.xchg_timeout_ms * 1000000ull;
    a.xlocal = ctx->x_win.as<rg::XWin>();
    a.xpeers = ctx->x_peers.as<rg::XWin* const>();
    const cudaError_t e = rg::launch_joint_spec(a, ctx->variant == rg::kTanhFma, ctx->j_src,
                                                ctx->sm_count, ctx->stream);
    if (e != cudaSuccess) {
        ctx->j_src = -1;
        return fail(RG_E_CUDA, "joint search launch failed: %s", cudaGetErrorString(e));
    }
    return rg_joint_end(ctx, out);
}

int32_t rg_bisect_joint(rg_ctx* ctx, const rg_problem* prob, const double* x0, double v_prev,
                        double r, int32_t n_kappa, const double* dist, int64_t n_sim,
                        int64_t horizon, const rg_scenarios* rng, rg_bisect_result* out,
                        int32_t flags) {
    if (!ctx || !prob) return fail(RG_E_ARGS, "null argument");
    const int depth = rg::joint_spec_depth(n_sim, ctx->sm_count);
    // a persistent search whose kappa = 1 probe goes to the time-split kernel with the RNG
    // generates its scenarios in the kernels (a steady-state search then stages nothing)
    const bool probe_rng = rng && !dist && !(flags & (RG_JOINT_ITER | RG_STAGE_RNG)) &&
                           depth > 0 && !ctx->tune.no_ts && !ctx->tune.no_ts_probe &&
                           prob->ss_v_lower <= r && r <= prob->ss_v_upper &&
                           (n_sim + 31) / 32 <= (int64_t)rg::kTsUnits * ctx->sm_count;
    int32_t rc = rg_joint_begin(ctx, prob, x0, v_prev, r, n_kappa, dist, n_sim, horizon, rng,
                                flags | (probe_rng ? kJointPreferFused : 0));
    if (rc) return rc;
    if (!(flags & RG_JOINT_ITER) && depth > 0 && n_kappa + 1 <= rg::kJointMaxRounds) {
        // the whole search in one cooperative launch, speculating `depth` levels per round;
        // its kappa = 1 probe first on the time-split kernel when v = r passes the gate (a
        // steady-state search is the probe alone; the kernel starts after its verdict)
        rg::JointArgs& ja = ctx->j_args;
        ja.probe_out = nullptr;
        ja.probe_viol = nullptr;
        if (ctx->j_src >= 0 && !ctx->tune.no_ts && !ctx->tune.no_ts_probe &&
            ja.p.vlo <= r && r <= ja.p.vhi &&
            (n_sim + 31) / 32 <= (int64_t)rg::kTsUnits * ctx->sm_count) {
            const unsigned *pok, *pearly;
            if ((rc = ts_probe(ctx, ja.p, ja.x0, v_prev, r, n_sim, ctx->j_src, ja.soa, ja.ld,
                               ja.stream, ja.k0, &pok, &pearly, &ja.probe_out,
                               &ja.probe_viol))) {
                ctx->j_src = -1;
                return rc;
            }
        }
        ctx->j_args.depth = depth;
        // the result lands in pinned host memory; the call spins on its token
        RG_CUDA(ctx->h_jout.ensure(sizeof(rg::JointOut)));
        rg::JointOut* jo = ctx->h_jout.as<rg::JointOut>();
        ctx->j_args.hout = jo;
        ctx->j_args.seq_token = ++ctx->seq_ctr;
        const cudaError_t e = rg::launch_joint_spec(ctx->j_args, ctx->variant == rg::kTanhFma,
                                                    ctx->j_src, ctx->sm_count, ctx->stream);
        ctx->j_args.hout = nullptr;
        if (e != cudaSuccess) {
            ctx->j_src = -1;
            return fail(RG_E_CUDA, "joint search launch failed: %s", cudaGetErrorString(e));
        }
        RG_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
        const cudaError_t w = wait_seq(ctx, &jo->seq, ctx->j_args.seq_token);
        if (w != cudaSuccess) {
            ctx->j_src = -1;
            RG_CUDA(w);
        }
        const bool xchg = ctx->j_args.xchg != 0;
        if (xchg) ctx->x_epoch += (unsigned long long)jo->rounds;  // one epoch per round
        ctx->j_src = -1;
        if (xchg && jo->xfail)
            return fail(RG_E_CUDA, "fused exchange: a peer's verdicts did not arrive within %lld "
                        "ms (every rank must run the same searches)",
                        (long long)ctx->tune.xchg_timeout_ms);
        if (out) {
            out->kappa = jo->kopt;
            out->found = jo->found;
            out->cells = (int64_t)jo->cells;
            out->early = (int64_t)jo->early;
            float ms = 0.f;
            out->kernel_ms = cudaEventSynchronize(ctx->ev1) == cudaSuccess &&
                                     cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1) == cudaSuccess
                                 ? ms
                                 : 0.f;
            cudaGetLastError();
        }
        return RG_OK;
    }
    for (int32_t it = -1; it < n_kappa; ++it)
        if ((rc = rg_joint_iter(ctx, it, 1))) return rc;
    return rg_joint_end(ctx, out);
}

}  // extern "C"

// One episode's candidate rows on the host, exactly as the device (and governor.py:286-317)
// evaluates them: v_i = update_setpoint(v_prev, r, i/(M-1)), the steady-state gate as the
// verified setpoint interval, duplicates mapped to the first gated row with the same v.
// Returns the number of simulated rows; src[i] = -2 gated out, -1 simulated, q duplicate.
// The setpoints are monotone in i except where rounding at kappa = 1 (exact r) breaks it,
// so a new value is compared with the previous distinct one and, only once the sequence
// stops being strictly monotone, with every earlier one.
static int32_t episode_rows(const rg::ProblemDev& p, double v_prev, double r, int32_t M,
                            int* src, double* v) {
    int32_t n = 0, last = -1;
    int dir = 0;          // +1 / -1 once two distinct gated values were seen
    bool monotone = true;
    for (int32_t i = 0; i < M; ++i) {
        const double vi = rg::update_setpoint(v_prev, r, rg::dvd((double)i, (double)(M - 1)));
        v[i] = vi;
        if (!(p.vlo <= vi && vi <= p.vhi)) {  // NaN -> gated out, like ConstraintSet.contains
            src[i] = -2;
            continue;
        }
        int dup = -1;
        if (last >= 0) {
            if (v[last] == vi) {
                dup = src[last] >= 0 ? src[last] : last;
            } else {
                const int d = vi > v[last] ? 1 : -1;
                if (dir == 0) dir = d;
                if (d != dir) monotone = false;
                if (!monotone) {
                    for (int32_t q = 0; q < i; ++q)
                        if (src[q] == -1 && v[q] == vi) {
                            dup = q;
                            break;
                        }
                }
            }
        }
        src[i] = dup;
        if (dup < 0) ++n;
        last = i;
    }
    return n;
}

extern "C" {

int32_t rg_grid_step_batch(rg_ctx* ctx, const rg_problem* prob, int32_t n_episodes,
                           const double* x0, const double* v_prev, const double* r,
                           const uint64_t* seeds, int64_t k0, int64_t n_sim, const double* lo,
                           const double* span, int32_t m_grid, int32_t prefix_mode,
                           int32_t* row_out, double* kappa_out, double* v_out,
                           int64_t* early_out, uint32_t* row_viol, int32_t flags) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    rg::BatchArgs a{};
    if ((rc = make_problem(prob, &a.p))) return rc;
    if (n_episodes < 1 || n_episodes > (1 << 24))
        return fail(RG_E_ARGS, "n_episodes must be in [1, 2^24], got %d", n_episodes);
    if (m_grid < 2 || m_grid > 65535) return fail(RG_E_ARGS, "m_grid must be in [2, 65535]");
    if (n_sim < 1 || k0 < 0) return fail(RG_E_ARGS, "bad scenario range");
    if (!x0 || !v_prev || !r || !seeds || !lo || !span || !row_out || !kappa_out || !v_out)
        return fail(RG_E_ARGS, "null buffer");
    const int64_t E = n_episodes, M = m_grid;
    for (int64_t e = 0; e < E; ++e) {
        if (!(isfinite(x0[3 * e]) && isfinite(x0[3 * e + 1]) && isfinite(x0[3 * e + 2]) &&
              isfinite(v_prev[e]) && isfinite(r[e])))
            return fail(RG_E_ARGS, "episode %lld: state, v_prev and r must be finite",
                        (long long)e);
    }
    const int tpb = ctx->tune.force_tpb ? ctx->tune.force_tpb : 64;  // always multi-wave
    const int bpr = (int)((n_sim + tpb - 1) / tpb);
    // host: every episode's rows, and the compacted pairs (episode-major)
    ctx->b_src.resize((size_t)E * M);
    ctx->b_v.resize((size_t)M);
    ctx->b_first.resize((size_t)E + 1);
    int64_t P = 0;
    for (int64_t e = 0; e < E; ++e) {
        ctx->b_first[e] = P;
        P += episode_rows(a.p, v_prev[e], r[e], m_grid, ctx->b_src.data() + e * M,
                          ctx->b_v.data());
    }
    ctx->b_first[E] = P;
    // one pinned staging block, one host-to-device copy:
    // [x0 3E | v_prev E | r E | hs E | pair_v P] doubles, [row_src E*M | pair_e P | pair_i P |
    // expect E] 32-bit words
    const size_t nd = (size_t)E * 6 + (size_t)P;
    const size_t nw = (size_t)E * M + 2 * (size_t)P + (size_t)E;
    const size_t in_bytes = nd * sizeof(double) + nw * sizeof(int32_t);
    const size_t out_bytes = (size_t)E * (3 * sizeof(double) + sizeof(int));
    const size_t viol_bytes_all = row_viol ? (size_t)E * M * sizeof(unsigned) : 0;
    RG_CUDA(ctx->h_stage.ensure(in_bytes + out_bytes + viol_bytes_all + 64));
    double* hd = ctx->h_stage.as<double>();
    memcpy(hd, x0, (size_t)E * 3 * sizeof(double));
    memcpy(hd + 3 * E, v_prev, (size_t)E * sizeof(double));
    memcpy(hd + 4 * E, r, (size_t)E * sizeof(double));
    uint64_t* hhs = reinterpret_cast<uint64_t*>(hd + 5 * E);
    for (int64_t e = 0; e < E; ++e) hhs[e] = rg::splitmix64(seeds[e]);
    double* hpv = hd + 6 * E;
    int32_t* hw = reinterpret_cast<int32_t*>(hd + nd);
    memcpy(hw, ctx->b_src.data(), (size_t)E * M * sizeof(int32_t));
    int32_t* hpe = hw + E * M;
    int32_t* hpi = hpe + P;
    uint32_t* hexp = reinterpret_cast<uint32_t*>(hpi + P);
    for (int64_t e = 0; e < E; ++e) {
        const int* src = ctx->b_src.data() + e * M;
        int64_t q = ctx->b_first[e];
        for (int32_t i = 0; i < M; ++i) {
            if (src[i] != -1) continue;
            hpe[q] = (int32_t)e;
            hpi[q] = i;
            hpv[q] = rg::update_setpoint(v_prev[e], r[e], rg::dvd((double)i, (double)(M - 1)));
            ++q;
        }
        hexp[e] = (uint32_t)((ctx->b_first[e + 1] - ctx->b_first[e]) * bpr);
    }
    if (E > ctx->batch_cap || E * M > ctx->batch_cap_m) {
        const int64_t cap = std::max<int64_t>(E, 64), capm = std::max<int64_t>(E * M, 64 * 32);
        RG_CUDA(ctx->e_viol.ensure(capm * sizeof(unsigned)));
        RG_CUDA(ctx->e_violout.ensure(capm * sizeof(unsigned)));
        RG_CUDA(ctx->e_early.ensure(cap * sizeof(unsigned long long)));
        RG_CUDA(ctx->e_ticket.ensure(cap * sizeof(unsigned)));
        RG_CUDA(ctx->e_out.ensure(cap * (sizeof(int) + 3 * sizeof(double))));
        RG_CUDA(cudaMemsetAsync(ctx->e_viol.p, 0, ctx->e_viol.bytes, ctx->stream));
        RG_CUDA(cudaMemsetAsync(ctx->e_early.p, 0, ctx->e_early.bytes, ctx->stream));
        RG_CUDA(cudaMemsetAsync(ctx->e_ticket.p, 0, ctx->e_ticket.bytes, ctx->stream));
        ctx->batch_cap = (int)cap;
        ctx->batch_cap_m = capm;
    }
    RG_CUDA(ctx->e_in.ensure(in_bytes));
    RG_CUDA(cudaMemcpyAsync(ctx->e_in.p, hd, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
    const double* din = ctx->e_in.as<double>();
    const int32_t* dw = reinterpret_cast<const int32_t*>(din + nd);
    a.x0 = din;
    a.v_prev = din + 3 * E;
    a.r = din + 4 * E;
    a.hs = reinterpret_cast<const uint64_t*>(din + 5 * E);
    a.pair_v = din + 6 * E;
    a.row_src = dw;
    a.pair_e = dw + E * M;
    a.pair_i = a.pair_e + P;
    a.expect = reinterpret_cast<const unsigned*>(a.pair_i + P);
    a.n_ep = n_episodes;
    a.m_grid = m_grid;
    a.prefix_mode = prefix_mode ? 1 : 0;
    a.n_sim = n_sim;
    a.k0 = k0;
    for (int c = 0; c < 3; ++c) {
        a.lo[c] = lo[c];
        a.span[c] = span[c];
    }
    a.viol = ctx->e_viol.as<unsigned>();
    a.early = ctx->e_early.as<unsigned long long>();
    a.ticket = ctx->e_ticket.as<unsigned>();
    char* dout = ctx->e_out.as<char>();
    a.kappa_out = reinterpret_cast<double*>(dout);
    a.v_out = a.kappa_out + E;
    a.early_out = reinterpret_cast<long long*>(a.v_out + E);
    a.row_out = reinterpret_cast<int*>(a.early_out + E);
    a.viol_out = row_viol ? ctx->e_violout.as<unsigned>() : nullptr;
    a.tpb = tpb;
    a.bpr = bpr;
    const bool fma = ctx->variant == rg::kTanhFma, poll = (flags & RG_ABANDON) != 0;
    // Scenario source.  Staged, each episode's block is generated once into SoA and
    // shared by its live rows; fused, every cell hashes its own disturbances.  Staging
    // pays 48 bytes of HBM traffic per scenario-step on top of the same hashing, so it
    // wins only when several rows share a block: fused up to 2 live rows per episode
    // (a closed loop has ~1.05), staged above (the bench snapshot: 32).
    const int64_t ld = (n_sim + 31) / 32 * 32;
    const int64_t ep_stride = (int64_t)prob->j_star * 3 * ld;
    const int64_t per_chunk = kStageMaxScenarioSteps / std::max<int64_t>(1, n_sim * prob->j_star);
    const bool staged = !(flags & RG_FUSED_RNG) && per_chunk >= 1 &&
                        ((flags & RG_STAGE_RNG) || P > 2 * E);
    if (staged) {
        int64_t ec = std::min<int64_t>(E, per_chunk);
        if (ctx->tune.batch_chunk > 0)  // tests: force several chunks
            ec = std::max<int64_t>(1, std::min<int64_t>(ec, ctx->tune.batch_chunk));
        RG_CUDA(ctx->soa.ensure((size_t)ec * ep_stride * sizeof(double)));
        a.soa = ctx->soa.as<double>();
        a.ld = ld;
        a.ep_stride = ep_stride;
        for (int64_t e0 = 0; e0 < E; e0 += ec) {
            const int64_t e1 = std::min<int64_t>(E, e0 + ec);
            const int64_t p0 = ctx->b_first[e0], np = ctx->b_first[e1] - p0;
            if (np == 0) continue;
            RG_CUDA(rg::launch_gen_soa_batch(a.hs + e0, lo, span, k0, n_sim, prob->j_star, ld,
                                             (int32_t)(e1 - e0), ep_stride, ctx->soa.as<double>(),
                                             ctx->stream));
            a.e0 = (int32_t)e0;
            a.p0 = p0;
            RG_CUDA(rg::launch_grid_batch(a, np, fma, poll, ctx->stream));
        }
    } else {
        a.soa = nullptr;
        a.p0 = 0;
        RG_CUDA(rg::launch_grid_batch(a, P, fma, poll, ctx->stream));
    }
    char* hout = reinterpret_cast<char*>(ctx->h_stage.as<char>() + in_bytes);
    RG_CUDA(cudaMemcpyAsync(hout, dout, out_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    unsigned* hviol = reinterpret_cast<unsigned*>(hout + out_bytes);
    if (row_viol)
        RG_CUDA(cudaMemcpyAsync(hviol, a.viol_out, (size_t)E * M * sizeof(unsigned),
                                cudaMemcpyDeviceToHost, ctx->stream));
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    const double* hk = reinterpret_cast<const double*>(hout);
    const long long* he = reinterpret_cast<const long long*>(hk + 2 * E);
    const int* hr = reinterpret_cast<const int*>(hk + 3 * E);
    for (int64_t e = 0; e < E; ++e) {
        if (ctx->b_first[e + 1] > ctx->b_first[e]) {
            kappa_out[e] = hk[e];
            v_out[e] = hk[E + e];
            if (early_out) early_out[e] = he[e];
            row_out[e] = hr[e];
            if (row_viol) memcpy(row_viol + e * M, hviol + e * M, (size_t)M * sizeof(unsigned));
        } else {  // every row gated out: nothing ran, hold (governor.py:562-573)
            kappa_out[e] = 0.0;
            v_out[e] = v_prev[e];
            if (early_out) early_out[e] = 0;
            row_out[e] = -1;
            if (row_viol)
                for (int64_t q = 0; q < M; ++q) row_viol[e * M + q] = 0xffffffffu;
        }
    }
    return RG_OK;
}

}  // extern "C"

namespace {

// [n_sim][horizon][n] (host or device) -> SoA d[(j*n+i)*ld + k], rows j < j_star.
__global__ void k_to_soa_w(const double* __restrict__ src, double* __restrict__ dst,
                           int64_t n_sim, int64_t horizon, int n, int32_t j_star, int64_t ld) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t j = blockIdx.y;
    if (k >= n_sim) return;
    for (int i = 0; i < n; ++i)
        dst[((int64_t)j * n + i) * ld + k] = src[(k * horizon + j) * n + i];
}

int32_t make_linear(const rg_linear_plant* pl, const rg_problem* prob, const double* x0,
                    rg::LinArgs* a) {
    if (!pl || !x0) return fail(RG_E_ARGS, "null argument");
    if (pl->n < 1 || pl->n > 4) return fail(RG_E_ARGS, "linear plant state dim must be 1..4, got %d", pl->n);
    int32_t rc = make_problem(prob, &a->p);
    if (rc) return rc;
    a->L.n = pl->n;
    for (int i = 0; i < 16; ++i) a->L.A[i] = pl->A[i];
    for (int i = 0; i < 4; ++i) {
        a->L.B[i] = pl->B[i];
        a->L.C[i] = pl->C[i];
        a->x0[i] = i < pl->n ? x0[i] : 0.0;
    }
    a->L.D = pl->D;
    a->L.gain = pl->dc_gain;
    a->L.tlo = pl->ss_lower;
    a->L.thi = pl->ss_upper;
    for (int i = 0; i < pl->n; ++i)
        if (!isfinite(x0[i])) return fail(RG_E_ARGS, "state entries must be finite");
    return RG_OK;
}

int32_t linear_source(rg_ctx* ctx, const rg_linear_plant* pl, const double* dist, int64_t n_sim,
                      int64_t horizon, const rg_scenarios* rng, int32_t flags, rg::LinArgs* a) {
    const int n = pl->n;
    const int32_t J = a->p.j_star;
    if (dist) {
        if (horizon < (int64_t)J + 1)
            return fail(RG_E_ARGS, "scenario horizon %lld too short: need >= j_star+1 = %d",
                        (long long)horizon, J + 1);
        const size_t raw = (size_t)n_sim * horizon * n * sizeof(double);
        const double* d = dist;
        if (!(flags & RG_DEVICE_PTRS)) {
            RG_CUDA(ctx->dist_raw.ensure(raw));
            RG_CUDA(cudaMemcpyAsync(ctx->dist_raw.p, dist, raw, cudaMemcpyHostToDevice,
                                    ctx->stream));
            d = ctx->dist_raw.as<double>();
        }
        a->ld = (n_sim + 31) / 32 * 32;
        RG_CUDA(ctx->soa.ensure((size_t)J * n * a->ld * sizeof(double)));
        dim3 grid((unsigned)((n_sim + 127) / 128), (unsigned)J);
        k_to_soa_w<<<grid, 128, 0, ctx->stream>>>(d, ctx->soa.as<double>(), n_sim, horizon, n, J,
                                                  a->ld);
        RG_CUDA(cudaGetLastError());
        a->soa = ctx->soa.as<double>();
    } else {
        if (!rng) return fail(RG_E_ARGS, "need a scenario tensor or an RNG stream");
        a->hs = rg::splitmix64(rng->seed);
        a->k0 = rng->k0;
        for (int i = 0; i < 4; ++i) {
            a->lo[i] = rng->lo[i];
            a->span[i] = rng->span[i];
        }
        a->soa = nullptr;
    }
    return RG_OK;
}

}  // namespace

extern "C" {

int32_t rg_fill_linear(rg_ctx* ctx, const rg_linear_plant* plant, const rg_problem* prob,
                       const double* x0, const double* v_rows, int32_t m_rows,
                       const int32_t* rows, int32_t n_rows, const double* dist, int64_t n_sim,
                       int64_t horizon, const rg_scenarios* rng, uint8_t* S, int32_t* steps,
                       int32_t flags) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    rg::LinArgs a{};
    if ((rc = make_linear(plant, prob, x0, &a))) return rc;
    if (!v_rows || (n_rows > 0 && !rows) || !S || !steps) return fail(RG_E_ARGS, "null buffer");
    if (m_rows < 1 || n_rows < 0 || n_rows > m_rows || n_sim < 1)
        return fail(RG_E_ARGS, "bad sizes");
    for (int32_t q = 0; q < n_rows; ++q)
        if (rows[q] < 0 || rows[q] >= m_rows) return fail(RG_E_ARGS, "row index out of range");
    if (n_rows == 0) return RG_OK;
    if ((rc = linear_source(ctx, plant, dist, n_sim, horizon, rng, flags, &a))) return rc;
    RG_CUDA(ctx->vrows.ensure(m_rows * sizeof(double)));
    RG_CUDA(ctx->rows.ensure(n_rows * sizeof(int32_t)));
    RG_CUDA(cudaMemcpyAsync(ctx->vrows.p, v_rows, m_rows * sizeof(double),
                            cudaMemcpyHostToDevice, ctx->stream));
    RG_CUDA(cudaMemcpyAsync(ctx->rows.p, rows, n_rows * sizeof(int32_t), cudaMemcpyHostToDevice,
                            ctx->stream));
    a.v_rows = ctx->vrows.as<double>();
    a.rows = ctx->rows.as<int32_t>();
    a.n_rows = n_rows;
    a.n_sim = n_sim;
    const size_t cells = (size_t)m_rows * n_sim;
    RG_CUDA(ctx->S.ensure(cells));
    RG_CUDA(ctx->steps.ensure(cells * sizeof(int32_t)));
    a.S = ctx->S.as<uint8_t>();
    a.steps = ctx->steps.as<int32_t>();
    a.tpb = tpb_for(ctx, n_sim, n_rows);
    RG_CUDA(rg::launch_fill_lin(a, ctx->stream));
    for (int32_t q = 0; q < n_rows;) {  // one copy per run of consecutive active rows
        int32_t e = q + 1;
        while (e < n_rows && rows[e] == rows[e - 1] + 1) ++e;
        const int64_t off = (int64_t)rows[q] * n_sim, cnt = (int64_t)(e - q) * n_sim;
        RG_CUDA(cudaMemcpyAsync(S + off, a.S + off, cnt, cudaMemcpyDeviceToHost, ctx->stream));
        RG_CUDA(cudaMemcpyAsync(steps + off, a.steps + off, cnt * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, ctx->stream));
        q = e;
    }
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    return RG_OK;
}

int32_t rg_bisect_linear(rg_ctx* ctx, const rg_linear_plant* plant, const rg_problem* prob,
                         const double* x0, double v_prev, double r, int32_t n_kappa,
                         const double* dist, int64_t n_sim, int64_t horizon,
                         const rg_scenarios* rng, double* kappa_k, int32_t* found_k,
                         int32_t* cells_k, int32_t* early_k, rg_bisect_result* out,
                         int32_t flags) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    rg::LinArgs a{};
    if ((rc = make_linear(plant, prob, x0, &a))) return rc;
    if (n_kappa < 1) return fail(RG_E_ARGS, "n_kappa must be >= 1, got %d", n_kappa);
    if (n_sim < 1) return fail(RG_E_ARGS, "n_sim must be >= 1");
    if (!isfinite(v_prev) || !isfinite(r)) return fail(RG_E_ARGS, "v_prev and r must be finite");
    if ((kappa_k || found_k || cells_k || early_k) && !(kappa_k && found_k && cells_k && early_k))
        return fail(RG_E_ARGS, "per-scenario outputs come as a set of four");
    if (dist || rng) {
        if ((rc = linear_source(ctx, plant, dist, n_sim, horizon, rng, flags, &a))) return rc;
    } else {  // nominal: the zero scenario, staged
        a.ld = 32;
        RG_CUDA(ctx->soa.ensure((size_t)a.p.j_star * plant->n * a.ld * sizeof(double)));
        RG_CUDA(cudaMemsetAsync(ctx->soa.p, 0, (size_t)a.p.j_star * plant->n * a.ld * sizeof(double),
                                ctx->stream));
        a.soa = ctx->soa.as<double>();
        n_sim = 1;
    }
    a.v_prev = v_prev;
    a.r = r;
    a.n_kappa = n_kappa;
    a.n_sim = n_sim;
    if (kappa_k) {
        RG_CUDA(ctx->kap_k.ensure(n_sim * sizeof(double)));
        RG_CUDA(ctx->fnd_k.ensure(n_sim * sizeof(int32_t)));
        RG_CUDA(ctx->cel_k.ensure(n_sim * sizeof(int32_t)));
        RG_CUDA(ctx->erl_k.ensure(n_sim * sizeof(int32_t)));
        a.kappa_k = ctx->kap_k.as<double>();
        a.found_k = ctx->fnd_k.as<int32_t>();
        a.cells_k = ctx->cel_k.as<int32_t>();
        a.early_k = ctx->erl_k.as<int32_t>();
    }
    a.acc = ctx->b_acc.as<rg::BisectAcc>();
    a.out = ctx->b_out.as<rg::BisectOut>();
    a.tpb = tpb_for(ctx, n_sim, 1);
    RG_CUDA(rg::launch_bisect_lin(a, ctx->stream));
    if (kappa_k) {
        RG_CUDA(cudaMemcpyAsync(kappa_k, a.kappa_k, n_sim * sizeof(double),
                                cudaMemcpyDeviceToHost, ctx->stream));
        RG_CUDA(cudaMemcpyAsync(found_k, a.found_k, n_sim * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, ctx->stream));
        RG_CUDA(cudaMemcpyAsync(cells_k, a.cells_k, n_sim * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, ctx->stream));
        RG_CUDA(cudaMemcpyAsync(early_k, a.early_k, n_sim * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, ctx->stream));
    }
    RG_CUDA(ctx->h_stage.ensure(sizeof(rg::BisectOut)));
    rg::BisectOut* ho = ctx->h_stage.as<rg::BisectOut>();
    RG_CUDA(cudaMemcpyAsync(ho, ctx->b_out.p, sizeof(rg::BisectOut), cudaMemcpyDeviceToHost,
                            ctx->stream));
    RG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (out) {
        out->kappa = ho->kappa;
        out->found = ho->found;
        out->cells = ho->cells;
        out->early = ho->early;
        out->kernel_ms = 0.f;
    }
    return RG_OK;
}

int32_t rg_fp64_peak(rg_ctx* ctx, double* flops_per_s) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    if (!flops_per_s) return fail(RG_E_ARGS, "null output");
    RG_CUDA(ctx->tmp_a.ensure(64));
    const int blocks = ctx->sm_count * 8, threads = 256, iters = 1 << 14;
    // warm-up, then the best of three
    RG_CUDA(rg::launch_dfma_peak(ctx->tmp_a.as<double>(), blocks, threads, 256, ctx->stream));
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        RG_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
        RG_CUDA(rg::launch_dfma_peak(ctx->tmp_a.as<double>(), blocks, threads, iters,
                                     ctx->stream));
        RG_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
        RG_CUDA(cudaEventSynchronize(ctx->ev1));
        float ms = 0.f;
        RG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        best = std::min(best, ms);
    }
    *flops_per_s = (double)blocks * threads * iters * 8.0 * 2.0 / (best * 1e-3);
    return RG_OK;
}

// ---------------------------------------------------------------------------
// the closed loop in native code (harness.py:138-224)
// ---------------------------------------------------------------------------

}  // extern "C"

// SurrogateFuelCellPlant.step (dynamics.py:110-130, 228-231) in the reference's operation
// order -- the scalar form of dynamics.py: _surrogate_rk4 -- with numpy's tanh
// (rg_nptanh.h).  Host code is compiled with -ffp-contract=off: every operation rounds.
static void surrogate_plant_step(double h, const double* x, double v, double* out) {
    const double hh = 0.5 * h;
    const double x0 = x[0], x1 = x[1], x2 = x[2];
    const double k11 = -x1 + v;
    const double b1 = x1 + hh * k11;
    const double k21 = -b1 + v;
    const double c1 = x1 + hh * k21;
    const double k31 = -c1 + v;
    const double d1 = x1 + h * k31;
    const double k41 = -d1 + v;
    const double t1 = rg::np_tanh(x1), t2 = rg::np_tanh(b1), t3 = rg::np_tanh(c1),
                 t4 = rg::np_tanh(d1);
    const double k10 = -x0 + t1;
    const double k12 = -2.0 * x2 + x0;
    const double a0 = x0 + hh * k10, a2 = x2 + hh * k12;
    const double k20 = -a0 + t2;
    const double k22 = -2.0 * a2 + a0;
    const double b0 = x0 + hh * k20, b2 = x2 + hh * k22;
    const double k30 = -b0 + t3;
    const double k32 = -2.0 * b2 + b0;
    const double c0 = x0 + h * k30, c2 = x2 + h * k32;
    const double k40 = -c0 + t4;
    const double k42 = -2.0 * c2 + c0;
    const double c = h / 6.0;
    out[0] = x0 + c * (((k10 + 2.0 * k20) + 2.0 * k30) + k40);
    out[1] = x1 + c * (((k11 + 2.0 * k21) + 2.0 * k31) + k41);
    out[2] = x2 + c * (((k12 + 2.0 * k22) + 2.0 * k32) + k42);
}

// rg_closed_loop on the device (rg_ts.cu: k_loop_ts): the whole trace in one cooperative
// launch.  Inputs and outputs travel once; the plan of step 0 comes from the host (the
// same episode_rows), every later one from the kernel.  Returns 1 (with nothing done) when
// the device cannot co-schedule one block per SM, so the caller runs the per-step loop.
static int32_t closed_loop_device(rg_ctx* ctx, const rg_problem* prob, int32_t m_grid,
                                  int32_t prefix_mode, int32_t infeasible_error, const double* x,
                                  double v0, int32_t steps, const double* r,
                                  const double* d_true, uint64_t scen_seed, int64_t n_sim,
                                  const double* lo, const double* span, double* v_out,
                                  double* kappa_out, double* y_out, uint8_t* feasible_out,
                                  int64_t* sims_out, int64_t* early_out, int32_t* wall_us_out,
                                  double* x_out, rg_loop_result* res) {
    int32_t rc;
    rg::LoopArgs L{};
    rg::GridArgs& g = L.g;
    if ((rc = make_problem(prob, &g.p))) return rc;
    if ((rc = grow_grid(ctx, m_grid))) return rc;
    g.m_grid = m_grid;
    g.prefix_mode = prefix_mode ? 1 : 0;
    g.n_sim = n_sim;
    g.k0 = 0;
    g.listed = 1;
    for (int i = 0; i < 3; ++i) {
        g.stream.lo[i] = lo[i];
        g.stream.span[i] = span[i];
    }
    g.abandoned = ctx->g_aband.as<unsigned long long>();
    g.row_src = ctx->g_src.as<int>();
    g.ticket = ctx->g_ticket.as<unsigned>();
    g.pwords = (n_sim + 31) / 32;
    // one buffer: r, d_true | v, kappa, y, sims, early, ns | feasible | LoopCtl, barrier |
    // three accumulator sets (violations, early, overflows per row; zeroed)
    const size_t n = (size_t)steps;
    const size_t o_r = 0, o_d = o_r + 8 * n, o_v = o_d + 24 * n, o_k = o_v + 8 * n,
                 o_y = o_k + 8 * n, o_s = o_y + 8 * n, o_e = o_s + 8 * n, o_ns = o_e + 8 * n,
                 o_f = o_ns + 8 * n, o_c = (o_f + n + 255) / 256 * 256,
                 o_b = o_c + (sizeof(rg::LoopCtl) + 255) / 256 * 256, o_acc = o_b + 256,
                 acc_bytes = 3 * (size_t)m_grid * (4 + 8 + 8), total = o_acc + acc_bytes;
    RG_CUDA(ctx->loop_buf.ensure(total));
    char* d = ctx->loop_buf.as<char>();
    g.early = reinterpret_cast<unsigned long long*>(d + o_acc);
    g.ovf = g.early + 3 * m_grid;
    g.viol = reinterpret_cast<unsigned*>(g.ovf + 3 * m_grid);
    rg::LoopCtl c0{};
    for (int i = 0; i < 3; ++i) c0.x[i] = x[i];
    c0.v_prev = v0;
    c0.r = r[0];
    c0.hs = rg::splitmix64(scen_seed);
    {
        int src[rg::kListMax];
        double vv[rg::kListMax];
        episode_rows(g.p, v0, r[0], m_grid, src, vv);
        c0.list_n = 0;
        for (int32_t q = 0; q < m_grid; ++q) {
            c0.src_tab[q] = src[q];
            if (src[q] == -1) c0.row_list[c0.list_n++] = q;
        }
    }
    c0.abort_step = -1;
    cudaStream_t st = ctx->stream;
    RG_CUDA(cudaMemcpyAsync(d + o_r, r, 8 * n, cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemcpyAsync(d + o_d, d_true, 24 * n, cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemcpyAsync(d + o_c, &c0, sizeof c0, cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemsetAsync(d + o_b, 0, 256 + acc_bytes, st));
    L.ctl = reinterpret_cast<rg::LoopCtl*>(d + o_c);
    L.bar = reinterpret_cast<unsigned*>(d + o_b);
    L.r = reinterpret_cast<const double*>(d + o_r);
    L.d_true = reinterpret_cast<const double*>(d + o_d);
    L.scen_seed = scen_seed;
    L.steps = steps;
    L.infeasible_error = infeasible_error ? 1 : 0;
    L.v_out = reinterpret_cast<double*>(d + o_v);
    L.kappa_out = reinterpret_cast<double*>(d + o_k);
    L.y_out = reinterpret_cast<double*>(d + o_y);
    L.sims_out = reinterpret_cast<long long*>(d + o_s);
    L.early_out = reinterpret_cast<long long*>(d + o_e);
    L.ns_out = reinterpret_cast<long long*>(d + o_ns);
    L.feas_out = reinterpret_cast<unsigned char*>(d + o_f);
    // waiting blocks poll the barrier at most every 256 ns (1024: no difference at C3 or 1k)
    L.spin_cap_ns = 256u;
    const cudaError_t e =
        rg::launch_loop_ts(L, ctx->variant == rg::kTanhFma, ctx->sm_count, st);
    if (e == cudaErrorCooperativeLaunchTooLarge) {
        cudaGetLastError();
        return 1;
    }
    RG_CUDA(e);
    ctx->grid_step_kernels += 1;
    rg::LoopCtl c{};
    RG_CUDA(cudaMemcpyAsync(&c, d + o_c, sizeof c, cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
    const size_t done = (size_t)c.steps_done;
    auto fetch = [&](void* dst, size_t off, size_t bytes) -> cudaError_t {
        return dst && bytes ? cudaMemcpy(dst, d + off, bytes, cudaMemcpyDeviceToHost)
                            : cudaSuccess;
    };
    RG_CUDA(fetch(v_out, o_v, 8 * done));
    RG_CUDA(fetch(kappa_out, o_k, 8 * done));
    RG_CUDA(fetch(y_out, o_y, 8 * done));
    RG_CUDA(fetch(feasible_out, o_f, done));
    static_assert(sizeof(int64_t) == sizeof(long long), "int64 outputs");
    RG_CUDA(fetch(sims_out, o_s, 8 * done));
    RG_CUDA(fetch(early_out, o_e, 8 * done));
    if (wall_us_out && done) {  // the device time of each governor step
        std::vector<long long> ns(done);
        RG_CUDA(fetch(ns.data(), o_ns, 8 * done));
        for (size_t t = 0; t < done; ++t) wall_us_out[t] = (int32_t)(ns[t] / 1000);
    }
    res->steps_done = c.steps_done;
    res->abort_kind = c.abort_kind;
    res->abort_step = c.abort_kind ? c.abort_step : -1;
    res->abort_index = c.abort_index;
    res->abort_value = c.abort_value;
    // the final state, where the per-step loop reports it (the end, or leaving the box)
    if (x_out && (c.abort_kind == 0 || c.abort_kind == RG_LOOP_LEFT_BOX))
        memcpy(x_out, c.x_final, sizeof c.x_final);
    ctx->last_grid_kernel = 1;
    ctx->last_zero_copy = false;
    ctx->last_m = -1;  // no grid step result to fetch
    return RG_OK;
}

extern "C" {

int32_t rg_np_tanh(const double* x, double* y, int64_t n) {
    if ((!x || !y) && n > 0) return fail(RG_E_ARGS, "null array");
    for (int64_t i = 0; i < n; ++i) y[i] = rg::np_tanh(x[i]);
    return RG_OK;
}

int32_t rg_plant_step(double step_size, const double* x, double v, double* out) {
    if (!x || !out) return fail(RG_E_ARGS, "null array");
    surrogate_plant_step(step_size, x, v, out);
    return RG_OK;
}

int32_t rg_closed_loop_bisection(rg_ctx* ctx, const rg_problem* prob, int32_t n_kappa,
                                 const double* x0, double v0, int32_t steps, const double* r,
                                 const double* d_true, double* kappa_out, double* v_out,
                                 double* y_out, uint8_t* feasible_out, int64_t* cells_out,
                                 int64_t* early_out, int32_t* wall_us_out, double* x_out,
                                 rg_loop_result* res) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    if (!prob || !x0 || !r || !d_true || !res) return fail(RG_E_ARGS, "null argument");
    if (steps < 1) return fail(RG_E_ARGS, "steps must be >= 1, got %d", steps);
    if (n_kappa < 1) return fail(RG_E_ARGS, "n_kappa must be >= 1, got %d", n_kappa);
    if (!(isfinite(x0[0]) && isfinite(x0[1]) && isfinite(x0[2])) || !isfinite(v0))
        return fail(RG_E_ARGS, "state entries must be finite");
    for (int32_t t = 0; t < steps; ++t)
        if (!isfinite(r[t])) return fail(RG_E_ARGS, "v_prev and r must be finite");
    rg::LoopBisArgs B{};
    rg::GridArgs& g = B.g;
    if ((rc = make_problem(prob, &g.p))) return rc;
    g.m_grid = 2;  // unused: every unit takes its kappa from the bisection
    g.n_sim = 1;
    g.k0 = 0;
    g.pwords = 1;
    *res = rg_loop_result{};
    res->abort_step = -1;
    // one buffer: r, d_true | kappa, v, y, cells, early, ns | feasible | LoopCtl | counters
    const size_t n = (size_t)steps;
    const size_t o_r = 0, o_d = o_r + 8 * n, o_k = o_d + 24 * n, o_v = o_k + 8 * n,
                 o_y = o_v + 8 * n, o_c = o_y + 8 * n, o_e = o_c + 8 * n, o_ns = o_e + 8 * n,
                 o_f = o_ns + 8 * n, o_ctl = (o_f + n + 255) / 256 * 256,
                 o_acc = o_ctl + (sizeof(rg::LoopCtl) + 255) / 256 * 256, total = o_acc + 256;
    RG_CUDA(ctx->loop_buf.ensure(total));
    char* d = ctx->loop_buf.as<char>();
    g.early = reinterpret_cast<unsigned long long*>(d + o_acc);
    g.ovf = g.early + 1;
    g.viol = reinterpret_cast<unsigned*>(g.ovf + 1);
    rg::LoopCtl c0{};
    for (int i = 0; i < 3; ++i) c0.x[i] = x0[i];
    c0.v_prev = v0;
    c0.abort_step = -1;
    cudaStream_t st = ctx->stream;
    RG_CUDA(cudaMemcpyAsync(d + o_r, r, 8 * n, cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemcpyAsync(d + o_d, d_true, 24 * n, cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemcpyAsync(d + o_ctl, &c0, sizeof c0, cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemsetAsync(d + o_acc, 0, 256, st));
    B.ctl = reinterpret_cast<rg::LoopCtl*>(d + o_ctl);
    B.r = reinterpret_cast<const double*>(d + o_r);
    B.d_true = reinterpret_cast<const double*>(d + o_d);
    B.steps = steps;
    B.n_kappa = n_kappa;
    B.kappa_out = reinterpret_cast<double*>(d + o_k);
    B.v_out = reinterpret_cast<double*>(d + o_v);
    B.y_out = reinterpret_cast<double*>(d + o_y);
    B.cells_out = reinterpret_cast<long long*>(d + o_c);
    B.early_out = reinterpret_cast<long long*>(d + o_e);
    B.ns_out = reinterpret_cast<long long*>(d + o_ns);
    B.feas_out = reinterpret_cast<unsigned char*>(d + o_f);
    RG_CUDA(rg::launch_loop_bisect(B, ctx->variant == rg::kTanhFma, st));
    rg::LoopCtl c{};
    RG_CUDA(cudaMemcpyAsync(&c, d + o_ctl, sizeof c, cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
    const size_t done = (size_t)c.steps_done;
    auto fetch = [&](void* dst, size_t off, size_t bytes) -> cudaError_t {
        return dst && bytes ? cudaMemcpy(dst, d + off, bytes, cudaMemcpyDeviceToHost)
                            : cudaSuccess;
    };
    RG_CUDA(fetch(kappa_out, o_k, 8 * done));
    RG_CUDA(fetch(v_out, o_v, 8 * done));
    RG_CUDA(fetch(y_out, o_y, 8 * done));
    RG_CUDA(fetch(feasible_out, o_f, done));
    RG_CUDA(fetch(cells_out, o_c, 8 * done));
    RG_CUDA(fetch(early_out, o_e, 8 * done));
    if (wall_us_out && done) {
        std::vector<long long> ns(done);
        RG_CUDA(fetch(ns.data(), o_ns, 8 * done));
        for (size_t t = 0; t < done; ++t) wall_us_out[t] = (int32_t)(ns[t] / 1000);
    }
    res->steps_done = c.steps_done;
    res->abort_kind = c.abort_kind;
    res->abort_step = c.abort_kind ? c.abort_step : -1;
    res->abort_index = c.abort_index;
    res->abort_value = c.abort_value;
    if (x_out && c.abort_kind == 0) memcpy(x_out, c.x_final, sizeof c.x_final);
    ctx->last_m = -1;
    return RG_OK;
}

int32_t rg_closed_loop(rg_ctx* ctx, const rg_problem* prob, int32_t m_grid, int32_t prefix_mode,
                       int32_t infeasible_error, const double* x0, double v0, int32_t steps,
                       const double* r, const double* d_true, uint64_t scen_seed, int64_t n_sim,
                       const double* lo, const double* span, double* v_out, double* kappa_out,
                       double* y_out, uint8_t* feasible_out, int64_t* sims_out,
                       int64_t* early_out, int32_t* wall_us_out, double* x_out,
                       rg_loop_result* res) {
    int32_t rc = enter(ctx);
    if (rc) return rc;
    if (!prob || !x0 || !r || !d_true || !lo || !span || !res)
        return fail(RG_E_ARGS, "null argument");
    if (steps < 1) return fail(RG_E_ARGS, "steps must be >= 1, got %d", steps);
    if (m_grid < 2) return fail(RG_E_ARGS, "m_grid must be >= 2, got %d", m_grid);
    if (n_sim < 1) return fail(RG_E_ARGS, "n_sim must be >= 1");
    double x[3] = {x0[0], x0[1], x0[2]};
    if (!(isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2])) || !isfinite(v0))
        return fail(RG_E_ARGS, "state entries must be finite");
    *res = rg_loop_result{};
    res->abort_step = -1;
    // the whole trace on the device when it runs on the time-split form with host-planned rows
    // (the options that disable those keep the per-step loop), every reference is finite and
    // a one-row step fits one pass (above that a step's k_grid launch beats many passes)
    ctx->last_loop_device = 0;
    bool dev_ok = !ctx->tune.no_device_loop && !ctx->tune.no_ts && !ctx->tune.no_row_plan &&
                  m_grid <= rg::kListMax &&
                  (n_sim + 31) / 32 <= (int64_t)rg::kTsUnits * ctx->sm_count && isfinite(v0);
    for (int32_t t = 0; dev_ok && t < steps; ++t) dev_ok = isfinite(r[t]);
    if (dev_ok) {
        rc = closed_loop_device(ctx, prob, m_grid, prefix_mode, infeasible_error, x, v0, steps, r,
                                d_true, scen_seed, n_sim, lo, span, v_out, kappa_out, y_out,
                                feasible_out, sims_out, early_out, wall_us_out, x_out, res);
        if (rc <= 0) {
            if (rc == 0) ctx->last_loop_device = 1;
            return rc;
        }
        *res = rg_loop_result{};
        res->abort_step = -1;
    }
    double v_prev = v0;
    const double h = prob->step_size;
    const double den = (double)(m_grid - 1);
    for (int32_t t = 0; t < steps; ++t) {
        const double rt = r[t];
        // the step's scenario set: seed derive_seed(seed, "scenarios") + t (harness.py:197)
        rg_scenarios sc{};
        sc.seed = scen_seed + (uint64_t)t;
        sc.k0 = 0;
        sc.n_sim = n_sim;
        for (int i = 0; i < 3; ++i) {
            sc.lo[i] = lo[i];
            sc.span[i] = span[i];
        }
        rg_grid_result gr{};
        const auto w0 = std::chrono::steady_clock::now();
        if ((rc = rg_grid_step(ctx, prob, x, v_prev, rt, m_grid, prefix_mode, nullptr, n_sim, 0,
                               &sc, nullptr, nullptr, &gr, RG_NO_TIMING)))
            return rc;
        const int32_t wall_us = (int32_t)std::chrono::duration_cast<std::chrono::microseconds>(
                                    std::chrono::steady_clock::now() - w0)
                                    .count();
        double v, kappa;
        bool feas;
        if (gr.row < 0) {  // governor.py:562-569
            if (infeasible_error) {
                res->abort_kind = RG_LOOP_INFEASIBLE;
                res->abort_step = t;
                return RG_OK;
            }
            v = v_prev;
            kappa = 0.0;
            feas = false;
        } else {  // kappa = grid[row] = row / (M - 1); governor.py:571-579
            kappa = rg::dvd((double)gr.row, den);
            v = rg::update_setpoint(v_prev, rt, kappa);
            v_prev = v;
            feas = true;
        }
        if (v_out) v_out[t] = v;
        if (kappa_out) kappa_out[t] = kappa;
        if (y_out) y_out[t] = x[0];  // plant.output(x, v) = x1 before the plant step
        if (feasible_out) feasible_out[t] = feas ? 1 : 0;
        if (sims_out) sims_out[t] = gr.sims_run;
        if (early_out) early_out[t] = gr.early_terms;
        if (wall_us_out) wall_us_out[t] = wall_us;
        res->steps_done = t + 1;
        // the true plant, then its disturbance (harness.py:215-224)
        double nx[3];
        surrogate_plant_step(h, x, v, nx);
        for (int i = 0; i < 3; ++i) {
            if (!isfinite(nx[i]) || fabs(nx[i]) > 1e6) {  // dynamics.py STATE_ABORT_LIMIT
                res->abort_kind = RG_LOOP_OVERFLOW;
                res->abort_step = t;
                res->abort_index = i;
                res->abort_value = nx[i];
                return RG_OK;
            }
        }
        for (int i = 0; i < 3; ++i) x[i] = nx[i] + d_true[(int64_t)t * 3 + i];
        for (int i = 0; i < 3; ++i) {
            if (!isfinite(x[i]) || fabs(x[i]) > 1e6) {  // harness.py STATE_LIMIT
                res->abort_kind = RG_LOOP_LEFT_BOX;
                res->abort_step = t;
                res->abort_index = i;
                res->abort_value = x[i];
                if (x_out) memcpy(x_out, x, sizeof x);
                return RG_OK;
            }
        }
    }
    if (x_out) memcpy(x_out, x, sizeof x);
    return RG_OK;
}

}  // extern "C"
