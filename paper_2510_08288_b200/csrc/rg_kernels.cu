// rg_kernels.cu -- sm_100a kernels of the robust Reference Governor hot path.
//
//   k_sample      scenario tensor from the counter RNG (disturbance.py:179-203)
//   k_to_soa      [k][j][i] host-layout tensor -> SoA d[(j*3+i)*ld + k]
//   k_fill        parity fill: status/steps per (active row, scenario) cell
//                 (kernels.py:121-162 / backend_gpu.fill seam)
//   k_grid        fused robust grid step (governor.py:245-377, 520-579):
//                 ss gate + dedup per row, rollout with fused RNG or staged
//                 SoA, warp-ballot feasibility reduction into per-row counters,
//                 optional P bitmask, last-block extraction of the best row
//   k_bisect      exact Alg. 2 (governor.py:380-430, 469-517): one thread per
//                 scenario runs its own bisection; min/AND/sum reductions
//   k_tanh        device tanh for the bit-parity self-test
//
// Layout: one thread per (row, scenario) cell, scenarios on the fast axis so a
// warp is 32 consecutive scenarios of one candidate setpoint: their
// trajectories stay close, so the data-dependent branches of tanh/expm1 and
// the early exits mostly agree across the warp.
#include "rg_kernels.h"

#include <cuda_runtime.h>

#include <mutex>

#include "rg_cell.cuh"
#include "rg_decoupled.cuh"
#include "rg_ws.cuh"

#ifndef RG_GRID_MINB
#define RG_GRID_MINB 1
#endif
// phase-decoupled grid kernel geometry: cells per block, steps per chunk, threads
#ifndef RG_DEC_C
#define RG_DEC_C 32
#endif
#ifndef RG_WS_T
#define RG_WS_T 4
#endif
#ifndef RG_GRID_WARP
#define RG_GRID_WARP 1  // k_grid, one lane per cell: warp-uniform rollout (rollout<..., WARP>)
#endif
#ifndef RG_WS_W
#define RG_WS_W 2
#endif
#ifndef RG_DEC_T
#define RG_DEC_T 16
#endif
#ifndef RG_DEC_TB
#define RG_DEC_TB 128
#endif

namespace rg {

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// warp-aggregated add of a per-lane predicate count into a 64-bit counter
__device__ __forceinline__ void warp_count_add(bool pred, unsigned long long* ctr) {
    const unsigned m = __ballot_sync(0xffffffffu, pred);
    if (lane_id() == 0 && m) atomicAdd(ctr, (unsigned long long)__popc(m));
}

__device__ __forceinline__ CellConst make_cell(const ProblemDev& p) {
    CellConst c;
    c.h = p.h;
    c.hh = p.hh;
    c.c = p.c;
    c.ylo = p.ylo;
    c.yhi = p.yhi;
    c.j_star = p.j_star;
    return c;
}

__device__ __forceinline__ bool ss_gate(double v, const ProblemDev& p) {
    return p.vlo <= v && v <= p.vhi;  // NaN -> false, like ConstraintSet.contains
}

// ---------------------------------------------------------------------------
// scenario generation
// ---------------------------------------------------------------------------

__global__ void k_sample(SampleArgs a) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (k, j)
    const int64_t total = a.n_sim * a.horizon;
    if (idx >= total) return;
    const int64_t k = idx / a.horizon;
    const int64_t j = idx - k * a.horizon;
    const uint64_t K = splitmix64(a.hs ^ (uint64_t)(a.k0 + k));
    const uint64_t J = splitmix64(K ^ (uint64_t)j);
    double* o = a.out + idx * a.width;
    for (int i = 0; i < a.width; ++i) {
        const double u = unit_double(splitmix64(J ^ (uint64_t)i));
        o[i] = add(a.lo[i], mul(a.span[i], u));
    }
}

// counter RNG straight into the SoA layout d[(j*3+i)*ld + k], rows j < j_star:
// one thread per (scenario, step); lanes run over scenarios, so stores coalesce.
__global__ void k_gen_soa(ScenarioStream st, int64_t k0, int64_t n_sim, int32_t j_star,
                          int64_t ld, double* __restrict__ dst) {
    // a grid step launched behind this kernel with programmatic stream
    // serialization may start its prologue now; it waits (griddepcontrol.wait)
    // for this grid's completion before it reads the block
    asm volatile("griddepcontrol.launch_dependents;");
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t j = blockIdx.y;
    if (k >= n_sim || j >= j_star) return;
    const uint64_t K = scenario_key(st, (uint64_t)(k0 + k));
    double d0, d1, d2;
    disturbance_at(st, K, (uint64_t)j, d0, d1, d2);
    double* o = dst + (int64_t)j * 3 * ld + k;
    o[0] = d0;
    o[ld] = d1;
    o[2 * ld] = d2;
}

// k_gen_soa for a batch of episodes (blockIdx.z), each with its own stream key hs[z]
// and a block of its own at dst + z * ep_stride.
__global__ void k_gen_soa_batch(const uint64_t* __restrict__ hs, double3 lo, double3 span,
                                int64_t k0, int64_t n_sim, int32_t j_star, int64_t ld,
                                int64_t ep_stride, double* __restrict__ dst) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t j = blockIdx.y;
    if (k >= n_sim || j >= j_star) return;
    ScenarioStream st;
    st.hs = hs[blockIdx.z];
    st.lo[0] = lo.x;
    st.lo[1] = lo.y;
    st.lo[2] = lo.z;
    st.span[0] = span.x;
    st.span[1] = span.y;
    st.span[2] = span.z;
    const uint64_t K = scenario_key(st, (uint64_t)(k0 + k));
    double d0, d1, d2;
    disturbance_at(st, K, (uint64_t)j, d0, d1, d2);
    double* o = dst + (int64_t)blockIdx.z * ep_stride + (int64_t)j * 3 * ld + k;
    o[0] = d0;
    o[ld] = d1;
    o[2 * ld] = d2;
}

// tile transpose of [n_sim][horizon][3] (rows j < j_star) into d[(j*3+i)*ld + k]
__global__ void k_to_soa(const double* __restrict__ src, double* __restrict__ dst,
                         int64_t n_sim, int64_t horizon, int32_t j_star, int64_t ld) {
    __shared__ double tile[32][32 * 3 + 1];
    const int64_t k0 = (int64_t)blockIdx.x * 32;
    const int32_t j0 = blockIdx.y * 32;
    // load: warp w reads scenario k0+w, 32 steps x 3 comps (96 contiguous doubles)
    for (int w = threadIdx.y; w < 32; w += blockDim.y) {
        const int64_t k = k0 + w;
        for (int e = threadIdx.x; e < 96; e += 32) {
            const int32_t j = j0 + e / 3;
            double v = 0.0;
            if (k < n_sim && j < j_star) v = src[(k * horizon + j) * 3 + (e % 3)];
            tile[w][e] = v;
        }
    }
    __syncthreads();
    // store: lanes run over k (coalesced), rows over (j, i)
    for (int r = threadIdx.y; r < 96; r += blockDim.y) {
        const int32_t j = j0 + r / 3;
        const int i = r % 3;
        const int64_t k = k0 + threadIdx.x;
        if (j < j_star && k < ld) dst[((int64_t)j * 3 + i) * ld + k] = tile[threadIdx.x][r];
    }
}

// ---------------------------------------------------------------------------
// parity fill: status/steps for every (active row, scenario)
// ---------------------------------------------------------------------------

template <bool FMA, bool RNG, int LPC>
__global__ void __launch_bounds__(128, RG_GRID_MINB) k_fill(FillArgs a) {
    const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPC;
    const bool live = k < a.n_sim;
    constexpr bool W = LPC == 1 && RG_GRID_WARP;  // whole warps run the rollout
    if (LPC == 1 && !W && !live) return;
    const int32_t row = a.rows[blockIdx.y];
    const double v = a.v_rows[row];
    const CellConst c = make_cell(a.p);
    const int64_t kk = live ? k : 0;  // out-of-range lanes replay scenario 0
    int32_t steps = 0;
    int st;
    if (RNG) {
        RngSource src{a.stream, scenario_key(a.stream, (uint64_t)(a.k0 + kk))};
        st = rollout<FMA, false, LPC, RngSource, W>(c, a.x0[0], a.x0[1], a.x0[2], v, src, steps,
                                                    nullptr, live);
    } else {
        __shared__ double ring[2 * 3 * kRingStride];
        SoaSource src{a.soa + kk, a.ld, ring + threadIdx.x};
        st = rollout<FMA, false, LPC, SoaSource, W>(c, a.x0[0], a.x0[1], a.x0[2], v, src, steps,
                                                    nullptr, live);
    }
    if (live && threadIdx.x % LPC == 0) {
        a.S[(int64_t)row * a.n_sim + k] = (uint8_t)st;
        a.steps[(int64_t)row * a.n_sim + k] = steps;
    }
}

// ---------------------------------------------------------------------------
// fused robust grid step
// ---------------------------------------------------------------------------

// Row status for the grid: -2 pruned by the steady-state gate, -1 simulated,
// >= 0 duplicate of that (earlier, simulated) row.  governor.py:302-317.
__device__ int row_source(const GridArgs& a, int i, double* v_out) {
    const double kap_i = dvd((double)i, (double)(a.m_grid - 1));
    const double v = update_setpoint(a.v_prev, a.r, kap_i);
    *v_out = v;
    if (!ss_gate(v, a.p)) return -2;
    for (int q = 0; q < i; ++q) {
        const double vq = update_setpoint(a.v_prev, a.r, dvd((double)q, (double)(a.m_grid - 1)));
        if (ss_gate(vq, a.p) && vq == v) return q;
    }
    return -1;
}

// row_source with the first warp: lane q evaluates candidate q's setpoint, a
// ballot finds the first equal gated row (same result, no serial loop of
// divisions in front of every block's rollout).  All 32 lanes must call it.
__device__ int row_source_warp(const GridArgs& a, int i, double* v_out) {
    const int lane = threadIdx.x & 31;
    const double den = (double)(a.m_grid - 1);
    const double v = update_setpoint(a.v_prev, a.r, dvd((double)i, den));
    *v_out = v;
    if (!ss_gate(v, a.p)) return -2;
    for (int q0 = 0; q0 < i; q0 += 32) {
        const int q = q0 + lane;
        bool hit = false;
        if (q < i) {
            const double vq = update_setpoint(a.v_prev, a.r, dvd((double)q, den));
            hit = ss_gate(vq, a.p) && vq == v;
        }
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (m) return q0 + __ffs(m) - 1;
    }
    return -1;
}

// Device-side span of a grid step for the diagnostics (kernel_us) without
// host event records: each block's first thread lowers t0 to its start time,
// the finalizing block reads it against its own end time and re-arms t0.
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void grid_clock_start(const GridArgs& a) {
    if (a.t0) atomicMin(a.t0, global_ns());
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// Last block out extracts the best row (governor.py:351-377) and resets the
// accumulators for the next launch.  The first warp reads 32 rows at a time
// (one per lane) and reduces with ballots and shuffles, so the step's tail is
// a few L2 round trips rather than one chain of loads per row.
__device__ __forceinline__ void grid_finalize(const GridArgs& a) {
    __shared__ bool s_last;
    __shared__ unsigned long long s_tfin;  // globaltimer when this block won the ticket
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned total = gridDim.x * gridDim.y;
        s_last = atomicAdd(a.ticket, 1u) == total - 1;
        s_tfin = global_ns();
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (a.pbits_host) {  // zero-copy result: the P bits go to pinned host memory in one pass
        // eight independent L2 loads in flight per thread, then the eight host stores
        const int64_t nw = (int64_t)a.m_grid * a.pwords;
        const int64_t step = blockDim.x;
        for (int64_t q0 = threadIdx.x; q0 < nw; q0 += 8 * step) {
            unsigned w[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t q = q0 + u * step;
                w[u] = q < nw ? __ldcg(a.pbits + q) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t q = q0 + u * step;
                if (q < nw) a.pbits_host[q] = w[u];
            }
        }
        __syncthreads();
    }
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int best = -1;
        bool open = true;  // prefix mode: every row so far was feasible
        int n_active = 0, pruned = 0, dup = 0;
        unsigned long long early = 0, ovf = 0, aband = 0;
        for (int q0 = 0; q0 < a.m_grid; q0 += 32) {
            const int q = q0 + lane;
            const bool in = q < a.m_grid;
            int sq = -2;
            unsigned vq = 0u;
            unsigned long long ab = 0ull, ea = 0ull, ov = 0ull;
            if (in) {
                sq = ((volatile int*)a.row_src)[q];
                vq = ((volatile unsigned*)a.viol)[q];
                ab = ((volatile unsigned long long*)a.abandoned)[q];
                ea = ((volatile unsigned long long*)a.early)[q];
                ov = ((volatile unsigned long long*)a.ovf)[q];
            }
            if (in && sq >= 0) {  // a duplicate row takes its source row's verdict
                vq = ((volatile unsigned*)a.viol)[sq];
                ab = ((volatile unsigned long long*)a.abandoned)[sq];
            }
            const bool act = in && sq == -1;
            const bool full = in && sq != -2 && vq == 0u && ab == 0ull;
            n_active += __popc(__ballot_sync(0xffffffffu, act));
            pruned += __popc(__ballot_sync(0xffffffffu, in && sq == -2));
            dup += __popc(__ballot_sync(0xffffffffu, in && sq >= 0));
            early += warp_sum_u64(act ? ea : 0ull);
            ovf += warp_sum_u64(act ? ov : 0ull);
            aband += warp_sum_u64(act ? ab : 0ull);
            if (in) a.viol_out[q] = sq == -2 ? 0xffffffffu : vq;
            const unsigned fm = __ballot_sync(0xffffffffu, full);
            if (a.prefix_mode) {
                if (open) {  // the run of feasible rows from row 0 (governor.py:370-375)
                    const int run = ~fm == 0u ? 32 : __ffs(~fm) - 1;
                    if (run > 0) best = q0 + run - 1;
                    open = run == 32;
                }
            } else if (fm) {
                best = q0 + 31 - __clz(fm);
            }
        }
        if (lane == 0) {
            a.out->row = best;
            a.out->n_active = n_active;
            a.out->ss_pruned_rows = pruned;
            a.out->dedup_rows = dup;
            a.out->early_terms = (long long)early;
            a.out->overflows = (long long)ovf;
            a.out->abandoned = (long long)aband;
            a.out->sims_run = (long long)n_active * a.n_sim;
            if (a.t0) {
                const unsigned long long now = global_ns();
                a.out->kernel_ns = now - *(volatile unsigned long long*)a.t0;
                a.out->reduce_ns = now - s_tfin;
                *a.t0 = ~0ull;
            }
            // publish: every result word above (and every block's P bits) before seq
            __threadfence_system();
            *(volatile unsigned long long*)&a.out->seq = a.seq_token;
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < a.m_grid; q += blockDim.x) {
        a.viol[q] = 0u;
        a.early[q] = 0ull;
        a.ovf[q] = 0ull;
        a.abandoned[q] = 0ull;
    }
    if (threadIdx.x == 0) *a.ticket = 0u;
}

// MOD: the tanh forms' operand-modifier variant (rg_math.cuh), for the
// issue-bound multi-wave steps; the single-wave (latency-bound) step keeps MOD off.
// S2: the two-steps-per-iteration rollout (rollout2) for the latency-bound
// single-wave step over a staged block (blocks of at most 256 threads).
template <bool FMA, bool RNG, bool POLL, int LPC, bool MOD = false, bool S2 = false>
__global__ void __launch_bounds__(256, RG_GRID_MINB) k_grid(GridArgs a) {
    __shared__ int s_src;
    __shared__ double s_v;
    const int i = blockIdx.y;
    if (threadIdx.x < 32) {
        double v;
        const int src = row_source_warp(a, i, &v);
        if (threadIdx.x == 0) {
            grid_clock_start(a);
            s_src = src;
            s_v = v;
            if (blockIdx.x == 0) a.row_src[i] = src;
        }
    }
    __syncthreads();
    // staged scenarios: the generator launched just before may still be running
    // (programmatic dependent launch); no-op otherwise
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int src_i = s_src;
    const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPC;
    const bool lead = threadIdx.x % LPC == 0;
    if (src_i == -1) {
        const bool live = k < a.n_sim;
        const int64_t kk = live ? k : 0;
        int st = kOk;
        int32_t steps = a.p.j_star;
        constexpr bool W = LPC == 1 && RG_GRID_WARP;  // whole warps run the rollout
        if constexpr (S2) {
            static_assert(!RNG && LPC == 1, "the two-step rollout reads a staged block");
            __shared__ double ring4[4 * 3 * kRing4Stride];
            Soa4Source src;
            src.d = a.soa + kk;
            src.ld = a.ld;
            src.ring = ring4 + threadIdx.x;
            st = rollout2<FMA, POLL>(make_cell(a.p), a.x0[0], a.x0[1], a.x0[2], s_v, src, steps,
                                     a.viol + i, live);
        } else if (live || LPC > 1 || W) {
            const CellConst c = make_cell(a.p);
            if (RNG) {
                RngSource src{a.stream, scenario_key(a.stream, (uint64_t)(a.k0 + kk))};
                st = rollout<FMA, POLL, LPC, RngSource, W, false, MOD>(c, a.x0[0], a.x0[1], a.x0[2], s_v,
                                                           src, steps, a.viol + i, live);
            } else {
                __shared__ double ring[2 * 3 * kRingStride];
                SoaSource src{a.soa + kk, a.ld, ring + threadIdx.x};
                st = rollout<FMA, POLL, LPC, SoaSource, W, false, MOD>(c, a.x0[0], a.x0[1], a.x0[2], s_v,
                                                           src, steps, a.viol + i, live);
            }
        }
        const bool cnt = live && lead;
        const bool bad = cnt && st != kOk && st != kAbandoned;
        const unsigned bad_mask = __ballot_sync(0xffffffffu, bad);
        if (lane_id() == 0 && bad_mask) atomicAdd(a.viol + i, (unsigned)__popc(bad_mask));
        warp_count_add(cnt && st != kAbandoned && steps < a.p.j_star, a.early + i);
        warp_count_add(cnt && st == kOverflow, a.ovf + i);
        warp_count_add(cnt && st == kAbandoned, a.abandoned + i);
        if (a.pbits) {
            if (LPC == 1) {
                const unsigned ok_mask = __ballot_sync(0xffffffffu, live && st == kOk);
                if (lane_id() == 0 && (k - lane_id()) < a.n_sim)
                    a.pbits[(int64_t)i * a.pwords + (k >> 5)] = ok_mask;
            } else if (cnt && st == kOk) {  // words pre-zeroed by the host
                atomicOr(a.pbits + (int64_t)i * a.pwords + (k >> 5), 1u << (k & 31));
            }
        }
    } else if (LPC == 1 && a.pbits && lane_id() == 0 && (k - lane_id()) < a.n_sim) {
        // pruned or duplicate row: no simulated bits (the host expands duplicates)
        a.pbits[(int64_t)i * a.pwords + (k >> 5)] = 0u;
    }
    grid_finalize(a);
}

// Phase-decoupled grid step (rg_decoupled.cuh): C scenarios of one row per
// block, chunks of T steps; same accumulators, bits and finalize as k_grid.
template <bool FMA, bool RNG, bool POLL, int C, int T, int TB>
__global__ void __launch_bounds__(TB) k_grid_dec(GridArgs a) {
    __shared__ DecSmem<C, T> sm;
    __shared__ uint64_t kkey[C];
    __shared__ int s_src;
    __shared__ double s_v;
    const int i = blockIdx.y;
    if (threadIdx.x < 32) {
        double v;
        const int src = row_source_warp(a, i, &v);
        if (threadIdx.x == 0) {
            grid_clock_start(a);
            s_src = src;
            s_v = v;
            if (blockIdx.x == 0) a.row_src[i] = src;
        }
    }
    const int64_t kbase = (int64_t)blockIdx.x * C;
    if (RNG && threadIdx.x < C)
        kkey[threadIdx.x] = scenario_key(a.stream, (uint64_t)(a.k0 + kbase + threadIdx.x));
    __syncthreads();
    const int64_t k = kbase + threadIdx.x;
    const bool cell_warp = threadIdx.x < C;
    if (s_src == -1) {
        int st;
        int32_t steps;
        rollout_decoupled<FMA, POLL, RNG, C, T>(sm, make_cell(a.p), a.x0[0], a.x0[1], a.x0[2],
                                                 s_v, kbase, a.n_sim, a.soa, a.ld, a.stream,
                                                 kkey, a.viol + i, st, steps);
        if (cell_warp) {
            const bool live = k < a.n_sim;
            const bool bad = live && st != kOk && st != kAbandoned;
            const unsigned bad_mask = __ballot_sync(0xffffffffu, bad);
            if (lane_id() == 0 && bad_mask) atomicAdd(a.viol + i, (unsigned)__popc(bad_mask));
            warp_count_add(live && st != kAbandoned && steps < a.p.j_star, a.early + i);
            warp_count_add(live && st == kOverflow, a.ovf + i);
            warp_count_add(live && st == kAbandoned, a.abandoned + i);
            if (a.pbits) {
                const unsigned ok_mask = __ballot_sync(0xffffffffu, live && st == kOk);
                if (lane_id() == 0 && (k - lane_id()) < a.n_sim)
                    a.pbits[(int64_t)i * a.pwords + (k >> 5)] = ok_mask;
            }
        }
    } else if (cell_warp && a.pbits && lane_id() == 0 && (k - lane_id()) < a.n_sim) {
        a.pbits[(int64_t)i * a.pwords + (k >> 5)] = 0u;
    }
    grid_finalize(a);
}

// Warp-specialised grid step (rg_ws.cuh): 32 scenarios of one row per block,
// one sequence warp plus W tanh warps; same accumulators, bits and finalize.
template <bool FMA, bool RNG, bool POLL, int T, int W>
__global__ void __launch_bounds__(32 * (1 + W)) k_grid_ws(GridArgs a) {
    __shared__ WsSmem<T> sm;
    __shared__ int s_src;
    __shared__ double s_v;
    const int i = blockIdx.y;
    if (threadIdx.x < 32) {
        double v;
        const int src = row_source_warp(a, i, &v);
        if (threadIdx.x == 0) {
            grid_clock_start(a);
            s_src = src;
            s_v = v;
            if (blockIdx.x == 0) a.row_src[i] = src;
        }
    }
    __syncthreads();
    const int64_t kbase = (int64_t)blockIdx.x * 32;
    const int64_t k = kbase + threadIdx.x;
    const bool seq_warp = threadIdx.x < 32;
    if (s_src == -1) {
        int st = kOk;
        int32_t steps = a.p.j_star;
        rollout_ws<FMA, POLL, RNG, T, W>(sm, make_cell(a.p), a.x0[0], a.x0[1], a.x0[2], s_v,
                                         kbase, a.n_sim, a.soa, a.ld, a.stream, a.viol + i, st,
                                         steps);
        if (seq_warp) {
            const bool live = k < a.n_sim;
            const bool bad = live && st != kOk && st != kAbandoned;
            const unsigned bad_mask = __ballot_sync(0xffffffffu, bad);
            if (lane_id() == 0 && bad_mask) atomicAdd(a.viol + i, (unsigned)__popc(bad_mask));
            warp_count_add(live && st != kAbandoned && steps < a.p.j_star, a.early + i);
            warp_count_add(live && st == kOverflow, a.ovf + i);
            warp_count_add(live && st == kAbandoned, a.abandoned + i);
            if (a.pbits) {
                const unsigned ok_mask = __ballot_sync(0xffffffffu, live && st == kOk);
                if (lane_id() == 0 && kbase < a.n_sim)
                    a.pbits[(int64_t)i * a.pwords + (kbase >> 5)] = ok_mask;
            }
        }
    } else if (seq_warp && a.pbits && lane_id() == 0 && kbase < a.n_sim) {
        a.pbits[(int64_t)i * a.pwords + (kbase >> 5)] = 0u;
    }
    grid_finalize(a);
}

// ---------------------------------------------------------------------------
// batched grid step: E independent governor instances in one launch
// ---------------------------------------------------------------------------

// Launch bounds: at most 168 registers (3 blocks of 128 threads per SM), so the
// 64-thread blocks keep 12 warps per SM (3 per SMSP) in this always multi-wave kernel.
template <bool FMA, bool POLL, int LPC, bool SOA = false>
__global__ void __launch_bounds__(128, 3) k_grid_batch(BatchArgs a) {
    __shared__ int s_src;
    __shared__ double s_v;
    __shared__ bool s_last;
    const int e = a.e0 + (int)blockIdx.z;
    const int i = blockIdx.y;
    const int M = a.m_grid;
    const double vp = a.v_prev[e], rr = a.r[e];
    if (threadIdx.x == 0) {
        const double v = update_setpoint(vp, rr, dvd((double)i, (double)(M - 1)));
        int src = ss_gate(v, a.p) ? -1 : -2;
        for (int q = 0; src == -1 && q < i; ++q) {
            const double vq = update_setpoint(vp, rr, dvd((double)q, (double)(M - 1)));
            if (ss_gate(vq, a.p) && vq == v) src = q;
        }
        s_src = src;
        s_v = v;
        if (blockIdx.x == 0) a.row_src[(int64_t)e * M + i] = src;
    }
    __syncthreads();
    const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPC;
    const bool lead = threadIdx.x % LPC == 0;
    unsigned* viol = a.viol + (int64_t)e * M;
    if (s_src == -1) {
        const bool live = k < a.n_sim;
        int st = kOk;
        int32_t steps = a.p.j_star;
        constexpr bool W = LPC == 1 && RG_GRID_WARP;  // whole warps run the rollout
        if (live || LPC > 1 || W) {
            const double* x0 = a.x0 + 3 * (int64_t)e;
            if constexpr (SOA) {  // staged block of this episode (k_gen_soa_batch)
                __shared__ double ring[2 * 3 * kRingStride];
                SoaSource src{a.soa + (int64_t)blockIdx.z * a.ep_stride + (live ? k : 0), a.ld,
                              ring + threadIdx.x};
                st = rollout<FMA, POLL, LPC, SoaSource, W, false, true>(make_cell(a.p), x0[0], x0[1], x0[2],
                                                           s_v, src, steps, viol + i, live);
            } else {
                ScenarioStream ss;
                ss.hs = a.hs[e];
                for (int c = 0; c < 3; ++c) {
                    ss.lo[c] = a.lo[c];
                    ss.span[c] = a.span[c];
                }
                RngSource src{ss, scenario_key(ss, (uint64_t)(a.k0 + (live ? k : 0)))};
                st = rollout<FMA, POLL, LPC, RngSource, W, false, true>(make_cell(a.p), x0[0], x0[1], x0[2],
                                                           s_v, src, steps, viol + i, live);
            }
        }
        const bool cnt = live && lead;
        const unsigned bad = __ballot_sync(0xffffffffu, cnt && st != kOk && st != kAbandoned);
        if (lane_id() == 0 && bad) atomicAdd(viol + i, (unsigned)__popc(bad));
        warp_count_add(cnt && st != kAbandoned && steps < a.p.j_star, a.early + e);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(a.ticket + e, 1u) == gridDim.x * gridDim.y - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x == 0) {
        const int* rs = a.row_src + (int64_t)e * M;
        int best = -1;
        for (int q = 0; q < M; ++q) {
            const int s = ((volatile const int*)rs)[q];
            const bool full = s != -2 && ((volatile unsigned*)viol)[s < 0 ? q : s] == 0u;
            if (a.viol_out)
                a.viol_out[(int64_t)e * M + q] =
                    s == -2 ? 0xffffffffu : ((volatile unsigned*)viol)[s < 0 ? q : s];
            if (a.prefix_mode) {
                if (best == q - 1 && full) best = q;
            } else if (full) {
                best = q;
            }
        }
        a.row_out[e] = best;
        const double kap = best < 0 ? 0.0 : dvd((double)best, (double)(M - 1));
        a.kappa_out[e] = kap;
        a.v_out[e] = best < 0 ? vp : update_setpoint(vp, rr, kap);
        a.early_out[e] = (long long)((volatile unsigned long long*)a.early)[e];
    }
    __syncthreads();
    for (int q = threadIdx.x; q < M; q += blockDim.x) viol[q] = 0u;
    if (threadIdx.x == 0) {
        a.early[e] = 0ull;
        a.ticket[e] = 0u;
    }
}

// ---------------------------------------------------------------------------
// joint bisection: every scenario tests the same kappa per iteration
// ---------------------------------------------------------------------------

// The iteration's candidate, as governor.py:407-431 walks it: kappa = 1 first
// (it < 0), then the midpoint of the bracket.
__device__ __forceinline__ double joint_kappa(const volatile JointState* st, int it) {
    return it < 0 ? 1.0 : mul(0.5, add(st->lo, st->hi));
}

// The decision after an iteration (governor.py:412-431 applied to the joint
// verdict): kappa = 1 feasible ends the search; otherwise a feasible midpoint
// raises the lower end, an infeasible one lowers the upper end.  Cells and
// early terminations count like Alg. 2 summed over scenarios (a gated-out
// candidate is an early termination of every scenario).
__device__ void joint_decide(const JointArgs& a, int it, double kappa, bool gated_in,
                             unsigned long long early_here) {
    volatile JointState* st = a.st;
    const bool feas = gated_in && st->viol == 0u;
    st->cells += (unsigned long long)a.n_sim;
    st->early += gated_in ? early_here : (unsigned long long)a.n_sim;
    if (it < 0) {
        if (feas) {
            st->kopt = 1.0;
            st->found = 1;
            st->done = 1;
        }
    } else if (feas) {
        st->kopt = kappa;
        st->found = 1;
        st->lo = kappa;
    } else {
        st->hi = kappa;
    }
    if (it == a.n_kappa - 1) st->done = 1;
    st->viol = 0u;
}

template <bool FMA, int SRC>  // SRC: 0 zero (nominal), 1 rng, 2 soa
__global__ void __launch_bounds__(256, RG_GRID_MINB) k_joint_roll(JointArgs a, int it) {
    __shared__ int s_run;  // 0 search finished, 1 candidate gated out, 2 roll out
    __shared__ double s_v, s_kappa;
    __shared__ bool s_last;
    __shared__ unsigned long long s_early;
    if (threadIdx.x == 0) {
        const volatile JointState* st = a.st;
        if (st->done) {
            s_run = 0;
        } else {
            const double kappa = joint_kappa(st, it);
            const double v = update_setpoint(a.v_prev, a.r, kappa);
            s_kappa = kappa;
            s_v = v;
            s_run = ss_gate(v, a.p) ? 2 : 1;
        }
    }
    __syncthreads();
    const int run = s_run;
    if (run == 0) return;
    if (run == 2) {
        const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        const bool live = k < a.n_sim;
        const int64_t kk = live ? k : 0;
        const CellConst c = make_cell(a.p);
        int32_t steps = 0;
        int st;
        unsigned* flag = &a.st->viol;
        if (SRC == 1) {
            RngSource src{a.stream, scenario_key(a.stream, (uint64_t)(a.k0 + kk))};
            st = rollout<FMA, true, 1, RngSource, true, true>(c, a.x0[0], a.x0[1], a.x0[2], s_v,
                                                              src, steps, flag, live);
        } else if (SRC == 2) {
            __shared__ double ring[2 * 3 * kRingStride];
            SoaSource src{a.soa + kk, a.ld, ring + threadIdx.x};
            st = rollout<FMA, true, 1, SoaSource, true, true>(c, a.x0[0], a.x0[1], a.x0[2], s_v,
                                                              src, steps, flag, live);
        } else {
            st = rollout<FMA, true, 1, ZeroSource, true, true>(c, a.x0[0], a.x0[1], a.x0[2],
                                                               s_v, ZeroSource{}, steps, flag,
                                                               live);
        }
        // the flag is raised inside the rollout at the violating step; a cell
        // that starts outside the set never enters the loop, so raise it here too
        const bool bad = live && st != kOk && st != kAbandoned;
        if (__ballot_sync(0xffffffffu, bad) && lane_id() == 0) atomicOr(flag, 1u);
        warp_count_add(bad && steps < a.p.j_star, &a.st->early);
    }
    if (!a.fold) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&a.st->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    __threadfence();
    // the early terminations of this iteration were accumulated into st->early
    // directly; joint_decide adds none for a rolled-out candidate
    a.st->ticket = 0u;
    joint_decide(a, it, s_kappa, run == 2, 0ull);
}

// Decision kernel for the sharded form: runs after the all-reduce of st->viol.
__global__ void k_joint_decide(JointArgs a, int it) {
    const volatile JointState* st = a.st;
    if (st->done) return;
    const double kappa = joint_kappa(st, it);
    const double v = update_setpoint(a.v_prev, a.r, kappa);
    joint_decide(a, it, kappa, ss_gate(v, a.p), 0ull);
}

// ---------------------------------------------------------------------------
// exact Alg. 2: per-scenario bisection
// ---------------------------------------------------------------------------

template <bool FMA, int SRC, int LPC>  // SRC: 0 zero (nominal), 1 rng, 2 soa
__global__ void __launch_bounds__(256, RG_GRID_MINB) k_bisect(BisectArgs a) {
    const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPC;
    const bool live = k < a.n_sim;
    const bool lead = threadIdx.x % LPC == 0;
    double kopt = 1.0;
    int found = 1, cells = 0, early = 0;
    // U: every lane of the warp walks the candidates (LPC > 1 shuffles, or the
    // warp-uniform one-lane-per-cell rollout); finished lanes keep it company
    constexpr bool W = LPC == 1 && RG_GRID_WARP;
    constexpr bool U = LPC > 1 || W;
    if (live || U) {
        const int64_t kk = live ? k : 0;
        const CellConst c = make_cell(a.p);
        RngSource rsrc{};
        SoaSource ssrc{};
        __shared__ double ring[2 * 3 * kRingStride];
        if (SRC == 1) rsrc = RngSource{a.stream, scenario_key(a.stream, (uint64_t)(a.k0 + kk))};
        if (SRC == 2) ssrc = SoaSource{a.soa + kk, a.ld, ring + threadIdx.x};
        double klo = 0.0, khi = 1.0;
        kopt = 0.0;
        found = 0;
        // With LPC > 1 the rollouts shuffle across the whole warp, so every
        // lane walks every candidate; finished or gated-out cells pass
        // live = false and only keep the warp company.
        bool fin = !live;
        for (int it = -1; it < a.n_kappa; ++it) {
            if (!U) {
                if (fin) break;
            } else if (__all_sync(0xffffffffu, fin)) {
                break;
            }
            const double kappa = it < 0 ? 1.0 : mul(0.5, add(klo, khi));
            const double v = update_setpoint(a.v_prev, a.r, kappa);
            const bool run = !fin && ss_gate(v, a.p);
            bool ok = false;
            int32_t sr = 0;
            if (run || U) {
                int st;
                if (SRC == 1)
                    st = rollout<FMA, false, LPC, RngSource, W>(c, a.x0[0], a.x0[1], a.x0[2], v,
                                                                rsrc, sr, nullptr, run);
                else if (SRC == 2)
                    st = rollout<FMA, false, LPC, SoaSource, W>(c, a.x0[0], a.x0[1], a.x0[2], v,
                                                                ssrc, sr, nullptr, run);
                else
                    st = rollout<FMA, false, LPC, ZeroSource, W>(c, a.x0[0], a.x0[1], a.x0[2],
                                                                 v, ZeroSource{}, sr, nullptr,
                                                                 run);
                ok = run && st == kOk;
                if (!run) sr = 0;
            }
            if (fin) continue;
            if (a.path_kappa && lead) {
                a.path_kappa[k * (a.n_kappa + 1) + cells] = kappa;
                a.path_ok[k * (a.n_kappa + 1) + cells] = ok ? 1 : 0;
            }
            cells += 1;
            if (sr < a.p.j_star && !ok) early += 1;
            if (it < 0) {
                if (ok) {
                    kopt = 1.0;
                    found = 1;
                    fin = true;
                }
                continue;
            }
            if (ok) {
                kopt = kappa;
                found = 1;
                klo = kappa;
            } else {
                khi = kappa;
            }
        }
        if (a.kappa_k && live && lead) {
            a.kappa_k[k] = kopt;
            a.found_k[k] = found;
            a.cells_k[k] = cells;
            a.early_k[k] = early;
        }
        if (!(live && lead)) {  // neutral elements of the reductions
            kopt = 1.0;
            found = 1;
            cells = 0;
            early = 0;
        }
    }
    // reductions: min kappa (non-negative doubles order like their bits), AND found,
    // sums of cells and early terminations
    unsigned long long kb = (unsigned long long)__double_as_longlong(kopt);
    int all_found = found;
    long long sc = cells, se = early;
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long ob = __shfl_down_sync(0xffffffffu, kb, off);
        kb = ob < kb ? ob : kb;
        all_found &= __shfl_down_sync(0xffffffffu, all_found, off);
        sc += __shfl_down_sync(0xffffffffu, sc, off);
        se += __shfl_down_sync(0xffffffffu, se, off);
    }
    if (lane_id() == 0) {
        atomicMin(&a.acc->kappa_bits, kb);
        if (!all_found) atomicAnd(&a.acc->found, 0);
        atomicAdd(&a.acc->cells, (unsigned long long)sc);
        atomicAdd(&a.acc->early, (unsigned long long)se);
    }
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&a.acc->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    __threadfence();
    volatile BisectAcc* acc = a.acc;
    a.out->kappa = __longlong_as_double((long long)acc->kappa_bits);
    a.out->found = acc->found;
    a.out->cells = (long long)acc->cells;
    a.out->early = (long long)acc->early;
    a.out->seq += 1;
    acc->kappa_bits = 0x3ff0000000000000ull;  // 1.0
    acc->found = 1;
    acc->cells = 0ull;
    acc->early = 0ull;
    acc->ticket = 0u;
}

// ---------------------------------------------------------------------------
// linear plant: parity fill and exact Alg. 2
// ---------------------------------------------------------------------------

__global__ void k_gen_soa_w(uint64_t hs, double4 lo4, double4 span4, int width, int64_t k0,
                            int64_t n_sim, int32_t j_star, int64_t ld, double* __restrict__ dst) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t j = blockIdx.y;
    if (k >= n_sim || j >= j_star) return;
    const double lo[4] = {lo4.x, lo4.y, lo4.z, lo4.w};
    const double span[4] = {span4.x, span4.y, span4.z, span4.w};
    const uint64_t K = splitmix64(hs ^ (uint64_t)(k0 + k));
    const uint64_t J = splitmix64(K ^ (uint64_t)j);
    for (int i = 0; i < width; ++i)
        dst[((int64_t)j * width + i) * ld + k] =
            add(lo[i], mul(span[i], unit_double(splitmix64(J ^ (uint64_t)i))));
}

template <int N>
__device__ __forceinline__ int lin_cell(const LinArgs& a, const CellConst& c, int64_t k, double v,
                                        int32_t& steps) {
    if (a.soa) {
        LinSoaSource<N> src{a.soa + k, a.ld};
        return rollout_lin<N, false>(a.L, c, a.x0, v, src, steps);
    }
    LinRngSource<N> src;
    src.K = splitmix64(a.hs ^ (uint64_t)(a.k0 + k));
    for (int i = 0; i < 4; ++i) {
        src.lo[i] = a.lo[i];
        src.span[i] = a.span[i];
    }
    return rollout_lin<N, true>(a.L, c, a.x0, v, src, steps);
}

template <int N>
__global__ void __launch_bounds__(128) k_fill_lin(LinArgs a) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.n_sim) return;
    const int32_t row = a.rows[blockIdx.y];
    int32_t steps = 0;
    const int st = lin_cell<N>(a, make_cell(a.p), k, a.v_rows[row], steps);
    a.S[(int64_t)row * a.n_sim + k] = (uint8_t)st;
    a.steps[(int64_t)row * a.n_sim + k] = steps;
}

template <int N>
__global__ void __launch_bounds__(128) k_bisect_lin(LinArgs a) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = k < a.n_sim;
    double kopt = 1.0;
    int found = 1, cells = 0, early = 0;
    if (live) {
        const CellConst c = make_cell(a.p);
        double klo = 0.0, khi = 1.0;
        kopt = 0.0;
        found = 0;
        for (int it = -1; it < a.n_kappa; ++it) {
            const double kappa = it < 0 ? 1.0 : mul(0.5, add(klo, khi));
            const double v = update_setpoint(a.v_prev, a.r, kappa);
            bool ok = false;
            int32_t sr = 0;
            const double yss = mul(a.L.gain, v);  // LinearOraclePlant.steady_state_output
            if (a.L.tlo <= yss && yss <= a.L.thi) ok = lin_cell<N>(a, c, k, v, sr) == kOk;
            cells += 1;
            if (sr < a.p.j_star && !ok) early += 1;
            if (it < 0) {
                if (ok) {
                    kopt = 1.0;
                    found = 1;
                    break;
                }
                continue;
            }
            if (ok) {
                kopt = kappa;
                found = 1;
                klo = kappa;
            } else {
                khi = kappa;
            }
        }
        if (a.kappa_k) {
            a.kappa_k[k] = kopt;
            a.found_k[k] = found;
            a.cells_k[k] = cells;
            a.early_k[k] = early;
        }
    }
    unsigned long long kb = (unsigned long long)__double_as_longlong(kopt);
    int all_found = found;
    long long sc = cells, se = early;
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long ob = __shfl_down_sync(0xffffffffu, kb, off);
        kb = ob < kb ? ob : kb;
        all_found &= __shfl_down_sync(0xffffffffu, all_found, off);
        sc += __shfl_down_sync(0xffffffffu, sc, off);
        se += __shfl_down_sync(0xffffffffu, se, off);
    }
    if (lane_id() == 0) {
        atomicMin(&a.acc->kappa_bits, kb);
        if (!all_found) atomicAnd(&a.acc->found, 0);
        atomicAdd(&a.acc->cells, (unsigned long long)sc);
        atomicAdd(&a.acc->early, (unsigned long long)se);
    }
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&a.acc->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    __threadfence();
    volatile BisectAcc* acc = a.acc;
    a.out->kappa = __longlong_as_double((long long)acc->kappa_bits);
    a.out->found = acc->found;
    a.out->cells = (long long)acc->cells;
    a.out->early = (long long)acc->early;
    a.out->seq += 1;
    acc->kappa_bits = 0x3ff0000000000000ull;
    acc->found = 1;
    acc->cells = 0ull;
    acc->early = 0ull;
    acc->ticket = 0u;
}

// ---------------------------------------------------------------------------
// tanh self-test
// ---------------------------------------------------------------------------

template <bool FMA>
__global__ void k_tanh(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = tanh_glibc<FMA>(x[i]);
}

// the rollout's lockstep form (tanh4 / tanh_core), four arguments per thread
template <bool FMA>
__global__ void k_tanh4(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i >= n) return;
    double a[4], z[4];
    for (int q = 0; q < 4; ++q) a[q] = i + q < n ? x[i + q] : 0.0;
    tanh4_auto<FMA>(a[0], a[1], a[2], a[3], z[0], z[1], z[2], z[3]);
    for (int q = 0; q < 4; ++q)
        if (i + q < n) y[i + q] = z[q];
}

// FP64 issue-rate probe: independent DFMA chains (the roofline denominator)
__global__ void k_dfma_peak(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1.0, x2 = x0 + 2.0, x3 = x0 + 3.0;
    double x4 = x0 + 4.0, x5 = x0 + 5.0, x6 = x0 + 6.0, x7 = x0 + 7.0;
    for (int i = 0; i < iters; ++i) {
        x0 = __fma_rn(x0, a, b);
        x1 = __fma_rn(x1, a, b);
        x2 = __fma_rn(x2, a, b);
        x3 = __fma_rn(x3, a, b);
        x4 = __fma_rn(x4, a, b);
        x5 = __fma_rn(x5, a, b);
        x6 = __fma_rn(x6, a, b);
        x7 = __fma_rn(x7, a, b);
    }
    const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

static inline unsigned blocks_for(int64_t n, int tpb) { return (unsigned)((n + tpb - 1) / tpb); }

cudaError_t launch_sample(const SampleArgs& a, cudaStream_t s) {
    const int64_t total = a.n_sim * a.horizon;
    if (total == 0) return cudaSuccess;
    k_sample<<<blocks_for(total, 256), 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_to_soa(const double* src, double* dst, int64_t n_sim, int64_t horizon,
                          int32_t j_star, int64_t ld, cudaStream_t s) {
    dim3 grid((unsigned)((ld + 31) / 32), (unsigned)((j_star + 31) / 32));
    k_to_soa<<<grid, dim3(32, 8), 0, s>>>(src, dst, n_sim, horizon, j_star, ld);
    return cudaGetLastError();
}

#define RG_DISPATCH_LPC(LPC_VAR, MACRO)   \
    do {                                   \
        if ((LPC_VAR) == 4) MACRO(4);      \
        else if ((LPC_VAR) == 2) MACRO(2); \
        else MACRO(1);                     \
    } while (0)

cudaError_t launch_fill(const FillArgs& a, bool fma, bool rng, int lpc, cudaStream_t s) {
    if (a.n_rows == 0 || a.n_sim == 0) return cudaSuccess;
    dim3 grid(blocks_for(a.n_sim * lpc, a.tpb), (unsigned)a.n_rows);
#define RG_FILL(L)                                                         \
    do {                                                                   \
        if (fma) {                                                         \
            if (rng) k_fill<true, true, L><<<grid, a.tpb, 0, s>>>(a);      \
            else     k_fill<true, false, L><<<grid, a.tpb, 0, s>>>(a);     \
        } else {                                                           \
            if (rng) k_fill<false, true, L><<<grid, a.tpb, 0, s>>>(a);     \
            else     k_fill<false, false, L><<<grid, a.tpb, 0, s>>>(a);    \
        }                                                                  \
    } while (0)
    RG_DISPATCH_LPC(lpc, RG_FILL);
#undef RG_FILL
    return cudaGetLastError();
}

// Launch with programmatic stream serialization (PDL) when `pdl`: the grid may
// start while the previous kernel on the stream (k_gen_soa) is still running.
template <class Kern, class Args>
cudaError_t launch_ex(Kern kern, dim3 grid, int block, size_t smem, cudaStream_t s, bool pdl,
                      const Args& a) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl ? attr : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

// The single-wave placement's occupancy pin: `total` bytes of shared memory per
// block (more than half an SM's), of which the kernel's static shared memory is a
// part.  Sets *dyn to the dynamic remainder and opts the kernel in to it, once per
// kernel and device.  total <= 0: no pin (*dyn = 0).
cudaError_t pin_smem(const void* fn, int total, int* dyn) {
    *dyn = 0;
    if (total <= 0) return cudaSuccess;
    struct Entry {
        const void* fn;
        int dev, total, dyn;
    };
    static Entry tab[256];
    static int n = 0;
    static std::mutex mu;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < n; ++i)
        if (tab[i].fn == fn && tab[i].dev == dev && tab[i].total == total) {
            *dyn = tab[i].dyn;
            return cudaSuccess;
        }
    cudaFuncAttributes attr;
    if ((e = cudaFuncGetAttributes(&attr, fn)) != cudaSuccess) return e;
    const int d = total > (int)attr.sharedSizeBytes ? total - (int)attr.sharedSizeBytes : 0;
    if (d > 0 &&
        (e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, d)) !=
            cudaSuccess)
        return e;
    if (n < 256) tab[n++] = Entry{fn, dev, total, d};
    *dyn = d;
    return cudaSuccess;
}

cudaError_t launch_grid(const GridArgs& a, bool fma, bool rng, bool poll, int lpc,
                        cudaStream_t s) {
    dim3 grid(blocks_for(a.n_sim * lpc, a.tpb), (unsigned)a.m_grid);
    cudaError_t e = cudaSuccess;
#define RG_GRID_M(F, R, P, L, M, S)                                                      \
    do {                                                                                 \
        int dyn = 0;                                                                     \
        if ((e = pin_smem((const void*)k_grid<F, R, P, L, M, S>, a.smem_dyn, &dyn)) !=    \
            cudaSuccess)                                                                 \
            break;                                                                       \
        e = launch_ex(k_grid<F, R, P, L, M, S>, grid, a.tpb, (size_t)dyn, s, a.pdl != 0, \
                      a);                                                                \
    } while (0)
    // one lane per cell: above one wave (issue-bound) the operand-modifier tanh forms,
    // in one wave over a staged block (latency-bound) the two-step rollout
#define RG_GRID(F, R, P, L)                                                              \
    do {                                                                                 \
        if (L == 1 && a.smem_dyn == 0) RG_GRID_M(F, R, P, 1, true, false);               \
        else if (L == 1 && !R && a.tpb <= kRing4Stride && !a.no_s2)                      \
            RG_GRID_M(F, false, P, 1, false, true);                                      \
        else RG_GRID_M(F, R, P, L, false, false);                                        \
    } while (0)
#define RG_GRID_L(L)                                                             \
    do {                                                                         \
        if (fma) {                                                               \
            if (rng) { if (poll) RG_GRID(true, true, true, L); else RG_GRID(true, true, false, L); }   \
            else     { if (poll) RG_GRID(true, false, true, L); else RG_GRID(true, false, false, L); } \
        } else {                                                                 \
            if (rng) { if (poll) RG_GRID(false, true, true, L); else RG_GRID(false, true, false, L); } \
            else     { if (poll) RG_GRID(false, false, true, L); else RG_GRID(false, false, false, L); } \
        }                                                                        \
    } while (0)
    RG_DISPATCH_LPC(lpc, RG_GRID_L);
#undef RG_GRID_L
#undef RG_GRID
#undef RG_GRID_M
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_grid_ws(const GridArgs& a, bool fma, bool rng, bool poll, cudaStream_t s) {
    constexpr int T = RG_WS_T, W = RG_WS_W;
    dim3 grid((unsigned)((a.n_sim + 31) / 32), (unsigned)a.m_grid);
#define RG_WS(F, R, P) k_grid_ws<F, R, P, T, W><<<grid, 32 * (1 + W), 0, s>>>(a)
    if (fma) {
        if (rng) { if (poll) RG_WS(true, true, true); else RG_WS(true, true, false); }
        else     { if (poll) RG_WS(true, false, true); else RG_WS(true, false, false); }
    } else {
        if (rng) { if (poll) RG_WS(false, true, true); else RG_WS(false, true, false); }
        else     { if (poll) RG_WS(false, false, true); else RG_WS(false, false, false); }
    }
#undef RG_WS
    return cudaGetLastError();
}

cudaError_t launch_grid_dec(const GridArgs& a, bool fma, bool rng, bool poll, cudaStream_t s) {
    constexpr int C = RG_DEC_C, T = RG_DEC_T, TB = RG_DEC_TB;
    dim3 grid((unsigned)((a.n_sim + C - 1) / C), (unsigned)a.m_grid);
#define RG_DEC(F, R, P) k_grid_dec<F, R, P, C, T, TB><<<grid, TB, 0, s>>>(a)
    if (fma) {
        if (rng) { if (poll) RG_DEC(true, true, true); else RG_DEC(true, true, false); }
        else     { if (poll) RG_DEC(true, false, true); else RG_DEC(true, false, false); }
    } else {
        if (rng) { if (poll) RG_DEC(false, true, true); else RG_DEC(false, true, false); }
        else     { if (poll) RG_DEC(false, false, true); else RG_DEC(false, false, false); }
    }
#undef RG_DEC
    return cudaGetLastError();
}

cudaError_t launch_grid_batch(const BatchArgs& a, bool fma, bool poll, int lpc, cudaStream_t s) {
    dim3 grid(blocks_for(a.n_sim * lpc, a.tpb), (unsigned)a.m_grid, (unsigned)a.n_ep);
#define RG_BATCH(L)                                                              \
    do {                                                                         \
        if (fma) {                                                               \
            if (poll) k_grid_batch<true, true, L><<<grid, a.tpb, 0, s>>>(a);     \
            else      k_grid_batch<true, false, L><<<grid, a.tpb, 0, s>>>(a);    \
        } else {                                                                 \
            if (poll) k_grid_batch<false, true, L><<<grid, a.tpb, 0, s>>>(a);    \
            else      k_grid_batch<false, false, L><<<grid, a.tpb, 0, s>>>(a);   \
        }                                                                        \
    } while (0)
    if (a.soa) {  // staged episodes: one lane per cell only
        if (fma) {
            if (poll) k_grid_batch<true, true, 1, true><<<grid, a.tpb, 0, s>>>(a);
            else      k_grid_batch<true, false, 1, true><<<grid, a.tpb, 0, s>>>(a);
        } else {
            if (poll) k_grid_batch<false, true, 1, true><<<grid, a.tpb, 0, s>>>(a);
            else      k_grid_batch<false, false, 1, true><<<grid, a.tpb, 0, s>>>(a);
        }
        return cudaGetLastError();
    }
    RG_DISPATCH_LPC(lpc, RG_BATCH);
#undef RG_BATCH
    return cudaGetLastError();
}

cudaError_t launch_gen_soa_batch(const uint64_t* hs, const double* lo, const double* span,
                                 int64_t k0, int64_t n_sim, int32_t j_star, int64_t ld,
                                 int32_t n_ep, int64_t ep_stride, double* dst, cudaStream_t s) {
    dim3 grid(blocks_for(n_sim, 128), (unsigned)j_star, (unsigned)n_ep);
    k_gen_soa_batch<<<grid, 128, 0, s>>>(hs, make_double3(lo[0], lo[1], lo[2]),
                                          make_double3(span[0], span[1], span[2]), k0, n_sim,
                                          j_star, ld, ep_stride, dst);
    return cudaGetLastError();
}

cudaError_t launch_joint_roll(const JointArgs& a, int it, bool fma, int src, cudaStream_t s) {
    const unsigned blocks = (unsigned)((a.n_sim + a.tpb - 1) / a.tpb);
    cudaError_t e = cudaSuccess;
#define RG_J(F, S)                                                                      \
    do {                                                                                \
        int dyn = 0;                                                                    \
        if ((e = pin_smem((const void*)k_joint_roll<F, S>, a.smem_dyn, &dyn)) != cudaSuccess) \
            return e;                                                                   \
        k_joint_roll<F, S><<<blocks, a.tpb, (size_t)dyn, s>>>(a, it);                   \
    } while (0)
    if (fma) {
        if (src == 1) RG_J(true, 1); else if (src == 2) RG_J(true, 2); else RG_J(true, 0);
    } else {
        if (src == 1) RG_J(false, 1); else if (src == 2) RG_J(false, 2); else RG_J(false, 0);
    }
#undef RG_J
    return cudaGetLastError();
}

cudaError_t launch_joint_decide(const JointArgs& a, int it, cudaStream_t s) {
    k_joint_decide<<<1, 1, 0, s>>>(a, it);
    return cudaGetLastError();
}

cudaError_t launch_bisect(const BisectArgs& a, bool fma, int src, int lpc, cudaStream_t s) {
    const unsigned g = blocks_for(a.n_sim * lpc, a.tpb);
    cudaError_t e = cudaSuccess;
#define RG_BIS(F, S, L)                                                                 \
    do {                                                                                \
        int dyn = 0;                                                                    \
        if ((e = pin_smem((const void*)k_bisect<F, S, L>, a.smem_dyn, &dyn)) != cudaSuccess) \
            return e;                                                                   \
        k_bisect<F, S, L><<<g, a.tpb, (size_t)dyn, s>>>(a);                             \
    } while (0)
#define RG_BIS_L(L)                                                              \
    do {                                                                         \
        if (fma) {                                                               \
            if (src == 0) RG_BIS(true, 0, L); else if (src == 1) RG_BIS(true, 1, L); else RG_BIS(true, 2, L);    \
        } else {                                                                 \
            if (src == 0) RG_BIS(false, 0, L); else if (src == 1) RG_BIS(false, 1, L); else RG_BIS(false, 2, L); \
        }                                                                        \
    } while (0)
    RG_DISPATCH_LPC(lpc, RG_BIS_L);
#undef RG_BIS_L
#undef RG_BIS
    return cudaGetLastError();
}

cudaError_t launch_tanh(const double* x, double* y, int64_t n, bool fma, bool lockstep,
                        cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (lockstep) {
        const unsigned g = blocks_for((n + 3) / 4, 256);
        if (fma) k_tanh4<true><<<g, 256, 0, s>>>(x, y, n);
        else     k_tanh4<false><<<g, 256, 0, s>>>(x, y, n);
    } else {
        if (fma) k_tanh<true><<<blocks_for(n, 256), 256, 0, s>>>(x, y, n);
        else     k_tanh<false><<<blocks_for(n, 256), 256, 0, s>>>(x, y, n);
    }
    return cudaGetLastError();
}

cudaError_t launch_fill_lin(const LinArgs& a, cudaStream_t s) {
    if (a.n_rows == 0 || a.n_sim == 0) return cudaSuccess;
    dim3 grid(blocks_for(a.n_sim, a.tpb), (unsigned)a.n_rows);
    switch (a.L.n) {
        case 1: k_fill_lin<1><<<grid, a.tpb, 0, s>>>(a); break;
        case 2: k_fill_lin<2><<<grid, a.tpb, 0, s>>>(a); break;
        case 3: k_fill_lin<3><<<grid, a.tpb, 0, s>>>(a); break;
        default: k_fill_lin<4><<<grid, a.tpb, 0, s>>>(a); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_bisect_lin(const LinArgs& a, cudaStream_t s) {
    const unsigned g = blocks_for(a.n_sim, a.tpb);
    switch (a.L.n) {
        case 1: k_bisect_lin<1><<<g, a.tpb, 0, s>>>(a); break;
        case 2: k_bisect_lin<2><<<g, a.tpb, 0, s>>>(a); break;
        case 3: k_bisect_lin<3><<<g, a.tpb, 0, s>>>(a); break;
        default: k_bisect_lin<4><<<g, a.tpb, 0, s>>>(a); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_gen_soa_w(uint64_t hs, const double* lo, const double* span, int width,
                             int64_t k0, int64_t n_sim, int32_t j_star, int64_t ld, double* dst,
                             cudaStream_t s) {
    double4 l4 = make_double4(lo[0], width > 1 ? lo[1] : 0, width > 2 ? lo[2] : 0,
                              width > 3 ? lo[3] : 0);
    double4 s4 = make_double4(span[0], width > 1 ? span[1] : 0, width > 2 ? span[2] : 0,
                              width > 3 ? span[3] : 0);
    dim3 grid(blocks_for(n_sim, 128), (unsigned)j_star);
    k_gen_soa_w<<<grid, 128, 0, s>>>(hs, l4, s4, width, k0, n_sim, j_star, ld, dst);
    return cudaGetLastError();
}

cudaError_t launch_gen_soa(const ScenarioStream& st, int64_t k0, int64_t n_sim, int32_t j_star,
                           int64_t ld, double* dst, cudaStream_t s) {
    dim3 grid(blocks_for(n_sim, 128), (unsigned)j_star);
    k_gen_soa<<<grid, 128, 0, s>>>(st, k0, n_sim, j_star, ld, dst);
    return cudaGetLastError();
}

cudaError_t launch_dfma_peak(double* out, int blocks, int threads, int iters, cudaStream_t s) {
    k_dfma_peak<<<blocks, threads, 0, s>>>(out, iters, 0.999999, 1e-7);
    return cudaGetLastError();
}

}  // namespace rg
