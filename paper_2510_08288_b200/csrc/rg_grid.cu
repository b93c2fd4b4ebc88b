// rg_grid.cu -- the fused robust grid step (governor.py:245-377, 520-579):
//   k_grid   steady-state gate + dedup per row, rollout with fused RNG or staged
//            SoA, warp-ballot feasibility reduction into per-row counters,
//            optional P bitmask, last-block extraction of the best row
// Layout: one thread per (row, scenario) cell, scenarios on the fast axis so a
// warp is 32 consecutive scenarios of one candidate setpoint: their
// trajectories stay close, so the data-dependent branches of tanh/expm1 and
// the early exits mostly agree across the warp.
#include "rg_common.cuh"

namespace rg {

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
__device__ __forceinline__ void grid_clock_start(const GridArgs& a) {
    if (a.t0) atomicMin(a.t0, global_ns());
}


// The finalizing block of a fused-exchange step (RG_XCHG, m_grid <= kXMaxRows): this shard's
// per-row words (a gated-out row -1, else the shard's violating-scenario count; duplicates
// carry their source's) go to every rank's window over NVLink, then this rank waits for
// every rank's words of the same epoch in its own window and extracts the row from the MAX
// (0 exactly for the rows feasible on every shard), as the NCCL path does after its
// all-reduce.  The stats stay this shard's.  A peer missing for xtimeout_ns marks the step
// failed instead of hanging the GPU.
__device__ __forceinline__ void grid_finalize_xchg(const GridArgs& a, unsigned long long t_fin) {
    __shared__ int s_w[kXMaxRows];
    __shared__ int s_src[kXMaxRows];
    __shared__ bool s_fail;
    const int M = a.m_grid;
    const int par = (int)(a.xepoch & 1ull);
    if (threadIdx.x < M) {
        const int q = threadIdx.x;
        const int sq = a.listed ? a.src_tab[q] : ((volatile int*)a.row_src)[q];
        const unsigned vq = ((volatile unsigned*)a.viol)[sq >= 0 ? sq : q];
        s_src[q] = sq;
        s_w[q] = sq == -2 ? -1 : (int)min(vq, 0x7fffffffu);
    }
    if (threadIdx.x == 0) s_fail = false;
    __syncthreads();
    // this shard's words into every rank's window (peer stores over NVLink)
    for (int t = threadIdx.x; t < a.xworld * M; t += blockDim.x) {
        const int r = t / M, q = t - r * M;
        a.xpeers[r]->words[par][a.xrank][q] = s_w[q];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x < a.xworld)
        st_release_sys(&a.xpeers[threadIdx.x]->flag[par][a.xrank], a.xepoch);
    // every rank's words of this epoch in our window
    if (threadIdx.x < a.xworld) {
        const unsigned long long* f = &a.xlocal->flag[par][threadIdx.x];
        const unsigned long long t0 = global_ns();
        while (ld_acquire_sys(f) < a.xepoch) {
            if (global_ns() - t0 > a.xtimeout_ns) {
                s_fail = true;
                break;
            }
            __nanosleep(100);
        }
    }
    __syncthreads();
    if (threadIdx.x < M) {
        int g = -1;
        for (int r = 0; r < a.xworld; ++r)
            g = max(g, ((volatile int*)a.xlocal->words[par][r])[threadIdx.x]);
        s_w[threadIdx.x] = g;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int best = -1, n_active = 0, pruned = 0, dup = 0;
        unsigned long long early = 0, ovf = 0, aband = 0;
        bool open = true;
        for (int q = 0; q < M; ++q) {
            const int sq = s_src[q];
            const bool full = sq != -2 && s_w[q] == 0;
            a.viol_out[q] = (unsigned)s_w[q];
            n_active += sq == -1;
            pruned += sq == -2;
            dup += sq >= 0;
            if (sq == -1) {
                early += ((volatile unsigned long long*)a.early)[q];
                ovf += ((volatile unsigned long long*)a.ovf)[q];
                aband += ((volatile unsigned long long*)a.abandoned)[q];
            }
            if (a.prefix_mode) {
                if (open && full) best = q;
                open = open && full;
            } else if (full) {
                best = q;
            }
        }
        a.out->row = best;
        a.out->n_active = n_active;
        a.out->ss_pruned_rows = pruned;
        a.out->dedup_rows = dup;
        a.out->early_terms = (long long)early;
        a.out->overflows = (long long)ovf;
        a.out->abandoned = (long long)aband;
        a.out->sims_run = (long long)n_active * a.n_sim;
        a.out->xchg_failed = s_fail ? 1 : 0;
        if (a.t0) {
            const unsigned long long now = global_ns();
            a.out->kernel_ns = now - *(volatile unsigned long long*)a.t0;
            a.out->reduce_ns = now - t_fin;
            *a.t0 = ~0ull;
        }
        __threadfence_system();
        *(volatile unsigned long long*)&a.out->seq = a.seq_token;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < M; q += blockDim.x) {
        a.viol[q] = 0u;
        a.early[q] = 0ull;
        a.ovf[q] = 0ull;
        a.abandoned[q] = 0ull;
    }
    if (threadIdx.x == 0) *a.ticket = 0u;
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
    if (a.xchg) {
        grid_finalize_xchg(a, s_tfin);
        return;
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
                sq = a.listed ? a.src_tab[q] : ((volatile int*)a.row_src)[q];
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
            a.out->xchg_failed = 0;
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
template <bool FMA, bool RNG, bool POLL, bool MOD = false, bool S2 = false>
__global__ void __launch_bounds__(256, RG_GRID_MINB) k_grid(GridArgs a) {
    __shared__ int s_src;
    __shared__ double s_v;
    const int i = a.listed ? a.row_list[blockIdx.y] : (int)blockIdx.y;
    if (threadIdx.x < 32) {
        double v;
        int src;
        if (a.listed) {  // a simulated row of the host's plan: its setpoint, as row_source
            v = update_setpoint(a.v_prev, a.r, dvd((double)i, (double)(a.m_grid - 1)));
            src = -1;
        } else {
            src = row_source_warp(a, i, &v);
        }
        if (threadIdx.x == 0) {
            grid_clock_start(a);
            s_src = src;
            s_v = v;
            if (blockIdx.x == 0) a.row_src[i] = src;
        }
    }
    __syncthreads();
    if (S2 && a.gen) {
        // the generator fused in: this block's share of the scenario block (consecutive
        // threads take consecutive scenarios: coalesced stores), then every block waits
        // for every share
        const int64_t total = a.n_sim * a.p.j_star;
        const int64_t nth = (int64_t)gridDim.x * gridDim.y * blockDim.x;
        int64_t idx = ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
        for (; idx < total; idx += nth) {
            const int64_t j = idx / a.n_sim;
            const int64_t kq = idx - j * a.n_sim;
            const uint64_t K = scenario_key(a.stream, (uint64_t)(a.k0 + kq));
            double d0, d1, d2;
            disturbance_at(a.stream, K, (uint64_t)j, d0, d1, d2);
            double* o = a.soa_w + j * 3 * a.ld + kq;
            o[0] = d0;
            o[a.ld] = d1;
            o[2 * a.ld] = d2;
        }
        grid_barrier(a.bar, a.bar + 1, gridDim.x * gridDim.y);
    } else {
        // staged scenarios: the generator launched just before may still be running
        // (programmatic dependent launch); no-op otherwise
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    const int src_i = s_src;
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (src_i == -1) {
        const bool live = k < a.n_sim;
        const int64_t kk = live ? k : 0;
        int st = kOk;
        int32_t steps = a.p.j_star;
        if constexpr (S2) {
            static_assert(!RNG, "the two-step rollout reads a staged block");
            __shared__ double ring4[4 * 3 * kRing4Stride];
            Soa4Source src;
            src.d = a.soa + kk;
            src.ld = a.ld;
            src.ring = ring4 + threadIdx.x;
            st = rollout2<FMA, POLL>(make_cell(a.p), a.x0[0], a.x0[1], a.x0[2], s_v, src, steps,
                                     a.viol + i, live);
        } else {  // whole warps run the rollout
            const CellConst c = make_cell(a.p);
            if (RNG) {
                RngSource src{a.stream, scenario_key(a.stream, (uint64_t)(a.k0 + kk))};
                st = rollout<FMA, POLL, RngSource, true, false, MOD>(c, a.x0[0], a.x0[1], a.x0[2],
                                                                     s_v, src, steps, a.viol + i,
                                                                     live);
            } else {
                __shared__ double ring[2 * 3 * kRingStride];
                SoaSource src{a.soa + kk, a.ld, ring + threadIdx.x};
                st = rollout<FMA, POLL, SoaSource, true, false, MOD>(c, a.x0[0], a.x0[1], a.x0[2],
                                                                     s_v, src, steps, a.viol + i,
                                                                     live);
            }
        }
        const bool cnt = live;
        const bool bad = cnt && st != kOk && st != kAbandoned;
        const unsigned bad_mask = __ballot_sync(0xffffffffu, bad);
        if (lane_id() == 0 && bad_mask) atomicAdd(a.viol + i, (unsigned)__popc(bad_mask));
        warp_count_add(cnt && st != kAbandoned && steps < a.p.j_star, a.early + i);
        warp_count_add(cnt && st == kOverflow, a.ovf + i);
        warp_count_add(cnt && st == kAbandoned, a.abandoned + i);
        if (a.pbits) {
            const unsigned ok_mask = __ballot_sync(0xffffffffu, live && st == kOk);
            if (lane_id() == 0 && (k - lane_id()) < a.n_sim)
                a.pbits[(int64_t)i * a.pwords + (k >> 5)] = ok_mask;
        }
    } else if (a.pbits && lane_id() == 0 && (k - lane_id()) < a.n_sim) {
        // pruned or duplicate row: no simulated bits (the host expands duplicates)
        a.pbits[(int64_t)i * a.pwords + (k >> 5)] = 0u;
    }
    grid_finalize(a);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

cudaError_t launch_grid(const GridArgs& a, bool fma, bool rng, bool poll, cudaStream_t s) {
    dim3 grid(blocks_for(a.n_sim, a.tpb), (unsigned)(a.listed ? a.list_n : a.m_grid));
    // the fused generator exists only in the single-wave two-step form
    if (a.gen && !(a.smem_dyn != 0 && !rng && a.tpb <= kRing4Stride && !a.no_s2))
        return cudaErrorInvalidValue;
    cudaError_t e = cudaSuccess;
#define RG_GRID_M(F, R, P, M, S)                                                        \
    do {                                                                                \
        int dyn = 0;                                                                    \
        if ((e = pin_smem((const void*)k_grid<F, R, P, M, S>, a.smem_dyn, &dyn)) !=     \
            cudaSuccess)                                                                \
            break;                                                                      \
        e = launch_ex(k_grid<F, R, P, M, S>, grid, a.tpb, (size_t)dyn, s, a.pdl != 0, a, \
                      S && a.gen != 0);                                                  \
    } while (0)
    // above one wave (issue-bound) the operand-modifier tanh forms, in one wave over a
    // staged block (latency-bound) the two-step rollout
#define RG_GRID(F, R, P)                                                               \
    do {                                                                               \
        if (a.smem_dyn == 0) RG_GRID_M(F, R, P, true, false);                          \
        else if (!R && a.tpb <= kRing4Stride && !a.no_s2)                              \
            RG_GRID_M(F, false, P, false, true);                                       \
        else RG_GRID_M(F, R, P, false, false);                                         \
    } while (0)
    if (fma) {
        if (rng) { if (poll) RG_GRID(true, true, true); else RG_GRID(true, true, false); }
        else     { if (poll) RG_GRID(true, false, true); else RG_GRID(true, false, false); }
    } else {
        if (rng) { if (poll) RG_GRID(false, true, true); else RG_GRID(false, true, false); }
        else     { if (poll) RG_GRID(false, false, true); else RG_GRID(false, false, false); }
    }
#undef RG_GRID
#undef RG_GRID_M
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace rg
