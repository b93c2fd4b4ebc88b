// rg_grid.cu -- the fused robust grid step (governor.py:245-377, 520-579):
//   k_grid   steady-state gate + dedup per row, rollout with fused RNG or staged
//            SoA, warp-ballot feasibility reduction into per-row counters,
//            optional P bitmask, last-block extraction of the best row
// Layout: one thread per (row, scenario) cell, scenarios on the fast axis so a
// warp is 32 consecutive scenarios of one candidate setpoint: their
// trajectories stay close, so the data-dependent branches of tanh/expm1 and
// the early exits mostly agree across the warp.
#include "rg_grid.cuh"

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

// MOD: the tanh forms' operand-modifier variant (rg_math.cuh), for the
// issue-bound multi-wave steps; the single-wave (latency-bound) step keeps MOD off.
// S2: the two-steps-per-iteration rollout (rollout2) for the latency-bound
// single-wave step over a staged block (blocks of at most 256 threads).
#ifndef RG_GRID_MW_MINB
#define RG_GRID_MW_MINB RG_GRID_MINB
#endif
template <bool FMA, bool RNG, bool POLL, bool MOD = false, bool S2 = false>
__global__ void __launch_bounds__(256, S2 ? RG_GRID_MINB : RG_GRID_MW_MINB) k_grid(GridArgs a) {
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
            __shared__ double ring4[kRing4Pairs * 2 * 3 * kRing4Stride];
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
    zero_unlisted_pbits(a);
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
