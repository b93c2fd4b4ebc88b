// rg_batch.cu -- the batched robust grid step: E independent governor instances
// (episodes, BASELINE configs C3/C5) per launch, and their staged scenario blocks.
#include "rg_common.cuh"

namespace rg {

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

// ---------------------------------------------------------------------------
// batched grid step over the compacted (episode, row) pairs
// ---------------------------------------------------------------------------

// Launch bounds: at most 80 registers (6 blocks of 128 threads per SM; ptxas needs 80,
// no spills), so the 64-thread blocks keep up to 24 warps per SM in this always multi-wave
// kernel.  C5 per closed-loop step (scripts/ab_pairs_regs.sh): 3 blocks (154 registers)
// 179.7 ms, 4: 183.5, 5: 178.1, 6: 177.1-177.4, 8 (64 registers): 178.8 -- the FP64 pipe,
// not latency, bounds it (ncu: 69.6% busy at 3 warps per scheduler).
// The staged-block form (SOA) keeps 3 blocks: at 80 registers its ring addressing spills.
#ifndef RG_PAIRS_MINB
#define RG_PAIRS_MINB 6
#endif
template <bool FMA, bool POLL, bool SOA>
__global__ void __launch_bounds__(128, SOA ? 3 : RG_PAIRS_MINB) k_grid_pairs(BatchArgs a) {
    __shared__ bool s_last;
    const int64_t pair = a.p0 + blockIdx.x / (unsigned)a.bpr;
    const int64_t kb = blockIdx.x % (unsigned)a.bpr;
    const int e = a.pair_e[pair];
    const int i = a.pair_i[pair];
    const double v = a.pair_v[pair];
    const int M = a.m_grid;
    const int64_t k = kb * blockDim.x + threadIdx.x;
    unsigned* viol = a.viol + (int64_t)e * M;
    const bool live = k < a.n_sim;
    int st = kOk;
    int32_t steps = a.p.j_star;
    {  // whole warps run the rollout
        const double* x0 = a.x0 + 3 * (int64_t)e;
        if constexpr (SOA) {  // staged block of this episode (k_gen_soa_batch)
            __shared__ double ring[2 * 3 * kRingStride];
            SoaSource src{a.soa + (int64_t)(e - a.e0) * a.ep_stride + (live ? k : 0), a.ld,
                          ring + threadIdx.x};
            st = rollout<FMA, POLL, SoaSource, true, false, true>(
                make_cell(a.p), x0[0], x0[1], x0[2], v, src, steps, viol + i, live);
        } else {
            ScenarioStream ss;
            ss.hs = a.hs[e];
            for (int c = 0; c < 3; ++c) {
                ss.lo[c] = a.lo[c];
                ss.span[c] = a.span[c];
            }
            RngSource src{ss, scenario_key(ss, (uint64_t)(a.k0 + (live ? k : 0)))};
            st = rollout<FMA, POLL, RngSource, true, false, true>(
                make_cell(a.p), x0[0], x0[1], x0[2], v, src, steps, viol + i, live);
        }
    }
    const unsigned bad = __ballot_sync(0xffffffffu, live && st != kOk && st != kAbandoned);
    if (lane_id() == 0 && bad) atomicAdd(viol + i, (unsigned)__popc(bad));
    warp_count_add(live && st != kAbandoned && steps < a.p.j_star, a.early + e);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(a.ticket + e, 1u) == a.expect[e] - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // last block of episode e: extract its best row (governor.py:351-377), apply it
    if (threadIdx.x == 0) {
        const int* rs = a.row_src + (int64_t)e * M;
        const double vp = a.v_prev[e], rr = a.r[e];
        int best = -1;
        for (int q = 0; q < M; ++q) {
            const int s = rs[q];
            const unsigned vq = s == -2 ? 0xffffffffu : ((volatile unsigned*)viol)[s < 0 ? q : s];
            const bool full = s != -2 && vq == 0u;
            if (a.viol_out) a.viol_out[(int64_t)e * M + q] = vq;
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
// launchers
// ---------------------------------------------------------------------------

cudaError_t launch_grid_batch(const BatchArgs& a, int64_t n_pairs, bool fma, bool poll,
                              cudaStream_t s) {
    if (n_pairs <= 0) return cudaSuccess;
    const int64_t blocks = n_pairs * a.bpr;
    if (blocks > 0x7fffffffll) return cudaErrorInvalidConfiguration;
    const dim3 grid((unsigned)blocks);
#define RG_PAIRS(F, P, S) k_grid_pairs<F, P, S><<<grid, a.tpb, 0, s>>>(a)
    if (a.soa) {
        if (fma) { if (poll) RG_PAIRS(true, true, true); else RG_PAIRS(true, false, true); }
        else     { if (poll) RG_PAIRS(false, true, true); else RG_PAIRS(false, false, true); }
    } else {
        if (fma) { if (poll) RG_PAIRS(true, true, false); else RG_PAIRS(true, false, false); }
        else     { if (poll) RG_PAIRS(false, true, false); else RG_PAIRS(false, false, false); }
    }
#undef RG_PAIRS
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

}  // namespace rg
