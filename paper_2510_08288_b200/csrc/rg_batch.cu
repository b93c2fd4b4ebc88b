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
// batched grid step: E independent governor instances in one launch
// ---------------------------------------------------------------------------

// Launch bounds: at most 168 registers (3 blocks of 128 threads per SM), so the
// 64-thread blocks keep 12 warps per SM (3 per SMSP) in this always multi-wave kernel.
template <bool FMA, bool POLL, bool SOA = false>
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
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned* viol = a.viol + (int64_t)e * M;
    if (s_src == -1) {
        const bool live = k < a.n_sim;
        int st = kOk;
        int32_t steps = a.p.j_star;
        {  // whole warps run the rollout
            const double* x0 = a.x0 + 3 * (int64_t)e;
            if constexpr (SOA) {  // staged block of this episode (k_gen_soa_batch)
                __shared__ double ring[2 * 3 * kRingStride];
                SoaSource src{a.soa + (int64_t)blockIdx.z * a.ep_stride + (live ? k : 0), a.ld,
                              ring + threadIdx.x};
                st = rollout<FMA, POLL, SoaSource, true, false, true>(
                    make_cell(a.p), x0[0], x0[1], x0[2], s_v, src, steps, viol + i, live);
            } else {
                ScenarioStream ss;
                ss.hs = a.hs[e];
                for (int c = 0; c < 3; ++c) {
                    ss.lo[c] = a.lo[c];
                    ss.span[c] = a.span[c];
                }
                RngSource src{ss, scenario_key(ss, (uint64_t)(a.k0 + (live ? k : 0)))};
                st = rollout<FMA, POLL, RngSource, true, false, true>(
                    make_cell(a.p), x0[0], x0[1], x0[2], s_v, src, steps, viol + i, live);
            }
        }
        const bool cnt = live;
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
// launchers
// ---------------------------------------------------------------------------

cudaError_t launch_grid_batch(const BatchArgs& a, bool fma, bool poll, cudaStream_t s) {
    dim3 grid(blocks_for(a.n_sim, a.tpb), (unsigned)a.m_grid, (unsigned)a.n_ep);
    if (a.soa) {  // staged episode blocks
        if (fma) {
            if (poll) k_grid_batch<true, true, true><<<grid, a.tpb, 0, s>>>(a);
            else      k_grid_batch<true, false, true><<<grid, a.tpb, 0, s>>>(a);
        } else {
            if (poll) k_grid_batch<false, true, true><<<grid, a.tpb, 0, s>>>(a);
            else      k_grid_batch<false, false, true><<<grid, a.tpb, 0, s>>>(a);
        }
    } else if (fma) {
        if (poll) k_grid_batch<true, true, false><<<grid, a.tpb, 0, s>>>(a);
        else      k_grid_batch<true, false, false><<<grid, a.tpb, 0, s>>>(a);
    } else {
        if (poll) k_grid_batch<false, true, false><<<grid, a.tpb, 0, s>>>(a);
        else      k_grid_batch<false, false, false><<<grid, a.tpb, 0, s>>>(a);
    }
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
