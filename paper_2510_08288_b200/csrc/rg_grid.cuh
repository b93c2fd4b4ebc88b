// rg_grid.cuh -- the grid step's shared epilogue: the device-side span clock and the
// last-block extraction (grid_finalize, with its fused-exchange form), used by k_grid
// (rg_grid.cu) and k_grid_ts (rg_ts.cu).  Internal to the library.
#pragma once

#include "rg_common.cuh"

namespace rg {

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

// A host-planned step (listed) launches only the simulated rows; with P requested the
// gated-out and duplicate rows' words must still read zero (the host expands duplicates from
// their source rows).  Every block zeroes a grid-strided share of them before finalizing.
__device__ __forceinline__ void zero_unlisted_pbits(const GridArgs& a) {
    if (!a.listed || !a.pbits) return;
    const int64_t nth = (int64_t)gridDim.x * gridDim.y * blockDim.x;
    const int64_t t0 = ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
    for (int q = 0; q < a.m_grid; ++q) {
        if (a.src_tab[q] == -1) continue;
        for (int64_t w = t0; w < a.pwords; w += nth) a.pbits[(int64_t)q * a.pwords + w] = 0u;
    }
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

}  // namespace rg
