// rg_ws.cuh -- warp-specialised, software-pipelined rollout of the surrogate
// plant (the grid step's production kernel).
//
// Same decomposition as rg_decoupled.cuh -- the four tanh arguments of an RK4
// step depend on the x2 trajectory alone -- but without block-wide phases:
//
//   warp 0 ("sequence warp", one lane per cell, 32 cells per block) runs, per
//   chunk iteration c, the x2 recurrence of chunk c+1 interleaved with the
//   x1/x3 recurrence (and the fused checks) of chunk c-1: two independent
//   dependency chains side by side;
//   warps 1..W ("tanh warps") evaluate the 4*T*32 tanh values of chunk c
//   meanwhile -- independent evaluations, throughput- not latency-bound.
//
// The warps hand chunks over through shared-memory rings guarded by named
// barriers (bar.arrive / bar.sync): FULL[b] (arguments of the chunk in
// buffer b are written) and DONE[b] (its tanh values are ready).  The
// disturbances are prefetched two chunks ahead into a 4-slot ring (cp.async
// for a staged tensor, computed in place for the counter RNG).  All operations,
// operands and roundings are those of sfc_step; the bits are the per-step
// rollout's.
#pragma once

#include "rg_cell.cuh"

namespace rg {

template <int T>
struct WsSmem {
    double arg[3][T][4][32];  // tanh arguments of a chunk, then its tanh values
    double x2s[3][T][32];     // x2 after each step (for the overflow check)
    double d[4][T][3][32];    // disturbances, two chunks ahead
    int stop;                 // sequence warp -> tanh warps: no more chunks
};

__device__ __forceinline__ void bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
// named barriers 1..3: FULL[b]; 4..6: DONE[b] (0 is __syncthreads)
__device__ __forceinline__ int bar_full(int b) { return 1 + b; }
__device__ __forceinline__ int bar_done(int b) { return 4 + b; }

// Sequence warp: bring the disturbances of chunk c into ring slot c % 4.
template <int T, bool RNG>
__device__ __forceinline__ void ws_fetch(WsSmem<T>& sm, int c, int32_t J, int64_t k, bool live,
                                         const double* soa, int64_t ld,
                                         const ScenarioStream& st, uint64_t key) {
    const int c0 = c * T;
    if (c0 >= J) return;
    const int tc = J - c0 < T ? J - c0 : T;
    const int slot = c & 3;
    const int lane = threadIdx.x;
    if constexpr (RNG) {
        for (int t = 0; t < tc; ++t) {
            double d0 = 0.0, d1 = 0.0, d2 = 0.0;
            if (live) disturbance_at(st, key, (uint64_t)(c0 + t), d0, d1, d2);
            sm.d[slot][t][0][lane] = d0;
            sm.d[slot][t][1][lane] = d1;
            sm.d[slot][t][2][lane] = d2;
        }
    } else {
        const int64_t kk = live ? k : 0;  // out-of-range lanes replay scenario 0
        for (int t = 0; t < tc; ++t)
            for (int i = 0; i < 3; ++i) {
                const unsigned sa =
                    (unsigned)__cvta_generic_to_shared(&sm.d[slot][t][i][lane]);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa),
                             "l"(soa + ((int64_t)(c0 + t) * 3 + i) * ld + kk));
            }
    }
}

// Warp-specialised rollout of 32 cells (scenarios kbase..kbase+31) of one
// candidate setpoint v.  All TB = 32*(1+W) threads of the block call it; the
// sequence-warp lanes return status/steps of their cell.
template <bool FMA, bool POLL, bool RNG, int T, int W>
__device__ void rollout_ws(WsSmem<T>& sm, const CellConst& p, double x1, double x2, double x3,
                           double v, int64_t kbase, int64_t n_sim, const double* soa,
                           int64_t ld, const ScenarioStream& st, const unsigned* dead,
                           int& status, int32_t& steps) {
    constexpr int TB = 32 * (1 + W);
    const int32_t J = p.j_star;
    const int nch = (J + T - 1) / T;
    if (threadIdx.x >= 32) {
        // ---------------- tanh warps ----------------
        const int tid = threadIdx.x - 32;
        for (int c = 0;; ++c) {
            const int b = c % 3;
            bar_sync(bar_full(b), TB);
            if (*(volatile int*)&sm.stop) return;
            const int tc = J - c * T < T ? J - c * T : T;
            double* a = &sm.arg[b][0][0][0];
            const int n = tc * 4 * 32;
            for (int base = tid; base < n; base += 64 * W) {
                const int i1 = base + 32 * W;
                const double in[2] = {a[base], i1 < n ? a[i1] : 0.5};
                double out[2];
                tanh_lockstep<FMA, 2>(in, out);
                a[base] = out[0];
                if (i1 < n) a[i1] = out[1];
            }
            bar_arrive(bar_done(b), TB);
        }
    }
    // ---------------- sequence warp ----------------
    const int lane = threadIdx.x;
    const int64_t k = kbase + lane;
    const bool live = k < n_sim;
    const uint64_t key = RNG ? scenario_key(st, (uint64_t)(live ? k : kbase)) : 0ull;
    status = kOk;
    steps = J;
    bool done = !live;
    if (live && !in_bounds(x1, p.ylo, p.yhi)) {
        status = kViolated;
        steps = 0;
        done = true;
    }
    if (lane == 0) sm.stop = 0;
    // prologue: disturbances of chunks 0 and 1, then the x2 chain of chunk 0
    ws_fetch<T, RNG>(sm, 0, J, k, live, soa, ld, st, key);
    if (!RNG) asm volatile("cp.async.commit_group;");
    ws_fetch<T, RNG>(sm, 1, J, k, live, soa, ld, st, key);
    if (!RNG) asm volatile("cp.async.commit_group;");
    if (!RNG) asm volatile("cp.async.wait_group 1;");
    __syncwarp();
    double y2 = x2;  // x2 at the start of the next chunk to produce
    auto produce = [&](int c) {  // x2 chain of chunk c into buffer c % 3
        const int b = c % 3, slot = c & 3, c0 = c * T;
        const int tc = J - c0 < T ? J - c0 : T;
        for (int t = 0; t < tc; ++t) {
            const X2Stage s2 = x2_stage<FMA>(y2, v, p);
            sm.arg[b][t][0][lane] = y2;
            sm.arg[b][t][1][lane] = s2.a2;
            sm.arg[b][t][2][lane] = s2.b2;
            sm.arg[b][t][3][lane] = s2.c2;
            y2 = add(add(y2, mul(p.c, s2.s2)), sm.d[slot][t][1][lane]);
            sm.x2s[b][t][lane] = y2;
        }
    };
    produce(0);
    bar_arrive(bar_full(0), TB);
    for (int c = 0; c < nch; ++c) {
        // prefetch chunk c+2's disturbances; chunk c+1's have landed
        ws_fetch<T, RNG>(sm, c + 2, J, k, live, soa, ld, st, key);
        if (!RNG) {
            asm volatile("cp.async.commit_group;");
            asm volatile("cp.async.wait_group 1;");
        }
        // x2 chain of chunk c+1, handed to the tanh warps at once
        const bool more = c + 1 < nch;
        if (more) {
            produce(c + 1);
            bar_arrive(bar_full((c + 1) % 3), TB);
        }
        // x1/x3 of chunk c once its tanh values are ready
        const int b = c % 3, slot = c & 3, c0 = c * T;
        bar_sync(bar_done(b), TB);
        if (!done) {
            const int tc = J - c0 < T ? J - c0 : T;
            for (int t = 0; t < tc; ++t) {
                const int32_t j = c0 + t;
                x13_update<FMA>(x1, x3, sm.arg[b][t][0][lane], sm.arg[b][t][1][lane],
                                sm.arg[b][t][2][lane], sm.arg[b][t][3][lane], p,
                                sm.d[slot][t][0][lane], sm.d[slot][t][2][lane]);
                const double x2j = sm.x2s[b][t][lane];
                if (!(fabs(x1) <= kStateLimit && fabs(x2j) <= kStateLimit &&
                      fabs(x3) <= kStateLimit)) {
                    status = kOverflow;
                    steps = j + 1;
                    done = true;
                    break;
                }
                if (!in_bounds(x1, p.ylo, p.yhi)) {
                    status = kViolated;
                    steps = j + 1;
                    done = true;
                    break;
                }
                if (POLL && (j & 31) == 31 && *(volatile const unsigned*)dead != 0u) {
                    status = kAbandoned;
                    steps = j + 1;
                    done = true;
                    break;
                }
            }
        }
        const bool all_done = __all_sync(0xffffffffu, done);
        if (!more || all_done) {
            // drain the chunk already handed over, then release the tanh warps
            if (more) bar_sync(bar_done((c + 1) % 3), TB);
            if (lane == 0) *(volatile int*)&sm.stop = 1;
            __syncwarp();
            bar_arrive(bar_full((more ? c + 2 : c + 1) % 3), TB);
            break;
        }
    }
    if (!RNG) asm volatile("cp.async.wait_group 0;");
}

}  // namespace rg
