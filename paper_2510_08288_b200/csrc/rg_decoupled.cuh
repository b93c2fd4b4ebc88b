// rg_decoupled.cuh -- phase-decoupled rollout of the surrogate plant.
//
// dx2/dt = -x2 + v does not involve x1 or x3, and the four tanh arguments of
// an RK4 step (x2, a2, b2, c2) depend on the x2 trajectory alone.  So a block
// advances its cells through the horizon in chunks of T steps, three phases per
// chunk:
//   1. cell threads run the x2 recurrence for T steps (13 dependent FP64 ops per
//      step) and write the 4T tanh arguments, plus x2 after every step, to
//      shared memory;
//   2. every thread of the block evaluates those tanh values in place: 4*T*C
//      independent evaluations with no chain between them -- this is where the
//      FP64 work is, and it runs at pipe throughput instead of chain latency;
//   3. cell threads run the x1/x3 recurrence for T steps with the fused
//      overflow/bound checks (exactly the reference's order per step).
// The operations, their operands and their roundings are those of sfc_step;
// only independent chains are reordered, so every bit (status, steps, the
// returned verdicts) equals the per-step rollout.  Work past an early exit is
// wasted, never observed.
#pragma once

#include "rg_cell.cuh"

namespace rg {

// C = cells per block (one warp of cell threads per 32 cells), T = steps per chunk.
template <int C, int T>
struct DecSmem {
    double arg[T][4][C];   // tanh arguments, overwritten by tanh values in phase 2
    double x2s[T][C];      // x2 after each step of the chunk (for the overflow check)
    double d[T][3][C];     // the chunk's disturbances
};

// Stage the chunk's disturbances into shared memory (all threads cooperate).
template <int C, int T, bool RNG>
__device__ __forceinline__ void dec_stage(DecSmem<C, T>& sm, int32_t c0, int32_t tc,
                                          int64_t kbase, int64_t n_sim, const double* soa,
                                          int64_t ld, const ScenarioStream& st,
                                          const uint64_t* kkey) {
    if constexpr (RNG) {
        for (int idx = threadIdx.x; idx < tc * C; idx += blockDim.x) {
            const int t = idx / C, c = idx - t * C;
            double d0 = 0.0, d1 = 0.0, d2 = 0.0;
            if (kbase + c < n_sim) disturbance_at(st, kkey[c], (uint64_t)(c0 + t), d0, d1, d2);
            sm.d[t][0][c] = d0;
            sm.d[t][1][c] = d1;
            sm.d[t][2][c] = d2;
        }
    } else {
        for (int idx = threadIdx.x; idx < tc * 3 * C; idx += blockDim.x) {
            const int c = idx % C, ti = idx / C;  // ti = t*3 + i
            const int64_t k = kbase + c;
            sm.d[0][0][ti * C + c] =
                k < n_sim ? __ldg(soa + ((int64_t)(c0 + ti / 3) * 3 + ti % 3) * ld + k) : 0.0;
        }
    }
}

// Phase 2: tanh of every staged argument, in place, by all threads of the block.
template <bool FMA, int C, int T>
__device__ __forceinline__ void dec_tanh(DecSmem<C, T>& sm, int tc) {
    double* a = &sm.arg[0][0][0];
    const int n = tc * 4 * C;
    for (int base = threadIdx.x; base < n; base += 2 * blockDim.x) {
        const int i1 = base + blockDim.x;
        const double in[2] = {a[base], i1 < n ? a[i1] : 0.5};
        double out[2];
        tanh_lockstep<FMA, 2>(in, out);
        a[base] = out[0];
        if (i1 < n) a[i1] = out[1];
    }
}

// Rollout of C cells of one candidate setpoint v.  Cell threads are
// threadIdx.x < C (cell c = scenario kbase + c); all threads must call it.
// Returns, in the cell threads, status and steps like rollout().
template <bool FMA, bool POLL, bool RNG, int C, int T>
__device__ __forceinline__ void rollout_decoupled(DecSmem<C, T>& sm, const CellConst& p, double x1,
                                                  double x2, double x3, double v, int64_t kbase,
                                                  int64_t n_sim, const double* soa, int64_t ld,
                                                  const ScenarioStream& st,
                                                  const uint64_t* kkey, const unsigned* dead,
                                                  int& status, int32_t& steps) {
    const int c = threadIdx.x;
    const bool cell_thread = c < C;
    const bool live = cell_thread && kbase + c < n_sim;
    const int32_t J = p.j_star;
    status = kOk;
    steps = J;
    bool done = !live;
    if (live && !in_bounds(x1, p.ylo, p.yhi)) {
        status = kViolated;
        steps = 0;
        done = true;
    }
    for (int32_t c0 = 0; c0 < J; c0 += T) {
        if (__syncthreads_and(done || !cell_thread)) break;  // every cell finished
        const int tc = J - c0 < T ? J - c0 : T;
        dec_stage<C, T, RNG>(sm, c0, tc, kbase, n_sim, soa, ld, st, kkey);
        __syncthreads();
        // phase 1: x2 chain
        if (cell_thread && !done) {
            double y2 = x2;
            for (int t = 0; t < tc; ++t) {
                const X2Stage s2 = x2_stage<FMA>(y2, v, p);
                sm.arg[t][0][c] = y2;
                sm.arg[t][1][c] = s2.a2;
                sm.arg[t][2][c] = s2.b2;
                sm.arg[t][3][c] = s2.c2;
                y2 = add(add(y2, mul(p.c, s2.s2)), sm.d[t][1][c]);
                sm.x2s[t][c] = y2;
            }
            x2 = y2;
        }
        __syncthreads();
        // phase 2: the chunk's tanh values
        dec_tanh<FMA, C, T>(sm, tc);
        __syncthreads();
        // phase 3: x1/x3 chain with the fused checks, per step in the reference's order
        if (cell_thread && !done) {
            for (int t = 0; t < tc; ++t) {
                const int32_t j = c0 + t;
                x13_update<FMA>(x1, x3, sm.arg[t][0][c], sm.arg[t][1][c], sm.arg[t][2][c],
                                sm.arg[t][3][c], p, sm.d[t][0][c], sm.d[t][2][c]);
                const double x2j = sm.x2s[t][c];
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
    }
}

}  // namespace rg
