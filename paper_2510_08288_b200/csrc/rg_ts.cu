// rg_ts.cu -- the time-split grid step (k_grid_ts) for steps with few simulated cells.
//
// A closed-loop governor step simulates about one candidate row:
// 10k scenarios are 313 warps, half a warp per SM sub-partition, and one warp running a
// whole rollout (k_grid) is bound by the latency of its per-step chain (~790 cycles per
// RK4 step, four tanh deep).  But only the x2 recurrence (dx2/dt = -x2 + v: the tanh
// arguments) and the x1/x3 recurrences are sequential: the four tanh of every step depend
// on the x2 chain alone (rg_cell.cuh), so other warps can evaluate them, ahead of the
// x1/x3 chain that consumes them.
//
// k_grid_ts splits each cell's rollout over three kinds of warps, per block of up to
// kTsUnits units (a unit = 32 scenarios of one simulated row, one P-bit word):
//   P (one per unit)  the x2 chain: writes each step's four tanh arguments and the
//                     consumer's disturbances d0/d2 into a shared-memory chunk slot;
//   T (kTsTanhWarps)  evaluate the slot's tanh (tanhN_with, the same warp-uniform forms as
//                     the rollouts) in place, 32 lanes of one unit and step per batch;
//   C (one per unit)  the x1/x3 chain and the per-step checks, reading the slot's tanh
//                     values one step ahead; then the unit's verdicts into the per-row
//                     counters and the P bits.
// Chunks of kTsChunk steps cycle through kTsSlots slots with named barriers per slot:
// FULL_G (P -> T), FULL_T (T -> C), EMPTY (C -> P).  Every operation, operand and
// rounding is the reference's (sfc_step); only which warp performs it changes, so the
// verdicts are bit-identical to k_grid's (tests/test_gpu_kernels.py: test_time_split_*,
// and the whole 2000-step C3 golden trace runs through here).  No cell exits early: a
// finished cell's state runs on unobserved to the end, so status and step count are the
// reference's and the counters k_grid's.
//
// Measured (profiles/r02_ab_time_split.txt, r02_ts_timeline_*.txt; RG_TS_TIMELINE build):
// a one-row step is 0.054 ms at 1k scenarios (k_grid 0.099) and 0.099 ms at 10k (0.120);
// C3 0.139-0.143 ms per closed-loop step (0.167).  At 10k the tanh warps are the busy
// stage (~3.2k of ~3.5k cycles per chunk: the 17-24 batches of a block over 12 warps);
// at 1k the producer (the prefetched loads land in the registers its chain reads, so the
// next chunk's loads issue after this chunk's stores) sets the ~2.6k-cycle period.
// Variants measured and not kept: tanh warps on two sub-partitions and the chains alone on
// the others (10k 0.124 ms), the chains alone on one sub-partition (0.106), cp.async
// staging of the disturbances with four slots (0.103), 8 tanh warps (0.104-0.108).
//
// Used for host-planned (listed) steps without polling whose units fit one wave
// (rg_capi.cu: use_ts); the scenario block is the staged SoA, padded by kTsPadSteps steps
// so the producer's look-ahead loads never leave the buffer.
#include "rg_grid.cuh"

namespace rg {

namespace {

__device__ __forceinline__ void nb_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nb_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// bar.arrive that passes two doubles through (bit-exact moves): the computation that
// depends on them cannot be scheduled above the arrive
__device__ __forceinline__ void nb_arrive_pass(int id, int n, double& x, double& y) {
    asm volatile("bar.arrive %2, %3;\n\tmov.b64 %0, %0;\n\tmov.b64 %1, %1;"
                 : "+d"(x), "+d"(y) : "r"(id), "r"(n) : "memory");
}
// shared-memory load in program order (volatile): a chunk's values are all loaded up
// front instead of one latency at a time next to their uses
__device__ __forceinline__ double lds_v(const double* p) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return v;
}

constexpr int TW = kTsTanhWarps, RW = kTsUnits, CH = kTsChunk, S = kTsSlots;
constexpr int kG = CH * 4 * RW * 32;  // doubles: tanh arguments / values of a slot
constexpr int kD = CH * 2 * RW * 32;  // doubles: d0, d2 of a slot
constexpr int kSlot = kG + kD;
// named barriers (0 is __syncthreads): FULL_G 1..S, FULL_T S+1..2S, EMPTY 2S+1..3S
constexpr int kBarG = 1, kBarT = 1 + S, kBarE = 1 + 2 * S;
constexpr int nG = (TW + RW) * 32, nT = (TW + RW) * 32, nE = 2 * RW * 32;
static_assert(3 * S < 16, "named barriers");
static_assert(kTsThreads == (TW + 2 * RW) * 32, "block shape");
static_assert(kTsSmemDyn == S * kSlot * 8 + S * RW * 32 * 4, "shared memory");
static_assert(kTsPadSteps >= 2 * CH, "look-ahead padding");

}  // namespace

#ifdef RG_TS_TIMELINE
// Instrumented build only (make EXTRA=-DRG_TS_TIMELINE): block 0's per-warp, per-chunk
// clock64 stamps [warp][chunk][2] -- T: (go, done), P: (start, arrive), C: (go, done) --
// read back with rg_ts_timeline (scripts/prof_ts.py).
__device__ long long g_ts_tl[kTsThreads / 32][64][2];
#define RG_TS_STAMP(g, k, t)                                                            \
    do {                                                                               \
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (g) < 64) g_ts_tl[warp][g][k] = (t); \
    } while (0)
__device__ __forceinline__ long long ts_clock_after(const unsigned* w) {
    const unsigned x = *(volatile const unsigned*)w;  // issued after the barrier
    long long t = clock64();
    if (x == 0x9e3779b9u) t += 1;  // depends on the load: the barrier is behind us
    return t;
}
#define RG_TS_STAMP_AFTER(g, k) RG_TS_STAMP(g, k, ts_clock_after(OV))
#else
#define RG_TS_STAMP(g, k, t) \
    do {                     \
    } while (0)
#define RG_TS_STAMP_AFTER(g, k) RG_TS_STAMP(g, k, 0)
#endif

// RNG: the producer generates each step's disturbances with the counter RNG (the
// reference's generator, rg_rng.cuh) instead of reading the staged block -- no generator
// kernel before the step, no scenario block in memory.
template <bool FMA, bool RNG>
__global__ void __launch_bounds__(kTsThreads, 1) k_grid_ts(GridArgs a) {
    extern __shared__ double sm[];
    unsigned* OV = reinterpret_cast<unsigned*>(sm + S * kSlot);  // [S][RW][32]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) grid_clock_start(a);
    const int W = (int)((a.n_sim + 31) / 32);
    const int n_rows = a.listed ? a.list_n : a.m_grid;
    const int64_t units = (int64_t)n_rows * W;
    const int u0 = (int)(blockIdx.x * units / gridDim.x);
    const int u1 = (int)((blockIdx.x + 1) * units / gridDim.x);
    const int rw = u1 - u0;
    const int J = a.p.j_star;
    const int nch = (J + CH - 1) / CH;
    // the staged scenario block may still be being written (PDL behind k_gen_soa)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (warp < TW) {
        // T: slot by slot, batches (unit rr, step st) round-robin over the T warps
        const int nbat = rw * CH;
        int slot = 0;
        for (int g = 0; g < nch; ++g) {
            nb_sync(kBarG + slot, nG);
            RG_TS_STAMP_AFTER(g, 0);
            double* Gs = sm + slot * kSlot;
            for (int b = warp; b < nbat; b += TW) {
                const int rr = b / CH, st = b % CH;
                double x[4], z[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) x[q] = Gs[((st * 4 + q) * RW + rr) * 32 + lane];
                tanhN_with<FMA, true, 4>(x, z, [] {});
#pragma unroll
                for (int q = 0; q < 4; ++q) Gs[((st * 4 + q) * RW + rr) * 32 + lane] = z[q];
            }
            RG_TS_STAMP(g, 1, clock64());
            nb_arrive(kBarT + slot, nT);
            slot = slot == S - 1 ? 0 : slot + 1;
        }
    } else {
        const bool is_p = warp < TW + RW;
        const int r = is_p ? warp - TW : warp - TW - RW;
        const int ridx = r * 32 + lane;
        if (r >= rw) {  // no unit in this block: keep the barrier counts
            int slot = 0;
            for (int g = 0; g < nch; ++g) {
                if (is_p) {
                    if (g >= S) nb_sync(kBarE + slot, nE);
                    nb_arrive(kBarG + slot, nG);
                } else {
                    nb_sync(kBarT + slot, nT);
                    nb_arrive(kBarE + slot, nE);
                }
                slot = slot == S - 1 ? 0 : slot + 1;
            }
        } else {
            const int u = u0 + r;
            const int q = u / W;
            const int i = a.listed ? a.row_list[q] : q;  // the grid row
            const int wd = u - q * W;                     // its P-bit word
            const int64_t sc = (int64_t)wd * 32 + lane;
            const bool live = sc < a.n_sim;
            const CellConst p = make_cell(a.p);
            const int64_t ld = a.ld, st3 = 3 * a.ld;
            if (is_p && RNG) {
                // P with the fused counter RNG: step j's three disturbances from the
                // scenario key, off the x2 chain's dependencies
                const double v =
                    update_setpoint(a.v_prev, a.r, dvd((double)i, (double)(a.m_grid - 1)));
                const uint64_t K = scenario_key(a.stream, (uint64_t)(a.k0 + (live ? sc : 0)));
                double x2p = a.x0[1];
                int slot = 0;
                for (int g = 0; g < nch; ++g) {
                    RG_TS_STAMP(g, 0, clock64());
                    if (g >= S) nb_sync(kBarE + slot, nE);  // C is done with chunk g - S
                    double* Ss = sm + slot * kSlot;
                    unsigned ov = 0u;
#pragma unroll
                    for (int s = 0; s < CH; ++s) {
                        double d0, d1, d2;
                        disturbance_at(a.stream, K, (uint64_t)(g * CH + s), d0, d1, d2);
                        const X2Stage st = x2_stage<FMA>(x2p, v, p);
                        Ss[(s * 4 + 0) * RW * 32 + ridx] = x2p;
                        Ss[(s * 4 + 1) * RW * 32 + ridx] = st.a2;
                        Ss[(s * 4 + 2) * RW * 32 + ridx] = st.b2;
                        Ss[(s * 4 + 3) * RW * 32 + ridx] = st.c2;
                        Ss[kG + (s * 2 + 0) * RW * 32 + ridx] = d0;
                        Ss[kG + (s * 2 + 1) * RW * 32 + ridx] = d2;
                        x2p = add(add(x2p, mul(p.c, st.s2)), d1);
                        ov |= (fabs(x2p) <= kStateLimit ? 0u : 1u) << s;
                    }
                    OV[slot * RW * 32 + ridx] = ov;
                    RG_TS_STAMP(g, 1, clock64());
                    nb_arrive(kBarG + slot, nG);
                    slot = slot == S - 1 ? 0 : slot + 1;
                }
            } else if (is_p) {
                // P: the x2 chain.  Registers one chunk ahead: this chunk's d1 (the chain)
                // and d0/d2 (staged for C); the next chunk's load while this one runs.
                const double v =
                    update_setpoint(a.v_prev, a.r, dvd((double)i, (double)(a.m_grid - 1)));
                const double* d = a.soa + (live ? sc : 0);
                double x2p = a.x0[1];
                double d1c[CH], d0c[CH], d2c[CH];
#pragma unroll
                for (int s = 0; s < CH; ++s) {
                    d1c[s] = __ldg(d + s * st3 + ld);
                    d0c[s] = __ldg(d + s * st3);
                    d2c[s] = __ldg(d + s * st3 + 2 * ld);
                }
                int slot = 0;
                for (int g = 0; g < nch; ++g) {
                    double d0n[CH], d2n[CH], d1n[CH];
#pragma unroll
                    for (int s = 0; s < CH; ++s) {  // chunk g+1 (inside the padding at the end)
                        d0n[s] = __ldg(d + (CH + s) * st3);
                        d2n[s] = __ldg(d + (CH + s) * st3 + 2 * ld);
                        d1n[s] = __ldg(d + (CH + s) * st3 + ld);
                    }
                    RG_TS_STAMP(g, 0, clock64());
                    if (g >= S) nb_sync(kBarE + slot, nE);  // C is done with chunk g - S
                    double* Ss = sm + slot * kSlot;
                    unsigned ov = 0u;
#pragma unroll
                    for (int s = 0; s < CH; ++s) {
                        const X2Stage st = x2_stage<FMA>(x2p, v, p);
                        Ss[(s * 4 + 0) * RW * 32 + ridx] = x2p;
                        Ss[(s * 4 + 1) * RW * 32 + ridx] = st.a2;
                        Ss[(s * 4 + 2) * RW * 32 + ridx] = st.b2;
                        Ss[(s * 4 + 3) * RW * 32 + ridx] = st.c2;
                        Ss[kG + (s * 2 + 0) * RW * 32 + ridx] = d0c[s];
                        Ss[kG + (s * 2 + 1) * RW * 32 + ridx] = d2c[s];
                        x2p = add(add(x2p, mul(p.c, st.s2)), d1c[s]);
                        // step s's overflow test on x2 (x2 after the step)
                        ov |= (fabs(x2p) <= kStateLimit ? 0u : 1u) << s;
                    }
#pragma unroll
                    for (int s = 0; s < CH; ++s) {
                        d0c[s] = d0n[s];
                        d2c[s] = d2n[s];
                        d1c[s] = d1n[s];
                    }
                    OV[slot * RW * 32 + ridx] = ov;
                    RG_TS_STAMP(g, 1, clock64());
                    nb_arrive(kBarG + slot, nG);
                    d += CH * st3;
                    slot = slot == S - 1 ? 0 : slot + 1;
                }
            } else {
                // C: the x1/x3 chain, the reference's checks in its order (overflow, then
                // the output bound), status and step count of the first failing step
                double x1 = a.x0[0], x3 = a.x0[2];
                int status = kOk, steps = J;
                bool done = !live;
                if (live && !in_bounds(x1, p.ylo, p.yhi)) {
                    steps = 0;
                    status = kViolated;
                    done = true;
                }
                int slot = 0;
                for (int g = 0; g < nch; ++g) {
                    nb_sync(kBarT + slot, nT);
                    RG_TS_STAMP_AFTER(g, 0);
                    const double* Cs = sm + slot * kSlot + ridx;
                    const unsigned ovc = OV[slot * RW * 32 + ridx];
                    // one step of look-ahead: step s+1's six values load while step s runs
                    double tn[4], dn[2];
                    auto load = [&](int s) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) tn[k] = lds_v(Cs + (s * 4 + k) * RW * 32);
                        dn[0] = lds_v(Cs + kG + (s * 2 + 0) * RW * 32);
                        dn[1] = lds_v(Cs + kG + (s * 2 + 1) * RW * 32);
                    };
                    load(0);
#pragma unroll
                    for (int s = 0; s < CH; ++s) {
                        const double t1 = tn[0], t2 = tn[1], t3 = tn[2], t4 = tn[3];
                        const double d0 = dn[0], d2 = dn[1];
                        if (s + 1 < CH) {
                            load(s + 1);
                        } else {
                            // the slot is read out (bar.arrive orders the loads before it):
                            // P may refill it
                            nb_arrive_pass(kBarE + slot, nE, x1, x3);
                        }
                        const int j = g * CH + s;
                        x13_update<FMA>(x1, x3, t1, t2, t3, t4, p, d0, d2);
                        const bool ovf = !(fabs(x1) <= kStateLimit && !((ovc >> s) & 1u) &&
                                           fabs(x3) <= kStateLimit);
                        const bool bnd = !in_bounds(x1, p.ylo, p.yhi);
                        const bool now = !done && j < J && (ovf || bnd);
                        status = now ? (ovf ? kOverflow : kViolated) : status;
                        steps = now ? j + 1 : steps;
                        done = done || now;
                    }
                    RG_TS_STAMP(g, 1, clock64() + (long long)(x1 == 12345.0));
                    slot = slot == S - 1 ? 0 : slot + 1;
                }
                // the unit's verdicts, as k_grid's warp epilogue
                const bool bad = live && status != kOk;
                const unsigned bad_mask = __ballot_sync(0xffffffffu, bad);
                if (lane == 0 && bad_mask) atomicAdd(a.viol + i, (unsigned)__popc(bad_mask));
                warp_count_add(live && steps < J, a.early + i);
                warp_count_add(live && status == kOverflow, a.ovf + i);
                if (a.pbits) {
                    const unsigned ok_mask = __ballot_sync(0xffffffffu, live && status == kOk);
                    if (lane == 0) a.pbits[(int64_t)i * a.pwords + wd] = ok_mask;
                }
            }
        }
    }
    grid_finalize(a);
}

#ifdef RG_TS_TIMELINE
extern "C" __attribute__((visibility("default"))) int rg_ts_timeline(long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_ts_tl, sizeof(g_ts_tl));
}
#endif

// Blocks for `units` units: one wave of at most kTsUnits units per block, at least one
// block per SM while there are units to spread.
int ts_blocks(int64_t units, int sms) {
    const int64_t by_units = (units + kTsUnits - 1) / kTsUnits;
    return (int)std::max<int64_t>(std::min<int64_t>(sms, units), by_units);
}

cudaError_t launch_grid_ts(const GridArgs& a, bool fma, bool rng, int sms, cudaStream_t s) {
    const int64_t units = (int64_t)(a.listed ? a.list_n : a.m_grid) * ((a.n_sim + 31) / 32);
    const int nblk = ts_blocks(units, sms);
#define RG_TS_LAUNCH(F, R)                                                                 \
    do {                                                                                   \
        int dyn = 0;                                                                       \
        /* pin_smem takes the block's total: the static part (the finalize's) is < 4 KB */ \
        cudaError_t e = pin_smem((const void*)k_grid_ts<F, R>, kTsSmemDyn + 4096, &dyn);  \
        if (e != cudaSuccess) return e;                                                    \
        e = launch_ex(k_grid_ts<F, R>, dim3(nblk), kTsThreads, (size_t)dyn, s,             \
                      !R && a.pdl != 0, a);                                                \
        if (e != cudaSuccess) return e;                                                    \
    } while (0)
    if (fma) {
        if (rng) RG_TS_LAUNCH(true, true);
        else RG_TS_LAUNCH(true, false);
    } else {
        if (rng) RG_TS_LAUNCH(false, true);
        else RG_TS_LAUNCH(false, false);
    }
#undef RG_TS_LAUNCH
    return cudaGetLastError();
}

}  // namespace rg
