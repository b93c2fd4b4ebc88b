// rg_bisect.cu -- the bisection searches: exact Alg. 2 (k_bisect, governor.py:380-430,
// 469-517: one thread per scenario runs its own bisection; min/AND/sum reductions)
// and the joint search (k_joint_roll / k_joint_decide: one candidate for every
// scenario per iteration, OR-reduced violation flag).
#include "rg_common.cuh"

namespace rg {

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
            st = rollout<FMA, true, RngSource, true, true>(c, a.x0[0], a.x0[1], a.x0[2], s_v,
                                                              src, steps, flag, live);
        } else if (SRC == 2) {
            __shared__ double ring[2 * 3 * kRingStride];
            SoaSource src{a.soa + kk, a.ld, ring + threadIdx.x};
            st = rollout<FMA, true, SoaSource, true, true>(c, a.x0[0], a.x0[1], a.x0[2], s_v,
                                                              src, steps, flag, live);
        } else {
            st = rollout<FMA, true, ZeroSource, true, true>(c, a.x0[0], a.x0[1], a.x0[2],
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

template <bool FMA, int SRC>  // SRC: 0 zero (nominal), 1 rng, 2 soa
__global__ void __launch_bounds__(256, RG_GRID_MINB) k_bisect(BisectArgs a) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = k < a.n_sim;
    constexpr bool lead = true;
    double kopt = 1.0;
    int found = 1, cells = 0, early = 0;
    // every lane of the warp walks the candidates (the warp-uniform rollout);
    // finished lanes keep it company
    constexpr bool U = true;
    {
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
        // Every lane walks every candidate; finished or gated-out cells pass
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
                    st = rollout<FMA, false, RngSource, true>(c, a.x0[0], a.x0[1], a.x0[2], v,
                                                              rsrc, sr, nullptr, run);
                else if (SRC == 2)
                    st = rollout<FMA, false, SoaSource, true>(c, a.x0[0], a.x0[1], a.x0[2], v,
                                                              ssrc, sr, nullptr, run);
                else
                    st = rollout<FMA, false, ZeroSource, true>(c, a.x0[0], a.x0[1], a.x0[2],
                                                               v, ZeroSource{}, sr, nullptr, run);
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
// launchers
// ---------------------------------------------------------------------------

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

cudaError_t launch_bisect(const BisectArgs& a, bool fma, int src, cudaStream_t s) {
    const unsigned g = blocks_for(a.n_sim, a.tpb);
    cudaError_t e = cudaSuccess;
#define RG_BIS(F, S)                                                                    \
    do {                                                                                \
        int dyn = 0;                                                                    \
        if ((e = pin_smem((const void*)k_bisect<F, S>, a.smem_dyn, &dyn)) != cudaSuccess) \
            return e;                                                                   \
        k_bisect<F, S><<<g, a.tpb, (size_t)dyn, s>>>(a);                                \
    } while (0)
    if (fma) {
        if (src == 0) RG_BIS(true, 0); else if (src == 1) RG_BIS(true, 1); else RG_BIS(true, 2);
    } else {
        if (src == 0) RG_BIS(false, 0); else if (src == 1) RG_BIS(false, 1); else RG_BIS(false, 2);
    }
#undef RG_BIS
    return cudaGetLastError();
}

}  // namespace rg
