// rg_bisect.cu -- the bisection searches: exact Alg. 2 (k_bisect, governor.py:380-430,
// 469-517: one thread per scenario runs its own bisection; min/AND/sum reductions)
// and the joint search (k_joint_roll / k_joint_decide: one candidate for every
// scenario per iteration, OR-reduced violation flag).
#include "rg_common.cuh"

#include <algorithm>

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

// ---------------------------------------------------------------------------
// joint search as ONE persistent kernel with speculative levels (north star: "the search
// never round-trips to the host").
//
// A bisection path is sequential: candidate i+1 depends on candidate i's verdict.  But
// the steady-state gate is known up front (gated candidates are infeasible without a
// rollout), and below one wave most of the GPU is idle while one candidate's 32-scenario
// tiles run latency-bound.  So each round rolls out a small tree of candidates at once:
// the first gate-passing candidate on the current path, and for each of its two
// possible verdicts the next gate-passing candidate after it, to `depth` levels (1, 3 or
// 7 candidates).  After a grid barrier every block walks the tree with the violation
// words, exactly the decisions governor.py:407-431 would take, and continues from where
// the walk leaves the tree.  Candidates off the walked path are never consulted; a
// candidate's rollouts abandon early when the candidate itself violates, or when an
// ancestor whose feasible branch holds it violates (it can then no longer be on the
// path).  Every candidate that is consulted has its exact verdict, so kappa, found and
// the rollout count equal the one-candidate-per-iteration search; only the
// (timing-dependent) early-termination count of the abandoning search may differ.
// ---------------------------------------------------------------------------

// The search state between candidates (governor.py:407-431 on the joint verdicts).
struct Bracket {
    double lo, hi, kopt, kappa, v;  // kappa / v: the candidate waiting for a verdict
    unsigned long long cells, early;  // sims_run and the gated candidates' early count
    int it, found, done;
};

// Apply a verdict to the waiting candidate (one iteration of the walk).
__device__ __forceinline__ void bracket_apply(Bracket& b, bool feas, const JointArgs& a) {
    b.cells += (unsigned long long)a.n_sim;
    if (b.it < 0) {
        if (feas) {
            b.kopt = 1.0;
            b.found = 1;
            b.done = 1;
        }
    } else if (feas) {
        b.kopt = b.kappa;
        b.found = 1;
        b.lo = b.kappa;
    } else {
        b.hi = b.kappa;
    }
    b.it += 1;
    if (b.it >= a.n_kappa) b.done = 1;
}

// Walk through gated candidates (infeasible without a rollout, every scenario an early
// termination) to the next candidate that needs a rollout, or to the end of the search.
__device__ __forceinline__ void bracket_advance(Bracket& b, const JointArgs& a) {
    while (!b.done) {
        b.kappa = b.it < 0 ? 1.0 : mul(0.5, add(b.lo, b.hi));
        b.v = update_setpoint(a.v_prev, a.r, b.kappa);
        if (ss_gate(b.v, a.p)) return;
        b.early += (unsigned long long)a.n_sim;
        bracket_apply(b, false, a);
    }
}

__device__ __forceinline__ bool in_subtree(int y, int root) {  // heap order
    while (y > root) y = (y - 1) >> 1;
    return y == root;
}

template <bool FMA, int SRC>  // SRC: 0 zero (nominal), 1 rng, 2 soa
__global__ void __launch_bounds__(256, 1) k_joint_spec(JointArgs a) {
    JointState* st = a.st;
    const unsigned lane = threadIdx.x & 31u;
    const unsigned warp = threadIdx.x >> 5;
    const int64_t n_tiles = (a.n_sim + 31) / 32;
    const int64_t slots = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int nodes = (1 << a.depth) - 1;
    const CellConst c = make_cell(a.p);
    __shared__ double ring[2 * 3 * kRingStride];
    __shared__ Bracket tree[kJointNodes];
    __shared__ int active[kJointNodes];  // node ids that need rollouts, in heap order
    __shared__ int n_active;
    __shared__ Bracket cur;
    if (threadIdx.x == 0) {
        Bracket b{};
        b.lo = 0.0;
        b.hi = 1.0;
        b.it = -1;
        bracket_advance(b, a);
        if (a.probe_out && !b.done && b.it < 0) {  // the probe's verdict and early count
            b.early += (unsigned long long)((const volatile GridOut*)a.probe_out)->early_terms;
            bracket_apply(b, *(const volatile unsigned*)a.probe_viol == 0u, a);
            bracket_advance(b, a);
        }
        cur = b;
    }
    __syncthreads();
    int round = 0;
    for (; !cur.done && round < kJointMaxRounds; ++round) {
        // the speculation tree of this round (every block builds the same one)
        if (threadIdx.x == 0) {
            int na = 0;
            bool exists[kJointNodes];
            for (int n = 0; n < nodes; ++n) {
                exists[n] = n == 0 || (exists[(n - 1) >> 1] && !tree[(n - 1) >> 1].done);
                if (!exists[n]) continue;
                if (n == 0) {
                    tree[0] = cur;
                } else {
                    Bracket b = tree[(n - 1) >> 1];
                    bracket_apply(b, (n & 1) != 0, a);  // odd: the feasible branch
                    bracket_advance(b, a);
                    tree[n] = b;
                }
                if (!tree[n].done) active[na++] = n;
            }
            n_active = na;
        }
        __syncthreads();
        unsigned* viol = st->sviol + round * 8;
        unsigned* dead = st->sdead + round * 8;
        unsigned long long* early = st->searly + round * 8;
        const int64_t items = (int64_t)n_active * n_tiles;
        // first item of every warp slot spread across the blocks (SMs) first, then
        // dynamic items from the round's counter
        int64_t t = (int64_t)warp * gridDim.x + blockIdx.x;
        while (t < items) {
            const int node = active[t / n_tiles];
            const double v = tree[node].v;
            unsigned* poll = dead + node;
            if (!*(volatile unsigned*)poll) {
                const int64_t k = (t % n_tiles) * 32 + lane;
                const bool live = k < a.n_sim;
                const int64_t kk = live ? k : 0;
                int32_t steps = 0;
                int stt;
                if constexpr (SRC == 1) {
                    RngSource src{a.stream, scenario_key(a.stream, (uint64_t)(a.k0 + kk))};
                    stt = rollout<FMA, true, RngSource, true, true>(c, a.x0[0], a.x0[1], a.x0[2],
                                                                     v, src, steps, poll, live);
                } else if constexpr (SRC == 2) {
                    SoaSource src{a.soa + kk, a.ld, ring + threadIdx.x};
                    stt = rollout<FMA, true, SoaSource, true, true>(c, a.x0[0], a.x0[1], a.x0[2],
                                                                     v, src, steps, poll, live);
                } else {
                    stt = rollout<FMA, true, ZeroSource, true, true>(c, a.x0[0], a.x0[1],
                                                                      a.x0[2], v, ZeroSource{},
                                                                      steps, poll, live);
                }
                const bool bad = live && stt != kOk && stt != kAbandoned;
                if (__ballot_sync(0xffffffffu, bad) && lane == 0) {
                    atomicOr(viol + node, 1u);
                    atomicOr(poll, 1u);
                    // this candidate is infeasible: the candidates of its feasible branch
                    // can no longer be on the path
                    for (int y = 2 * node + 1; y < nodes; ++y)
                        if (in_subtree(y, 2 * node + 1)) atomicOr(dead + y, 1u);
                }
                warp_count_add(bad && steps < a.p.j_star, early + node);
            }
            if (slots >= items) break;  // every item had its own warp slot
            int64_t nxt = 0;
            if (lane == 0) nxt = slots + (int64_t)atomicAdd(&st->sitem[round], 1u);
            t = __shfl_sync(0xffffffffu, nxt, 0);
        }
        grid_barrier(&st->bar_count, &st->bar_gen, gridDim.x);
        __shared__ unsigned s_gv[kJointNodes];  // the verdicts the walk reads
        if (a.xchg) {
            // the shards' verdicts: block 0 sends this shard's to every rank's window, every
            // block waits for every rank's and ORs them (epoch xepoch0 + round, parity buffers)
            const unsigned long long ep = a.xepoch0 + (unsigned long long)round;
            const int par = (int)(ep & 1ull);
            if (blockIdx.x == 0) {
                for (int t = threadIdx.x; t < a.xworld * nodes; t += blockDim.x) {
                    const int r = t / nodes, q = t - r * nodes;
                    a.xpeers[r]->words[par][a.xrank][q] = *(volatile unsigned*)(viol + q) != 0u;
                }
                __threadfence_system();
                __syncthreads();
                if (threadIdx.x < a.xworld)
                    st_release_sys(&a.xpeers[threadIdx.x]->flag[par][a.xrank], ep);
            }
            if (threadIdx.x < a.xworld) {
                const unsigned long long* f = &a.xlocal->flag[par][threadIdx.x];
                const unsigned long long t0 = global_ns();
                while (ld_acquire_sys(f) < ep) {
                    if (global_ns() - t0 > a.xtimeout_ns) {
                        st->xfail = 1;
                        break;
                    }
                    __nanosleep(100);
                }
            }
            __syncthreads();
            if (threadIdx.x < nodes) {
                int g = 0;
                for (int r = 0; r < a.xworld; ++r)
                    g |= ((volatile int*)a.xlocal->words[par][r])[threadIdx.x];
                s_gv[threadIdx.x] = (unsigned)g;
            }
        } else if (threadIdx.x < nodes) {
            s_gv[threadIdx.x] = *(volatile unsigned*)(viol + threadIdx.x);
        }
        __syncthreads();
        // the walk: the decisions the one-candidate search takes, while they stay in the tree
        if (threadIdx.x == 0) {
            int n = 0;
            Bracket b = tree[0];
            while (true) {
                const bool feas = s_gv[n] == 0u;
                b.early += *(volatile unsigned long long*)(early + n);
                const int nx = feas ? 2 * n + 1 : 2 * n + 2;
                if (nx < nodes) {
                    const unsigned long long e = b.early;
                    b = tree[nx];  // = advance(apply(tree[n], feas)), plus the early counts
                    b.early += e - tree[n].early;
                    if (b.done) break;
                    n = nx;
                } else {
                    bracket_apply(b, feas, a);
                    bracket_advance(b, a);
                    break;
                }
            }
            cur = b;
        }
        __syncthreads();
    }
    // every block has read every word it needs; the last block out publishes and resets
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&st->exit_ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int q = threadIdx.x; q < round * 8; q += blockDim.x) {
        st->sviol[q] = 0u;
        st->sdead[q] = 0u;
        st->searly[q] = 0ull;
    }
    for (int q = threadIdx.x; q < round; q += blockDim.x) st->sitem[q] = 0u;
    if (threadIdx.x == 0) {
        volatile JointState* vs = st;
        vs->kopt = cur.kopt;
        vs->found = cur.found;
        vs->done = 1;
        vs->cells = cur.cells;
        vs->early = cur.early;
        vs->rounds = round;
        vs->exit_ticket = 0u;
        vs->seq = vs->seq + 1;
        if (a.hout) {
            volatile JointOut* ho = a.hout;
            ho->kopt = cur.kopt;
            ho->found = cur.found;
            ho->cells = cur.cells;
            ho->early = cur.early;
            ho->rounds = round;
            ho->xfail = vs->xfail;
            __threadfence_system();
            ho->seq = a.seq_token;
        }
    }
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
            if (it < 0 && a.probe_ok) {
                // the kappa = 1 probe was rolled out ahead (rg_bisect: the time-split kernel,
                // used only when v = r passes the gate): its verdict and early bit
                const unsigned bit = 1u << (kk & 31);
                ok = run && (a.probe_ok[kk >> 5] & bit) != 0u;
                sr = run && (a.probe_early[kk >> 5] & bit) != 0u ? 0 : a.p.j_star;
            } else if (run || U) {
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
    if (a.host_out) __threadfence_system();  // the fields before the token
    *(volatile unsigned long long*)&a.out->seq = a.seq_token;
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

int joint_spec_depth(int64_t n_sim, int sm_count) {
    const int64_t tiles = (n_sim + 31) / 32;
    const int64_t wave = 8 * (int64_t)sm_count;  // two warps per SM sub-partition
    for (int d = 3; d >= 1; --d)
        if (((int64_t)1 << d) - 1 <= wave / std::max<int64_t>(tiles, 1)) return d;
    return 0;
}

cudaError_t launch_joint_spec(const JointArgs& a, bool fma, int src, int sm_count,
                              cudaStream_t s) {
    constexpr int kThreads = 256;
    const void* fn;
    if (fma) fn = src == 1 ? (const void*)k_joint_spec<true, 1>
                           : src == 2 ? (const void*)k_joint_spec<true, 2>
                                      : (const void*)k_joint_spec<true, 0>;
    else fn = src == 1 ? (const void*)k_joint_spec<false, 1>
                       : src == 2 ? (const void*)k_joint_spec<false, 2>
                                  : (const void*)k_joint_spec<false, 0>;
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
    // one block per SM at most; warp w of block b takes item w * blocks + b first, so the
    // items land one warp per SM sub-partition before any gets a second
    const int64_t items = (((int64_t)1 << a.depth) - 1) * ((a.n_sim + 31) / 32);
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(items, sm_count));
    JointArgs args = a;
    void* params[] = {&args};
    return cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(kThreads), params, 0, s);
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
