// Prototype: the time-split rollout (warp-specialised recurrence / tanh warps).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --fmad=false -lineinfo \
//        -Xptxas -v -I paper_2510_08288_b200/csrc -o scripts/micro/ts_proto scripts/micro/ts_proto.cu
// Run on the B200: scripts/micro/ts_proto [n_sim] [m_rows] [transient]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <random>
#include <algorithm>

#include "rg_cell.cuh"

using namespace rg;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

struct TsArgs {
    const double* soa;
    int64_t ld;
    int32_t n_sim, W, units;
    const double* vrow;
    double x0[3];
    CellConst p;
    int* status;
    int* steps;
    long long* prof;  // [block][warp][2]: cycles waiting, cycles total (k_ts3, if set)
    long long* tl;    // block 0 timeline: [warp][chunk][2]
};

__device__ __forceinline__ void nb_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// bar.sync that also yields a zero the caller folds into later shared-memory addresses:
// loads through lds_nc() (no memory clobber) may then move freely past unrelated stores
// but never above the barrier
__device__ __forceinline__ uint32_t nb_sync_tok(int id, int n) {
    uint32_t z;
    asm volatile("bar.sync %1, %2;\n\tmov.u32 %0, 0;" : "=r"(z) : "r"(id), "r"(n) : "memory");
    return z;
}
__device__ __forceinline__ double lds_nc(uint32_t addr) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}
// the cycle count after a barrier: waits for a shared load issued after the barrier so a
// deferred-blocking BAR.SYNC is really behind us
__device__ __forceinline__ long long clock_after(const unsigned* sm_word) {
    const unsigned x = *(volatile const unsigned*)sm_word;
    long long t = clock64();
    if (x == 0x9e3779b9u) t += 1;
    return t;
}
__device__ __forceinline__ void nb_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// TW tanh warps (first), RW recurrence warps; chunks of CH steps; N-wide tanh batches
// (N/4 steps of one recurrence warp's 32 cells); a ring of 3 chunk slots.
template <int TW, int RW, int CH, int N>
__global__ void __launch_bounds__((TW + RW) * 32, 1) k_ts(TsArgs a) {
    constexpr int kT = (TW + RW) * 32;
    constexpr int S = 3;
    constexpr int kSlot = CH * 4 * RW * 32;  // doubles per slot
    constexpr int SPB = N / 4;               // steps per batch
    static_assert(CH % SPB == 0, "batch steps divide the chunk");
    extern __shared__ double sm[];
    double* G = sm;
    unsigned* OV = reinterpret_cast<unsigned*>(sm + S * kSlot);  // [S][RW][32]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int u0 = (int)((int64_t)blockIdx.x * a.units / gridDim.x);
    const int u1 = (int)((int64_t)(blockIdx.x + 1) * a.units / gridDim.x);
    const int ntile = (u1 - u0 + RW - 1) / RW;
    const int J = a.p.j_star;
    const int nch = (J + CH - 1) / CH;
    const int total = ntile * nch;
    if (warp < TW) {
        for (int g = 0; g < total; ++g) {
            const int slot = g % S;
            const int tile = g / nch;
            const int rw = min(RW, u1 - u0 - tile * RW);
            nb_sync(1 + slot, kT);
            double* Gs = G + slot * kSlot;
            const int nbat = rw * (CH / SPB);
            for (int b = warp; b < nbat; b += TW) {
                const int r = b / (CH / SPB);
                const int s0 = (b % (CH / SPB)) * SPB;
                double x[N], z[N];
#pragma unroll
                for (int q = 0; q < N; ++q)
                    x[q] = Gs[(((s0 + q / 4) * 4 + (q % 4)) * RW + r) * 32 + lane];
                tanhN_with<true, true, N>(x, z, [] {});
#pragma unroll
                for (int q = 0; q < N; ++q)
                    Gs[(((s0 + q / 4) * 4 + (q % 4)) * RW + r) * 32 + lane] = z[q];
            }
            nb_arrive(1 + S + slot, kT);
        }
        return;
    }
    const int r = warp - TW;
    const CellConst p = a.p;
    // producer (x2 chain) and consumer (x1/x3 chains) positions
    double x2p = 0.0, vp = 0.0;
    int64_t scen_p = 0;
    bool live_p = false;
    double x1 = 0.0, x3 = 0.0;
    int64_t scen_c = 0;
    int cell_c = -1;
    bool live_c = false, done = true;
    int status = kOk, steps = J;
    auto unit_of = [&](int tile) { return u0 + tile * RW + r; };
    // the producer's unit for chunk g (called before a tile's chunk 0)
    auto produce_reset = [&](int g) {
        const int tile = g / nch;
        const int u = unit_of(tile);
        live_p = u < u1;
        const int row = live_p ? u / a.W : 0;
        vp = a.vrow[row];
        x2p = a.x0[1];
    };
    // step s of chunk g's x2 chain, tanh arguments into the slot (branch-free)
    auto produce = [&](int g, int s, unsigned& ovbits, double d1) {
        double* Gs = G + (g % S) * kSlot;
        const X2Stage st = x2_stage<true>(x2p, vp, p);
        Gs[((s * 4 + 0) * RW + r) * 32 + lane] = x2p;
        Gs[((s * 4 + 1) * RW + r) * 32 + lane] = st.a2;
        Gs[((s * 4 + 2) * RW + r) * 32 + lane] = st.b2;
        Gs[((s * 4 + 3) * RW + r) * 32 + lane] = st.c2;
        x2p = add(add(x2p, mul(p.c, st.s2)), d1);
        ovbits |= (fabs(x2p) <= kStateLimit ? 0u : 1u) << s;
    };
    // scenario of the producer's unit for chunk g (the disturbances are loaded before the
    // chunk's first step resets the producer)
    auto scen_of = [&](int g) -> int64_t {
        const int tile = g / nch;
        const int u = unit_of(tile);
        if (u >= u1) return 0;
        const int row = u / a.W;
        const int sc = (u - row * a.W) * 32 + lane;
        return sc < a.n_sim ? sc : 0;
    };
    auto load_d1 = [&](int g, double (&d)[CH]) {
        const int c = g % nch;
        const int64_t sc = scen_of(g);
#pragma unroll
        for (int s = 0; s < CH; ++s) {
            const int j = min(c * CH + s, J - 1);
            d[s] = __ldg(a.soa + (int64_t)j * 3 * a.ld + a.ld + sc);
        }
    };
    // prologue: chunks 0 and 1
    for (int g = 0; g < 2 && g < total; ++g) {
        unsigned ov = 0u;
        double pd[CH];
        load_d1(g, pd);
        if (g % nch == 0) produce_reset(g);
#pragma unroll
        for (int s = 0; s < CH; ++s) produce(g, s, ov, pd[s]);
        OV[((g % S) * RW + r) * 32 + lane] = ov;
        nb_arrive(1 + (g % S), kT);
    }
    for (int g = 0; g < total; ++g) {
        const int slot = g % S;
        const int tile = g / nch, c = g - tile * nch;
        const bool prod = g + 2 < total;
        // a recurrence warp without a unit in this tile only keeps the barriers
        const bool idle = unit_of(tile) >= u1 && (g + 2 >= total || unit_of((g + 2) / nch) >= u1);
        if (idle) {
            nb_sync(1 + S + slot, kT);
            if (prod) nb_arrive(1 + ((g + 2) % S), kT);
            continue;
        }
        // this iteration's disturbances, in flight across the barrier wait
        double pd1[CH], cd0[CH], cd2[CH];
        load_d1(min(g + 2, total - 1), pd1);  // past the end: produced into a dead slot
        {
            const int64_t sc = scen_of(g);
#pragma unroll
            for (int s = 0; s < CH; ++s) {
                const int j = min(c * CH + s, J - 1);
                const double* dp = a.soa + (int64_t)j * 3 * a.ld + sc;
                cd0[s] = __ldg(dp);
                cd2[s] = __ldg(dp + 2 * a.ld);
            }
        }
        const uint32_t tok = nb_sync_tok(1 + S + slot, kT);
        if (c == 0) {
            const int u = unit_of(tile);
            const bool uv = u < u1;
            const int row = uv ? u / a.W : 0;
            const int sc = (uv ? (u - row * a.W) * 32 : 0) + lane;
            live_c = uv && sc < a.n_sim;
            scen_c = live_c ? sc : 0;
            cell_c = live_c ? row * a.n_sim + sc : -1;
            x1 = a.x0[0];
            x3 = a.x0[2];
            status = kOk;
            steps = J;
            done = !live_c;
            if (live_c && !in_bounds(x1, p.ylo, p.yhi)) {
                steps = 0;
                status = kViolated;
                done = true;
            }
        }
        const uint32_t gsa = (uint32_t)__cvta_generic_to_shared(G + slot * kSlot) + tok;
        const unsigned ovc = OV[(slot * RW + r) * 32 + lane];
        unsigned ovp = 0u;
        if ((g + 2) % nch == 0) produce_reset(g + 2);
#pragma unroll
        for (int s = 0; s < CH; ++s) {
            produce(g + 2, s, ovp, pd1[s]);
            const int j = c * CH + s;
            const double t1 = lds_nc(gsa + 8 * (((s * 4 + 0) * RW + r) * 32 + lane));
            const double t2 = lds_nc(gsa + 8 * (((s * 4 + 1) * RW + r) * 32 + lane));
            const double t3 = lds_nc(gsa + 8 * (((s * 4 + 2) * RW + r) * 32 + lane));
            const double t4 = lds_nc(gsa + 8 * (((s * 4 + 3) * RW + r) * 32 + lane));
            const double d0 = cd0[s], d2 = cd2[s];
            double y1 = x1, y3 = x3;
            x13_update<true>(y1, y3, t1, t2, t3, t4, p, d0, d2);
            const bool ovf = !(fabs(y1) <= kStateLimit && !((ovc >> s) & 1u) &&
                               fabs(y3) <= kStateLimit);
            const bool bnd = !in_bounds(y1, p.ylo, p.yhi);
            const bool act = !done && j < J;
            x1 = y1;  // a finished cell's state runs on unobserved
            x3 = y3;
            const bool now = act && (ovf || bnd);
            status = now ? (ovf ? kOverflow : kViolated) : status;
            steps = now ? j + 1 : steps;
            done = done || now;
        }
        if (prod) {
            OV[(((g + 2) % S) * RW + r) * 32 + lane] = ovp;
            nb_arrive(1 + ((g + 2) % S), kT);
        }
        if (c == nch - 1 && cell_c >= 0) {
            a.status[cell_c] = status;
            a.steps[cell_c] = steps;
        }
    }
}

// v2, the latency regime: at most RW units per block (one tile), the producer also stages
// the consumer's d0/d2 into the slot, its own d1 one chunk ahead in registers; no integer
// division inside the loop.
template <int TW, int RW, int CH>
__global__ void __launch_bounds__((TW + RW) * 32, 1) k_ts2(TsArgs a) {
    constexpr int kT = (TW + RW) * 32;
    constexpr int S = 3;
    constexpr int kG = CH * 4 * RW * 32;
    constexpr int kD = CH * 2 * RW * 32;
    constexpr int kSlot = kG + kD;
    extern __shared__ double sm[];
    unsigned* OV = reinterpret_cast<unsigned*>(sm + S * kSlot);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int u0 = (int)((int64_t)blockIdx.x * a.units / gridDim.x);
    const int u1 = (int)((int64_t)(blockIdx.x + 1) * a.units / gridDim.x);
    const int rw = u1 - u0;
    const int J = a.p.j_star;
    const int nch = (J + CH - 1) / CH;
    if (warp < TW) {
        const int nbat = rw * CH;
        int slot = 0;
        for (int g = 0; g < nch; ++g) {
            nb_sync(1 + slot, kT);
            double* Gs = sm + slot * kSlot;
            for (int b = warp; b < nbat; b += TW) {
                const int rr = b / CH, st = b % CH;
                double x[4], z[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) x[q] = Gs[((st * 4 + q) * RW + rr) * 32 + lane];
                tanhN_with<true, true, 4>(x, z, [] {});
#pragma unroll
                for (int q = 0; q < 4; ++q) Gs[((st * 4 + q) * RW + rr) * 32 + lane] = z[q];
            }
            nb_arrive(1 + S + slot, kT);
            slot = slot == S - 1 ? 0 : slot + 1;
        }
        return;
    }
    const int r = warp - TW;
    if (r >= rw) {  // no unit: keep the barrier counts
        for (int g = 0; g < 2 && g < nch; ++g) nb_arrive(1 + g, kT);
        for (int g = 0; g < nch; ++g) {
            nb_sync(1 + S + g % S, kT);
            if (g + 2 < nch) nb_arrive(1 + (g + 2) % S, kT);
        }
        return;
    }
    const int u = u0 + r;
    const int row = u / a.W;
    const int sc = (u - row * a.W) * 32 + lane;
    const bool live = sc < a.n_sim;
    const double v = a.vrow[row];
    const CellConst p = a.p;
    const double* db = a.soa + (live ? sc : 0);
    const int64_t st3 = 3 * a.ld, ld = a.ld;
    auto dp = [&](int j) { return db + (int64_t)(j < J ? j : J - 1) * st3; };
    const int ridx = r * 32 + lane;  // [.][RW][32] offset
    double x2p = a.x0[1];
    auto produce = [&](double* Ss, int s, double d1, unsigned& ov) {
        const X2Stage q = x2_stage<true>(x2p, v, p);
        Ss[(s * 4 + 0) * RW * 32 + ridx] = x2p;
        Ss[(s * 4 + 1) * RW * 32 + ridx] = q.a2;
        Ss[(s * 4 + 2) * RW * 32 + ridx] = q.b2;
        Ss[(s * 4 + 3) * RW * 32 + ridx] = q.c2;
        x2p = add(add(x2p, mul(p.c, q.s2)), d1);
        ov |= (fabs(x2p) <= kStateLimit ? 0u : 1u) << s;
    };
    // prologue: chunks 0 and 1
    for (int g = 0; g < 2 && g < nch; ++g) {
        double* Ss = sm + g * kSlot;
        unsigned ov = 0u;
#pragma unroll
        for (int s = 0; s < CH; ++s) {
            const double* q = dp(g * CH + s);
            produce(Ss, s, __ldg(q + ld), ov);
            Ss[kG + (s * 2 + 0) * RW * 32 + ridx] = __ldg(q);
            Ss[kG + (s * 2 + 1) * RW * 32 + ridx] = __ldg(q + 2 * ld);
        }
        OV[g * RW * 32 + ridx] = ov;
        nb_arrive(1 + g, kT);
    }
    double d1c[CH];
#pragma unroll
    for (int s = 0; s < CH; ++s) d1c[s] = __ldg(dp(2 * CH + s) + ld);
    double x1 = a.x0[0], x3 = a.x0[2];
    int status = kOk, steps = J;
    bool done = !live;
    if (live && !in_bounds(x1, p.ylo, p.yhi)) {
        steps = 0;
        status = kViolated;
        done = true;
    }
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
    int sc_ = 0, sp_ = 2;  // consumer / producer slots
    for (int g = 0; g < nch; ++g) {
        const bool prod = g + 2 < nch;
        double d0p[CH], d2p[CH], d1n[CH];
#pragma unroll
        for (int s = 0; s < CH; ++s) {
            const double* q = dp((g + 2) * CH + s);
            d0p[s] = __ldg(q);
            d2p[s] = __ldg(q + 2 * ld);
            d1n[s] = __ldg(dp((g + 3) * CH + s) + ld);
        }
        const uint32_t tok = nb_sync_tok(1 + S + sc_, kT);
        const uint32_t ca = sbase + 8u * (uint32_t)(sc_ * kSlot + ridx) + tok;
        const unsigned ovc = OV[sc_ * RW * 32 + ridx];
        double* Sp = sm + sp_ * kSlot;
        unsigned ovp = 0u;
#pragma unroll
        for (int s = 0; s < CH; ++s) {
            produce(Sp, s, d1c[s], ovp);
            const int j = g * CH + s;
            const double t1 = lds_nc(ca + 8u * ((s * 4 + 0) * RW * 32));
            const double t2 = lds_nc(ca + 8u * ((s * 4 + 1) * RW * 32));
            const double t3 = lds_nc(ca + 8u * ((s * 4 + 2) * RW * 32));
            const double t4 = lds_nc(ca + 8u * ((s * 4 + 3) * RW * 32));
            const double d0 = lds_nc(ca + 8u * (kG + (s * 2 + 0) * RW * 32));
            const double d2 = lds_nc(ca + 8u * (kG + (s * 2 + 1) * RW * 32));
            x13_update<true>(x1, x3, t1, t2, t3, t4, p, d0, d2);
            const bool ovf = !(fabs(x1) <= kStateLimit && !((ovc >> s) & 1u) &&
                               fabs(x3) <= kStateLimit);
            const bool bnd = !in_bounds(x1, p.ylo, p.yhi);
            const bool now = !done && j < J && (ovf || bnd);
            status = now ? (ovf ? kOverflow : kViolated) : status;
            steps = now ? j + 1 : steps;
            done = done || now;
        }
#pragma unroll
        for (int s = 0; s < CH; ++s) {
            Sp[kG + (s * 2 + 0) * RW * 32 + ridx] = d0p[s];
            Sp[kG + (s * 2 + 1) * RW * 32 + ridx] = d2p[s];
            d1c[s] = d1n[s];
        }
        OV[sp_ * RW * 32 + ridx] = ovp;
        if (prod) nb_arrive(1 + sp_, kT);
        sc_ = sc_ == S - 1 ? 0 : sc_ + 1;
        sp_ = sp_ == S - 1 ? 0 : sp_ + 1;
    }
    if (live) {
        a.status[(int64_t)row * a.n_sim + sc] = status;
        a.steps[(int64_t)row * a.n_sim + sc] = steps;
    }
}

template <int TW, int RW, int CH>
float run_ts2(const TsArgs& a, int sms, int reps) {
    constexpr int kT = (TW + RW) * 32;
    const size_t smem = 3 * (size_t)CH * 6 * RW * 32 * 8 + 3 * RW * 32 * 4;
    CK(cudaFuncSetAttribute(k_ts2<TW, RW, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
    const int nblk = std::max(std::min(sms, a.units), (a.units + RW - 1) / RW);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    k_ts2<TW, RW, CH><<<nblk, kT, smem>>>(a);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> ts;
    for (int i = 0; i < reps; ++i) {
        CK(cudaEventRecord(e0));
        k_ts2<TW, RW, CH><<<nblk, kT, smem>>>(a);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
}

// v3: producer (x2 chain) and consumer (x1/x3 chains) in separate warps.  Per unit one P
// warp and one C warp; barriers per slot: FULL_G (P -> T), FULL_T (T -> C), EMPTY (C -> P).
// The scenario tensor is padded by 3 chunks of steps (reads past J land in the padding).
template <int TW, int RW, int CH>
__global__ void __launch_bounds__((TW + 2 * RW) * 32, 1) k_ts3(TsArgs a) {
    constexpr int S = 3;
    constexpr int kG = CH * 4 * RW * 32;
    constexpr int kD = CH * 2 * RW * 32;
    constexpr int kSlot = kG + kD;
    constexpr int nG = (TW + RW) * 32, nT = (TW + RW) * 32, nE = 2 * RW * 32;
    extern __shared__ double sm[];
    unsigned* OV = reinterpret_cast<unsigned*>(sm + S * kSlot);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int u0 = (int)((int64_t)blockIdx.x * a.units / gridDim.x);
    const int u1 = (int)((int64_t)(blockIdx.x + 1) * a.units / gridDim.x);
    const int rw = u1 - u0;
    const int J = a.p.j_star;
    const int nch = (J + CH - 1) / CH;
    // barrier ids: FULL_G 1..3, FULL_T 4..6, EMPTY 7..9
    long long t_wait = 0, t_start = clock64();
    auto prof_out = [&]() {
        if (a.prof && lane == 0) {
            a.prof[((int64_t)blockIdx.x * 32 + warp) * 2] = t_wait;
            a.prof[((int64_t)blockIdx.x * 32 + warp) * 2 + 1] = clock64() - t_start;
        }
    };
    if (warp < TW) {
        const int nbat = rw * CH;
        int slot = 0;
        for (int g = 0; g < nch; ++g) {
            { const long long t0 = clock64(); nb_sync(1 + slot, nG); const long long t1 = clock_after(OV); t_wait += t1 - t0;
              if (a.tl && blockIdx.x == 0 && lane == 0 && g < 64) a.tl[(warp * 64 + g) * 2] = t1; }
            double* Gs = sm + slot * kSlot;
            for (int b = warp; b < nbat; b += TW) {
                const int rr = b / CH, st = b % CH;
                double x[4], z[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) x[q] = Gs[((st * 4 + q) * RW + rr) * 32 + lane];
                tanhN_with<true, true, 4>(x, z, [] {});
#pragma unroll
                for (int q = 0; q < 4; ++q) Gs[((st * 4 + q) * RW + rr) * 32 + lane] = z[q];
            }
            if (a.tl && blockIdx.x == 0 && lane == 0 && g < 64) a.tl[(warp * 64 + g) * 2 + 1] = clock64();
            nb_arrive(4 + slot, nT);
            slot = slot == S - 1 ? 0 : slot + 1;
        }
        prof_out();
        return;
    }
    const bool is_p = warp < TW + RW;
    const int r = is_p ? warp - TW : warp - TW - RW;
    const int ridx = r * 32 + lane;
    if (r >= rw) {  // no unit: keep the barrier counts
        int slot = 0;
        for (int g = 0; g < nch; ++g) {
            if (is_p) {
                if (g >= S) nb_sync(7 + slot, nE);
                nb_arrive(1 + slot, nG);
            } else {
                nb_sync(4 + slot, nT);
                nb_arrive(7 + slot, nE);
            }
            slot = slot == S - 1 ? 0 : slot + 1;
        }
        return;
    }
    const int u = u0 + r;
    const int row = u / a.W;
    const int sc = (u - row * a.W) * 32 + lane;
    const bool live = sc < a.n_sim;
    const CellConst p = a.p;
    const int64_t ld = a.ld, st3 = 3 * a.ld;
    if (is_p) {
        const double v = a.vrow[row];
        const double* d = a.soa + (live ? sc : 0);  // step 0
        double x2p = a.x0[1];
        // registers one chunk ahead: this chunk's d1 (the chain) and d0/d2 (staged for the
        // consumer); the next chunk's are loaded while this one runs
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
            for (int s = 0; s < CH; ++s) {
                d0n[s] = __ldg(d + (CH + s) * st3);
                d2n[s] = __ldg(d + (CH + s) * st3 + 2 * ld);
                d1n[s] = __ldg(d + (CH + s) * st3 + ld);
            }
            if (a.tl && blockIdx.x == 0 && lane == 0 && g < 64) a.tl[(warp * 64 + g) * 2] = clock64();
            if (g >= S) { const long long t0 = clock64(); nb_sync(7 + slot, nE); t_wait += clock_after(OV) - t0; }
            double* Ss = sm + slot * kSlot;
            unsigned ov = 0u;
#pragma unroll
            for (int s = 0; s < CH; ++s) {
                const X2Stage q = x2_stage<true>(x2p, v, p);
                Ss[(s * 4 + 0) * RW * 32 + ridx] = x2p;
                Ss[(s * 4 + 1) * RW * 32 + ridx] = q.a2;
                Ss[(s * 4 + 2) * RW * 32 + ridx] = q.b2;
                Ss[(s * 4 + 3) * RW * 32 + ridx] = q.c2;
                Ss[kG + (s * 2 + 0) * RW * 32 + ridx] = d0c[s];
                Ss[kG + (s * 2 + 1) * RW * 32 + ridx] = d2c[s];
                x2p = add(add(x2p, mul(p.c, q.s2)), d1c[s]);
                ov |= (fabs(x2p) <= kStateLimit ? 0u : 1u) << s;
            }
#pragma unroll
            for (int s = 0; s < CH; ++s) {
                d0c[s] = d0n[s];
                d2c[s] = d2n[s];
                d1c[s] = d1n[s];
            }
            OV[slot * RW * 32 + ridx] = ov;
            if (a.tl && blockIdx.x == 0 && lane == 0 && g < 64) a.tl[(warp * 64 + g) * 2 + 1] = clock64();
            nb_arrive(1 + slot, nG);
            d += CH * st3;
            slot = slot == S - 1 ? 0 : slot + 1;
        }
        prof_out();
        return;
    }
    // consumer
    double x1 = a.x0[0], x3 = a.x0[2];
    int status = kOk, steps = J;
    bool done = !live;
    if (live && !in_bounds(x1, p.ylo, p.yhi)) {
        steps = 0;
        status = kViolated;
        done = true;
    }
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
    int slot = 0;
    for (int g = 0; g < nch; ++g) {
        const long long t0 = clock64();
        const uint32_t tok = nb_sync_tok(4 + slot, nT);
        const long long t1 = clock_after(OV);
        t_wait += t1 - t0;
        if (a.tl && blockIdx.x == 0 && lane == 0 && g < 64) a.tl[(warp * 64 + g) * 2] = t1;
        const uint32_t ca = sbase + 8u * (uint32_t)(slot * kSlot + ridx) + tok;
        const unsigned ovc = OV[slot * RW * 32 + ridx];
        double t[CH][4], dd[CH][2];
#pragma unroll
        for (int s = 0; s < CH; ++s) {
#pragma unroll
            for (int k = 0; k < 4; ++k) t[s][k] = lds_nc(ca + 8u * ((s * 4 + k) * RW * 32));
            dd[s][0] = lds_nc(ca + 8u * (kG + (s * 2 + 0) * RW * 32));
            dd[s][1] = lds_nc(ca + 8u * (kG + (s * 2 + 1) * RW * 32));
        }
        // the slot is read out: the producer may refill it
        asm volatile("" ::: "memory");
        nb_arrive(7 + slot, nE);
#pragma unroll
        for (int s = 0; s < CH; ++s) {
            const int j = g * CH + s;
            x13_update<true>(x1, x3, t[s][0], t[s][1], t[s][2], t[s][3], p, dd[s][0], dd[s][1]);
            const bool ovf = !(fabs(x1) <= kStateLimit && !((ovc >> s) & 1u) &&
                               fabs(x3) <= kStateLimit);
            const bool bnd = !in_bounds(x1, p.ylo, p.yhi);
            const bool now = !done && j < J && (ovf || bnd);
            status = now ? (ovf ? kOverflow : kViolated) : status;
            steps = now ? j + 1 : steps;
            done = done || now;
        }
        if (a.tl && blockIdx.x == 0 && lane == 0 && g < 64) a.tl[(warp * 64 + g) * 2 + 1] = clock64() + (long long)(x1 == 12345.0);
        slot = slot == S - 1 ? 0 : slot + 1;
    }
    prof_out();
    if (live) {
        a.status[(int64_t)row * a.n_sim + sc] = status;
        a.steps[(int64_t)row * a.n_sim + sc] = steps;
    }
}

template <int TW, int RW, int CH>
float run_ts3(const TsArgs& a, int sms, int reps) {
    constexpr int kT = (TW + 2 * RW) * 32;
    const size_t smem = 3 * (size_t)CH * 6 * RW * 32 * 8 + 3 * RW * 32 * 4;
    CK(cudaFuncSetAttribute(k_ts3<TW, RW, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
    const int nblk = std::max(std::min(sms, a.units), (a.units + RW - 1) / RW);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    k_ts3<TW, RW, CH><<<nblk, kT, smem>>>(a);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> ts;
    for (int i = 0; i < reps; ++i) {
        CK(cudaEventRecord(e0));
        k_ts3<TW, RW, CH><<<nblk, kT, smem>>>(a);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
}

// reference: one thread per cell, the plain rollout over global memory
struct GSource {
    const double* d;
    int64_t ld;
    __device__ D3 load(int32_t j) const {
        const double* q = d + (int64_t)j * 3 * ld;
        return D3{q[0], q[ld], q[2 * ld]};
    }
};

__global__ void k_ref(TsArgs a, int M) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)M * a.n_sim) return;
    const int row = (int)(t / a.n_sim), sc = (int)(t % a.n_sim);
    GSource src{a.soa + sc, a.ld};
    int32_t steps = 0;
    const int st = rollout<true, false, GSource>(a.p, a.x0[0], a.x0[1], a.x0[2], a.vrow[row],
                                                   src, steps, nullptr, true);
    a.status[t] = st;
    a.steps[t] = steps;
}

template <int TW, int RW, int CH, int N>
float run_ts(const TsArgs& a, int nblk, int reps) {
    constexpr int kT = (TW + RW) * 32;
    const size_t smem = 3 * (size_t)CH * 4 * RW * 32 * 8 + 3 * RW * 32 * 4;
    CK(cudaFuncSetAttribute(k_ts<TW, RW, CH, N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    k_ts<TW, RW, CH, N><<<nblk, kT, smem>>>(a);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> ts;
    for (int i = 0; i < reps; ++i) {
        CK(cudaEventRecord(e0));
        k_ts<TW, RW, CH, N><<<nblk, kT, smem>>>(a);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
}

int main(int argc, char** argv) {
    const int n_sim = argc > 1 ? atoi(argv[1]) : 1000;
    const int M = argc > 2 ? atoi(argv[2]) : 32;
    const int transient = argc > 3 ? atoi(argv[3]) : 0;
    const int J = 256;
    const int64_t ld = (n_sim + 31) / 32 * 32;
    std::vector<double> h_soa((size_t)(J + 32) * 3 * ld, 0.0);
    std::mt19937_64 rng(7);
    const double amp = transient ? 0.02 : 0.001;
    std::uniform_real_distribution<double> U(-amp, amp);
    for (int j = 0; j < J; ++j)
        for (int c = 0; c < 3; ++c)
            for (int s = 0; s < n_sim; ++s) h_soa[((size_t)j * 3 + c) * ld + s] = U(rng);
    std::vector<double> vrow(M);
    for (int i = 0; i < M; ++i) vrow[i] = (transient ? 2.5 : 0.5) * (M > 1 ? i / (double)(M - 1) : 0.5);
    TsArgs a{};
    a.tl = nullptr;
    a.prof = nullptr;
    double *d_soa, *d_v;
    int *st_ref, *sp_ref, *st_ts, *sp_ts;
    CK(cudaMalloc(&d_soa, h_soa.size() * 8));
    CK(cudaMemcpy(d_soa, h_soa.data(), h_soa.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&d_v, M * 8));
    CK(cudaMemcpy(d_v, vrow.data(), M * 8, cudaMemcpyHostToDevice));
    const size_t ncell = (size_t)M * n_sim;
    CK(cudaMalloc(&st_ref, ncell * 4));
    CK(cudaMalloc(&sp_ref, ncell * 4));
    CK(cudaMalloc(&st_ts, ncell * 4));
    CK(cudaMalloc(&sp_ts, ncell * 4));
    a.soa = d_soa;
    a.ld = ld;
    a.n_sim = n_sim;
    a.W = (n_sim + 31) / 32;
    a.units = M * a.W;
    a.vrow = d_v;
    a.x0[0] = transient ? 0.3 : 0.0;
    a.x0[1] = transient ? -0.2 : 0.0;
    a.x0[2] = transient ? 0.1 : 0.0;
    a.p.h = 0.05;
    a.p.hh = 0.5 * 0.05;
    a.p.c = 0.05 / 6.0;
    a.p.ylo = -0.855;
    a.p.yhi = 0.855;
    a.p.j_star = J;
    a.status = st_ref;
    a.steps = sp_ref;
    k_ref<<<(unsigned)((ncell + 127) / 128), 128>>>(a, M);
    CK(cudaDeviceSynchronize());
    std::vector<int> h_st(ncell), h_sp(ncell), r_st(ncell), r_sp(ncell);
    CK(cudaMemcpy(r_st.data(), st_ref, ncell * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r_sp.data(), sp_ref, ncell * 4, cudaMemcpyDeviceToHost));
    int hist[4] = {0, 0, 0, 0};
    for (size_t i = 0; i < ncell; ++i) hist[r_st[i] & 3]++;
    printf("n_sim=%d M=%d transient=%d units=%d ref status: viol %d ok %d ovf %d\n", n_sim, M,
           transient, a.units, hist[0], hist[1], hist[2]);
    a.status = st_ts;
    a.steps = sp_ts;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    auto check = [&](const char* tag, float ms) {
        CK(cudaMemcpy(h_st.data(), st_ts, ncell * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(h_sp.data(), sp_ts, ncell * 4, cudaMemcpyDeviceToHost));
        size_t bad = 0;
        for (size_t i = 0; i < ncell; ++i) bad += h_st[i] != r_st[i] || h_sp[i] != r_sp[i];
        printf("%-28s %8.2f us  mismatches %zu\n", tag, ms * 1e3, bad);
        CK(cudaMemset(st_ts, 0xff, ncell * 4));
    };
    const int nblk = std::min(sms, a.units);
    long long* d_prof;
    CK(cudaMalloc(&d_prof, 4096 * 32 * 2 * 8));
    CK(cudaMemset(d_prof, 0, 4096 * 32 * 2 * 8));
    a.prof = d_prof;
    long long* d_tl;
    CK(cudaMalloc(&d_tl, 32 * 64 * 2 * 8));
    CK(cudaMemset(d_tl, 0, 32 * 64 * 2 * 8));
    a.tl = d_tl;
    check("v3 TW12 RW3 CH8", run_ts3<12, 3, 8>(a, sms, 50));
    {
        std::vector<long long> tl(32 * 64 * 2);
        CK(cudaMemcpy(tl.data(), d_tl, tl.size() * 8, cudaMemcpyDeviceToHost));
        const long long base = tl[(12 * 64 + 0) * 2];
        printf("  timeline (kcycles from P0 start): chunk: P0[start,arrive] T0[go,done] C0[go,done]\n");
        for (int g = 0; g < 32; g += 1)
            printf("   %2d: P %.2f %.2f | T %.2f %.2f | C %.2f %.2f\n", g,
                   (tl[(12 * 64 + g) * 2] - base) / 1e3, (tl[(12 * 64 + g) * 2 + 1] - base) / 1e3,
                   (tl[(0 * 64 + g) * 2] - base) / 1e3, (tl[(0 * 64 + g) * 2 + 1] - base) / 1e3,
                   (tl[(15 * 64 + g) * 2] - base) / 1e3, (tl[(15 * 64 + g) * 2 + 1] - base) / 1e3);
    }
    a.tl = nullptr;
    check("v3 TW8 RW3 CH8", run_ts3<8, 3, 8>(a, sms, 50));
    {
        std::vector<long long> hp(32 * 2 * 2);
        CK(cudaMemcpy(hp.data(), d_prof, hp.size() * 8, cudaMemcpyDeviceToHost));
        for (int b = 0; b < 2; ++b) {
            printf("  block %d (warp: wait/total kcycles):", b);
            for (int w = 0; w < 14; ++w)
                printf(" %s%d %.1f/%.1f", w < 8 ? "T" : (w < 11 ? "P" : "C"), w,
                       hp[(b * 32 + w) * 2] / 1e3, hp[(b * 32 + w) * 2 + 1] / 1e3);
            printf("\n");
        }
    }
    a.prof = nullptr;
    check("v3 TW4 RW3 CH8", run_ts3<4, 3, 8>(a, sms, 50));
    check("v3 TW4 RW1 CH8", run_ts3<4, 1, 8>(a, sms, 50));
    check("v3 TW8 RW1 CH8", run_ts3<8, 1, 8>(a, sms, 50));
    check("v3 TW8 RW3 CH4", run_ts3<8, 3, 4>(a, sms, 50));
    check("v2 TW8 RW3 CH8", run_ts2<8, 3, 8>(a, sms, 50));
    check("TW8 RW7 CH8 N4", run_ts<8, 7, 8, 4>(a, nblk, 50));
    // reference timing
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    a.status = st_ref;
    a.steps = sp_ref;
    std::vector<float> tr;
    for (int i = 0; i < 20; ++i) {
        CK(cudaEventRecord(e0));
        k_ref<<<(unsigned)((ncell + 127) / 128), 128>>>(a, M);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        tr.push_back(ms);
    }
    std::sort(tr.begin(), tr.end());
    printf("%-28s %8.2f us\n", "plain rollout (reference)", tr[10] * 1e3);
    return 0;
}
