// rg_cell.cuh -- one (candidate setpoint, scenario) cell of the surrogate
// fuel-cell plant on the device: kernels.py:47-86 (_cell_sfc).
//
// The state lives in registers for the whole horizon; the output-bound and
// overflow checks are fused into every step and exit early, so no trajectory
// is ever written to memory.  Arithmetic is the reference's exactly: 58
// separately rounded IEEE operations per step in Python's evaluation order
// plus four calls of the bit-exact glibc tanh port (rg_math.cuh).
//
// Reordering for ILP without changing a bit: the four tanh arguments
// (x2, a2, b2, c2) depend only on the x2 chain (dx2/dt = -x2 + v), so the
// chain is computed first and the four tanh evaluations are independent of
// each other -- the scheduler can overlap them.  Every individual operation,
// and the operands it rounds, is unchanged.
#pragma once

#include "rg_math.cuh"
#include "rg_rng.cuh"

#include <type_traits>

#ifndef RG_UNROLL
#define RG_UNROLL 2
#endif
#define RG_PRAGMA(x) _Pragma(#x)
#define RG_UNROLL_PRAGMA(n) RG_PRAGMA(unroll n)

namespace rg {

enum CellStatus : int { kViolated = 0, kOk = 1, kOverflow = 2, kAbandoned = 3 };

constexpr double kStateLimit = 1e6;  // kernels.py:42

struct CellConst {
    double h;    // plant.step_size
    double hh;   // 0.5 * h  (Python evaluates 0.5 * h * k as (0.5*h)*k)
    double c;    // h / 6.0
    double ylo;  // cset.lower
    double yhi;  // cset.upper
    int32_t j_star;
};

RG_HD bool in_bounds(double y, double lo, double hi) { return lo <= y && y <= hi; }

// x_{j+1} = RK4(x_j, v) + d_j with Python's operation order (kernels.py:56-79).
// Reference form: used by the host self-test and as the specification of the
// pipelined rollout below.
template <bool FMA>
RG_HD void sfc_step(double& x1, double& x2, double& x3, double v, const CellConst& p,
                    double d0, double d1, double d2) {
    const double h = p.h, hh = p.hh;
    const double k12 = add(-x2, v);
    const double a2 = add(x2, mul(hh, k12));
    const double k22 = add(-a2, v);
    const double b2 = add(x2, mul(hh, k22));
    const double k32 = add(-b2, v);
    const double c2 = add(x2, mul(h, k32));
    const double k42 = add(-c2, v);
    double t1, t2, t3, t4;
    tanh4<FMA>(x2, a2, b2, c2, t1, t2, t3, t4);
    const double k11 = add(-x1, t1);
    const double k13 = add(mul(-2.0, x3), x1);
    const double a1 = add(x1, mul(hh, k11));
    const double a3 = add(x3, mul(hh, k13));
    const double k21 = add(-a1, t2);
    const double k23 = add(mul(-2.0, a3), a1);
    const double b1 = add(x1, mul(hh, k21));
    const double b3 = add(x3, mul(hh, k23));
    const double k31 = add(-b1, t3);
    const double k33 = add(mul(-2.0, b3), b1);
    const double c1 = add(x1, mul(h, k31));
    const double c3 = add(x3, mul(h, k33));
    const double k41 = add(-c1, t4);
    const double k43 = add(mul(-2.0, c3), c1);
    const double s1 = add(add(add(k11, mul(2.0, k21)), mul(2.0, k31)), k41);
    const double s2 = add(add(add(k12, mul(2.0, k22)), mul(2.0, k32)), k42);
    const double s3 = add(add(add(k13, mul(2.0, k23)), mul(2.0, k33)), k43);
    x1 = add(add(x1, mul(p.c, s1)), d0);
    x2 = add(add(x2, mul(p.c, s2)), d1);
    x3 = add(add(x3, mul(p.c, s3)), d2);
}

// The step's products by +-2 are exact (a power-of-two scaling), so the
// reference's add(mul(2, b), a) rounds once, exactly like fma(2, b, a): one
// FP64 instruction instead of two, the same bits.  The one exception is a
// product that overflows, which needs a state component beyond 2^1021 at
// the start of a step -- only possible in an absurd initial state (every later
// state passed the 1e6 check).  Such a step ends with a component far beyond
// STATE_LIMIT (or inf/NaN) under either evaluation, so status and step count
// are still the reference's.
RG_HD double sum2(double a, double b) { return fma_(2.0, b, a); }      // a + 2*b
RG_HD double neg2_add(double b, double a) { return fma_(-2.0, b, a); }  // -2*b + a

// The x2 sub-chain of one step: dx2/dt = -x2 + v does not involve x1 or x3,
// so the stage values a2, b2, c2 (the tanh arguments) and the increment s2
// depend on x2 alone.
struct X2Stage {
    double a2, b2, c2, s2;
};

template <bool FMA>
RG_HD X2Stage x2_stage(double x2, double v, const CellConst& p) {
    X2Stage r;
    const double k12 = add(-x2, v);
    r.a2 = add(x2, mul(p.hh, k12));
    const double k22 = add(-r.a2, v);
    r.b2 = add(x2, mul(p.hh, k22));
    const double k32 = add(-r.b2, v);
    r.c2 = add(x2, mul(p.h, k32));
    const double k42 = add(-r.c2, v);
    r.s2 = add(sum2(sum2(k12, k22), k32), k42);
    return r;
}

// The x1/x3 part of one step given the step's four tanh values.
template <bool FMA>
RG_HD void x13_update(double& x1, double& x3, double t1, double t2, double t3, double t4,
                      const CellConst& p, double d0, double d2) {
    const double h = p.h, hh = p.hh;
    const double k11 = add(-x1, t1);
    const double k13 = neg2_add(x3, x1);
    const double a1 = add(x1, mul(hh, k11));
    const double a3 = add(x3, mul(hh, k13));
    const double k21 = add(-a1, t2);
    const double k23 = neg2_add(a3, a1);
    const double b1 = add(x1, mul(hh, k21));
    const double b3 = add(x3, mul(hh, k23));
    const double k31 = add(-b1, t3);
    const double k33 = neg2_add(b3, b1);
    const double c1 = add(x1, mul(h, k31));
    const double c3 = add(x3, mul(h, k33));
    const double k41 = add(-c1, t4);
    const double k43 = neg2_add(c3, c1);
    const double s1 = add(sum2(sum2(k11, k21), k31), k41);
    const double s3 = add(sum2(sum2(k13, k23), k33), k43);
    x1 = add(add(x1, mul(p.c, s1)), d0);
    x3 = add(add(x3, mul(p.c, s3)), d2);
}

// ---- disturbance sources ---------------------------------------------------

struct D3 {
    double d0, d1, d2;
};

constexpr int kRingStride = 256;  // max threads per block of the rollout kernels

// Fused counter RNG: the scenario tensor never exists in memory.
struct RngSource {
    ScenarioStream s;
    uint64_t K;  // sm(sm(seed) ^ k)
    RG_HD D3 load(int32_t j) const {
        D3 r;
        disturbance_at(s, K, (uint64_t)j, r.d0, r.d1, r.d2);
        return r;
    }
};

// Staged structure-of-arrays tensor d[(j*3 + i) * ld + k] (coalesced across k).
// The rollout streams it through a two-slot per-thread ring in shared memory
// filled with cp.async two steps ahead of use, so no register ever waits on
// an in-flight L2 load (ring layout [slot][comp][thread]: conflict-free).
struct SoaSource {
    const double* d;  // already offset by k
    int64_t ld;       // padded scenario count
    double* ring;     // &ring[0][0][threadIdx.x] of a [2][3][RING_STRIDE] array
    __device__ __forceinline__ D3 load(int32_t j) const {
        const double* p = d + (int64_t)j * 3 * ld;
        return D3{__ldg(p), __ldg(p + ld), __ldg(p + 2 * ld)};
    }
    __device__ __forceinline__ void issue(int32_t j, int slot) const {
        const double* p = d + (int64_t)j * 3 * ld;
        double* r = ring + slot * 3 * kRingStride;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(r + i * kRingStride);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(p + i * ld));
        }
    }
    __device__ __forceinline__ D3 read(int slot) const {
        const double* r = ring + slot * 3 * kRingStride;
        return D3{r[0], r[kRingStride], r[2 * kRingStride]};
    }
    // issue() from a precomputed step pointer p = d + j*3*ld (the rollout
    // walks the steps in order, so it advances p instead of multiplying)
    __device__ __forceinline__ void issue_at(const double* p, int slot) const {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(ring + slot * 3 * kRingStride);
        const double* p1 = p + ld;
        const double* p2 = p1 + ld;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(p));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa + 8 * kRingStride),
                     "l"(p1));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa + 16 * kRingStride),
                     "l"(p2));
    }
};

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// Nominal prediction (bisection_rg: zero disturbance, governor.py:448).
struct ZeroSource {
    RG_HD D3 load(int32_t) const { return D3{0.0, 0.0, 0.0}; }
};

// The four tanh values of one step.  LPC lanes cooperate on a cell: with
// LPC = 2 each lane of a pair evaluates two of the four (in lockstep) and the
// pair swaps results with one shuffle per value; with LPC = 4 each lane
// evaluates one.  ptxas serialises independent tanh chains inside a thread,
// so spreading them over lanes turns ILP the compiler will not schedule into
// TLP the warp schedulers do.  Every lane ends with all four values.
template <bool FMA, int LPC>
__device__ __forceinline__ void step_tanh(double x2, double a2, double b2, double c2,
                                          double& u1, double& u2, double& u3, double& u4) {
    if constexpr (LPC == 1) {
        tanh4_auto<FMA>(x2, a2, b2, c2, u1, u2, u3, u4);
    } else if constexpr (LPC == 2) {
        const bool q = (threadIdx.x & 1u) != 0;
        const double in[2] = {q ? a2 : x2, q ? c2 : b2};
        double out[2];
        tanh_lockstep<FMA, 2>(in, out);
        const double o0 = __shfl_xor_sync(0xffffffffu, out[0], 1);
        const double o1 = __shfl_xor_sync(0xffffffffu, out[1], 1);
        u1 = q ? o0 : out[0];
        u2 = q ? out[0] : o0;
        u3 = q ? o1 : out[1];
        u4 = q ? out[1] : o1;
    } else {
        const unsigned q = threadIdx.x & 3u;
        const double in[1] = {q == 0 ? x2 : (q == 1 ? a2 : (q == 2 ? b2 : c2))};
        double out[1];
        tanh_lockstep<FMA, 1>(in, out);
        const int base = (int)(threadIdx.x & 31u) & ~3;
        u1 = __shfl_sync(0xffffffffu, out[0], base + 0);
        u2 = __shfl_sync(0xffffffffu, out[0], base + 1);
        u3 = __shfl_sync(0xffffffffu, out[0], base + 2);
        u4 = __shfl_sync(0xffffffffu, out[0], base + 3);
    }
}

// One cell.  POLL: every 32 steps check a row-level "already infeasible"
// flag and abandon (used only when the caller wants verdicts, not P).
//
// Software-pipelined two steps deep (see the loop): every value is still
// produced by the reference's operations on the reference's operands, so the
// bits are those of sfc_step.  Steps past an early exit or past the horizon are
// computed speculatively and never observed.
//
// LPC > 1: all 32 lanes of the warp run the loop until every cell of the warp
// is done (lanes of finished or out-of-range cells keep computing throwaway
// values), so the shuffles in step_tanh always see full warps.  `live` marks
// lanes whose cell exists.
//
// WARP (LPC = 1 only): the caller guarantees that all 32 lanes call, and the
// lanes then run as one: out-of-range and finished lanes keep computing
// throwaway values until every lane is done, the exit and the tanh range vote
// are full-warp votes, and the per-step checks are predicated into the
// iteration's single basic block (no divergent branches inside the loop).
//
// RAISE (with WARP and POLL): a lane whose cell violates or overflows sets
// *dead at once, so the other cells sharing the flag abandon at their next
// poll (the joint bisection's OR-reduced violation flag).
template <bool FMA, bool POLL, int LPC, class Src, bool WARP = false, bool RAISE = false,
          bool MOD = false>
__device__ __forceinline__ int rollout(const CellConst& p, double x1, double x2, double x3,
                                       double v, const Src& src, int32_t& steps,
                                       const unsigned int* dead, bool live = true) {
    static_assert(!RAISE || (WARP && POLL), "RAISE needs the polled warp-uniform form");
    static_assert(!WARP || LPC == 1, "WARP is the one-lane-per-cell form");
    constexpr bool kUniform = WARP || LPC > 1;  // all lanes run the loop together
    const int32_t J = p.j_star;
    constexpr bool kRing = std::is_same<Src, SoaSource>::value;
    int status = kOk;
    steps = J;
    bool done = !live;
    if (live && !in_bounds(x1, p.ylo, p.yhi)) {
        steps = 0;
        status = kViolated;
        done = true;
    }
    if constexpr (!kUniform) {
        if (done) return status;
    } else {
        if (__all_sync(0xffffffffu, done)) return status;
    }
    // Pipelined two steps deep: iteration j finishes x1/x3 of step j (tanh
    // values from iteration j-1), evaluates the four tanh of step j+1
    // (arguments from iteration j-1) and runs the x2 chain of step j+2.  The
    // three pieces are mutually independent, so the tanh chains no longer
    // wait behind the x2 recurrence inside an iteration.
    // staged source: the next step to issue, as a pointer (steps 2, 3, ..., J-1, J-1, ...)
    const double* nxt = nullptr;
    const double* last = nullptr;
    int64_t stride = 0;
    if constexpr (kRing) {
        stride = 3 * src.ld;
        nxt = src.d + (J > 2 ? 2 : J - 1) * stride;
        last = src.d + (int64_t)(J - 1) * stride;
    }
    auto fetch = [&](int32_t j) -> D3 {  // disturbances of step min(j, J-1)
        if constexpr (kRing) {
            cp_async_wait<1>();          // step j landed (issued two fetches ago)
            const D3 r = src.read(j & 1);
            src.issue_at(nxt, j & 1);    // step min(j + 2, J - 1)
            nxt = nxt == last ? nxt : nxt + stride;
            cp_async_commit();
            return r;
        } else {
            return src.load(j < J ? j : J - 1);
        }
    };
    if constexpr (kRing) {
        src.issue(0, 0);
        cp_async_commit();
        src.issue(J > 1 ? 1 : 0, 1);
        cp_async_commit();
    }
    const D3 dj0 = fetch(0);
    const D3 dj1 = fetch(1);
    // step 0: tanh values, x2 after step 0
    const X2Stage s0 = x2_stage<FMA>(x2, v, p);
    double t1, t2, t3, t4;
    step_tanh<FMA, LPC>(x2, s0.a2, s0.b2, s0.c2, t1, t2, t3, t4);
    const double y1 = add(add(x2, mul(p.c, s0.s2)), dj0.d1);
    // step 1: tanh arguments, x2 after step 1
    const X2Stage s1 = x2_stage<FMA>(y1, v, p);
    double g0 = y1, g1 = s1.a2, g2 = s1.b2, g3 = s1.c2;  // tanh arguments of step j+1
    double y2 = add(add(y1, mul(p.c, s1.s2)), dj1.d1);  // x2 before step j+2
    double dA0 = dj0.d0, dA2 = dj0.d2;  // x1/x3 disturbances of step j
    double dB0 = dj1.d0, dB2 = dj1.d2;  // ... and of step j+1
    RG_UNROLL_PRAGMA(RG_UNROLL)
    for (int32_t j = 0; j < J; ++j) {
        const D3 dn = fetch(j + 2);
        // step j+2's x2 chain and step j's x1/x3: independent of the tanh
        // values of step j+1 evaluated alongside (speculative past an exit)
        X2Stage sn;
        double y3;
        bool bad_ovf, bad_bnd;
        auto side = [&]() {
            sn = x2_stage<FMA>(y2, v, p);
            y3 = add(add(y2, mul(p.c, sn.s2)), dn.d1);
            x13_update<FMA>(x1, x3, t1, t2, t3, t4, p, dA0, dA2);
            // step j's checks (x2 after step j is g0), as predicates
            bad_ovf = !(fabs(x1) <= kStateLimit && fabs(g0) <= kStateLimit &&
                        fabs(x3) <= kStateLimit);
            bad_bnd = !in_bounds(x1, p.ylo, p.yhi);
        };
        double u1, u2, u3, u4;
        if constexpr (LPC == 1) {
            tanh4_with<FMA, WARP, decltype(side)&, MOD>(g0, g1, g2, g3, u1, u2, u3, u4, side);
        } else {
            step_tanh<FMA, LPC>(g0, g1, g2, g3, u1, u2, u3, u4);
            side();
        }
        if constexpr (WARP) {
            // the reference's order: overflow, then the output bound, then the poll
            bool aband = false;
            if (POLL && (j & 31) == 31) aband = *(volatile const unsigned int*)dead != 0u;
            const bool now = !done && (bad_ovf || bad_bnd || aband);
            const int code = bad_ovf ? kOverflow : (bad_bnd ? kViolated : kAbandoned);
            status = now ? code : status;
            steps = now ? j + 1 : steps;
            done = done || now;
            if (RAISE && now && code != kAbandoned) atomicOr((unsigned int*)dead, 1u);
        } else if (!done) {
            if (bad_ovf) {
                steps = j + 1;
                status = kOverflow;
                done = true;
            } else if (bad_bnd) {
                steps = j + 1;
                status = kViolated;
                done = true;
            } else if (POLL && (j & 31) == 31 &&
                       *(volatile const unsigned int*)dead != 0u) {
                steps = j + 1;
                status = kAbandoned;
                done = true;
            }
        }
        if constexpr (!kUniform) {
            if (done) break;
        } else {
            if (__all_sync(0xffffffffu, done)) break;
        }
        t1 = u1;
        t2 = u2;
        t3 = u3;
        t4 = u4;
        g0 = y2;
        g1 = sn.a2;
        g2 = sn.b2;
        g3 = sn.c2;
        y2 = y3;
        dA0 = dB0;
        dA2 = dB2;
        dB0 = dn.d0;
        dB2 = dn.d2;
    }
    if constexpr (kRing) cp_async_wait<0>();  // no copy may land after we leave
    return status;
}

// ---- linear plant: kernels.py:90-118 (_cell_lin) ----------------------------
//
// x+ = A x + B v + d, y = C x + D v with n <= 4 states; numba evaluates
// `s += A[i, l] * x[l]` as a separate multiply and add, in this order.

struct LinPlant {
    int32_t n;
    double A[16];  // row-major n x n
    double B[4], C[4], D;
    double gain, tlo, thi;  // steady-state gate: tlo <= gain * v <= thi
};

template <int N>
struct LinSoaSource {  // d[(j*N + i) * ld + k]
    const double* d;
    int64_t ld;
    __device__ __forceinline__ double at(int32_t j, int i) const {
        return __ldg(d + ((int64_t)j * N + i) * ld);
    }
};

template <int N>
struct LinRngSource {
    uint64_t K;
    double lo[4], span[4];
    __device__ __forceinline__ void step(int32_t j, double (&d)[N]) const {
        const uint64_t J = splitmix64(K ^ (uint64_t)j);
#pragma unroll
        for (int i = 0; i < N; ++i)
            d[i] = add(lo[i], mul(span[i], unit_double(splitmix64(J ^ (uint64_t)i))));
    }
};

template <int N>
__device__ __forceinline__ double lin_output(const LinPlant& L, const double (&x)[N], double v) {
    double y = mul(L.D, v);
#pragma unroll
    for (int l = 0; l < N; ++l) y = add(y, mul(L.C[l], x[l]));
    return y;
}

template <int N, bool RNG, class Src>
__device__ int rollout_lin(const LinPlant& L, const CellConst& p, const double* x0, double v,
                           const Src& src, int32_t& steps) {
    double x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = x0[i];
    if (!in_bounds(lin_output<N>(L, x, v), p.ylo, p.yhi)) {
        steps = 0;
        return kViolated;
    }
    for (int32_t j = 0; j < p.j_star; ++j) {
        double d[N];
        if constexpr (RNG) {
            src.step(j, d);
        } else {
#pragma unroll
            for (int i = 0; i < N; ++i) d[i] = src.at(j, i);
        }
        double xn[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
            double s = mul(L.B[i], v);
#pragma unroll
            for (int l = 0; l < N; ++l) s = add(s, mul(L.A[i * N + l], x[l]));
            xn[i] = add(s, d[i]);
        }
        bool ok = true;
#pragma unroll
        for (int i = 0; i < N; ++i) {
            x[i] = xn[i];
            ok = ok && fabs(x[i]) <= kStateLimit;
        }
        if (!ok) {
            steps = j + 1;
            return kOverflow;
        }
        if (!in_bounds(lin_output<N>(L, x, v), p.ylo, p.yhi)) {
            steps = j + 1;
            return kViolated;
        }
    }
    steps = p.j_star;
    return kOk;
}

// governor.py:151-159: exact at both endpoints, three roundings otherwise.
RG_HD double update_setpoint(double v_prev, double r, double kappa) {
    if (kappa == 0.0) return v_prev;
    if (kappa == 1.0) return r;
    return add(v_prev, mul(kappa, sub(r, v_prev)));
}

}  // namespace rg
