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

// One cell.  POLL: every 32 steps check a row-level "already infeasible"
// flag and abandon (used only when the caller wants verdicts, not P).
//
// Software-pipelined two steps deep (see the loop): every value is still
// produced by the reference's operations on the reference's operands, so the
// bits are those of sfc_step.  Steps past an early exit or past the horizon are
// computed speculatively and never observed.
//
// WARP: the caller guarantees that all 32 lanes call, and the
// lanes then run as one: out-of-range and finished lanes keep computing
// throwaway values until every lane is done, the exit and the tanh range vote
// are full-warp votes, and the per-step checks are predicated into the
// iteration's single basic block (no divergent branches inside the loop).
//
// RAISE (with WARP and POLL): a lane whose cell violates or overflows sets
// *dead at once, so the other cells sharing the flag abandon at their next
// poll (the joint bisection's OR-reduced violation flag).
template <bool FMA, bool POLL, class Src, bool WARP = false, bool RAISE = false,
          bool MOD = false>
__device__ __forceinline__ int rollout(const CellConst& p, double x1, double x2, double x3,
                                       double v, const Src& src, int32_t& steps,
                                       const unsigned int* dead, bool live = true) {
    static_assert(!RAISE || (WARP && POLL), "RAISE needs the polled warp-uniform form");
    constexpr bool kUniform = WARP;  // all lanes run the loop together
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
    tanh4_auto<FMA>(x2, s0.a2, s0.b2, s0.c2, t1, t2, t3, t4);
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
        tanh4_with<FMA, WARP, decltype(side)&, MOD>(g0, g1, g2, g3, u1, u2, u3, u4, side);
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

// ---- two RK4 steps per loop iteration (the single-wave grid step) ------------
//
// At one or two resident warps per SM sub-partition (the C2 step) the rollout is
// latency-bound: rollout()'s iteration holds four tanh chains of ~30 dependent
// FP64 operations each.  rollout2 runs two steps per iteration, pipelined one
// step deeper: iteration j (j even) finishes x1/x3 of steps j and j+1 (tanh
// values from iteration j-2), evaluates the eight tanh of steps j+2 and j+3 side
// by side (arguments from iteration j-2) and runs the x2 chain of steps j+4 and
// j+5.  Twice the independent work per basic block at the same chain length.
// Every operation, operand and rounding is still sfc_step's.
//
// Sources: start() gives steps 0..3, next(j) steps j+4 and j+5 (clamped to J-1),
// into registers.  The staged source is a per-lane ring of two slot pairs in
// shared memory ([pair][slot][comp][lane], conflict-free): in iteration j one pair
// is read (steps j+4, j+5) and the other, read in iteration j-2, receives the
// cp.async copies of steps j+6, j+7; then the pairs swap roles.

constexpr int kRing4Stride = 256;  // threads per block of the two-step rollout, at most
#ifndef RG_RING_PAIRS
#define RG_RING_PAIRS 2
#endif
constexpr int kRing4Pairs = RG_RING_PAIRS;  // slot pairs in flight (2: double buffering)

struct Soa4Source {
    const double* d;  // already offset by k
    int64_t ld;
    double* ring;     // &ring[0][0][0][threadIdx.x] of a [kRing4Pairs][2][3][kRing4Stride] array
    const double* nxt = nullptr;   // next step to issue (clamped walk)
    const double* last = nullptr;  // step J-1
    int64_t stride = 0;
    uint32_t base = 0;  // shared-memory address of this lane's pair 0, slot 0, component 0
    uint32_t rd = 0;    // byte offset of the pair read in this iteration
    static constexpr uint32_t kComp = 8 * kRing4Stride, kSlot = 3 * kComp, kPair = 2 * kSlot;
    __device__ __forceinline__ void init(int32_t J) {
        stride = 3 * ld;
        nxt = d;
        last = d + (int64_t)(J - 1) * stride;
        base = (uint32_t)__cvta_generic_to_shared(ring);
        rd = 0;
    }
    __device__ __forceinline__ void issue_one(uint32_t sa) {
        const double* p1 = nxt + ld;
        const double* p2 = p1 + ld;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(nxt));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa + kComp), "l"(p1));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa + 2 * kComp), "l"(p2));
        nxt = nxt == last ? nxt : nxt + stride;
    }
    // the next two steps (in order) into the slot pair at byte offset `pair`
    __device__ __forceinline__ void issue_pair(uint32_t pair) {
        const uint32_t sa = base + pair;
        issue_one(sa);
        issue_one(sa + kSlot);
        asm volatile("cp.async.commit_group;");
    }
    // the oldest pair in flight has landed (kRing4Pairs - 2 younger groups may still fly)
    __device__ __forceinline__ void wait() {
        asm volatile("cp.async.wait_group %0;" ::"n"(kRing4Pairs - 2));
    }
    __device__ __forceinline__ static double lds(uint32_t a) {
        double v;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
        return v;
    }
    __device__ __forceinline__ void read_slot(uint32_t a, double (&o)[3]) const {
        o[0] = lds(a);
        o[1] = lds(a + kComp);
        o[2] = lds(a + 2 * kComp);
    }
    __device__ __forceinline__ uint32_t after(uint32_t off) const {
        return off + kPair == kRing4Pairs * kPair ? 0u : off + kPair;
    }
    // prologue: step pairs 0 .. kRing4Pairs-1 issued, pair 0 (steps 0, 1) read; pair 1 is
    // read by next(-2)
    __device__ __forceinline__ void start(double (&dd)[2][3]) {
#pragma unroll
        for (int q = 0; q < kRing4Pairs; ++q) issue_pair(q * kPair);
        asm volatile("cp.async.wait_group %0;" ::"n"(kRing4Pairs - 1));
        read_slot(base, dd[0]);
        read_slot(base + kSlot, dd[1]);
        rd = kPair;
    }
    // iteration j: pair (j+4)/2 (steps j+4, j+5) read from offset rd; the pair read in
    // iteration j-2 (the one before rd, now free) receives steps j+2+2*kRing4Pairs, +1
    __device__ __forceinline__ void next(int32_t, double (&e4)[3], double (&e5)[3]) {
        wait();
        const uint32_t a = base + rd;
        read_slot(a, e4);
        read_slot(a + kSlot, e5);
        if constexpr (kRing4Pairs == 2) {  // double buffering: the pairs swap roles
            rd = kPair - rd;
            issue_pair(rd);
        } else {
            const uint32_t freed = rd == 0 ? (kRing4Pairs - 1) * kPair : rd - kPair;
            rd = after(rd);
            issue_pair(freed);
        }
    }
    __device__ __forceinline__ void finish() { asm volatile("cp.async.wait_group 0;"); }
};

struct Rng4Source {  // fused counter RNG (micro-benchmarks)
    ScenarioStream st;
    uint64_t K;
    int32_t J = 0;
    __device__ __forceinline__ void init(int32_t j_star) { J = j_star; }
    __device__ __forceinline__ void at(int32_t s, double (&o)[3]) const {
        disturbance_at(st, K, (uint64_t)(s < J ? s : J - 1), o[0], o[1], o[2]);
    }
    __device__ __forceinline__ void start(double (&d)[2][3]) {
        at(0, d[0]);
        at(1, d[1]);
    }
    __device__ __forceinline__ void next(int32_t j, double (&e4)[3], double (&e5)[3]) {
        at(j + 4, e4);
        at(j + 5, e5);
    }
    __device__ __forceinline__ void finish() {}
};

struct Zero4Source {  // nominal prediction / micro-benchmarks
    __device__ __forceinline__ void init(int32_t) {}
    __device__ __forceinline__ void start(double (&d)[2][3]) {
        for (int s = 0; s < 2; ++s) d[s][0] = d[s][1] = d[s][2] = 0.0;
    }
    __device__ __forceinline__ void next(int32_t, double (&e4)[3], double (&e5)[3]) {
        e4[0] = e4[1] = e4[2] = e5[0] = e5[1] = e5[2] = 0.0;
    }
    __device__ __forceinline__ void finish() {}
};

// RAISE (with POLL): a lane whose cell violates or overflows sets *dead at once, as
// rollout<..., RAISE> does (the joint search's OR-reduced flag).
template <bool FMA, bool POLL, class Src, bool RAISE = false>
struct Rollout2 {
    static_assert(!RAISE || POLL, "RAISE needs the polled form");
    const CellConst& p;
    const double v;
    Src& src;
    const unsigned int* dead;
    int32_t J;
    double x1, x3;
    double y;         // x2 before step j+4
    double x2n1;      // x2 after step j (the first tanh argument of step j+1)
    double T[8];      // tanh values of steps j, j+1
    double G[8];      // tanh arguments of steps j+2, j+3
    double D[4];      // d0, d2 of steps j, j+1
    double Dn[4];     // d0, d2 of steps j+2, j+3
    int status = kOk;
    int32_t steps = 0;
    bool done = false;

    __device__ __forceinline__ Rollout2(const CellConst& p_, double v_, Src& src_,
                                        const unsigned int* dead_)
        : p(p_), v(v_), src(src_), dead(dead_), J(p_.j_star) {}

    // iteration j (even): true once every lane of the warp is done
    __device__ __forceinline__ bool iter(int32_t j) {
        double e4[3], e5[3];
        src.next(j, e4, e5);
        double Gn[8];
        double yn, x1j, x3j;
        auto side = [&]() {
            const X2Stage s4 = x2_stage<FMA>(y, v, p);
            const double y5 = add(add(y, mul(p.c, s4.s2)), e4[1]);
            const X2Stage s5 = x2_stage<FMA>(y5, v, p);
            yn = add(add(y5, mul(p.c, s5.s2)), e5[1]);
            Gn[0] = y;
            Gn[1] = s4.a2;
            Gn[2] = s4.b2;
            Gn[3] = s4.c2;
            Gn[4] = y5;
            Gn[5] = s5.a2;
            Gn[6] = s5.b2;
            Gn[7] = s5.c2;
            double u1 = x1, u3 = x3;
            x13_update<FMA>(u1, u3, T[0], T[1], T[2], T[3], p, D[0], D[1]);
            x1j = u1;
            x3j = u3;
            x13_update<FMA>(u1, u3, T[4], T[5], T[6], T[7], p, D[2], D[3]);
            // the pipeline-fill iteration (j = -2) has no steps j, j+1: its x1/x3
            // update runs on unset tanh values and is dropped
            x1 = j >= 0 ? u1 : x1;
            x3 = j >= 0 ? u3 : x3;
        };
        double U[8];
        tanhN_with<FMA, true, 8>(G, U, side);
        {  // step j: overflow, then the output bound (x2 after step j is x2n1)
            const bool ovf = !(fabs(x1j) <= kStateLimit && fabs(x2n1) <= kStateLimit &&
                               fabs(x3j) <= kStateLimit);
            const bool bnd = !in_bounds(x1j, p.ylo, p.yhi);
            const bool now = !done && j >= 0 && (ovf || bnd);
            status = now ? (ovf ? kOverflow : kViolated) : status;
            steps = now ? j + 1 : steps;
            done = done || now;
            if (RAISE && now) atomicOr((unsigned int*)dead, 1u);
        }
        {  // step j+1 inside the horizon: overflow, bound, then the poll (x2 after it: G[0])
            const bool ovf = !(fabs(x1) <= kStateLimit && fabs(G[0]) <= kStateLimit &&
                               fabs(x3) <= kStateLimit);
            const bool bnd = !in_bounds(x1, p.ylo, p.yhi);
            bool aband = false;
            if (POLL && ((j + 1) & 31) == 31) aband = *(volatile const unsigned int*)dead != 0u;
            const bool now = !done && j >= 0 && j + 1 < J && (ovf || bnd || aband);
            status = now ? (ovf ? kOverflow : (bnd ? kViolated : kAbandoned)) : status;
            steps = now ? j + 2 : steps;
            done = done || now;
            if (RAISE && now && (ovf || bnd)) atomicOr((unsigned int*)dead, 1u);
        }
        if (__all_sync(0xffffffffu, done)) return true;
#pragma unroll
        for (int q = 0; q < 8; ++q) T[q] = U[q];
        x2n1 = G[4];
#pragma unroll
        for (int q = 0; q < 8; ++q) G[q] = Gn[q];
        y = yn;
#pragma unroll
        for (int q = 0; q < 4; ++q) D[q] = Dn[q];
        Dn[0] = e4[0];
        Dn[1] = e4[2];
        Dn[2] = e5[0];
        Dn[3] = e5[2];
        return false;
    }

    __device__ __forceinline__ int run(double x1_0, double x2_0, double x3_0, bool live,
                                       int32_t& steps_out) {
        x1 = x1_0;
        x3 = x3_0;
        steps = J;
        done = !live;
        if (live && !in_bounds(x1, p.ylo, p.yhi)) {
            steps = 0;
            status = kViolated;
            done = true;
        }
        if (__all_sync(0xffffffffu, done)) {
            steps_out = steps;
            return status;
        }
        // prologue: the x2 chain of steps 0 and 1 (the tanh arguments G); the loop
        // starts with a pipeline-fill iteration j = -2 that evaluates their tanh and
        // the x2 chain of steps 2, 3 (so the tanh block has one copy in the code)
        src.init(J);
        double d[2][3];
        src.start(d);
        double yy = x2_0;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const X2Stage st = x2_stage<FMA>(yy, v, p);
            G[4 * s] = yy;
            G[4 * s + 1] = st.a2;
            G[4 * s + 2] = st.b2;
            G[4 * s + 3] = st.c2;
            yy = add(add(yy, mul(p.c, st.s2)), d[s][1]);
        }
        y = yy;
#pragma unroll
        for (int q = 0; q < 8; ++q) T[q] = 0.0;
        x2n1 = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) D[q] = 0.0;
        Dn[0] = d[0][0];
        Dn[1] = d[0][2];
        Dn[2] = d[1][0];
        Dn[3] = d[1][2];
        for (int32_t j = -2; j < J; j += 2)
            if (iter(j)) break;
        src.finish();  // no copy may land after we leave
        steps_out = steps;
        return status;
    }
};

// One cell, warp-uniform (all 32 lanes call, like rollout<..., WARP>), two steps per
// iteration; same status / steps semantics as rollout.
template <bool FMA, bool POLL, class Src, bool RAISE = false>
__device__ __forceinline__ int rollout2(const CellConst& p, double x1, double x2, double x3,
                                        double v, Src& src, int32_t& steps,
                                        const unsigned int* dead, bool live) {
    Rollout2<FMA, POLL, Src, RAISE> r(p, v, src, dead);
    return r.run(x1, x2, x3, live, steps);
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
