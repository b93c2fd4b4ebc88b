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
template <bool FMA>
RG_HD void sfc_step(double& x1, double& x2, double& x3, double v, const CellConst& p,
                    double d0, double d1, double d2) {
    const double h = p.h, hh = p.hh;
    // x2 chain (no tanh): k12, a2, k22, b2, k32, c2, k42
    const double k12 = add(-x2, v);
    const double a2 = add(x2, mul(hh, k12));
    const double k22 = add(-a2, v);
    const double b2 = add(x2, mul(hh, k22));
    const double k32 = add(-b2, v);
    const double c2 = add(x2, mul(h, k32));
    const double k42 = add(-c2, v);
    // four independent tanh evaluations
    const double t1 = tanh_glibc<FMA>(x2);
    const double t2 = tanh_glibc<FMA>(a2);
    const double t3 = tanh_glibc<FMA>(b2);
    const double t4 = tanh_glibc<FMA>(c2);
    // x1 / x3 chains
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
    // x + c*(((k1 + 2 k2) + 2 k3) + k4) + d
    const double s1 = add(add(add(k11, mul(2.0, k21)), mul(2.0, k31)), k41);
    const double s2 = add(add(add(k12, mul(2.0, k22)), mul(2.0, k32)), k42);
    const double s3 = add(add(add(k13, mul(2.0, k23)), mul(2.0, k33)), k43);
    x1 = add(add(x1, mul(p.c, s1)), d0);
    x2 = add(add(x2, mul(p.c, s2)), d1);
    x3 = add(add(x3, mul(p.c, s3)), d2);
}

// ---- disturbance sources ---------------------------------------------------

// Fused counter RNG: the scenario tensor never exists in memory.
struct RngSource {
    ScenarioStream s;
    uint64_t K;  // sm(sm(seed) ^ k)
    RG_HD void get(int32_t j, double& d0, double& d1, double& d2) const {
        disturbance_at(s, K, (uint64_t)j, d0, d1, d2);
    }
};

// Staged structure-of-arrays tensor d[(j*3 + i) * ld + k] (coalesced across k).
struct SoaSource {
    const double* d;  // already offset by k
    int64_t ld;       // padded scenario count
    __device__ __forceinline__ void get(int32_t j, double& d0, double& d1, double& d2) const {
        const double* p = d + (int64_t)j * 3 * ld;
        d0 = __ldg(p);
        d1 = __ldg(p + ld);
        d2 = __ldg(p + 2 * ld);
    }
};

// Nominal prediction (bisection_rg: zero disturbance, governor.py:448).
struct ZeroSource {
    RG_HD void get(int32_t, double& d0, double& d1, double& d2) const { d0 = d1 = d2 = 0.0; }
};

// One cell.  POLL: every 32 steps check a row-level "already infeasible"
// flag and abandon (used only when the caller wants verdicts, not P).
template <bool FMA, bool POLL, class Src>
__device__ __forceinline__ int rollout(const CellConst& p, double x1, double x2, double x3,
                                       double v, const Src& src, int32_t& steps,
                                       const unsigned int* dead) {
    if (!in_bounds(x1, p.ylo, p.yhi)) {
        steps = 0;
        return kViolated;
    }
    for (int32_t j = 0; j < p.j_star; ++j) {
        double d0, d1, d2;
        src.get(j, d0, d1, d2);
        sfc_step<FMA>(x1, x2, x3, v, p, d0, d1, d2);
        if (!(fabs(x1) <= kStateLimit && fabs(x2) <= kStateLimit && fabs(x3) <= kStateLimit)) {
            steps = j + 1;
            return kOverflow;
        }
        if (!in_bounds(x1, p.ylo, p.yhi)) {
            steps = j + 1;
            return kViolated;
        }
        if (POLL && (j & 31) == 31) {
            if (*(volatile const unsigned int*)dead != 0u) {
                steps = j + 1;
                return kAbandoned;
            }
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
