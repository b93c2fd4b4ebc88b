// rg_rng.cuh -- the reference's counter-based disturbance generator
// (disturbance.py:35-92, 179-203), host and device.
//
// u(seed, k, j, i) = (sm(sm(sm(sm(seed) ^ k) ^ j) ^ i) >> 11) * 2^-53 and the
// disturbance entry is lo_i + span_i * u (two IEEE roundings, as numpy does).
// All integer arithmetic wraps mod 2^64 like the numpy uint64 mirror.
// The chain factorises: K_k = sm(sm(seed) ^ k) once per scenario,
// J = sm(K_k ^ j) once per scenario-step, then one sm per state component --
// the rollout kernels generate a step's three entries from one J.
#pragma once

#include "rg_math.cuh"

namespace rg {

RG_HD uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// (H >> 11) * 2^-53: the 53-bit integer converts exactly; the scale is exact.
RG_HD double unit_double(uint64_t h) {
#if defined(__CUDA_ARCH__)
    return __dmul_rn(__ull2double_rn(h >> 11), 0x1p-53);
#else
    return (double)(h >> 11) * 0x1p-53;
#endif
}

// Per-shard constants of a scenario set: hs = sm(seed), lo/span per state.
struct ScenarioStream {
    uint64_t hs;
    double lo[3];
    double span[3];
};

RG_HD uint64_t scenario_key(const ScenarioStream& s, uint64_t k) { return splitmix64(s.hs ^ k); }

// The three disturbance entries of scenario key K at step j.
RG_HD void disturbance_at(const ScenarioStream& s, uint64_t K, uint64_t j, double& d0,
                          double& d1, double& d2) {
    const uint64_t J = splitmix64(K ^ j);
    d0 = add(s.lo[0], mul(s.span[0], unit_double(splitmix64(J ^ 0ull))));
    d1 = add(s.lo[1], mul(s.span[1], unit_double(splitmix64(J ^ 1ull))));
    d2 = add(s.lo[2], mul(s.span[2], unit_double(splitmix64(J ^ 2ull))));
}

}  // namespace rg
