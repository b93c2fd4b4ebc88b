// Rollout throughput vs warps per SM sub-partition: one block per SM (forced by
// dynamic shared memory), 128*W threads, every thread one cell of the bench
// snapshot (x0 = 0, v in [0.25, 0.5], zero disturbance).  Prints cycles per
// step per SMSP and per warp.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2510_08288_b200/csrc/rg_cell.cuh"

using namespace rg;

// SRC: 0 zero, 1 staged SoA through the cp.async ring, 2 fused counter RNG
// STEP2: rollout2 (two steps per iteration) instead of rollout
template <bool WARP, int SRC, bool STEP2 = false>
__global__ void __launch_bounds__(STEP2 ? 256 : 512, 1) probe(int J, int* out, const double* soa, int64_t ld) {
    extern __shared__ double dyn[];
    CellConst c;
    c.h = 0.01; c.hh = 0.005; c.c = 0.01 / 6.0; c.ylo = -0.9; c.yhi = 0.9; c.j_star = J;
    const double v = 0.5 * (0.5 + 0.5 * (threadIdx.x & 31) / 31.0);
    int32_t steps = 0;
    int st;
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (STEP2) {
        if (SRC == 0) {
            Zero4Source src;
            st = rollout2<true, false>(c, 0.0, 0.0, 0.0, v, src, steps, nullptr, true);
        } else if (SRC == 1) {
            Soa4Source src;
            src.d = soa + k;
            src.ld = ld;
            src.ring = dyn + threadIdx.x;  // [4][3][256] needs blockDim <= 256
            st = rollout2<true, false>(c, 0.0, 0.0, 0.0, v, src, steps, nullptr, true);
        } else {
            ScenarioStream ss;
            ss.hs = 12345;
            for (int q = 0; q < 3; ++q) { ss.lo[q] = -0.001; ss.span[q] = 0.002; }
            Rng4Source src{ss, scenario_key(ss, (uint64_t)k), 0};
            st = rollout2<true, false>(c, 0.0, 0.0, 0.0, v, src, steps, nullptr, true);
        }
    } else if (SRC == 0) {
        st = rollout<true, false, 1, ZeroSource, WARP>(c, 0.0, 0.0, 0.0, v, ZeroSource{}, steps,
                                                       nullptr, true);
    } else if (SRC == 1) {
        SoaSource src{soa + k, ld, dyn + threadIdx.x};
        st = rollout<true, false, 1, SoaSource, WARP>(c, 0.0, 0.0, 0.0, v, src, steps, nullptr,
                                                      true);
    } else {
        ScenarioStream ss;
        ss.hs = 12345;
        for (int q = 0; q < 3; ++q) { ss.lo[q] = -0.001; ss.span[q] = 0.002; }
        RngSource src{ss, scenario_key(ss, (uint64_t)k)};
        st = rollout<true, false, 1, RngSource, WARP>(c, 0.0, 0.0, 0.0, v, src, steps, nullptr,
                                                      true);
    }
    if (st == 77 && steps == 3) out[0] = (int)dyn[0];
}

int main() {
    int* out; cudaMalloc(&out, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = 160 * 1024;
    cudaFuncSetAttribute(probe<true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<true, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<true, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<true, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int J = 1024;
    const int64_t ld = (int64_t)sms * 512;
    double* soa;
    cudaMalloc(&soa, (size_t)J * 3 * ld * sizeof(double));
    cudaMemset(soa, 0, (size_t)J * 3 * ld * sizeof(double));
    for (int W = 1; W <= 4; ++W) {
        for (int warp = 0; warp < 6; ++warp) {
            if (warp >= 3 && W > 2) continue;  // rollout2's ring: blocks of <= 256 threads
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            auto go = [&]() {
                if (warp == 0) probe<true, 0><<<sms, 128 * W, smem>>>(J, out, soa, ld);
                else if (warp == 1) probe<true, 1><<<sms, 128 * W, smem>>>(J, out, soa, ld);
                else if (warp == 2) probe<true, 2><<<sms, 128 * W, smem>>>(J, out, soa, ld);
                else if (warp == 3) probe<true, 0, true><<<sms, 128 * W, smem>>>(J, out, soa, ld);
                else if (warp == 4) probe<true, 1, true><<<sms, 128 * W, smem>>>(J, out, soa, ld);
                else probe<true, 2, true><<<sms, 128 * W, smem>>>(J, out, soa, ld);
            };
            go();
            cudaEventRecord(a);
            go();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            const double cyc = ms * 1e-3 * 1.965e9 / J;
            printf("W=%d warps/SMSP SRC=%d STEP2=%d: %.0f cycles/step per SMSP, %.0f per warp-step (%s)\n",
                   W, warp % 3, warp >= 3, cyc, cyc / W, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
