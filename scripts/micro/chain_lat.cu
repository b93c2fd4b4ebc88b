// Per-step latency of the RK4 recurrences on one warp (cycles per step):
// the x2 chain (x2_stage + update), the x1/x3 chain (x13_update), each with and without
// the per-step checks.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   --fmad=false -I paper_2510_08288_b200/csrc -o scripts/micro/chain_lat scripts/micro/chain_lat.cu
#include <cstdio>
#include "rg_cell.cuh"
using namespace rg;

template <int MODE>
__global__ void k_chain(const double* dv, double* out, long long* cyc, int J) {
    CellConst p;
    p.h = 0.05; p.hh = 0.025; p.c = 0.05 / 6.0; p.ylo = -0.855; p.yhi = 0.855; p.j_star = J;
    const int lane = threadIdx.x & 31;
    double x1 = dv[lane] * 0.1, x2 = dv[lane + 32] * 0.1, x3 = dv[lane + 64] * 0.1;
    const double v = 0.25 + dv[lane] * 1e-3;
    double t1 = 0.1, t2 = 0.11, t3 = 0.12, t4 = 0.13;
    int status = kOk, steps = J;
    bool done = false;
    const long long t0 = clock64();
    for (int j = 0; j < J; ++j) {
        const double d0 = dv[96 + (j & 31)] * 1e-3, d1 = dv[128 + (j & 31)] * 1e-3,
                     d2 = dv[160 + (j & 31)] * 1e-3;
        if (MODE == 0 || MODE == 2) {  // x2 chain
            const X2Stage q = x2_stage<true>(x2, v, p);
            x2 = add(add(x2, mul(p.c, q.s2)), d1);
            t1 += q.a2 * 1e-300;  // keep a2.. live cheaply
        }
        if (MODE == 1 || MODE == 2 || MODE == 3) {  // x1/x3 chain
            x13_update<true>(x1, x3, t1, t2, t3, t4, p, d0, d2);
            if (MODE == 3) {
                const bool ovf = !(fabs(x1) <= kStateLimit && fabs(x3) <= kStateLimit);
                const bool bnd = !in_bounds(x1, p.ylo, p.yhi);
                const bool now = !done && (ovf || bnd);
                status = now ? (ovf ? kOverflow : kViolated) : status;
                steps = now ? j + 1 : steps;
                done = done || now;
            }
        }
    }
    const long long t1c = clock64();
    out[threadIdx.x] = x1 + x2 + x3 + status + steps;
    if (threadIdx.x == 0) cyc[MODE] = t1c - t0;
}

int main() {
    double *dv, *out;
    long long* cyc;
    cudaMalloc(&dv, 256 * 8);
    cudaMemset(dv, 0, 256 * 8);
    cudaMalloc(&out, 64 * 8);
    cudaMalloc(&cyc, 8 * 8);
    const int J = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        k_chain<0><<<1, 32>>>(dv, out, cyc, J);
        k_chain<1><<<1, 32>>>(dv, out, cyc, J);
        k_chain<2><<<1, 32>>>(dv, out, cyc, J);
        k_chain<3><<<1, 32>>>(dv, out, cyc, J);
        cudaDeviceSynchronize();
    }
    long long h[4];
    cudaMemcpy(h, cyc, 4 * 8, cudaMemcpyDeviceToHost);
    printf("cycles per step, one warp: x2 chain %.1f | x1/x3 chain %.1f | both %.1f | x1/x3 + checks %.1f\n",
           h[0] / (double)J, h[1] / (double)J, h[2] / (double)J, h[3] / (double)J);
    return 0;
}
