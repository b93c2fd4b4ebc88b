// Does an FP64 warp-instruction with only 16 (or 8) active lanes issue faster than a full
// warp?  W warps per SMSP run independent DFMA chains with `act` active lanes each (the
// others exit at once); reports cycles per warp-instruction per SMSP.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, int iters, int act, long long* cyc) {
    const int lane = threadIdx.x & 31;
    if (lane >= act) return;
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4,
           x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    const double a = 0.999999, b = 1e-7;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    long long t1 = clock64();
    double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 12345.678) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 8); cudaMalloc(&cyc, 8 * 1024);
    const int iters = 1 << 14;
    for (int W : {1, 2, 4, 8}) {
        for (int act : {32, 16, 8, 1}) {
            // one block per SM, 4*W warps: W warps per SMSP
            k<<<148, 128 * W>>>(out, 64, act, cyc);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k<<<148, 128 * W>>>(out, iters, act, cyc);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            const double instr = (double)iters * 8 * W;  // warp-instructions per SMSP
            printf("W=%d act=%2d: %.3f ms, %.3f cycles per DFMA warp-instruction per SMSP (clock64 %.3f)\n",
                   W, act, ms, ms * 1e-3 * 1.965e9 / instr, (double)h / (iters * 8.0));
        }
    }
    return 0;
}
