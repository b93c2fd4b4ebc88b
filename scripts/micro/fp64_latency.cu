// Dependent-chain latency and throughput of the FP64 / conversion / MUFU ops the
// rollout uses, measured with clock64 in one warp (latency) and many warps (rate).
#include <cstdio>
#include <cuda_runtime.h>

#define CHAIN 512
template <int OP>
__global__ void lat(double* out, long long* cyc, double a, double b) {
    double x = a + threadIdx.x * 1e-12;
    int ix = (int)b;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < CHAIN; ++i) {
        if (OP == 0) x = __fma_rn(x, a, b);
        if (OP == 1) x = __dadd_rn(x, b);
        if (OP == 2) x = __dmul_rn(x, a);
        if (OP == 3) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
        if (OP == 4) { ix = __double2int_rz(x); x = (double)ix + a; }
        if (OP == 5) x = __ddiv_rn(b, x);
        if (OP == 6) { long long v = __double_as_longlong(x); v ^= (v >> 7); x = __longlong_as_double(v) ; x = __dadd_rn(x, 0.0); }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (x == 123.0) out[0] = x;
}

int main() {
    double* out; long long* cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 8 * 1024);
    const char* names[] = {"DFMA", "DADD", "DMUL", "MUFU.RCP64H", "F2I+I2F+DADD", "ddiv_rn", "int-xor+DADD"};
    for (int op = 0; op < 7; ++op) {
        long long h = 0;
        for (int rep = 0; rep < 3; ++rep) {
            switch (op) {
                case 0: lat<0><<<1, 32>>>(out, cyc, 0.999, 1e-3); break;
                case 1: lat<1><<<1, 32>>>(out, cyc, 0.999, 1e-3); break;
                case 2: lat<2><<<1, 32>>>(out, cyc, 0.999, 1e-3); break;
                case 3: lat<3><<<1, 32>>>(out, cyc, 0.999, 1e-3); break;
                case 4: lat<4><<<1, 32>>>(out, cyc, 0.5, 1e-3); break;
                case 5: lat<5><<<1, 32>>>(out, cyc, 0.999, 1.5); break;
                case 6: lat<6><<<1, 32>>>(out, cyc, 0.999, 1e-3); break;
            }
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        }
        printf("%-14s latency %.2f cycles/op (1 warp)\n", names[op], (double)h / CHAIN);
    }
    // throughput: many warps per SM, independent chains
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {1, 2, 4, 8, 16}) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        lat<0><<<sms, 32 * w>>>(out, cyc, 0.999, 1e-3);
        cudaEventRecord(e0);
        for (int r = 0; r < 10; ++r) lat<0><<<sms, 32 * w>>>(out, cyc, 0.999, 1e-3);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 10.0 * sms * 32 * w * CHAIN * 2;
        printf("DFMA chains: %2d warps/SM -> %.2f TFLOP/s\n", w, flops / (ms * 1e-3) / 1e12);
    }
    return 0;
}
