// Throughput (warp-instructions / clock / SM) of the instruction classes in the
// rollout's hot loop: independent chains, 16 warps per SM on every SM.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 2048
template <int OP>
__global__ void thr(double* out, double a, double b) {
    double x[8];
    int ix[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) { x[c] = a + (threadIdx.x + c) * 1e-9; ix[c] = threadIdx.x + c; }
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (OP == 0) x[c] = __fma_rn(x[c], a, b);
            if (OP == 1) x[c] = __dadd_rn(x[c], b);
            if (OP == 2) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[c])); x[c] = r; }
            if (OP == 3) { ix[c] = __double2int_rz(x[c]); x[c] = __longlong_as_double(((long long)ix[c] << 20) ^ __double_as_longlong(x[c])); }
            if (OP == 4) { x[c] = (double)ix[c]; ix[c] = ix[c] + __double2hiint(x[c]); }
            if (OP == 5) { bool p = x[c] > b; x[c] = p ? x[c] : b; }
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c] + ix[c];
    if (s == 1234.5) out[0] = s;
}

int main() {
    double* out; cudaMalloc(&out, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz
    const char* names[] = {"DFMA", "DADD", "MUFU.RCP64H", "F2I.F64 (+int)", "I2F.F64 (+int)", "DSETP+FSEL x2"};
    for (int op = 0; op < 6; ++op) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        auto launch = [&]() {
            switch (op) {
                case 0: thr<0><<<sms * 4, 128>>>(out, 0.999, 1e-3); break;
                case 1: thr<1><<<sms * 4, 128>>>(out, 0.999, 1e-3); break;
                case 2: thr<2><<<sms * 4, 128>>>(out, 0.999, 1e-3); break;
                case 3: thr<3><<<sms * 4, 128>>>(out, 1.5, 1e-3); break;
                case 4: thr<4><<<sms * 4, 128>>>(out, 0.999, 1e-3); break;
                case 5: thr<5><<<sms * 4, 128>>>(out, 0.999, 1e-3); break;
            }
        };
        launch();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double warp_instr = 5.0 * sms * 4 * 4 * (double)ITERS * 8;   // blocks*warps*iters*chains
        double clocks = ms * 1e-3 * 1.965e9;
        printf("%-18s %.3f warp-instr/clk/SM (%.1f ms)\n", names[op], warp_instr / clocks / sms, ms);
    }
    return 0;
}
