// Single-warp FP64 issue: cycles per DFMA for K independent chains with W warps
// per SM sub-partition (blocks of 128*W threads, one block per SM).
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
template <int K>
__global__ void ilp(double* out, double a, double b, long long* cyc) {
    double x[K];
#pragma unroll
    for (int c = 0; c < K; ++c) x[c] = a + (threadIdx.x + c) * 1e-9;
    const long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < K; ++c) x[c] = __fma_rn(x[c], a, b);
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < K; ++c) s += x[c];
    if (s == 1234.5) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int K>
void run(int sms, int W, double* out, long long* cyc) {
    ilp<K><<<sms, 128 * W>>>(out, 0.999, 1e-3, cyc);
    cudaDeviceSynchronize();
    ilp<K><<<sms, 128 * W>>>(out, 0.999, 1e-3, cyc);
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double per_warp = (double)c / (ITERS * (double)K);
    printf("K=%d chains  W=%d warps/SMSP: %.2f clk per DFMA per warp, SMSP rate %.3f DFMA/clk\n",
           K, W, per_warp, W / per_warp);
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int W : {1, 2, 4}) {
        run<1>(sms, W, out, cyc);
        run<2>(sms, W, out, cyc);
        run<4>(sms, W, out, cyc);
        run<8>(sms, W, out, cyc);
    }
    return 0;
}
