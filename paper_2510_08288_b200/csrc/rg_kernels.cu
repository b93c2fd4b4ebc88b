// rg_kernels.cu -- sm_100a kernels of the robust Reference Governor hot path:
// scenario generation, the parity fill and the auxiliary kernels.
//
//   k_sample      scenario tensor from the counter RNG (disturbance.py:179-203)
//   k_gen_soa     the same stream straight into the SoA block of the grid step
//   k_to_soa      [k][j][i] host-layout tensor -> SoA d[(j*3+i)*ld + k]
//   k_fill        parity fill: status/steps per (active row, scenario) cell
//                 (kernels.py:121-162 / backend_gpu.fill seam)
//   k_fill_lin / k_bisect_lin   the linear plant (kernels.py:90-118)
//   k_tanh        device tanh for the bit-parity self-test
//   k_dfma_peak   the FP64 roofline probe
// The fused grid step is rg_grid.cu, the batched step rg_batch.cu, the
// bisections rg_bisect.cu; shared helpers rg_common.cuh.
#include "rg_common.cuh"

#include <mutex>

namespace rg {

// ---------------------------------------------------------------------------
// scenario generation
// ---------------------------------------------------------------------------

__global__ void k_sample(SampleArgs a) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (k, j)
    const int64_t total = a.n_sim * a.horizon;
    if (idx >= total) return;
    const int64_t k = idx / a.horizon;
    const int64_t j = idx - k * a.horizon;
    const uint64_t K = splitmix64(a.hs ^ (uint64_t)(a.k0 + k));
    const uint64_t J = splitmix64(K ^ (uint64_t)j);
    double* o = a.out + idx * a.width;
    for (int i = 0; i < a.width; ++i) {
        const double u = unit_double(splitmix64(J ^ (uint64_t)i));
        o[i] = add(a.lo[i], mul(a.span[i], u));
    }
}

// counter RNG straight into the SoA layout d[(j*3+i)*ld + k], rows j < j_star:
// one thread per (scenario, step); lanes run over scenarios, so stores coalesce.
__global__ void k_gen_soa(ScenarioStream st, int64_t k0, int64_t n_sim, int32_t j_star,
                          int64_t ld, double* __restrict__ dst) {
    // a grid step launched behind this kernel with programmatic stream
    // serialization may start its prologue now; it waits (griddepcontrol.wait)
    // for this grid's completion before it reads the block
    asm volatile("griddepcontrol.launch_dependents;");
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t j = blockIdx.y;
    if (k >= n_sim || j >= j_star) return;
    const uint64_t K = scenario_key(st, (uint64_t)(k0 + k));
    double d0, d1, d2;
    disturbance_at(st, K, (uint64_t)j, d0, d1, d2);
    double* o = dst + (int64_t)j * 3 * ld + k;
    o[0] = d0;
    o[ld] = d1;
    o[2 * ld] = d2;
}

// tile transpose of [n_sim][horizon][3] (rows j < j_star) into d[(j*3+i)*ld + k], columns
// k < ncols (scenarios past n_sim are zero padding); a chunk of scenarios passes src and
// dst already offset to its first scenario
__global__ void k_to_soa(const double* __restrict__ src, double* __restrict__ dst,
                         int64_t n_sim, int64_t horizon, int32_t j_star, int64_t ld,
                         int64_t ncols) {
    __shared__ double tile[32][32 * 3 + 1];
    const int64_t k0 = (int64_t)blockIdx.x * 32;
    const int32_t j0 = blockIdx.y * 32;
    // load: warp w reads scenario k0+w, 32 steps x 3 comps (96 contiguous doubles)
    for (int w = threadIdx.y; w < 32; w += blockDim.y) {
        const int64_t k = k0 + w;
        for (int e = threadIdx.x; e < 96; e += 32) {
            const int32_t j = j0 + e / 3;
            double v = 0.0;
            if (k < n_sim && j < j_star) v = src[(k * horizon + j) * 3 + (e % 3)];
            tile[w][e] = v;
        }
    }
    __syncthreads();
    // store: lanes run over k (coalesced), rows over (j, i)
    for (int r = threadIdx.y; r < 96; r += blockDim.y) {
        const int32_t j = j0 + r / 3;
        const int i = r % 3;
        const int64_t k = k0 + threadIdx.x;
        if (j < j_star && k < ncols) dst[((int64_t)j * 3 + i) * ld + k] = tile[threadIdx.x][r];
    }
}

// ---------------------------------------------------------------------------
// parity fill: status/steps for every (active row, scenario)
// ---------------------------------------------------------------------------

template <bool FMA, bool RNG>
__global__ void __launch_bounds__(128, RG_GRID_MINB) k_fill(FillArgs a) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = k < a.n_sim;  // whole warps run the rollout (out-of-range lanes replay)
    const int32_t row = a.rows[blockIdx.y];
    const double v = a.v_rows[row];
    const CellConst c = make_cell(a.p);
    const int64_t kk = live ? k : 0;  // out-of-range lanes replay scenario 0
    int32_t steps = 0;
    int st;
    if (RNG) {
        RngSource src{a.stream, scenario_key(a.stream, (uint64_t)(a.k0 + kk))};
        st = rollout<FMA, false, RngSource, true>(c, a.x0[0], a.x0[1], a.x0[2], v, src, steps,
                                                  nullptr, live);
    } else {
        __shared__ double ring[2 * 3 * kRingStride];
        SoaSource src{a.soa + kk, a.ld, ring + threadIdx.x};
        st = rollout<FMA, false, SoaSource, true>(c, a.x0[0], a.x0[1], a.x0[2], v, src, steps,
                                                  nullptr, live);
    }
    if (live) {
        a.S[(int64_t)row * a.n_sim + k] = (uint8_t)st;
        a.steps[(int64_t)row * a.n_sim + k] = steps;
    }
}

// ---------------------------------------------------------------------------
// linear plant: parity fill and exact Alg. 2
// ---------------------------------------------------------------------------

__global__ void k_gen_soa_w(uint64_t hs, double4 lo4, double4 span4, int width, int64_t k0,
                            int64_t n_sim, int32_t j_star, int64_t ld, double* __restrict__ dst) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t j = blockIdx.y;
    if (k >= n_sim || j >= j_star) return;
    const double lo[4] = {lo4.x, lo4.y, lo4.z, lo4.w};
    const double span[4] = {span4.x, span4.y, span4.z, span4.w};
    const uint64_t K = splitmix64(hs ^ (uint64_t)(k0 + k));
    const uint64_t J = splitmix64(K ^ (uint64_t)j);
    for (int i = 0; i < width; ++i)
        dst[((int64_t)j * width + i) * ld + k] =
            add(lo[i], mul(span[i], unit_double(splitmix64(J ^ (uint64_t)i))));
}

template <int N>
__device__ __forceinline__ int lin_cell(const LinArgs& a, const CellConst& c, int64_t k, double v,
                                        int32_t& steps) {
    if (a.soa) {
        LinSoaSource<N> src{a.soa + k, a.ld};
        return rollout_lin<N, false>(a.L, c, a.x0, v, src, steps);
    }
    LinRngSource<N> src;
    src.K = splitmix64(a.hs ^ (uint64_t)(a.k0 + k));
    for (int i = 0; i < 4; ++i) {
        src.lo[i] = a.lo[i];
        src.span[i] = a.span[i];
    }
    return rollout_lin<N, true>(a.L, c, a.x0, v, src, steps);
}

template <int N>
__global__ void __launch_bounds__(128) k_fill_lin(LinArgs a) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.n_sim) return;
    const int32_t row = a.rows[blockIdx.y];
    int32_t steps = 0;
    const int st = lin_cell<N>(a, make_cell(a.p), k, a.v_rows[row], steps);
    a.S[(int64_t)row * a.n_sim + k] = (uint8_t)st;
    a.steps[(int64_t)row * a.n_sim + k] = steps;
}

template <int N>
__global__ void __launch_bounds__(128) k_bisect_lin(LinArgs a) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = k < a.n_sim;
    double kopt = 1.0;
    int found = 1, cells = 0, early = 0;
    if (live) {
        const CellConst c = make_cell(a.p);
        double klo = 0.0, khi = 1.0;
        kopt = 0.0;
        found = 0;
        for (int it = -1; it < a.n_kappa; ++it) {
            const double kappa = it < 0 ? 1.0 : mul(0.5, add(klo, khi));
            const double v = update_setpoint(a.v_prev, a.r, kappa);
            bool ok = false;
            int32_t sr = 0;
            const double yss = mul(a.L.gain, v);  // LinearOraclePlant.steady_state_output
            if (a.L.tlo <= yss && yss <= a.L.thi) ok = lin_cell<N>(a, c, k, v, sr) == kOk;
            cells += 1;
            if (sr < a.p.j_star && !ok) early += 1;
            if (it < 0) {
                if (ok) {
                    kopt = 1.0;
                    found = 1;
                    break;
                }
                continue;
            }
            if (ok) {
                kopt = kappa;
                found = 1;
                klo = kappa;
            } else {
                khi = kappa;
            }
        }
        if (a.kappa_k) {
            a.kappa_k[k] = kopt;
            a.found_k[k] = found;
            a.cells_k[k] = cells;
            a.early_k[k] = early;
        }
    }
    unsigned long long kb = (unsigned long long)__double_as_longlong(kopt);
    int all_found = found;
    long long sc = cells, se = early;
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long ob = __shfl_down_sync(0xffffffffu, kb, off);
        kb = ob < kb ? ob : kb;
        all_found &= __shfl_down_sync(0xffffffffu, all_found, off);
        sc += __shfl_down_sync(0xffffffffu, sc, off);
        se += __shfl_down_sync(0xffffffffu, se, off);
    }
    if (lane_id() == 0) {
        atomicMin(&a.acc->kappa_bits, kb);
        if (!all_found) atomicAnd(&a.acc->found, 0);
        atomicAdd(&a.acc->cells, (unsigned long long)sc);
        atomicAdd(&a.acc->early, (unsigned long long)se);
    }
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&a.acc->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    __threadfence();
    volatile BisectAcc* acc = a.acc;
    a.out->kappa = __longlong_as_double((long long)acc->kappa_bits);
    a.out->found = acc->found;
    a.out->cells = (long long)acc->cells;
    a.out->early = (long long)acc->early;
    a.out->seq += 1;
    acc->kappa_bits = 0x3ff0000000000000ull;
    acc->found = 1;
    acc->cells = 0ull;
    acc->early = 0ull;
    acc->ticket = 0u;
}

// ---------------------------------------------------------------------------
// tanh self-test
// ---------------------------------------------------------------------------

template <bool FMA>
__global__ void k_tanh(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = tanh_glibc<FMA>(x[i]);
}

// the rollout's lockstep form (tanh4 / tanh_core), four arguments per thread
template <bool FMA>
__global__ void k_tanh4(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i >= n) return;
    double a[4], z[4];
    for (int q = 0; q < 4; ++q) a[q] = i + q < n ? x[i + q] : 0.0;
    tanh4_auto<FMA>(a[0], a[1], a[2], a[3], z[0], z[1], z[2], z[3]);
    for (int q = 0; q < 4; ++q)
        if (i + q < n) y[i + q] = z[q];
}

// FP64 issue-rate probe: independent DFMA chains (the roofline denominator)
__global__ void k_dfma_peak(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1.0, x2 = x0 + 2.0, x3 = x0 + 3.0;
    double x4 = x0 + 4.0, x5 = x0 + 5.0, x6 = x0 + 6.0, x7 = x0 + 7.0;
    for (int i = 0; i < iters; ++i) {
        x0 = __fma_rn(x0, a, b);
        x1 = __fma_rn(x1, a, b);
        x2 = __fma_rn(x2, a, b);
        x3 = __fma_rn(x3, a, b);
        x4 = __fma_rn(x4, a, b);
        x5 = __fma_rn(x5, a, b);
        x6 = __fma_rn(x6, a, b);
        x7 = __fma_rn(x7, a, b);
    }
    const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

cudaError_t launch_sample(const SampleArgs& a, cudaStream_t s) {
    const int64_t total = a.n_sim * a.horizon;
    if (total == 0) return cudaSuccess;
    k_sample<<<blocks_for(total, 256), 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_to_soa(const double* src, double* dst, int64_t n_sim, int64_t horizon,
                          int32_t j_star, int64_t ld, cudaStream_t s, int64_t ncols) {
    if (ncols < 0) ncols = ld;
    dim3 grid((unsigned)((ncols + 31) / 32), (unsigned)((j_star + 31) / 32));
    k_to_soa<<<grid, dim3(32, 8), 0, s>>>(src, dst, n_sim, horizon, j_star, ld, ncols);
    return cudaGetLastError();
}

cudaError_t launch_fill(const FillArgs& a, bool fma, bool rng, cudaStream_t s) {
    if (a.n_rows == 0 || a.n_sim == 0) return cudaSuccess;
    dim3 grid(blocks_for(a.n_sim, a.tpb), (unsigned)a.n_rows);
    if (fma) {
        if (rng) k_fill<true, true><<<grid, a.tpb, 0, s>>>(a);
        else     k_fill<true, false><<<grid, a.tpb, 0, s>>>(a);
    } else {
        if (rng) k_fill<false, true><<<grid, a.tpb, 0, s>>>(a);
        else     k_fill<false, false><<<grid, a.tpb, 0, s>>>(a);
    }
    return cudaGetLastError();
}

// The single-wave placement's occupancy pin: `total` bytes of shared memory per
// block (more than half an SM's), of which the kernel's static shared memory is a
// part.  Sets *dyn to the dynamic remainder and opts the kernel in to it, once per
// kernel and device.  total <= 0: no pin (*dyn = 0).
cudaError_t pin_smem(const void* fn, int total, int* dyn) {
    *dyn = 0;
    if (total <= 0) return cudaSuccess;
    struct Entry {
        const void* fn;
        int dev, total, dyn;
    };
    static Entry tab[256];
    static int n = 0;
    static std::mutex mu;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < n; ++i)
        if (tab[i].fn == fn && tab[i].dev == dev && tab[i].total == total) {
            *dyn = tab[i].dyn;
            return cudaSuccess;
        }
    cudaFuncAttributes attr;
    if ((e = cudaFuncGetAttributes(&attr, fn)) != cudaSuccess) return e;
    const int d = total > (int)attr.sharedSizeBytes ? total - (int)attr.sharedSizeBytes : 0;
    if (d > 0 &&
        (e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, d)) !=
            cudaSuccess)
        return e;
    if (n < 256) tab[n++] = Entry{fn, dev, total, d};
    *dyn = d;
    return cudaSuccess;
}

cudaError_t launch_tanh(const double* x, double* y, int64_t n, bool fma, bool lockstep,
                        cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (lockstep) {
        const unsigned g = blocks_for((n + 3) / 4, 256);
        if (fma) k_tanh4<true><<<g, 256, 0, s>>>(x, y, n);
        else     k_tanh4<false><<<g, 256, 0, s>>>(x, y, n);
    } else {
        if (fma) k_tanh<true><<<blocks_for(n, 256), 256, 0, s>>>(x, y, n);
        else     k_tanh<false><<<blocks_for(n, 256), 256, 0, s>>>(x, y, n);
    }
    return cudaGetLastError();
}

cudaError_t launch_fill_lin(const LinArgs& a, cudaStream_t s) {
    if (a.n_rows == 0 || a.n_sim == 0) return cudaSuccess;
    dim3 grid(blocks_for(a.n_sim, a.tpb), (unsigned)a.n_rows);
    switch (a.L.n) {
        case 1: k_fill_lin<1><<<grid, a.tpb, 0, s>>>(a); break;
        case 2: k_fill_lin<2><<<grid, a.tpb, 0, s>>>(a); break;
        case 3: k_fill_lin<3><<<grid, a.tpb, 0, s>>>(a); break;
        default: k_fill_lin<4><<<grid, a.tpb, 0, s>>>(a); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_bisect_lin(const LinArgs& a, cudaStream_t s) {
    const unsigned g = blocks_for(a.n_sim, a.tpb);
    switch (a.L.n) {
        case 1: k_bisect_lin<1><<<g, a.tpb, 0, s>>>(a); break;
        case 2: k_bisect_lin<2><<<g, a.tpb, 0, s>>>(a); break;
        case 3: k_bisect_lin<3><<<g, a.tpb, 0, s>>>(a); break;
        default: k_bisect_lin<4><<<g, a.tpb, 0, s>>>(a); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_gen_soa_w(uint64_t hs, const double* lo, const double* span, int width,
                             int64_t k0, int64_t n_sim, int32_t j_star, int64_t ld, double* dst,
                             cudaStream_t s) {
    double4 l4 = make_double4(lo[0], width > 1 ? lo[1] : 0, width > 2 ? lo[2] : 0,
                              width > 3 ? lo[3] : 0);
    double4 s4 = make_double4(span[0], width > 1 ? span[1] : 0, width > 2 ? span[2] : 0,
                              width > 3 ? span[3] : 0);
    dim3 grid(blocks_for(n_sim, 128), (unsigned)j_star);
    k_gen_soa_w<<<grid, 128, 0, s>>>(hs, l4, s4, width, k0, n_sim, j_star, ld, dst);
    return cudaGetLastError();
}

cudaError_t launch_gen_soa(const ScenarioStream& st, int64_t k0, int64_t n_sim, int32_t j_star,
                           int64_t ld, double* dst, cudaStream_t s) {
    dim3 grid(blocks_for(n_sim, 128), (unsigned)j_star);
    k_gen_soa<<<grid, 128, 0, s>>>(st, k0, n_sim, j_star, ld, dst);
    return cudaGetLastError();
}

cudaError_t launch_dfma_peak(double* out, int blocks, int threads, int iters, cudaStream_t s) {
    k_dfma_peak<<<blocks, threads, 0, s>>>(out, iters, 0.999999, 1e-7);
    return cudaGetLastError();
}

}  // namespace rg
