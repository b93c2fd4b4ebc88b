// rg_common.cuh -- device helpers and launch utilities shared by the kernel
// translation units (rg_kernels.cu, rg_grid.cu, rg_batch.cu, rg_bisect.cu).
// Internal to the library.
#pragma once

#include <cuda_runtime.h>

#include "rg_cell.cuh"
#include "rg_kernels.h"

#ifndef RG_GRID_MINB
#define RG_GRID_MINB 1
#endif

namespace rg {

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// warp-aggregated add of a per-lane predicate count into a 64-bit counter
__device__ __forceinline__ void warp_count_add(bool pred, unsigned long long* ctr) {
    const unsigned m = __ballot_sync(0xffffffffu, pred);
    if (lane_id() == 0 && m) atomicAdd(ctr, (unsigned long long)__popc(m));
}

__device__ __forceinline__ CellConst make_cell(const ProblemDev& p) {
    CellConst c;
    c.h = p.h;
    c.hh = p.hh;
    c.c = p.c;
    c.ylo = p.ylo;
    c.yhi = p.yhi;
    c.j_star = p.j_star;
    return c;
}

__device__ __forceinline__ bool ss_gate(double v, const ProblemDev& p) {
    return p.vlo <= v && v <= p.vhi;  // NaN -> false, like ConstraintSet.contains
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// Sense-free grid barrier on (count, gen): the last arriver resets count, then bumps
// gen; the others spin on gen.  Requires every block of the grid to be resident.
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* vgen = gen;
        const unsigned g = *vgen;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *(volatile unsigned*)count = 0u;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*vgen == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

static inline unsigned blocks_for(int64_t n, int tpb) { return (unsigned)((n + tpb - 1) / tpb); }

// Launch with programmatic stream serialization (PDL) when `pdl`: the grid may start while
// the previous kernel on the stream (k_gen_soa) is still running.  `coop`: a cooperative
// launch (every block resident at once, or the launch fails), for kernels with a grid barrier.
template <class Kern, class Args>
cudaError_t launch_ex(Kern kern, dim3 grid, int block, size_t smem, cudaStream_t s, bool pdl,
                      const Args& a, bool coop = false) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int n = 0;
    if (pdl) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    if (coop) {
        attr[n].id = cudaLaunchAttributeCooperative;
        attr[n].val.cooperative = 1;
        ++n;
    }
    cfg.attrs = n ? attr : nullptr;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

// The single-wave placement's occupancy pin (rg_kernels.cu): `total` bytes of
// shared memory per block; *dyn receives the dynamic part to launch with.
cudaError_t pin_smem(const void* fn, int total, int* dyn);

}  // namespace rg
