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

static inline unsigned blocks_for(int64_t n, int tpb) { return (unsigned)((n + tpb - 1) / tpb); }

// Launch with programmatic stream serialization (PDL) when `pdl`: the grid may
// start while the previous kernel on the stream (k_gen_soa) is still running.
template <class Kern, class Args>
cudaError_t launch_ex(Kern kern, dim3 grid, int block, size_t smem, cudaStream_t s, bool pdl,
                      const Args& a) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl ? attr : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

// The single-wave placement's occupancy pin (rg_kernels.cu): `total` bytes of
// shared memory per block; *dyn receives the dynamic part to launch with.
cudaError_t pin_smem(const void* fn, int total, int* dyn);

}  // namespace rg
