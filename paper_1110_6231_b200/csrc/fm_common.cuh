// fm_common.cuh -- shared helpers for the B200 grid max-flow / assignment kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "flowmatch_b200.h"

void fm_set_error(const char *fmt, ...);

#define FM_CHECK_CUDA(call)                                                        \
    do {                                                                           \
        cudaError_t fm_err_ = (call);                                              \
        if (fm_err_ != cudaSuccess) {                                              \
            fm_set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,                \
                         cudaGetErrorString(fm_err_));                             \
            return FM_CUDA_ERROR;                                                  \
        }                                                                          \
    } while (0)

#define FM_CHECK_LAUNCH() FM_CHECK_CUDA(cudaGetLastError())

#define FM_TRY(expr)                                                               \
    do {                                                                           \
        int fm_rc_ = (expr);                                                       \
        if (fm_rc_ != FM_OK) return fm_rc_;                                        \
    } while (0)

// int32 loads that bypass L1: state words are updated by L2 atomics from other
// SMs, so a cached copy in this SM's L1 could be older than one the L2 holds.
__device__ __forceinline__ int32_t ld_cg(const int32_t *p) { return __ldcg(p); }
__device__ __forceinline__ int4 ld_cg4(const int32_t *p) { return __ldcg(reinterpret_cast<const int4 *>(p)); }

// block-wide sum of an int64 via warp shuffles + shared scratch; one atomic per block
template <int NWARPS>
__device__ __forceinline__ void block_add_i64(long long v, unsigned long long *dst) {
    __shared__ long long red[NWARPS];
    const int lane = threadIdx.x & 31;
    const int wid = (threadIdx.y * blockDim.x + threadIdx.x) >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();  // red[] may still be read by a previous call
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (wid == 0) {
        long long s = lane < NWARPS ? red[lane] : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0 && s != 0) atomicAdd(dst, (unsigned long long)s);
    }
}

struct FmTimer {
    cudaEvent_t a = nullptr, b = nullptr;
};
