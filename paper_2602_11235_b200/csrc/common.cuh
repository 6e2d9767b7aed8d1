// common.cuh — shared helpers for the MTFM sm_100a kernels.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace mtfm {

constexpr int kNumSMs = 148;

__host__ __device__ inline long long cdiv(long long a, long long b) { return (a + b - 1) / b; }
__host__ __device__ inline long long round_up(long long a, long long b) { return cdiv(a, b) * b; }

// ---------------------------------------------------------------- programmatic dependent launch
// Every kernel of the forward is launched with programmatic stream
// serialization: the next kernel's CTAs are scheduled as the predecessor's
// CTAs retire, run their prologue (barrier init, TMEM allocation, SMEM
// tables), and block in griddepcontrol.wait until the predecessor grid has
// completed and its writes are visible: launch latency and prologues overlap
// the predecessor's tail.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Measured: an explicit early trigger lets dependents flood the SMs while the
// persistent predecessor still runs (2% slower); without it the dependent grid
// is released as the predecessor's CTAs retire (2% faster than no PDL).
__device__ __forceinline__ void pdl_trigger() {
#ifdef MTFM_PDL_EARLY_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
// entry of a kernel that reads predecessor outputs from its first instruction on
#define MTFM_PDL_ENTRY()     \
    do {                     \
        ::mtfm::pdl_wait();    \
        ::mtfm::pdl_trigger(); \
    } while (0)

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

// Storage-type conversions used by the kernels templated on the activation
// type (float in the fp32 check mode, bf16 in the fast mode).
__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T>
__device__ __forceinline__ T from_f32(float x);
template <>
__device__ __forceinline__ float from_f32<float>(float x) {
    return x;
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) {
    return __float2bfloat16_rn(x);
}

// Precise sigmoid/silu (kernels.hpp:96-110 branch structure) for the fp32
// check mode; expf, not __expf.
__device__ __forceinline__ float sigmoid_precise(float x) {
    if (x >= 0.f) {
        const float e = expf(-x);
        return 1.f / (1.f + e);
    }
    const float e = expf(x);
    return e / (1.f + e);
}
__device__ __forceinline__ float silu_precise(float x) { return x * sigmoid_precise(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace mtfm
