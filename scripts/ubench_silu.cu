// ubench_silu.cu — throughput of SiLU formulations on one B200 (per-SM rate).
// Each thread evaluates silu on 2 independent streams of values, many
// iterations; reports elements / clk / SM. Variants:
//   tanh    : h + h*tanh.approx(h)                  (1 MUFU.TANH)
//   ex2rcp  : x * rcp(1 + ex2(-x*log2e))             (MUFU.EX2 + MUFU.RCP)
//   poly    : FMA-pipe only (FFMA2), exp2 by Cody-Waite + degree-5 poly,
//             reciprocal by bit-trick seed + 2 Newton steps
//   tanhbf  : tanh.approx.bf16x2
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 ubench_silu.cu -o ubench_silu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

__device__ __forceinline__ float silu_tanh(float x) {
    float h = 0.5f * x, t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(h));
    return fmaf(h, t, h);
}
__device__ __forceinline__ float silu_ex2rcp(float x) {
    float e, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-1.4426950408889634f * x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.f + e));
    return x * r;
}
// FMA-only: sigmoid via 2^(-x log2e) = 2^n * p(f), reciprocal Newton.
__device__ __forceinline__ float silu_poly(float x) {
    float t = fminf(fmaxf(-1.4426950408889634f * x, -126.f), 126.f);
    float n = rintf(t);
    float f = t - n;  // [-0.5, 0.5]
    float p = fmaf(f, 1.3333558e-3f, 9.6181291e-3f);
    p = fmaf(p, f, 5.5504109e-2f);
    p = fmaf(p, f, 2.4022651e-1f);
    p = fmaf(p, f, 6.9314718e-1f);
    p = fmaf(p, f, 1.0f);
    float e = __int_as_float(__float_as_int(p) + (static_cast<int>(n) << 23));
    float d = 1.f + e;
    float r = __int_as_float(0x7EF311C7 - __float_as_int(d));
    r = r * fmaf(-d, r, 2.f);
    r = r * fmaf(-d, r, 2.f);
    r = r * fmaf(-d, r, 2.f);
    return x * r;
}

template <int V>
__global__ void bench(float* out, int iters, long long* clk) {
    float a = 0.001f * threadIdx.x, b = -0.002f * threadIdx.x, c = 0.003f * threadIdx.x, d = -0.0005f * threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (V == 0) { a = silu_tanh(a + 0.5f); b = silu_tanh(b - 0.25f); c = silu_tanh(c + 0.1f); d = silu_tanh(d - 0.3f); }
        if (V == 1) { a = silu_ex2rcp(a + 0.5f); b = silu_ex2rcp(b - 0.25f); c = silu_ex2rcp(c + 0.1f); d = silu_ex2rcp(d - 0.3f); }
        if (V == 2) { a = silu_poly(a + 0.5f); b = silu_poly(b - 0.25f); c = silu_poly(c + 0.1f); d = silu_poly(d - 0.3f); }
        if (V == 4) {
            // tanh.approx.f16x2: h in f16, silu = h + h*tanh(h) in f32
            uint32_t ha, hb;
            asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(ha) : "f"(0.5f * a + 0.25f), "f"(0.5f * b - 0.125f));
            asm("tanh.approx.f16x2 %0, %0;" : "+r"(ha));
            asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hb) : "f"(0.5f * c + 0.05f), "f"(0.5f * d - 0.15f));
            asm("tanh.approx.f16x2 %0, %0;" : "+r"(hb));
            a = __half2float(__ushort_as_half(ha & 0xffff));
            b = __half2float(__ushort_as_half(ha >> 16));
            c = __half2float(__ushort_as_half(hb & 0xffff));
            d = __half2float(__ushort_as_half(hb >> 16));
        }
        if (V == 5) {
            uint32_t ha, hb;
            asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(ha) : "f"(0.5f * a + 0.25f), "f"(0.5f * b - 0.125f));
            asm("ex2.approx.f16x2 %0, %0;" : "+r"(ha));
            asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hb) : "f"(0.5f * c + 0.05f), "f"(0.5f * d - 0.15f));
            asm("ex2.approx.f16x2 %0, %0;" : "+r"(hb));
            a = __half2float(__ushort_as_half(ha & 0xffff));
            b = __half2float(__ushort_as_half(ha >> 16));
            c = __half2float(__ushort_as_half(hb & 0xffff));
            d = __half2float(__ushort_as_half(hb >> 16));
        }
        if (V == 3) {
            uint32_t ha, hb;
            asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(ha) : "f"(0.5f * a + 0.25f), "f"(0.5f * b - 0.125f));
            asm("tanh.approx.bf16x2 %0, %0;" : "+r"(ha));
            asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(hb) : "f"(0.5f * c + 0.05f), "f"(0.5f * d - 0.15f));
            asm("tanh.approx.bf16x2 %0, %0;" : "+r"(hb));
            a = __bfloat162float(__ushort_as_bfloat16(ha & 0xffff));
            b = __bfloat162float(__ushort_as_bfloat16(ha >> 16));
            c = __bfloat162float(__ushort_as_bfloat16(hb & 0xffff));
            d = __bfloat162float(__ushort_as_bfloat16(hb >> 16));
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
    if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
    float* out;
    long long* clk;
    cudaMalloc(&out, 148 * 1024 * 4 * 4);
    cudaMalloc(&clk, 8);
    const int iters = 4096;
    const char* names[6] = {"tanh", "ex2rcp", "poly", "tanhbf16x2", "tanhf16x2", "ex2f16x2"};
    for (int v = 0; v < 6; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            const int threads = 1024, blocks = 148 * 2;
            if (v == 0) bench<0><<<blocks, threads>>>(out, iters, clk);
            if (v == 1) bench<1><<<blocks, threads>>>(out, iters, clk);
            if (v == 2) bench<2><<<blocks, threads>>>(out, iters, clk);
            if (v == 3) bench<3><<<blocks, threads>>>(out, iters, clk);
            if (v == 4) bench<4><<<blocks, threads>>>(out, iters, clk);
            if (v == 5) bench<5><<<blocks, threads>>>(out, iters, clk);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            long long c;
            cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
            const double elems = 4.0 * iters * threads * blocks;
            if (rep)
                printf("%-11s %.3f ms  %.2f Gelem/s  %.2f elem/clk/SM (@%d block clk %lld)\n", names[v], ms,
                       elems / ms / 1e6, elems / (ms * 1e-3) / 148 / 1.965e9, blocks, c);
        }
    }
    return 0;
}
