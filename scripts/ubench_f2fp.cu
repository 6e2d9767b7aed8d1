// Throughput of cvt.rn.bf16x2.f32 (F2FP.BF16.F32.PACK_AB) vs MUFU.TANH, alone and mixed.
#include <cstdio>
#include <cstdint>
__global__ void k(float* out, int iters, int mode, long long* clk) {
    float a = threadIdx.x * 1e-3f, b = -a, c = a * 0.5f, d = b * 0.5f;
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t p0, p1;
        if (mode == 0 || mode == 2) {
            asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p0) : "f"(a), "f"(b));
            asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p1) : "f"(c), "f"(d));
            acc ^= p0 ^ p1;
            a += 1e-7f; c -= 1e-7f;
        }
        if (mode == 1 || mode == 2) {
            float t0_, t1_;
            asm volatile("tanh.approx.f32 %0, %1;" : "=f"(t0_) : "f"(b));
            asm volatile("tanh.approx.f32 %0, %1;" : "=f"(t1_) : "f"(d));
            b += t0_ * 1e-9f; d += t1_ * 1e-9f;
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d + acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
int main() {
    float* out; long long* clk;
    cudaMalloc(&out, 148 * 1024 * 4 * 2); cudaMalloc(&clk, 8);
    const char* nm[3] = {"cvt.bf16x2 only", "tanh only", "both"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) k<<<148 * 2, 1024>>>(out, 4096, mode, clk);
        cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
        // per SM: 2 blocks x 1024 threads x 4096 iters x 2 ops of each kind
        const double ops = 2.0 * 1024 * 4096 * 2;
        printf("%-16s %8.2f ops/clk/SM per kind\n", nm[mode], ops / c);
    }
}
