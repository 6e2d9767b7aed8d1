// Microbenchmark: TMEM load throughput (tcgen05.ld 32x32b) with W warps, alone
// and while one thread streams tcgen05.mma into another TMEM region; and MMA
// throughput alone. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2602_11235_b200/csrc
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace mtfm;

template <int X>
__device__ __forceinline__ uint32_t ld_x(uint32_t taddr);

template <>
__device__ __forceinline__ uint32_t ld_x<16>(uint32_t taddr) {
    float v[16];
    ptx::tmem_ld16(taddr, v);
    ptx::tmem_ld_wait();
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s ^= __float_as_uint(v[i]);
    return s;
}
template <>
__device__ __forceinline__ uint32_t ld_x<64>(uint32_t taddr) {
    float v[64];
#pragma unroll
    for (int k = 0; k < 4; ++k) ptx::tmem_ld16(taddr + 16 * k, *reinterpret_cast<float(*)[16]>(v + 16 * k));
    ptx::tmem_ld_wait();
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 64; ++i) s ^= __float_as_uint(v[i]);
    return s;
}
template <>
__device__ __forceinline__ uint32_t ld_x<32>(uint32_t taddr) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    ptx::tmem_ld_wait();
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) s ^= r[i];
    return s;
}

// mode 0: loads only; 1: loads + MMA stream; 2: MMA only
template <int X>
__global__ void __launch_bounds__(544, 1) kern(int ld_warps, int iters, int mode, int mma_n, int mma_iters,
                                               unsigned long long* cyc, uint32_t* sink) {
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t bar2;
    __shared__ __align__(8) uint64_t bar3;
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t mma_warp = 16;
    if (warp == 0) ptx::tmem_alloc<512>(&slot);
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::mbar_init(&bar2, 1);
        ptx::mbar_init(&bar3, 1);
        ptx::fence_mbar_init();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tbase = slot;
    if (mode >= 3 && mode != 5) {
        // random bf16 operands (power-realistic)
        uint32_t x = 0x9e3779b9u * (threadIdx.x + 1) + blockIdx.x;
        for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) {
            x ^= x << 13; x ^= x >> 17; x ^= x << 5;
            const uint32_t lo = 0x3c00u | (x & 0x807fu), hi = 0x3c00u | ((x >> 16) & 0x807fu);
            reinterpret_cast<uint32_t*>(sm)[i] = lo | (hi << 16);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
    }
    unsigned long long t0 = clock64();
    uint32_t s = 0;
    if (mode == 7 && warp < 12) {
        // 12 warps spinning on an mbarrier that completes only when the MMA warp finishes
        while (!ptx::mbar_try_wait(&bar3, 0)) {
        }
    } else if (mode == 4 && warp < 8) {
        // smem store traffic from 8 warps (epilogue staging analogue) into a separate 8 KB region
        uint4* dst = reinterpret_cast<uint4*>(sm + 49152) + (warp * 32 + lane) % 512;
        for (int it = 0; it < iters * 16; ++it) { *dst = make_uint4(it, it, it, it); __syncwarp(); }
        s ^= reinterpret_cast<uint32_t*>(sm + 49152)[lane];
    } else if (warp < (uint32_t)ld_warps && mode < 2) {
        const uint32_t q = warp & 3;
        const uint32_t lb = tbase + ((q * 32u) << 16) + 256;  // columns 256..511
        const uint32_t g = warp >> 2, ng = (ld_warps + 3) >> 2;
        for (int it = 0; it < iters; ++it) {
            for (uint32_t c = g * X; c < 256; c += ng * X) s ^= ld_x<X>(lb + c);
        }
    }
    if (warp == mma_warp && mode >= 1) {
        const uint32_t idesc = ptx::instr_desc_bf16(128, mma_n, false, false);
        const uint32_t sa = ptx::smem_u32(sm);
        if (ptx::elect_one()) {
            for (int it = 0; it < mma_iters; ++it) {
                const uint64_t da = ptx::smem_desc(sa + (it & 3) * 32, 16, 1024, 2);
                const uint64_t db = ptx::smem_desc(sa + 16384 + (it & 3) * 32, 16, 1024, 2);
                const uint32_t dcol = mode == 8 ? ((it >> 4) & 3) * 128 : 0;
                ptx::umma_bf16(tbase + dcol, da, db, idesc, mode == 8 ? (it & 15) != 0 : it > 0);
                if (mode == 8 && (it & 3) == 3) ptx::umma_commit(&bar2);
                if (mode == 5 && (it & 3) == 3) ptx::umma_commit(&bar2);
                if (mode == 6 && (it & 3) == 3) {
                    ptx::umma_commit(&bar2);
                    __syncwarp(__activemask());
                }
            }
            ptx::umma_commit(&bar);
        }
        __syncwarp();
        ptx::mbar_wait(&bar, 0);
        if (lane == 0) ptx::mbar_arrive(&bar3);
    }
    unsigned long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
    if (s == 0x12345678u) sink[0] = s;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<512>(tbase);
}

int main() {
    unsigned long long* cyc;
    uint32_t* sink;
    cudaMalloc(&cyc, 148 * 32 * 8);
    cudaMalloc(&sink, 4);
    const int smem = 64 * 1024;
    auto run = [&](auto kfn, int X, int ldw, int mode, int mma_n) {
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int iters = 200, mma_iters = 4000;
        for (int rep = 0; rep < 2; ++rep) kfn<<<148, 544, smem>>>(ldw, iters, mode, mma_n, mma_iters, cyc, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
        unsigned long long h[32];
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        unsigned long long ld_max = 0;
        for (int w = 0; w < ldw; ++w) ld_max = h[w] > ld_max ? h[w] : ld_max;
        const double bytes = (double)iters * 256 * 128 * 4;  // 256 columns x 128 lanes x 4 B per iteration
        if (mode < 2)
            printf("X=%2d warps=%2d mode=%d n=%3d: ld %.1f B/clk/SM (%llu clk)", X, ldw, mode, mma_n, bytes / ld_max, ld_max);
        if (mode != 0) {
            const double macs = (double)mma_iters * 128 * mma_n * 16;
            printf("  mma %.0f MAC/clk (%llu clk)", macs / h[16], h[16]);
        }
        printf("\n");
    };
    for (int w : {4, 8, 16}) {
        run(kern<16>, 16, w, 0, 128);
        run(kern<32>, 32, w, 0, 128);
        run(kern<64>, 64, w, 0, 128);
    }
    run(kern<16>, 16, 4, 2, 128);
    run(kern<16>, 16, 4, 2, 256);
    printf("random operands:\n");
    run(kern<16>, 16, 4, 3, 128);
    run(kern<16>, 16, 4, 3, 256);
    printf("commit every 4 MMAs:\n");
    run(kern<16>, 16, 4, 5, 128);
    printf("rotating accumulators every 16 MMAs (+commit per 4):\n");
    run(kern<16>, 16, 4, 8, 128);
    printf("12 warps spinning on mbarrier:\n");
    run(kern<16>, 16, 4, 7, 128);
    printf("random operands + STS traffic:\n");
    run(kern<16>, 16, 4, 4, 128);
    run(kern<16>, 16, 4, 4, 256);
    for (int w : {4, 8}) {
        run(kern<32>, 32, w, 1, 128);
        run(kern<32>, 32, w, 1, 256);
    }
    return 0;
}
