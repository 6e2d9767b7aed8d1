// probe_sparse.cu — establishes the TMEM layout of the 2:4 metadata consumed by
// tcgen05.mma.sp (kind::f16, M=128, K=32 logical) on the device itself.
//
// D = A_dec . B^T with B = identity (N = 32), so D is the decompressed A. The
// compressed A holds the value j+1 at physical column j of every row, so D shows
// where each kept element landed. One experiment per (lane, nibble) flips a single
// metadata nibble from the pattern (0,1) to (2,3); the (row, group) whose output
// changes is the place that nibble feeds. Output: one line per (lane, nibble).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 scripts/probe_sparse.cu -o gpurun_out/probe_sparse
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2602_11235_b200/csrc/ptx.cuh"

using namespace mtfm;

__device__ __forceinline__ uint32_t core_off(int r, int c, int lbo, int sbo) {
    return (r / 8) * sbo + (c / 8) * lbo + (r % 8) * 16 + (c % 8) * 2;
}

__global__ void probe(const uint32_t* meta, float* D, uint32_t idesc) {
    __shared__ __align__(1024) uint8_t sA[128 * 16 * 2];
    __shared__ __align__(1024) uint8_t sB[32 * 32 * 2];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 128 * 16; i += blockDim.x) {
        const int r = i / 16, c = i % 16;
        *reinterpret_cast<__nv_bfloat16*>(sA + core_off(r, c, 128, 256)) = __float2bfloat16(static_cast<float>(c + 1));
    }
    for (int i = tid; i < 32 * 32; i += blockDim.x) {
        const int n = i / 32, k = i % 32;
        *reinterpret_cast<__nv_bfloat16*>(sB + core_off(n, k, 128, 512)) = __float2bfloat16(n == k ? 1.f : 0.f);
    }
    ptx::fence_proxy_async_smem();
    if (warp == 0) ptx::tmem_alloc<64>(&slot);
    if (tid == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_mbar_init();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    {
        const uint32_t w = meta[warp * 32 + lane];
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((warp * 32u) << 16) + 32u),
                     "r"(w)
                     : "memory");
        ptx::tmem_st_wait();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (tid == 0) {
        const uint64_t ad = ptx::smem_desc(ptx::smem_u32(sA), 128, 256, 0);
        const uint64_t bd = ptx::smem_desc(ptx::smem_u32(sB), 128, 512, 0);
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%5], %3, {%6, %6, %6, %6}, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(0), "r"(tmem + 32u), "r"(0));
        ptx::umma_commit(&bar);
    }
    ptx::mbar_wait(&bar, 0);
    ptx::tc_fence_after();
    float v[32];
    ptx::tmem_ld16(tmem + ((warp * 32u) << 16), *reinterpret_cast<float(*)[16]>(v));
    ptx::tmem_ld16(tmem + ((warp * 32u) << 16) + 16, *reinterpret_cast<float(*)[16]>(v + 16));
    ptx::tmem_ld_wait();
    for (int n = 0; n < 32; ++n) D[(warp * 32 + lane) * 32 + n] = v[n];
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<64>(tmem);
}

int main() {
    const uint32_t idesc = (1u << 2) | ptx::instr_desc_bf16(128, 32, false, false);
    uint32_t* dm;
    float* dd;
    cudaMalloc(&dm, 128 * 4);
    cudaMalloc(&dd, 128 * 32 * 4);
    std::vector<uint32_t> meta(128);
    std::vector<float> D(128 * 32);
    auto run = [&]() {
        cudaMemcpy(dm, meta.data(), 128 * 4, cudaMemcpyHostToDevice);
        probe<<<1, 128>>>(dm, dd, idesc);
        const cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("cuda error %s\n", cudaGetErrorString(e));
            exit(1);
        }
        cudaMemcpy(D.data(), dd, 128 * 32 * 4, cudaMemcpyDeviceToHost);
    };
    // baseline: every nibble (0,1) = 0x4 in low-index-first encoding
    for (auto& w : meta) w = 0x44444444u;
    run();
    std::vector<float> base = D;
    printf("baseline row 0:");
    for (int n = 0; n < 32; ++n) printf(" %g", D[n]);
    printf("\nbaseline row 9:");
    for (int n = 0; n < 32; ++n) printf(" %g", D[9 * 32 + n]);
    printf("\n");
    for (int L = 0; L < 128; ++L)
        for (int q = 0; q < 8; ++q) {
            for (auto& w : meta) w = 0x44444444u;
            meta[L] = (meta[L] & ~(0xFu << (4 * q))) | (0xEu << (4 * q));
            run();
            printf("lane %3d nib %d ->", L, q);
            int hits = 0;
            for (int m = 0; m < 128; ++m)
                for (int g = 0; g < 8; ++g) {
                    bool diff = false;
                    for (int p = 0; p < 4; ++p) diff |= D[m * 32 + 4 * g + p] != base[m * 32 + 4 * g + p];
                    if (diff) {
                        ++hits;
                        printf(" (m%d g%d:", m, g);
                        for (int p = 0; p < 4; ++p) printf(" %g", D[m * 32 + 4 * g + p]);
                        printf(")");
                    }
                }
            printf(" hits=%d\n", hits);
        }
    return 0;
}
