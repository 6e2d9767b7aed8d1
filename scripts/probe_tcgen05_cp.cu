// probe_tcgen05_cp.cu — checks the shared-memory source layout of
// tcgen05.cp.cta_group::1.128x128b (row r of a 128 x 16 B matrix -> TMEM lane r,
// columns c..c+3) for a few descriptor encodings, by reading TMEM back.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 scripts/probe_tcgen05_cp.cu -o /tmp/probe_cp
#include <cstdio>
#include <vector>

#include "../paper_2602_11235_b200/csrc/ptx.cuh"

using namespace mtfm;

__global__ void probe(uint32_t lbo, uint32_t sbo, int layout_rows, uint32_t* out) {
    // layout_rows 0: row r at r * 16 (contiguous rows)
    // layout_rows 1: core matrices 8 rows x 16 B, row r at (r / 8) * sbo + (r % 8) * 16
    __shared__ __align__(1024) uint32_t s[128 * 4 * 4];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int r = tid; r < 128; r += blockDim.x)
        for (int c = 0; c < 4; ++c) {
            const uint32_t off = layout_rows == 0 ? r * 16 : (r / 8) * sbo + (r % 8) * 16;
            s[off / 4 + c] = (static_cast<uint32_t>(r) << 8) | c | 0xA0000000u;
        }
    ptx::fence_proxy_async_smem();
    if (warp == 0) ptx::tmem_alloc<32>(&slot);
    if (tid == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_mbar_init();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    if (tid == 0) {
        const uint64_t d = ptx::smem_desc(ptx::smem_u32(s), lbo, sbo, 0);
        asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tmem + 4u), "l"(d));
        ptx::umma_commit(&bar);
    }
    ptx::mbar_wait(&bar, 0);
    ptx::tc_fence_after();
    float v[16];
    ptx::tmem_ld16(tmem + ((warp * 32u) << 16), v);
    ptx::tmem_ld_wait();
    for (int c = 0; c < 4; ++c) out[(warp * 32 + lane) * 4 + c] = __float_as_uint(v[4 + c]);
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<32>(tmem);
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, 128 * 4 * 4);
    std::vector<uint32_t> h(128 * 4);
    struct V { uint32_t lbo, sbo; int rows; };
    const V vs[] = {{16, 128, 0}, {128, 16, 0}, {0, 128, 0}, {2048, 128, 0}, {16, 128, 1}, {128, 128, 1}, {2048, 128, 1}};
    for (const V& v : vs) {
        cudaMemset(d, 0, 128 * 16);
        probe<<<1, 128>>>(v.lbo, v.sbo, v.rows, d);
        const cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("lbo %u sbo %u rows %d: cuda error %s\n", v.lbo, v.sbo, v.rows, cudaGetErrorString(e));
            return 1;
        }
        cudaMemcpy(h.data(), d, 128 * 16, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int r = 0; r < 128; ++r)
            for (int c = 0; c < 4; ++c) bad += h[r * 4 + c] != ((static_cast<uint32_t>(r) << 8) | c | 0xA0000000u);
        printf("lbo %u sbo %u rows %d: mismatches %d; lane 0: %08x %08x %08x %08x lane 9: %08x %08x %08x %08x\n", v.lbo,
               v.sbo, v.rows, bad, h[0], h[1], h[2], h[3], h[36], h[37], h[38], h[39]);
    }
    return 0;
}
