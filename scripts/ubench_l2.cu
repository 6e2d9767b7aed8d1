// L2 -> SMEM bandwidth with TMA 2D loads: every CTA (one per SM) streams 16 KB
// boxes of one shared (L2-resident) bf16 matrix through a 4-stage ring.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2602_11235_b200/csrc ubench_l2.cu -o ubench_l2 -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace mtfm;

__global__ void __launch_bounds__(128) kern(const __grid_constant__ CUtensorMap tm, int rows_boxes, int iters,
                                            unsigned long long* out, int stages, int box_bytes, int issuers) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[16];
    if (threadIdx.x == 0) {
        for (int s = 0; s < 16; ++s) ptx::mbar_init(&bar[s], 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    unsigned long long t0 = clock64();
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0 && w < issuers) {
        // issuer w owns stages [w * stages, (w + 1) * stages) of the ring
        int issued = 0, done = 0;
        const int total = iters / issuers;
        uint64_t* bar_w = bar + w * stages;
        uint8_t* sm_w = sm + w * stages * box_bytes;
        while (done < total) {
            while (issued < total && issued - done < stages) {
                const int s = issued % stages;
                ptx::mbar_arrive_expect_tx(&bar_w[s], box_bytes);
                const int box = (issued * 7 + blockIdx.x * 131 + w * 17) % rows_boxes;
                ptx::tma_load_2d(sm_w + s * box_bytes, &tm, &bar_w[s], 0, box * (box_bytes / 128));
                ++issued;
            }
            const int s = done % stages;
            ptx::mbar_wait(&bar_w[s], (done / stages) & 1);
            ++done;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    EncFn enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    unsigned long long* out;
    cudaMalloc(&out, 148 * 8 * 4);
    struct Cfg { long long mb; int stages, box_rows, ctas, issuers; };
    for (Cfg c : {Cfg{4LL << 20, 8, 128, 148, 1}, Cfg{4LL << 20, 4, 128, 148, 2}, Cfg{4LL << 20, 3, 128, 148, 4},
                  Cfg{4LL << 20, 4, 256, 148, 2}, Cfg{4LL << 20, 2, 512, 148, 2}, Cfg{4LL << 20, 8, 32, 148, 1},
                  Cfg{4LL << 20, 8, 32, 148, 4}, Cfg{1LL << 30, 4, 128, 148, 2}}) {
        const long long mb = c.mb;
        void* buf;
        cudaMalloc(&buf, mb);
        cudaMemset(buf, 0, mb);
        const long long rows = mb / 128;  // 64 bf16 columns = 128 B per row
        CUtensorMap tm;
        cuuint64_t dims[2] = {64, (cuuint64_t)rows};
        cuuint64_t strides[1] = {128};
        cuuint32_t box[2] = {64, (cuuint32_t)c.box_rows};
        cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int box_bytes = c.box_rows * 128;
        const int smem = c.stages * box_bytes * c.issuers;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int iters = 2000;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            kern<<<c.ctas, 128, smem>>>(tm, (int)(rows / c.box_rows), iters * 16384 / box_bytes, out, c.stages,
                                         box_bytes, c.issuers);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep)
 printf("footprint %7lld KB stages %2d box %3d rows ctas %d issuers %d: %.1f TB/s aggregate\n", mb >> 10,
                       c.stages, c.box_rows, c.ctas, c.issuers, (double)c.ctas * iters * 16384 / (ms * 1e-3) / 1e12);
        }
        cudaFree(buf);
    }
    return 0;
}
