// TMA load issue rate from one thread: batch of B boxes (16 KB) issued back to
// back onto one mbarrier, then one wait; repeated. Variants: tensor map in
// param space (grid_constant) with / without prefetch.tensormap, or in global memory.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace mtfm;

__device__ __forceinline__ void body(const CUtensorMap* tm, int rows_boxes, int iters, int batch, int box_bytes,
                                     uint8_t* sm, uint64_t* bar, unsigned long long* out, int prefetch) {
    if (threadIdx.x == 0) {
        if (prefetch) ptx::tma_prefetch(tm);
        unsigned long long t0 = clock64(), t_issue = 0;
        for (int it = 0; it < iters; ++it) {
            unsigned long long a = clock64();
            ptx::mbar_arrive_expect_tx(bar, batch * box_bytes);
            for (int b = 0; b < batch; ++b) {
                const int box = (it * batch + b + blockIdx.x * 37) % rows_boxes;
                ptx::tma_load_2d(sm + b * box_bytes, tm, bar, 0, box * (box_bytes / 128));
            }
            t_issue += clock64() - a;
            ptx::mbar_wait(bar, it & 1);
        }
        out[blockIdx.x * 2] = clock64() - t0;
        out[blockIdx.x * 2 + 1] = t_issue;
    }
}
__global__ void __launch_bounds__(32) k_param(const __grid_constant__ CUtensorMap tm, int rows_boxes, int iters,
                                              int batch, int box_bytes, unsigned long long* out, int prefetch) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    __syncwarp();
    body(&tm, rows_boxes, iters, batch, box_bytes, sm, &bar, out, prefetch);
}
__global__ void __launch_bounds__(32) k_global(const CUtensorMap* tm, int rows_boxes, int iters, int batch,
                                               int box_bytes, unsigned long long* out, int prefetch) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    __syncwarp();
    body(tm, rows_boxes, iters, batch, box_bytes, sm, &bar, out, prefetch);
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    EncFn enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    unsigned long long* out;
    cudaMalloc(&out, 148 * 16);
    const long long bytes = 4LL << 20;
    void* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    CUtensorMap tm;
    cuuint64_t dims[2] = {64, (cuuint64_t)(bytes / 128)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap* dtm;
    cudaMalloc(&dtm, sizeof(tm));
    cudaMemcpy(dtm, &tm, sizeof(tm), cudaMemcpyHostToDevice);
    const int rows_boxes = (int)(bytes / 128 / 128);
    for (int variant = 0; variant < 3; ++variant)
        for (int batch : {1, 4, 8}) {
            const int box_bytes = 16384, iters = 2000 / batch, smem = batch * box_bytes;
            cudaFuncSetAttribute(k_param, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            cudaFuncSetAttribute(k_global, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            for (int rep = 0; rep < 2; ++rep) {
                if (variant == 2) k_global<<<148, 32, smem>>>(dtm, rows_boxes, iters, batch, box_bytes, out, 1);
                else k_param<<<148, 32, smem>>>(tm, rows_boxes, iters, batch, box_bytes, out, variant);
                cudaDeviceSynchronize();
            }
            unsigned long long h[2];
            cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
            const char* names[3] = {"param", "param+prefetch", "global+prefetch"};
            printf("%-16s batch %d: %.0f clk per box total, %.0f clk per box issue, %.1f B/clk/SM\n", names[variant],
                   batch, (double)h[0] / (iters * batch), (double)h[1] / (iters * batch),
                   (double)iters * batch * box_bytes / h[0]);
        }
    return 0;
}
