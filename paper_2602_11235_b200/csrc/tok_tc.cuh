// tok_tc.cuh — fused tokenizer MLP on tcgen05 (sm_100a), d_model = 256.
//
//   X[row_map[m]] = silu(E[m] W1 + b1) W2 + b2        (tokenizer.hpp:136-149)
//
// for every sequence source whose embedding concat fits one 64-wide k-block
// (k_pad <= 64). The 512-wide hidden layer never leaves the SM: per 128-row
// tile it is produced in 8 chunks of 64 columns,
//
//   GEMM1_c : Hacc[c%2] (TMEM fp32, 128 x 64)  = E_tile . W1[64c:64c+64]^T + b1_c
//   SiLU    : Hb[c%2]   (TMEM bf16, 128 x 64)  = silu(Hacc[c%2])
//   GEMM2_c : Y         (TMEM fp32, 128 x 256) += Hb[c%2] . W2[:, 64c:64c+64]^T   (A from TMEM)
//
// and Y (+ b2 through the ones-tile MMA) is scattered to the X rows. Versus
// the two-GEMM path this removes the 2 x (rows x 512 x 2 B) hidden-layer round
// trip through HBM.
//
// Roles (512 threads): warps 0..7 SiLU (two groups of 4, group g owns Hacc[g] /
// Hb[g], i.e. chunks c = g mod 2), warps 8..11 Y epilogue, warp 12 TMEM
// allocator, warp 14 TMA producer, warp 15 MMA issuer.
// TMEM columns: Y [0, 256), Hacc [256, 384), Hb [384, 448).
// SMEM: 2 x tile stages (E tile 16 KB + b2 tile 8 KB), 3 x chunk stages
// (W1 chunk 8 KB + W2 chunk 32 KB + b1 chunk 2 KB), ones tile, Y staging.
#pragma once

#include "common.cuh"
#include "ptx.cuh"

namespace mtfm {

constexpr int kTokMaxSrc = 8;

struct TokSource {
    CUtensorMap tma_e;    // E_s [M][k_pad] bf16, box {64, 128}, SW128 (columns >= k_pad zero-filled)
    CUtensorMap tma_w1;   // W1^T [512][k_pad] bf16, box {64, 64}, SW128
    CUtensorMap tma_w2;   // W2^T [256][512] bf16, box {64, 256}, SW128
    CUtensorMap tma_b1;   // b1 tile [512][16] bf16, box {16, 64}, SW32
    CUtensorMap tma_b2;   // b2 tile [256][16] bf16, box {16, 256}, SW32
    const int* row_map;   // X row of source row m
    int M;                // rows
    int k_steps;          // ceil(k_pad / 16)
    int tile_start;       // first global tile
};

struct TokArgs {
    TokSource s[kTokMaxSrc];
    int n_src;
    int n_tiles;
    float* X;             // [rows][256] fp32
};

namespace tok_detail {
constexpr int BM = 128, D = 256, HC = 64, NCH = 8;  // rows per tile, d_model, hidden chunk, chunks
constexpr int E_BYTES = BM * 64 * 2;                // 16 KB
constexpr int B2_BYTES = D * 32;                    // 8 KB
constexpr int XS_BYTES = E_BYTES + B2_BYTES;        // tile stage
constexpr int W1_BYTES = HC * 64 * 2;               // 8 KB
constexpr int W2_BYTES = D * 64 * 2;                // 32 KB
constexpr int B1_BYTES = HC * 32;                   // 2 KB
constexpr int WS_BYTES = 43 * 1024;                 // chunk stage (42 KB used)
constexpr int kXStages = 2, kWStages = 3;
constexpr int ONES_BYTES = 4096;
constexpr int STG_BYTES = 4 * 32 * 32 * 4;          // Y staging, one 32 x 32 fp32 block per Y warp
constexpr int BAR_BYTES = 1024;
constexpr int SMEM = 1024 + kXStages * XS_BYTES + kWStages * WS_BYTES + ONES_BYTES + STG_BYTES + BAR_BYTES;
static_assert(SMEM <= 227 * 1024, "tok SMEM budget");
constexpr uint32_t Y_COL = 0, HACC_COL = 256, HB_COL = 384;

__device__ __forceinline__ void decode(const TokArgs& a, int t, int& s, int& m0) {
    s = 0;
#pragma unroll 1
    for (int i = 1; i < a.n_src; ++i)
        if (t >= a.s[i].tile_start) s = i;
    m0 = (t - a.s[s].tile_start) * BM;
}
}  // namespace tok_detail

__global__ void __launch_bounds__(512, 1) tok_fused_kernel(const __grid_constant__ TokArgs args) {
    using namespace tok_detail;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* xs = base;                                  // tile stages
    uint8_t* ws = xs + kXStages * XS_BYTES;              // chunk stages
    uint8_t* ones = ws + kWStages * WS_BYTES;
    float* stg = reinterpret_cast<float*>(ones + ONES_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stg) + STG_BYTES);
    uint64_t* x_full = bars;             // [2]
    uint64_t* x_empty = bars + 2;        // [2]
    uint64_t* w_full = bars + 4;         // [3]
    uint64_t* w_empty = bars + 7;        // [3]
    uint64_t* hacc_full = bars + 10;     // [2]
    uint64_t* hacc_empty = bars + 12;    // [2]
    uint64_t* hb_full = bars + 14;       // [2]
    uint64_t* hb_empty = bars + 16;      // [2]
    uint64_t* y_full = bars + 18;
    uint64_t* y_empty = bars + 19;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    constexpr uint32_t kWarpMma = 15, kWarpTma = 14, kWarpAlloc = 12;

    for (int i = threadIdx.x; i < ONES_BYTES / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(ones)[i] = make_uint4(0x3f803f80u, 0u, 0u, 0u);
    ptx::fence_proxy_async_smem();
    if (warp == kWarpTma && lane == 0) {
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&x_full[i], 1);
            ptx::mbar_init(&x_empty[i], 1);
            ptx::mbar_init(&hacc_full[i], 1);
            ptx::mbar_init(&hacc_empty[i], 4);
            ptx::mbar_init(&hb_full[i], 4);
            ptx::mbar_init(&hb_empty[i], 1);
        }
        for (int i = 0; i < kWStages; ++i) {
            ptx::mbar_init(&w_full[i], 1);
            ptx::mbar_init(&w_empty[i], 1);
        }
        ptx::mbar_init(y_full, 1);
        ptx::mbar_init(y_empty, 4);
        ptx::fence_mbar_init();
        for (int i = 0; i < args.n_src; ++i) {
            ptx::tma_prefetch(&args.s[i].tma_e);
            ptx::tma_prefetch(&args.s[i].tma_w1);
            ptx::tma_prefetch(&args.s[i].tma_w2);
        }
    }
    if (warp == kWarpAlloc) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == kWarpTma) {
        // ------------------------------------------------ TMA producer
        if (ptx::elect_one()) {
            uint32_t n_t = 0, n_w = 0;
            for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++n_t) {
                int s, m0;
                decode(args, t, s, m0);
                const TokSource& src = args.s[s];
                const uint32_t xb = n_t & 1;
                ptx::mbar_wait(&x_empty[xb], ((n_t >> 1) & 1) ^ 1);
                ptx::mbar_arrive_expect_tx(&x_full[xb], XS_BYTES);
                ptx::tma_load_2d(xs + xb * XS_BYTES, &src.tma_e, &x_full[xb], 0, m0);
                ptx::tma_load_2d(xs + xb * XS_BYTES + E_BYTES, &src.tma_b2, &x_full[xb], 0, 0);
                for (int c = 0; c < NCH; ++c, ++n_w) {
                    const uint32_t wb = n_w % kWStages;
                    ptx::mbar_wait(&w_empty[wb], ((n_w / kWStages) & 1) ^ 1);
                    uint8_t* st = ws + wb * WS_BYTES;
                    ptx::mbar_arrive_expect_tx(&w_full[wb], W1_BYTES + W2_BYTES + B1_BYTES);
                    ptx::tma_load_2d(st, &src.tma_w1, &w_full[wb], 0, c * HC);
                    ptx::tma_load_2d(st + W1_BYTES, &src.tma_w2, &w_full[wb], c * HC, 0);
                    ptx::tma_load_2d(st + W1_BYTES + W2_BYTES, &src.tma_b1, &w_full[wb], 0, c * HC);
                }
            }
        }
    } else if (warp == kWarpMma) {
        // ------------------------------------------------ MMA issuer
        const uint32_t idesc1 = ptx::instr_desc_bf16(128, HC, false, false);
        const uint32_t idesc2 = ptx::instr_desc_bf16(128, D, false, false);
        const uint64_t ones_desc = ptx::smem_desc(ptx::smem_u32(ones), 16, 256, 6);
        uint32_t n_t = 0, n_w = 0, n_h = 0;  // tiles, chunk stages, hidden chunks (= n_w)
        // GEMM2 of hidden chunk h (stage wb) for tile n_t; c = chunk within the tile
        auto gemm2 = [&](uint32_t h, uint32_t wb, int c, const uint8_t* xst) {
            const uint32_t hb = h & 1;
            if (c == 0) {
                ptx::mbar_wait(y_empty, (n_t & 1) ^ 1);  // the previous tile's Y has been read out
                ptx::tc_fence_after();
            }
            ptx::mbar_wait(&hb_full[hb], (h >> 1) & 1);
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
                const uint32_t w2 = ptx::smem_u32(ws + wb * WS_BYTES + W1_BYTES);
#pragma unroll
                for (int k = 0; k < HC / 16; ++k)
                    ptx::umma_bf16_ts(tmem + Y_COL, tmem + HB_COL + hb * (HC / 2) + k * 8,
                                      ptx::smem_desc(w2 + k * 32, 16, 1024, 2), idesc2, (c > 0 || k > 0) ? 1u : 0u);
                if (c == NCH - 1) {
                    ptx::umma_bf16(tmem + Y_COL, ones_desc,
                                   ptx::smem_desc(ptx::smem_u32(xst + E_BYTES), 16, 256, 6), idesc2, 1u);
                }
                ptx::umma_commit(&hb_empty[hb]);
                ptx::umma_commit(&w_empty[wb]);
                if (c == NCH - 1) {
                    ptx::umma_commit(&x_empty[n_t & 1]);  // E tile and the b2 tile of this stage are consumed
                    ptx::umma_commit(y_full);
                }
            }
            __syncwarp();
        };
        for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++n_t) {
            int s, m0;
            tok_detail::decode(args, t, s, m0);
            const int k_steps = args.s[s].k_steps;
            const uint32_t xb = n_t & 1;
            uint8_t* xst = xs + xb * XS_BYTES;
            ptx::mbar_wait(&x_full[xb], (n_t >> 1) & 1);
            uint32_t prev_wb = 0;
            for (int c = 0; c < NCH; ++c, ++n_w, ++n_h) {
                const uint32_t wb = n_w % kWStages, hb = n_h & 1;
                // GEMM1 chunk c -> Hacc[hb]
                ptx::mbar_wait(&w_full[wb], (n_w / kWStages) & 1);
                ptx::mbar_wait(&hacc_empty[hb], ((n_h >> 1) & 1) ^ 1);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    const uint32_t e = ptx::smem_u32(xst), w1 = ptx::smem_u32(ws + wb * WS_BYTES);
                    for (int k = 0; k < k_steps; ++k)
                        ptx::umma_bf16(tmem + HACC_COL + hb * HC, ptx::smem_desc(e + k * 32, 16, 1024, 2),
                                       ptx::smem_desc(w1 + k * 32, 16, 1024, 2), idesc1, k > 0 ? 1u : 0u);
                    ptx::umma_bf16(tmem + HACC_COL + hb * HC, ones_desc,
                                   ptx::smem_desc(w1 + W1_BYTES + W2_BYTES, 16, 256, 6), idesc1, 1u);
                    ptx::umma_commit(&hacc_full[hb]);
                }
                __syncwarp();
                // GEMM2 of the previous chunk overlaps the SiLU of this one
                if (c > 0) gemm2(n_h - 1, prev_wb, c - 1, xst);
                prev_wb = wb;
            }
            gemm2(n_h - 1, prev_wb, NCH - 1, xst);
        }
    } else if (warp < 8) {
        // ------------------------------------------------ SiLU warps: Hacc -> silu -> bf16 Hb
        const uint32_t q = warp & 3, g = warp >> 2;
        const uint32_t lane_addr = (q * 32u) << 16;
        uint32_t k = 0;  // chunks of this group
        for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x) {
            for (int c = g; c < NCH; c += 2, ++k) {
                ptx::mbar_wait(&hacc_full[g], k & 1);
                ptx::tc_fence_after();
                uint32_t packed[HC / 2];
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    float v[32];
                    ptx::tmem_ld16(tmem + lane_addr + HACC_COL + g * HC + h2 * 32, *reinterpret_cast<float(*)[16]>(v));
                    ptx::tmem_ld16(tmem + lane_addr + HACC_COL + g * HC + h2 * 32 + 16,
                                   *reinterpret_cast<float(*)[16]>(v + 16));
                    ptx::tmem_ld_wait();
                    ptx::silu_bf16_batch<16>(v, packed + h2 * 16);
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&hacc_empty[g]);
                // Hb[g] must have been consumed by GEMM2 of this group's previous chunk
                ptx::mbar_wait(&hb_empty[g], (k & 1) ^ 1);
                ptx::tc_fence_after();
                ptx::tmem_st16(tmem + lane_addr + HB_COL + g * (HC / 2), *reinterpret_cast<uint32_t(*)[16]>(packed));
                ptx::tmem_st16(tmem + lane_addr + HB_COL + g * (HC / 2) + 16,
                               *reinterpret_cast<uint32_t(*)[16]>(packed + 16));
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&hb_full[g]);
            }
        }
    } else if (warp < 12) {
        // ------------------------------------------------ Y epilogue: TMEM -> X rows (fp32)
        const uint32_t q = warp & 3;
        const uint32_t lane_addr = (q * 32u) << 16;
        float* sb = stg + q * 32 * 32;
        const int sub = lane >> 3, ch = lane & 7;
        uint32_t n_t = 0;
        for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++n_t) {
            int s, m0;
            tok_detail::decode(args, t, s, m0);
            const TokSource& src = args.s[s];
            const int rbase = m0 + q * 32;
            int orow[8];
#pragma unroll
            for (int gg = 0; gg < 8; ++gg) {
                const int m = rbase + 4 * gg + sub;
                orow[gg] = m < src.M ? __ldg(src.row_map + m) : -1;
            }
            ptx::mbar_wait(y_full, n_t & 1);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int cb = 0; cb < D / 32; ++cb) {
                float v[32];
                ptx::tmem_ld16(tmem + lane_addr + Y_COL + cb * 32, *reinterpret_cast<float(*)[16]>(v));
                ptx::tmem_ld16(tmem + lane_addr + Y_COL + cb * 32 + 16, *reinterpret_cast<float(*)[16]>(v + 16));
                ptx::tmem_ld_wait();
                if (cb == D / 32 - 1) {
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(y_empty);  // Y is free for the next tile's GEMM2
                }
                // 32 x 32 block through XOR-swizzled SMEM: lane = row on the way in,
                // 4 rows x 128 B per warp store on the way out
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    *reinterpret_cast<float4*>(sb + lane * 32 + ((kk ^ (lane & 7)) << 2)) =
                        make_float4(v[4 * kk], v[4 * kk + 1], v[4 * kk + 2], v[4 * kk + 3]);
                __syncwarp();
#pragma unroll
                for (int gg = 0; gg < 8; ++gg) {
                    const int r = 4 * gg + sub;
                    const float4 w = *reinterpret_cast<const float4*>(sb + r * 32 + ((ch ^ (r & 7)) << 2));
                    if (orow[gg] >= 0)
                        __stcs(reinterpret_cast<float4*>(args.X + static_cast<long long>(orow[gg]) * D + cb * 32 + 4 * ch), w);
                }
                __syncwarp();
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kWarpAlloc) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

}  // namespace mtfm
