// tok_tc.cuh — fused tokenizer MLP on tcgen05 (sm_100a), d_model a multiple of 256.
//
//   X[row_map[m]] = silu(E[m] W1 + b1) W2 + b2        (tokenizer.hpp:136-149)
//
// for every sequence source whose embedding concat fits one 64-wide k-block
// (k_pad <= 64). The 2d-wide hidden layer never leaves the SM: per 128-row
// tile and 256-column output pass it is produced in 2d/64 chunks of 64 columns,
//
//   GEMM1_c : Hacc[c%2] (TMEM fp32, 128 x 64)  = E_tile . W1[64c:64c+64]^T + b1_c
//   SiLU    : Hb[c%4]   (TMEM bf16, 128 x 64)  = silu(Hacc[c%2])
//   GEMM2_c : Y         (TMEM fp32, 128 x 256) += Hb[c%4] . W2[n0:n0+256, 64c:64c+64]^T   (A from TMEM)
//
// and Y (+ b2 through the ones-tile MMA) is scattered to columns [n0, n0 + 256)
// of the X rows. Versus the two-GEMM path this removes the 2 x (rows x 2d x 2 B)
// hidden-layer round trip through HBM; for d > 256 every pass recomputes the
// hidden layer (Y is half of TMEM, so only 256 output columns fit), and x̂ (which
// needs whole rows) comes from the separate GLN pass.
//
// Roles (640 threads): warps 0..7 SiLU (two groups of 4, group g owns Hacc[g] /
// Hb[g], Hb[g + 2], i.e. chunks c = g mod 2), warps 8..11 and 16..19 Y epilogue
// (column halves), warp 12 TMEM allocator + GEMM1 issuer, warp 13 W2 producer,
// warp 14 tile + W1/b1 producer, warp 15 GEMM2 issuer. Two producer and two MMA
// threads: one thread issues a TMA load only every ~150-300 clk
// (scripts/ubench_tma.cu), and the per-chunk barrier waits of one MMA thread
// would serialise both GEMMs.
// TMEM columns: Y [0, 256), Hacc [256, 384), Hb [384, 512) (4 chunks: while the Y warps
// drain a tile, GEMM1 and the SiLU warps prepare half of the next tile's hidden layer).
// SMEM: 2 x tile stages (E tile 16 KB + the pass's b2 rows 8 KB), 3 x W1 chunk stages
// (8 KB + the chunk's b1 rows 2 KB), 3 x W2 chunk stages (32 KB), ones tile, Y / x̂ staging.
#pragma once

#include "common.cuh"
#include "ptx.cuh"

namespace mtfm {

constexpr int kTokMaxSrc = 8;
constexpr int kTokThreads = 640;

struct TokSource {
    CUtensorMap tma_e;    // E_s [M][k_pad] bf16, box {64, 128}, SW128 (columns >= k_pad zero-filled)
    CUtensorMap tma_w1;   // W1^T [2d][k_pad] bf16, box {64, 64}, SW128
    CUtensorMap tma_w2;   // W2^T [d][2d] bf16, box {64, 256}, SW128
    CUtensorMap tma_b1;   // b1 tile [2d][16] bf16, box {16, 64}, SW32 (one hidden chunk's rows)
    CUtensorMap tma_b2;   // b2 tile [d][16] bf16, box {16, 256}, SW32 (one output pass's rows)
    const int* row_map;   // X row of source row m
    int M;                // rows
    int k_steps;          // ceil(k_pad / 16)
    int tile_start;       // first global tile
    long long xhat_row0;  // >= 0: also write xhat = (y - mean) * rstd (bf16) to TokArgs::xhat rows xhat_row0 + m
};

struct TokArgs {
    TokSource s[kTokMaxSrc];
    int n_src;
    int n_tiles;          // work items: 128-row tiles x output passes
    int n_pass;           // d_model / 256: output column passes (each recomputes the hidden layer)
    int nch;              // hidden chunks: 2 d_model / 64
    int ldx;              // d_model
    float* X;             // [rows][d_model] fp32
    __nv_bfloat16* xhat;  // [rows][256] bf16, source order: the first target run's normalised context rows
    float eps;
};

namespace tok_detail {
constexpr int BM = 128, D = 256, HC = 64;          // rows per tile, output columns per pass, hidden chunk
constexpr int E_BYTES = BM * 64 * 2;                // 16 KB
constexpr int B2_BYTES = D * 32;                    // 8 KB: the pass's b2 rows [256][16]
constexpr int XS_BYTES = E_BYTES + B2_BYTES;        // tile stage
constexpr int W1_BYTES = HC * 64 * 2;               // 8 KB
constexpr int B1C_BYTES = HC * 32;                  // 2 KB: the chunk's b1 rows [64][16]
constexpr int W1S_BYTES = W1_BYTES + B1C_BYTES;     // W1 stage (multiple of 1 KB: SW128 alignment)
constexpr int W2_BYTES = D * 64 * 2;                // 32 KB
constexpr int kXStages = 2, kWStages = 3;
constexpr int ONES_BYTES = 4096;
// staging: 4 KB per Y warp (32 rows x 128 B of Y; 64 B of x̂), then the x̂ partial-sum exchange
constexpr int STG_BYTES = 8 * 4096;
constexpr int XCH_BYTES = 2 * 128 * 8;
constexpr int BAR_BYTES = 1024;
constexpr int SMEM = 1024 + kXStages * XS_BYTES + kWStages * (W1S_BYTES + W2_BYTES) + ONES_BYTES + STG_BYTES +
                     XCH_BYTES + BAR_BYTES;
static_assert(SMEM <= 227 * 1024, "tok SMEM budget");
constexpr int NHB = 4;  // Hb buffers: SiLU runs up to 4 chunks ahead of GEMM2 (through the Y drain)
constexpr uint32_t Y_COL = 0, HACC_COL = 256, HB_COL = 384;

// work item t -> source s, first row m0, first output column n_off
__device__ __forceinline__ void decode(const TokArgs& a, int t, int& s, int& m0, int& n_off) {
    const int tile = a.n_pass == 1 ? t : t / a.n_pass;
    n_off = (t - tile * a.n_pass) * D;
    s = 0;
#pragma unroll 1
    for (int i = 1; i < a.n_src; ++i)
        if (tile >= a.s[i].tile_start) s = i;
    m0 = (tile - a.s[s].tile_start) * BM;
}
}  // namespace tok_detail

__global__ void __launch_bounds__(kTokThreads, 1) tok_fused_kernel(const __grid_constant__ TokArgs args) {
    using namespace tok_detail;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* xs = base;                                  // tile stages
    uint8_t* w1s = xs + kXStages * XS_BYTES;             // W1 chunk stages
    uint8_t* w2s = w1s + kWStages * W1S_BYTES;           // W2 chunk stages
    uint8_t* ones = w2s + kWStages * W2_BYTES;
    float* stg = reinterpret_cast<float*>(ones + ONES_BYTES);
    float2* xch = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(stg) + STG_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stg) + STG_BYTES + XCH_BYTES);
    uint64_t* x_full = bars;             // [2]
    uint64_t* x_empty = bars + 2;        // [2]
    uint64_t* w1_full = bars + 4;        // [3]
    uint64_t* w1_empty = bars + 7;       // [3]
    uint64_t* hacc_full = bars + 10;     // [2]
    uint64_t* hacc_empty = bars + 12;    // [2]
    uint64_t* hb_full = bars + 14;       // [NHB]
    uint64_t* hb_empty = bars + 18;      // [NHB]
    uint64_t* y_full = bars + 22;
    uint64_t* y_empty = bars + 23;
    uint64_t* w2_full = bars + 24;       // [3]
    uint64_t* w2_empty = bars + 27;      // [3]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 30);

    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    constexpr uint32_t kWarpMma = 15, kWarpTma = 14, kWarpTmaW2 = 13, kWarpAlloc = 12;

    for (int i = threadIdx.x; i < ONES_BYTES / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(ones)[i] = make_uint4(0x3f803f80u, 0u, 0u, 0u);
    ptx::fence_proxy_async_smem();
    if (warp == kWarpTma && lane == 0) {
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&x_full[i], 1);
            ptx::mbar_init(&x_empty[i], 2);  // GEMM1 warp (E, b1) + GEMM2 warp (b2)
            ptx::mbar_init(&hacc_full[i], 1);
            ptx::mbar_init(&hacc_empty[i], 4);
        }
        for (int i = 0; i < NHB; ++i) {
            ptx::mbar_init(&hb_full[i], 4);
            ptx::mbar_init(&hb_empty[i], 1);
        }
        for (int i = 0; i < kWStages; ++i) {
            ptx::mbar_init(&w1_full[i], 1);
            ptx::mbar_init(&w1_empty[i], 1);
            ptx::mbar_init(&w2_full[i], 1);
            ptx::mbar_init(&w2_empty[i], 1);
        }
        ptx::mbar_init(y_full, 1);
        ptx::mbar_init(y_empty, 8);  // every draining warp arrives
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
    // prologue done (barriers, TMEM, SMEM tables): wait for the producer of our inputs
    MTFM_PDL_ENTRY();

    // Y drain by the 8 Y warps once a tile's GEMM2 is done: warp (quarter q, group g)
    // takes its 32 rows and the columns [128 g, 128 g + 128). Each 16-column block goes
    // through the warp's 2 KB staging slot (lane = row on the way in, 16 B chunks
    // XOR-swizzled by row; 4 lanes per row on the way out: 8 row segments of 64 B per
    // store instruction). x̂ needs whole-row statistics: the two warps of a quarter
    // swap their partial sums (both shifted by the row's first value, so that
    // |mean| >> std does not cancel in E[y^2] - mean^2). Y is handed back to the
    // GEMM2 warp as soon as each warp's TMEM reads are done.
    auto drain = [&](uint32_t n_t, int t, uint32_t q, uint32_t grp) {
        int s, m0, n_off;
        tok_detail::decode(args, t, s, m0, n_off);
        const TokSource& src = args.s[s];
        const uint32_t slot = grp * 4 + q;
        const uint32_t wst = ptx::smem_u32(stg) + slot * 4096u;
        const int c4 = lane & 3;         // 16 B chunk of a 64 B x̂ row segment (store phase)
        const int c8 = lane & 7;         // 16 B chunk of a 128 B X row segment (store phase)
        int orow[8];                     // X store phase rows 4i + lane / 8 of the warp's 32
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int m = m0 + static_cast<int>(q * 32) + 4 * i + (lane >> 3);
            orow[i] = m < src.M ? __ldg(src.row_map + m) : -1;
        }
        float* const X = args.X;
        const uint32_t lane_addr = (q * 32u) << 16;
        const int cb0 = static_cast<int>(grp) * (D / 64);
        const bool xh = src.xhat_row0 >= 0;
        float ssum = 0.f, ssq = 0.f, piv = 0.f;
        ptx::mbar_wait(y_full, n_t & 1);
        ptx::tc_fence_after();
        if (xh && grp == 1) piv = ptx::tmem_ld1(tmem + lane_addr + Y_COL);  // the row's first value
#pragma unroll 1
        for (int cb = cb0; cb < cb0 + D / 64; ++cb) {
            float v[32];
            ptx::tmem_ld16(tmem + lane_addr + Y_COL + cb * 32, *reinterpret_cast<float(*)[16]>(v));
            ptx::tmem_ld16(tmem + lane_addr + Y_COL + cb * 32 + 16, *reinterpret_cast<float(*)[16]>(v + 16));
            ptx::tmem_ld_wait();
            if (xh) {
                if (grp == 0 && cb == 0) piv = v[0];
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const float y = v[e] - piv;
                    ssum += y;
                    ssq = fmaf(y, y, ssq);
                }
            }
            if (!xh && cb == cb0 + D / 64 - 1) {
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(y_empty);  // Y is free for the next tile's GEMM2
            }
            // row r = lane, 16 B chunk j at (j ^ (r & 7)); then 8 lanes per row: four whole
            // 128 B row segments per store instruction
#pragma unroll
            for (int j = 0; j < 8; ++j)
                ptx::sts128(wst + lane * 128 + ((j ^ (lane & 7)) << 4), v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            __syncwarp();
            float4 w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int r = 4 * i + (lane >> 3);
                w[i] = ptx::lds128(wst + r * 128 + ((c8 ^ (r & 7)) << 4));
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (orow[i] >= 0)
                    __stcs(reinterpret_cast<float4*>(X + static_cast<long long>(orow[i]) * args.ldx + n_off + cb * 32 + c8 * 4),
                           w[i]);
            __syncwarp();
        }
        if (xh) {
            // whole-row statistics from the two halves (same summation order in both warps)
            xch[grp * 128 + q * 32 + lane] = make_float2(ssum, ssq);
            ptx::named_bar_sync(1 + q, 64);
            const float2 o = xch[(grp ^ 1) * 128 + q * 32 + lane];
            const float s_all = grp == 0 ? ssum + o.x : o.x + ssum;
            const float q_all = grp == 0 ? ssq + o.y : o.y + ssq;
            // second pass over the warp's columns in TMEM: xhat = (y - mean) * rstd (population
            // variance, GLN of hta.hpp:104-109 without the affine, which the folded K|V / f1
            // weights carry). Y goes back to the GEMM2 warp after this pass's last TMEM load.
            const float dm = s_all * (1.f / D);
            const float mean = piv + dm;
            const float var = fmaxf(q_all * (1.f / D) - dm * dm, 0.f);
            const float rstd = rsqrtf(var + args.eps);
#pragma unroll 1
            for (int cb = cb0; cb < cb0 + D / 64; ++cb) {
                float v[32];
                ptx::tmem_ld16(tmem + lane_addr + Y_COL + cb * 32, *reinterpret_cast<float(*)[16]>(v));
                ptx::tmem_ld16(tmem + lane_addr + Y_COL + cb * 32 + 16, *reinterpret_cast<float(*)[16]>(v + 16));
                ptx::tmem_ld_wait();
                if (cb == cb0 + D / 64 - 1) {
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(y_empty);  // Y is free for the next tile's GEMM2
                }
                // row r = lane, 16 B chunk j at (j ^ (r >> 1 & 3)) (conflict-free both ways);
                // then 4 lanes per row, 8 rows x 64 B per store instruction
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    ptx::sts128(wst + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4),
                                __uint_as_float(pack_bf16((v[8 * j] - mean) * rstd, (v[8 * j + 1] - mean) * rstd)),
                                __uint_as_float(pack_bf16((v[8 * j + 2] - mean) * rstd, (v[8 * j + 3] - mean) * rstd)),
                                __uint_as_float(pack_bf16((v[8 * j + 4] - mean) * rstd, (v[8 * j + 5] - mean) * rstd)),
                                __uint_as_float(pack_bf16((v[8 * j + 6] - mean) * rstd, (v[8 * j + 7] - mean) * rstd)));
                __syncwarp();
                float4 w[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int rr = 8 * i + (lane >> 2);
                    w[i] = ptx::lds128(wst + rr * 64 + ((c4 ^ ((rr >> 1) & 3)) << 4));
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int mr = m0 + static_cast<int>(q * 32) + 8 * i + (lane >> 2);
                    if (mr < src.M)
                        *reinterpret_cast<float4*>(args.xhat + (src.xhat_row0 + mr) * D + cb * 32 + c4 * 8) = w[i];
                }
                __syncwarp();
            }
        }
    };

    if (warp == kWarpTma) {
        // ------------------------------------------------ TMA producer
        if (ptx::elect_one()) {
            uint32_t n_t = 0, n_w = 0;
            for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++n_t) {
                int s, m0, n_off;
                decode(args, t, s, m0, n_off);
                const TokSource& src = args.s[s];
                const uint32_t xb = n_t & 1;
                ptx::mbar_wait(&x_empty[xb], ((n_t >> 1) & 1) ^ 1);
                uint8_t* xst = xs + xb * XS_BYTES;
                ptx::mbar_arrive_expect_tx(&x_full[xb], XS_BYTES);
                ptx::tma_load_2d(xst, &src.tma_e, &x_full[xb], 0, m0);
                ptx::tma_load_2d(xst + E_BYTES, &src.tma_b2, &x_full[xb], 0, n_off);
                for (int c = 0; c < args.nch; ++c, ++n_w) {
                    const uint32_t wb = n_w % kWStages;
                    ptx::mbar_wait(&w1_empty[wb], ((n_w / kWStages) & 1) ^ 1);
                    ptx::mbar_arrive_expect_tx(&w1_full[wb], W1S_BYTES);
                    ptx::tma_load_2d(w1s + wb * W1S_BYTES, &src.tma_w1, &w1_full[wb], 0, c * HC);
                    ptx::tma_load_2d(w1s + wb * W1S_BYTES + W1_BYTES, &src.tma_b1, &w1_full[wb], 0, c * HC);
                }
            }
        }
    } else if (warp == kWarpTmaW2) {
        // ------------------------------------------------ W2 producer
        if (ptx::elect_one()) {
            uint32_t n_w = 0;
            for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x) {
                int s, m0, n_off;
                decode(args, t, s, m0, n_off);
                const TokSource& src = args.s[s];
                for (int c = 0; c < args.nch; ++c, ++n_w) {
                    const uint32_t wb = n_w % kWStages;
                    ptx::mbar_wait(&w2_empty[wb], ((n_w / kWStages) & 1) ^ 1);
                    ptx::mbar_arrive_expect_tx(&w2_full[wb], W2_BYTES);
                    ptx::tma_load_2d(w2s + wb * W2_BYTES, &src.tma_w2, &w2_full[wb], c * HC, n_off);
                }
            }
        }
    } else if (warp == kWarpMma) {
        // ------------------------------------------------ GEMM2 issuer: Y += Hb . W2_c^T (+ b2)
        const uint32_t idesc2 = ptx::instr_desc_bf16(128, D, false, false);
        const uint64_t ones_desc = ptx::smem_desc(ptx::smem_u32(ones), 16, 256, 6);
        uint32_t n_t = 0, h = 0;
        for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++n_t) {
            const uint32_t xb = n_t & 1;
            uint8_t* xst = xs + xb * XS_BYTES;
            ptx::mbar_wait(&x_full[xb], (n_t >> 1) & 1);         // b2 tile
            ptx::mbar_wait(y_empty, (n_t & 1) ^ 1);              // the previous tile's Y has been read out
            for (int c = 0; c < args.nch; ++c, ++h) {
                const uint32_t hb = h % NHB, wb = h % kWStages;
                ptx::mbar_wait(&hb_full[hb], (h / NHB) & 1);
                ptx::mbar_wait(&w2_full[wb], (h / kWStages) & 1);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    const uint32_t w2 = ptx::smem_u32(w2s + wb * W2_BYTES);
#pragma unroll
                    for (int k = 0; k < HC / 16; ++k)
                        ptx::umma_bf16_ts(tmem + Y_COL, tmem + HB_COL + hb * (HC / 2) + k * 8,
                                          ptx::smem_desc(w2 + k * 32, 16, 1024, 2), idesc2, (c > 0 || k > 0) ? 1u : 0u);
                    if (c == args.nch - 1)
                        ptx::umma_bf16(tmem + Y_COL, ones_desc,
                                       ptx::smem_desc(ptx::smem_u32(xst + E_BYTES), 16, 256, 6), idesc2, 1u);
                    ptx::umma_commit(&hb_empty[hb]);
                    ptx::umma_commit(&w2_empty[wb]);
                    if (c == args.nch - 1) {
                        ptx::umma_commit(&x_empty[xb]);  // b2 tile consumed (the GEMM1 warp releases E)
                        ptx::umma_commit(y_full);
                    }
                }
                __syncwarp();
            }
        }
    } else if (warp == kWarpAlloc) {
        // ------------------------------------------------ GEMM1 issuer: Hacc = E . W1_c^T + b1_c
        // (a second MMA-issuing warp: the per-chunk waits and issues of the two
        // GEMMs overlap instead of adding up in one thread)
        const uint32_t idesc1 = ptx::instr_desc_bf16(128, HC, false, false);
        const uint64_t ones_desc = ptx::smem_desc(ptx::smem_u32(ones), 16, 256, 6);
        uint32_t n_t = 0, h = 0;
        for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++n_t) {
            int s, m0, n_off;
            tok_detail::decode(args, t, s, m0, n_off);
            const int k_steps = args.s[s].k_steps;
            const uint32_t xb = n_t & 1;
            uint8_t* xst = xs + xb * XS_BYTES;
            ptx::mbar_wait(&x_full[xb], (n_t >> 1) & 1);
            for (int c = 0; c < args.nch; ++c, ++h) {
                const uint32_t wb = h % kWStages, hb = h & 1;
                ptx::mbar_wait(&w1_full[wb], (h / kWStages) & 1);
                ptx::mbar_wait(&hacc_empty[hb], ((h >> 1) & 1) ^ 1);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    const uint32_t e = ptx::smem_u32(xst), w1 = ptx::smem_u32(w1s + wb * W1S_BYTES);
                    for (int k = 0; k < k_steps; ++k)
                        ptx::umma_bf16(tmem + HACC_COL + hb * HC, ptx::smem_desc(e + k * 32, 16, 1024, 2),
                                       ptx::smem_desc(w1 + k * 32, 16, 1024, 2), idesc1, k > 0 ? 1u : 0u);
                    // + b1 rows [64c, 64c + 64), loaded with the W1 chunk (SW32, 256 B per 8 rows)
                    ptx::umma_bf16(tmem + HACC_COL + hb * HC, ones_desc,
                                   ptx::smem_desc(ptx::smem_u32(w1s + wb * W1S_BYTES + W1_BYTES), 16, 256, 6), idesc1, 1u);
                    ptx::umma_commit(&hacc_full[hb]);
                    ptx::umma_commit(&w1_empty[wb]);
                    if (c == args.nch - 1) ptx::umma_commit(&x_empty[xb]);  // E tile consumed
                }
                __syncwarp();
            }
        }
    } else if (warp < 8) {
        // ------------------------------------------------ SiLU warps: Hacc -> silu -> bf16 Hb
        const uint32_t q = warp & 3, g = warp >> 2;
        const uint32_t lane_addr = (q * 32u) << 16;
        uint32_t k = 0;  // chunks of this group
        uint32_t n_t = 0;
        for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++n_t) {
            for (int c = g; c < args.nch; c += 2, ++k) {
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
                // this group's Hb buffers alternate g, g + 2 (chunk c -> c % NHB); the buffer must
                // have been consumed by GEMM2 of the chunk NHB before
                const uint32_t hbb = g + 2 * (k & 1);
                ptx::mbar_wait(&hb_empty[hbb], ((k >> 1) & 1) ^ 1);
                ptx::tc_fence_after();
                ptx::tmem_st16(tmem + lane_addr + HB_COL + hbb * (HC / 2), *reinterpret_cast<uint32_t(*)[16]>(packed));
                ptx::tmem_st16(tmem + lane_addr + HB_COL + hbb * (HC / 2) + 16,
                               *reinterpret_cast<uint32_t(*)[16]>(packed + 16));
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&hb_full[hbb]);
            }
        }
    } else if (warp < 12 || warp >= 16) {
        // ------------------------------------------------ Y epilogue (groups: warps 8..11, 16..19)
        uint32_t n_t = 0;
        for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++n_t) drain(n_t, t, warp & 3, warp >= 16 ? 1u : 0u);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kWarpAlloc) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

}  // namespace mtfm
