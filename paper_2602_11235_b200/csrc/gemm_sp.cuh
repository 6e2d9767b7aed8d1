// gemm_sp.cuh — 2:4-sparse tcgen05 GEMM (sm_100a, tcgen05.mma.sp kind::f16) for the
// pruned projections f1 / fuq / fkv / f2 (prune.hpp:33-103).
//
//   out[row(t)][f] = epilogue( sum_k W[f][k] X[t][k] + bias[f] )
//
// The pruned weight is the sparse A operand: M = 128 output features per tile, K
// logical, stored compressed (bf16 [N][K/2], the two kept values of every group of
// four in K order) plus metadata (two 2-bit indices per group). The activations X
// are the dense B operand, N = 128 tokens per tile. D = W X^T lands in TMEM with one
// feature per lane, so for a token the 32 lanes of a warp hold 32 consecutive
// features; the epilogue turns them into one 64 B (bf16) / 128 B (fp32) row segment per lane
// through a per-warp SMEM transpose, with the row scatter of the dense path.
//
// Metadata in TMEM (established on the device by scripts/probe_sparse.cu): one
// 32-bit column per MMA (M = 128, K = 32); row m, group g (of four logical K) sits
// in lane (m % 8) + 16 (m / 16) + 8 (g / 4), nibble 4 ((m / 8) % 2) + g % 4, with
// nibble = i0 | i1 << 2 (i0 < i1). In global memory one 128-K block of a feature
// tile is 128 lanes x 4 words (16 B per lane, 2 KB): it rides with the stage's TMA
// loads and is moved into TMEM by one tcgen05.cp 128x128b (row r -> lane r,
// checked by scripts/probe_tcgen05_cp.cu) issued ahead of the stage's four MMAs.
//
// Roles (480 threads): warps 0..11 epilogue (three groups of four, group g drains
// accumulator g), warp 12 TMEM allocator, warp 13 TMA producer, warp 14 MMA issuer.
#pragma once

#include "common.cuh"
#include "gemm_tc.cuh"
#include "ptx.cuh"

namespace mtfm {

struct SpProblem {
    CUtensorMap tma_w;      // compressed W [Np][Kp / 2] bf16, box {64, 128}, SW128
    CUtensorMap tma_x;      // X [M][K] bf16, box {64, 128}, SW128
    const uint32_t* meta;   // [Np / 128][Kp / 128][128 lanes][4 words]
    int M, N, K;            // tokens, features, logical K (multiple of 64)
    int kb;                 // 128-K blocks (Kp / 128)
    int tile_start;         // first global tile of this problem
    int tiles_f;            // feature tiles
    int epi;                // EPI_SILU_BF16 or EPI_RESID_F32
    const float* bias;      // [N] or null
    void* out;
    long long ldo;          // elements
    const int* row_map;     // optional output row of token t
    long long row_offset;   // added to the output row when row_map is null
};

struct SpArgs {
    int n_problems;
    int n_tiles;
    SpProblem p[kMaxProblems];
};

namespace sp_detail {
constexpr int BM = 128, BN = 128;
constexpr int W_BYTES = BM * 64 * 2;        // 128 features x 64 kept values (128 logical K)
constexpr int X_BYTES = 2 * BN * 64 * 2;    // 128 tokens x 128 logical K, two SW128 boxes
constexpr int E_BYTES = 128 * 16;           // metadata: 128 lanes x 4 words
constexpr int STAGE_BYTES = W_BYTES + X_BYTES + E_BYTES;
constexpr int kStages = 3;
constexpr int STG_LD = 36;                        // epilogue staging row: 32 fp32 + 16 B pad (conflict-free both ways)
constexpr int kAcc = 3;                           // TMEM accumulators = epilogue groups of 4 warps
constexpr int kEpiWarps = 4 * kAcc;
constexpr int STG_BYTES = kEpiWarps * 32 * STG_LD * 4;  // per epilogue warp: 32 tokens
constexpr int BAR_BYTES = 256;
constexpr int SMEM = 1024 + kStages * STAGE_BYTES + STG_BYTES + BAR_BYTES + kMaxProblems * 4;
constexpr int kThreads = 32 * (kEpiWarps + 3);
constexpr uint32_t ACC_COL = 0, META_COL = kAcc * BN;  // TMEM: kAcc 128-column accumulators, then 4 metadata columns per stage
static_assert(SMEM <= 227 * 1024, "sparse GEMM SMEM budget");

__device__ __forceinline__ void decode(const SpArgs& a, const int* ts, int t, int& pi, int& tt, int& ft) {
    pi = 0;
#pragma unroll 1
    for (int i = 1; i < a.n_problems; ++i)
        if (t >= ts[i]) pi = i;
    const int local = t - ts[pi];
    tt = local / a.p[pi].tiles_f;
    ft = local - tt * a.p[pi].tiles_f;
}

__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            ptx::smem_u32(smem)),
        "l"(reinterpret_cast<uint64_t>(gmem)), "r"(bytes), "r"(ptx::smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tmem_cp_128x128b(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(taddr), "l"(sdesc));
}

__device__ __forceinline__ void umma_sp_bf16(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc, uint32_t tmem_e,
                                             uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%5], %3, {%6, %6, %6, %6}, p;\n\t}" ::"r"(tmem_d),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(tmem_e), "r"(0));
}
}  // namespace sp_detail

__global__ void __launch_bounds__(sp_detail::kThreads, 1) gemm_sp_kernel(const __grid_constant__ SpArgs args) {
    using namespace sp_detail;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float* stg = reinterpret_cast<float*>(base + kStages * STAGE_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + kStages * STAGE_BYTES + STG_BYTES);
    uint64_t* full = bars;              // [kStages]
    uint64_t* empty = bars + kStages;   // [kStages]
    uint64_t* acc_full = bars + 2 * kStages;   // [kAcc]
    uint64_t* acc_empty = acc_full + kAcc;     // [kAcc]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + kAcc);
    int* s_ts = reinterpret_cast<int*>(base + kStages * STAGE_BYTES + STG_BYTES + BAR_BYTES);

    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    constexpr uint32_t kWarpAlloc = kEpiWarps, kWarpTma = kEpiWarps + 1, kWarpMma = kEpiWarps + 2;
    for (int i = threadIdx.x; i < args.n_problems; i += blockDim.x) s_ts[i] = args.p[i].tile_start;
    if (warp == kWarpTma && lane == 0) {
        for (int i = 0; i < kStages; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < kAcc; ++i) {
            ptx::mbar_init(&acc_full[i], 1);
            ptx::mbar_init(&acc_empty[i], 4);
        }
        ptx::fence_mbar_init();
        for (int i = 0; i < args.n_problems; ++i) {
            ptx::tma_prefetch(&args.p[i].tma_w);
            ptx::tma_prefetch(&args.p[i].tma_x);
        }
    }
    if (warp == kWarpAlloc) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    MTFM_PDL_ENTRY();

    if (warp == kWarpTma) {
        if (ptx::elect_one()) {
            uint32_t it = 0;
            for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x) {
                int pi, tt, ft;
                decode(args, s_ts, t, pi, tt, ft);
                const SpProblem& p = args.p[pi];
                for (int kb = 0; kb < p.kb; ++kb, ++it) {
                    const uint32_t s = it % kStages;
                    ptx::mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
                    uint8_t* st = base + s * STAGE_BYTES;
                    const bool two = p.K - kb * 128 >= 128;  // second 64-K box inside the matrix
                    ptx::mbar_arrive_expect_tx(&full[s], W_BYTES + (two ? 2 : 1) * (X_BYTES / 2) + E_BYTES);
                    ptx::tma_load_2d(st, &p.tma_w, &full[s], kb * 64, ft * BM);
                    ptx::tma_load_2d(st + W_BYTES, &p.tma_x, &full[s], kb * 128, tt * BN);
                    if (two) ptx::tma_load_2d(st + W_BYTES + X_BYTES / 2, &p.tma_x, &full[s], kb * 128 + 64, tt * BN);
                    bulk_g2s(st + W_BYTES + X_BYTES, p.meta + (static_cast<long long>(ft) * p.kb + kb) * 512, E_BYTES,
                             &full[s]);
                }
            }
        }
    } else if (warp == kWarpMma) {
        const uint32_t idesc = (1u << 2) | ptx::instr_desc_bf16(BM, BN, false, false);  // sparse flag
        uint32_t it = 0, n_t = 0;
        for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++n_t) {
            int pi, tt, ft;
            decode(args, s_ts, t, pi, tt, ft);
            const SpProblem& p = args.p[pi];
            const uint32_t acc = n_t % kAcc;
            ptx::mbar_wait(&acc_empty[acc], ((n_t / kAcc) & 1) ^ 1);
            ptx::tc_fence_after();
            for (int kb = 0; kb < p.kb; ++kb, ++it) {
                const uint32_t s = it % kStages;
                ptx::mbar_wait(&full[s], (it / kStages) & 1);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    const uint8_t* st = base + s * STAGE_BYTES;
                    const uint32_t meta_t = tmem + META_COL + 4 * s;
                    tmem_cp_128x128b(meta_t, ptx::smem_desc(ptx::smem_u32(st + W_BYTES + X_BYTES), 16, 128, 0));
                    const int n_mma = min(4, (p.K - kb * 128) / 32);
                    for (int j = 0; j < n_mma; ++j) {
                        const uint64_t ad = ptx::smem_desc(ptx::smem_u32(st) + j * 32, 16, 1024, 2);
                        const uint64_t bd =
                            ptx::smem_desc(ptx::smem_u32(st + W_BYTES + (j >> 1) * (X_BYTES / 2)) + (j & 1) * 64, 16,
                                           1024, 2);
                        // metadata column meta_t + j: even column address, odd one through the
                        // descriptor's id2 bit (an odd column address faults as misaligned)
                        umma_sp_bf16(tmem + ACC_COL + acc * BN, ad, bd, meta_t + (j & ~1), idesc | (j & 1),
                                     (kb > 0 || j > 0) ? 1u : 0u);
                    }
                    ptx::umma_commit(&empty[s]);
                    if (kb == p.kb - 1) ptx::umma_commit(&acc_full[acc]);
                }
                __syncwarp();
            }
        }
    } else if (warp < kEpiWarps) {
        // epilogue group g drains accumulator g (tiles n_t with n_t % kAcc == g); lane = feature.
        // SiLU -> bf16: per 32-token block through SMEM [token][feature], then lane = token writes
        // its 32 features (64 B) to its row (scattered through row_map; measured faster than
        // 4 lanes per row). Residual (contiguous rows): per token the warp's 32 features are one
        // 128 B segment, read and written straight from registers.
        const uint32_t g = warp >> 2, q = warp & 3;
        const uint32_t sw = ptx::smem_u32(stg) + warp * (32 * STG_LD * 4);
        uint32_t n_t = 0, k = 0;
        for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++n_t) {
            if (n_t % kAcc != g) continue;
            int pi, tt, ft;
            decode(args, s_ts, t, pi, tt, ft);
            const SpProblem& p = args.p[pi];
            const int f0 = ft * BM + static_cast<int>(q * 32);
            const int nval = min(max(p.N - f0, 0), 32);  // valid features of this warp (a multiple of 8)
            const bool fv = static_cast<int>(lane) < nval;
            const float bf = (p.bias && fv) ? __ldg(p.bias + f0 + lane) : 0.f;
            const bool silu = p.epi == EPI_SILU_BF16;
            // SiLU store phase: lane = token, its 32 features as 4 x 16 B to its (scattered) row
            long long rr[BN / 32];
            if (silu) {
#pragma unroll
                for (int cb = 0; cb < BN / 32; ++cb) {
                    const int tok = tt * BN + cb * 32 + static_cast<int>(lane);
                    rr[cb] = tok < p.M ? (p.row_map ? static_cast<long long>(__ldg(p.row_map + tok))
                                                    : p.row_offset + tok)
                                       : -1;
                }
            }
            ptx::mbar_wait(&acc_full[g], k & 1);
            ++k;
            ptx::tc_fence_after();
#pragma unroll
            for (int cb = 0; cb < BN / 32; ++cb) {
                float v[32];
                const uint32_t ta = tmem + ((q * 32u) << 16) + ACC_COL + g * BN + cb * 32;
                ptx::tmem_ld16(ta, *reinterpret_cast<float(*)[16]>(v));
                ptx::tmem_ld16(ta + 16, *reinterpret_cast<float(*)[16]>(v + 16));
                ptx::tmem_ld_wait();
                if (cb == BN / 32 - 1) {
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&acc_empty[g]);
                }
                const int tok0 = tt * BN + cb * 32;
                if (silu) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) ptx::sts32(sw + (j * STG_LD + lane) * 4, ptx::silu_fast(v[j] + bf));
                    __syncwarp();
                    float4 w[8];
#pragma unroll
                    for (int c = 0; c < 8; ++c) w[c] = ptx::lds128(sw + (lane * STG_LD + 4 * c) * 4);
                    const long long r = rr[cb];
                    if (r >= 0) {
                        __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out) + r * p.ldo + f0;
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            if (8 * c < nval)
                                *reinterpret_cast<uint4*>(o + 8 * c) =
                                    make_uint4(pack_bf16(w[2 * c].x, w[2 * c].y), pack_bf16(w[2 * c].z, w[2 * c].w),
                                               pack_bf16(w[2 * c + 1].x, w[2 * c + 1].y),
                                               pack_bf16(w[2 * c + 1].z, w[2 * c + 1].w));
                    }
                    __syncwarp();
                } else {
                    // residual rows first (32 independent 128 B loads in flight), then the stores
                    const int jn = min(32, p.M - tok0);
                    float* o = static_cast<float*>(p.out) + (p.row_offset + tok0) * p.ldo + f0 + lane;
                    float old[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) old[j] = (j < jn && fv) ? o[j * p.ldo] : 0.f;
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (j < jn && fv) o[j * p.ldo] = (v[j] + bf) + old[j];
                }
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

// Compressed 2:4 form of a K-major bf16 weight W [N][ldw] (K logical columns):
// comp [Np][Kp / 2] and metadata words in the gemm_sp layout; one thread per word
// (feature tile ft, 128-K block kb, lane, column c). Groups with more than two
// non-zeros are counted in *bad (the weight is not 2:4; the caller rejects it).
__global__ void sp_compress_kernel(const __nv_bfloat16* __restrict__ w, long long ldw, int N, int K, int Np, int KB,
                                   __nv_bfloat16* __restrict__ comp, uint32_t* __restrict__ meta,
                                   unsigned long long* bad) {
    const long long n_words = static_cast<long long>(Np / 128) * KB * 512;
    const long long Kh = static_cast<long long>(KB) * 64;  // compressed row length
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n_words;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i & 3), lane = static_cast<int>((i >> 2) & 127);
        const long long blk = i >> 9;
        const int kb = static_cast<int>(blk % KB), ft = static_cast<int>(blk / KB);
        uint32_t word = 0;
        for (int qn = 0; qn < 8; ++qn) {
            const int m = (lane & 7) + 8 * (qn >> 2) + 16 * (lane >> 4);
            const int gl = 4 * ((lane >> 3) & 1) + (qn & 3);
            const int n = ft * 128 + m;
            const int k0 = kb * 128 + c * 32 + gl * 4;
            float x[4];
            int nz[4], cnt = 0;
            for (int e = 0; e < 4; ++e) {
                x[e] = (n < N && k0 + e < K) ? __bfloat162float(w[static_cast<long long>(n) * ldw + k0 + e]) : 0.f;
                if (x[e] != 0.f) nz[cnt++] = e;
            }
            int i0, i1;
            if (cnt >= 2) {
                i0 = nz[0];
                i1 = nz[1];
                if (cnt > 2) atomicAdd(bad, 1ull);
            } else if (cnt == 1) {
                const int o = nz[0] == 0 ? 1 : 0;
                i0 = min(nz[0], o);
                i1 = max(nz[0], o);
            } else {
                i0 = 0;
                i1 = 1;
            }
            word |= static_cast<uint32_t>(i0 | (i1 << 2)) << (4 * qn);
            comp[static_cast<long long>(n) * Kh + k0 / 2] = __float2bfloat16_rn(x[i0]);
            comp[static_cast<long long>(n) * Kh + k0 / 2 + 1] = __float2bfloat16_rn(x[i1]);
        }
        meta[i] = word;
    }
}

}  // namespace mtfm
