// gemm_tc.cuh — grouped, persistent, warp-specialised tcgen05 GEMM (sm_100a).
//
//   C[m, n] = epilogue( sum_k A[m, k] * Bt[n, k] + bias[n] )
//
// A: bf16 row-major [M][K] (K-major), Bt: bf16 row-major [N][K] (the weight
// pre-transposed at upload, K-major). K is a multiple of 64 (buffers are
// zero-padded). One launch serves up to kMaxProblems independent problems
// (tokenizer sources, fuq+fkv of a target layer, ...): the persistent CTAs
// walk one global tile list, tile t -> (problem, m-block, n-block) with n
// fastest so the CTAs resident at one time share A tiles through L2.
//
// Roles (384 threads): warp 0 TMA producer, warp 1 MMA issuer (one elected
// lane), warp 2 TMEM allocator, warps 4..11 epilogue (two warps per TMEM lane
// quarter, each owning half the columns). Pipelines: kStages smem stages
// (full/empty mbarriers) and 2 TMEM accumulator stages (tmem_full/empty), so
// the epilogue of tile i overlaps the MMAs of tile i+1.
#pragma once

#include "common.cuh"
#include "ptx.cuh"

namespace mtfm {

enum GemmEpi : int {
    EPI_SILU_BF16 = 0,   // out_bf16[m][n] = silu(acc + bias)
    EPI_BIAS_F32 = 1,    // out_f32[row(m)][n] = acc + bias
    EPI_RESID_F32 = 2,   // out_f32[row(m)][n] = (acc + bias) + resid[row(m)][n]
    EPI_BIAS_BF16 = 3,   // out_bf16[m][n] = acc + bias
};

constexpr int kMaxProblems = 16;

struct GemmProblem {
    CUtensorMap tma_a;      // box {64, 128}, SW128
    CUtensorMap tma_b;      // box {64, BN}, SW128
    int M, N, K;
    int tile_start;         // first global tile of this problem
    int tiles_n;
    int epi;
    const float* bias;      // [N] (may be null)
    void* out;
    long long ldo;          // elements
    const int* row_map;     // optional output row indirection (f32 epilogues)
    long long row_offset;   // added to the output row when row_map is null
    const float* resid;     // EPI_RESID_F32
};

struct GemmArgs {
    int n_problems;
    int n_tiles;
    GemmProblem p[kMaxProblems];
};

namespace gemm_detail {

template <int BN>
struct Cfg {
    static constexpr int BM = 128, BK = 64;
    static constexpr int kStages = BN >= 256 ? 4 : 6;
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int TMEM_COLS = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
    static constexpr int SMEM = kStages * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr int kThreads = 384;
};

__device__ __forceinline__ void decode_tile(const GemmArgs& a, int t, int& pi, int& mb, int& nb) {
    pi = 0;
#pragma unroll 1
    for (int i = 1; i < a.n_problems; ++i)
        if (t >= a.p[i].tile_start) pi = i;
    const int local = t - a.p[pi].tile_start;
    mb = local / a.p[pi].tiles_n;
    nb = local - mb * a.p[pi].tiles_n;
}

}  // namespace gemm_detail

template <int BN>
__global__ void __launch_bounds__(384, 1) gemm_tc_kernel(const __grid_constant__ GemmArgs args) {
    using C = gemm_detail::Cfg<BN>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::kStages * C::STAGE_BYTES);
    uint64_t* empty_bar = full_bar + C::kStages;
    uint64_t* tfull_bar = empty_bar + C::kStages;
    uint64_t* tempty_bar = tfull_bar + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

    const uint32_t warp = ptx::warp_id();
    const uint32_t lane = ptx::lane_id();

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            ptx::mbar_init(&full_bar[s], 1);
            ptx::mbar_init(&empty_bar[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(&tfull_bar[s], 1);
            ptx::mbar_init(&tempty_bar[s], 8);  // one arrive per epilogue warp
        }
        ptx::fence_mbar_init();
        for (int i = 0; i < args.n_problems; ++i) {
            ptx::tma_prefetch(&args.p[i].tma_a);
            ptx::tma_prefetch(&args.p[i].tma_b);
        }
    }
    if (warp == 2) ptx::tmem_alloc<C::TMEM_COLS>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (ptx::elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x) {
                int pi, mb, nb;
                gemm_detail::decode_tile(args, t, pi, mb, nb);
                const GemmProblem& p = args.p[pi];
                const int kblocks = p.K / C::BK;
                for (int kb = 0; kb < kblocks; ++kb) {
                    ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * C::STAGE_BYTES;
                    uint8_t* sb = sa + C::A_BYTES;
                    ptx::mbar_arrive_expect_tx(&full_bar[stage], C::STAGE_BYTES);
                    ptx::tma_load_2d(sa, &p.tma_a, &full_bar[stage], kb * C::BK, mb * C::BM);
                    ptx::tma_load_2d(sb, &p.tma_b, &full_bar[stage], kb * C::BK, nb * BN);
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        const uint32_t idesc = ptx::instr_desc_bf16(128, BN, false, false);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x) {
            int pi, mb, nb;
            gemm_detail::decode_tile(args, t, pi, mb, nb);
            const int kblocks = args.p[pi].K / C::BK;
            ptx::mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
            ptx::tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * BN;
            for (int kb = 0; kb < kblocks; ++kb) {
                ptx::mbar_wait(&full_bar[stage], phase);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    const uint32_t sa = ptx::smem_u32(smem + stage * C::STAGE_BYTES);
                    const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
                    for (int k = 0; k < C::BK / 16; ++k) {
                        const uint64_t da = ptx::smem_desc(sa + k * 32, 16, 1024, 2);
                        const uint64_t db = ptx::smem_desc(sb + k * 32, 16, 1024, 2);
                        ptx::umma_bf16(d_tmem, da, db, idesc, (kb | k) != 0);
                    }
                    ptx::umma_commit(&empty_bar[stage]);
                    if (kb == kblocks - 1) ptx::umma_commit(&tfull_bar[acc]);
                }
                __syncwarp();
                if (++stage == C::kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {
        const uint32_t q = warp & 3;               // TMEM lane quarter
        const uint32_t half = (warp - 4) >> 2;     // column half
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x) {
            int pi, mb, nb;
            gemm_detail::decode_tile(args, t, pi, mb, nb);
            const GemmProblem& p = args.p[pi];
            ptx::mbar_wait(&tfull_bar[acc], acc_phase);
            ptx::tc_fence_after();
            const int m = mb * C::BM + q * 32 + lane;
            const bool row_ok = m < p.M;
            long long orow = 0;
            if (row_ok) orow = p.row_map ? static_cast<long long>(p.row_map[m]) : p.row_offset + m;
            const int n_begin = half * (BN / 2);
#pragma unroll 1
            for (int c = n_begin; c < n_begin + BN / 2; c += 16) {
                float v[16];
                ptx::tmem_ld16(tmem_base + ((q * 32u) << 16) + acc * BN + c, v);
                ptx::tmem_ld_wait();
                const int n0 = nb * BN + c;
                if (!row_ok || n0 >= p.N) continue;
                const int nvalid = min(16, p.N - n0);
                if (p.bias) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[i] += (i < nvalid) ? __ldg(p.bias + n0 + i) : 0.f;
                }
                if (p.epi == EPI_SILU_BF16 || p.epi == EPI_BIAS_BF16) {
                    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out) + orow * p.ldo + n0;
                    if (p.epi == EPI_SILU_BF16) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] = ptx::silu_f32(v[i]);
                    }
                    if (nvalid == 16 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
                        uint4 w0, w1;
                        w0.x = pack_bf16(v[0], v[1]);
                        w0.y = pack_bf16(v[2], v[3]);
                        w0.z = pack_bf16(v[4], v[5]);
                        w0.w = pack_bf16(v[6], v[7]);
                        w1.x = pack_bf16(v[8], v[9]);
                        w1.y = pack_bf16(v[10], v[11]);
                        w1.z = pack_bf16(v[12], v[13]);
                        w1.w = pack_bf16(v[14], v[15]);
                        reinterpret_cast<uint4*>(o)[0] = w0;
                        reinterpret_cast<uint4*>(o)[1] = w1;
                    } else {
                        for (int i = 0; i < nvalid; ++i) o[i] = __float2bfloat16_rn(v[i]);
                    }
                } else {
                    float* o = static_cast<float*>(p.out) + orow * p.ldo + n0;
                    if (p.epi == EPI_RESID_F32) {
                        const float* r = p.resid + orow * p.ldo + n0;
                        if (nvalid == 16 && (reinterpret_cast<uintptr_t>(r) & 15) == 0) {
#pragma unroll
                            for (int i = 0; i < 16; i += 4) {
                                float4 rr = *reinterpret_cast<const float4*>(r + i);
                                v[i] += rr.x;
                                v[i + 1] += rr.y;
                                v[i + 2] += rr.z;
                                v[i + 3] += rr.w;
                            }
                        } else {
                            for (int i = 0; i < nvalid; ++i) v[i] += r[i];
                        }
                    }
                    if (nvalid == 16 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
#pragma unroll
                        for (int i = 0; i < 16; i += 4)
                            *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                    } else {
                        for (int i = 0; i < nvalid; ++i) o[i] = v[i];
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty_bar[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<C::TMEM_COLS>(tmem_base);
    }
}

}  // namespace mtfm
