// gemm_tc.cuh — grouped, persistent, warp-specialised tcgen05 GEMM (sm_100a).
//
//   C[m, n] = epilogue( sum_k A[m, k] * Bt[n, k] + bias[n] )
//
// Bt: bf16 row-major [N][K] (the weight pre-transposed at upload, K-major) and
// A: bf16 row-major [M][K], both TMA-loaded (128 x 64 / BN x 64 per k-block,
// SW128 K-major in SMEM).
// One launch serves up to kMaxProblems independent problems (tokenizer
// sources, fkv+fuq of a target layer, ...): the persistent CTAs walk one
// global tile list, tile t -> (problem, m-block, n-block), n fastest, so the
// CTAs resident at one time share A tiles through L2.
//
// Roles (512 threads): warp 15 MMA issuer (one elected lane), warp 14 TMA,
// warp 13 TMEM allocator, warps 0..7 (0..11) epilogue (warp & 3 = TMEM lane
// quarter). The single-thread roles sit at
// the highest warp ids because the issue arbiter favours higher ids.
// Pipelines: kStages SMEM stages (full/empty mbarriers) and 2 TMEM
// accumulator stages (tmem_full/empty), so the epilogue of tile i overlaps
// the MMAs of tile i+1. The epilogue stages each 32 x 32 block through
// XOR-swizzled SMEM so global stores are 128-byte row segments.
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
    CUtensorMap tma_a;      // box {64, 128} (2D) or {64, 128, stage_kb} (3D k-block view), SW128
    CUtensorMap tma_b;      // box {64, BN} or {64, BN, stage_kb}, SW128
    CUtensorMap tma_c;      // output, box {32, 32}: bf16 SW64 / f32 SW128 (use_tma_c)
    int use_tma_c;          // plain row-major output rows [0, M): bulk-tensor stores
    int use_tma_r;          // EPI_RESID_F32 with resid == out: residual blocks TMA-prefetched via tma_c
    int use_scatter_c;      // bf16 output through row_map: staged like use_tma_c, then 128-byte row-segment stores
    int M, N, K;            // K padded to a multiple of 64
    int tile_start;         // first global tile of this problem
    int tiles_n;
    int epi;
    int has_bias;           // bias added by one extra K=16 MMA: ones(128 x 16) x bias_t(BN x 16)^T
    CUtensorMap tma_bias;   // bias_t bf16 [N][16] = (hi, lo, 0, ...), box {16, BN}, SW32
    void* out;
    long long ldo;          // elements
    const int* row_map;     // optional output row indirection (f32 epilogues)
    long long row_offset;   // added to the output row when row_map is null
    const float* resid;     // EPI_RESID_F32
};

// B-resident schedule: CTA b owns (problem pi, n-block nb) for the whole launch,
// keeps that weight slice in SMEM and walks m-blocks m0, m0 + mstep, ...
struct CtaWork {
    short pi, nb;
    int m0, mstep, mcount;
};

struct GemmArgs {
    int n_problems;
    int n_tiles;
    int b_res;        // 1: B-resident schedule (cta[]), 0: streaming over the global tile list
    int n_stages;     // SMEM pipeline stages
    int stage_kb;     // k-blocks per stage: > 1 only when every K is a multiple of 64 (3D tensor maps, one TMA per stage)
    int stage_bytes;  // stage_kb x (A_BYTES (+ B_BYTES when streaming B)) (+ bias tile)
    int bres_bytes;   // resident B slice bytes (b_res)
    int n_epi;        // epilogue warps: 8, or 12 when BN < 256 (more accumulators than 2 groups)
    int stg_warp;     // epilogue staging bytes per warp: 8 KB (2 fp32 blocks), 4 KB when every problem is a bf16 bulk store
    int bias_bytes;   // BN x 32 B bias tile: after the resident B slice (b_res) or at the end of every stage
    int cl;           // 2: CTA pairs (clusters) on m-block pairs share each B k-block by TMA multicast
                      // (streaming schedule, one k-block per stage; tile_start / n_tiles count pairs)
    GemmProblem p[kMaxProblems];
    CtaWork cta[kNumSMs];
};

namespace gemm_detail {

template <int BN>
struct Cfg {
    static constexpr int BM = 128, BK = 64;
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int kAcc = BN >= 256 ? 2 : 4;  // TMEM accumulator buffers
    static constexpr int TMEM_COLS = kAcc * BN <= 32 ? 32 : (kAcc * BN <= 64 ? 64 : (kAcc * BN <= 128 ? 128 : (kAcc * BN <= 256 ? 256 : 512)));
    static constexpr int STG_WARP = 2 * 32 * 32 * 4;  // per epilogue warp: 2 x (32 rows x 32 fp32)
    static constexpr int BAR_BYTES = 1024;  // mbarriers, TMEM slot, per-problem tables
    static constexpr int kMaxSmem = 227 * 1024;
    static constexpr int kThreads = 512;
};

// The tile sequence of this CTA (identical for every role).
// B-resident: the CTA's (problem, n-block, m-blocks) held in registers;
// streaming: global tile t -> (problem, m, n) through the SMEM tile_start table.
struct TileSeq {
    int t, i, tstep;
    int b_res, pi0, nb0, m0, mstep, mcount, n_tiles, n_problems, cl, rank;
    const int* tile_start;  // SMEM: first global tile of each problem
    const int* tiles_n;     // SMEM: n-blocks of each problem
    __device__ TileSeq(const GemmArgs& a, const int* ts, const int* tn)
        : t(blockIdx.x / a.cl), i(0), tstep(gridDim.x / a.cl), b_res(a.b_res), n_tiles(a.n_tiles),
          n_problems(a.n_problems), cl(a.cl), rank(blockIdx.x % a.cl), tile_start(ts), tiles_n(tn) {
        const CtaWork w = a.cta[blockIdx.x];
        pi0 = w.pi;
        nb0 = w.nb;
        m0 = w.m0;
        mstep = w.mstep;
        mcount = w.mcount;
    }
    __device__ __forceinline__ bool next(int& pi, int& mb, int& nb) {
        if (b_res) {
            if (i >= mcount) return false;
            pi = pi0;
            nb = nb0;
            mb = m0 + i * mstep;
            ++i;
            return true;
        }
        if (t >= n_tiles) return false;
        pi = 0;
#pragma unroll 1
        for (int k = 1; k < n_problems; ++k)
            if (t >= tile_start[k]) pi = k;
        const int local = t - tile_start[pi];
        mb = local / tiles_n[pi];
        nb = local - mb * tiles_n[pi];
        mb = mb * cl + rank;  // cluster: the pair's m-blocks (the second may lie past M: zero-filled, not stored)
        t += tstep;
        return true;
    }
    // advance past one tile without decoding it; false at the end of the sequence
    __device__ __forceinline__ bool skip() {
        if (b_res) return i++ < mcount;
        const bool more = t < n_tiles;
        t += tstep;
        return more;
    }
};

}  // namespace gemm_detail

template <int BN>
__global__ void __launch_bounds__(512, 1) gemm_tc_kernel(const __grid_constant__ GemmArgs args) {
    using C = gemm_detail::Cfg<BN>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem0 = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* bres = smem0;                               // resident B slice (+ its bias tile) (b_res)
    uint8_t* ones = smem0 + args.bres_bytes;             // 128 x 16 bf16 ones tile (SW32), A operand of the bias MMA
    uint8_t* smem = ones + 4096;                         // pipeline stages
    const int n_stages = args.n_stages;
    const int stage_bytes = args.stage_bytes;
    const int KS = args.stage_kb;
    float* stg_all = reinterpret_cast<float*>(smem + n_stages * stage_bytes);
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + n_stages * stage_bytes + args.n_epi * args.stg_warp);
    uint64_t* empty_bar = full_bar + 8;
    uint64_t* tfull_bar = empty_bar + 8;
    uint64_t* tempty_bar = tfull_bar + 4;
    uint64_t* res_bar = tempty_bar + 4;  // [12 epilogue warps][2 staging buffers]
    uint64_t* bres_bar = res_bar + 24;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres_bar + 1);
    int* s_tile_start = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(full_bar) + 512);
    int* s_tiles_n = s_tile_start + kMaxProblems;
    int* s_kblocks = s_tiles_n + kMaxProblems;
    int* s_has_bias = s_kblocks + kMaxProblems;
    if (threadIdx.x < static_cast<unsigned>(args.n_problems)) {
        const GemmProblem& p = args.p[threadIdx.x];
        s_tile_start[threadIdx.x] = p.tile_start;
        s_tiles_n[threadIdx.x] = p.tiles_n;
        s_kblocks[threadIdx.x] = p.K / C::BK;
        s_has_bias[threadIdx.x] = p.has_bias;
    }

    // ones tile: every 16-byte chunk = (1, 1, 0, ..., 0). With bias_t = (hi, lo, 0, ...)
    // the K=16 MMA adds hi + lo whichever chunk the swizzle puts first.
    for (int i = threadIdx.x; i < 4096 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(ones)[i] = make_uint4(0x3f803f80u, 0u, 0u, 0u);
    ptx::fence_proxy_async_smem();

    const uint32_t warp = ptx::warp_id();
    const uint32_t lane = ptx::lane_id();
    // Warp roles. The issue arbiter favours higher warp ids, so the latency-
    // critical single-thread roles sit at the top: 15 MMA issuer, 14 TMA
    // producer, 13 TMEM allocator; epilogue warps 0..n_epi-1 (warp & 3 = TMEM
    // lane quarter).
    constexpr uint32_t kWarpMma = 15, kWarpTma = 14, kWarpAlloc = 13, kWarpTma2 = 12;

    if (warp == kWarpTma && lane == 0) {
        for (int s = 0; s < n_stages; ++s) {
            ptx::mbar_init(&full_bar[s], 1);
            ptx::mbar_init(&empty_bar[s], args.cl);  // the MMA commit of every CTA of the cluster
        }
        ptx::mbar_init(bres_bar, 1);
        for (int s = 0; s < C::kAcc; ++s) {
            ptx::mbar_init(&tfull_bar[s], 1);
            ptx::mbar_init(&tempty_bar[s], 4);  // one arrive per warp of the epilogue group
        }
        for (int s = 0; s < 24; ++s) ptx::mbar_init(&res_bar[s], 1);
        ptx::fence_mbar_init();
        for (int i = 0; i < args.n_problems; ++i) {
            ptx::tma_prefetch(&args.p[i].tma_a);
            ptx::tma_prefetch(&args.p[i].tma_b);
        }
    }
    if (warp == kWarpAlloc) ptx::tmem_alloc<C::TMEM_COLS>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    if (args.cl > 1) ptx::cluster_sync();  // peers' barriers initialised before any multicast
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t cl_rank = args.cl > 1 ? ptx::cluster_ctarank() : 0;
    // prologue done (barriers, TMEM, SMEM tables): wait for the producer of our inputs
    MTFM_PDL_ENTRY();

    if (warp == kWarpTma || warp == kWarpTma2) {
        // ------------------------------------------------ TMA producers (A and B)
        // two issuing warps take alternate stages: one thread issues a TMA load only every
        // few hundred clocks (scripts/ubench_l2.cu: 8 TB/s aggregate L2 -> SMEM with one
        // issuer per SM, 16 TB/s with two)
        const int prod = warp == kWarpTma ? 0 : 1;
        if (ptx::elect_one()) {
            if (prod == 0 && args.b_res && args.cta[blockIdx.x].mcount > 0) {
                // resident weight slice: every k-block of this CTA's (problem, n-block), once
                const CtaWork& w = args.cta[blockIdx.x];
                const GemmProblem& p = args.p[w.pi];
                const int kblocks = p.K / C::BK;
                ptx::mbar_arrive_expect_tx(bres_bar, kblocks * C::B_BYTES + (p.has_bias ? BN * 32 : 0));
                for (int kb = 0; kb < kblocks; ++kb)
                    ptx::tma_load_2d(bres + kb * C::B_BYTES, &p.tma_b, bres_bar, kb * C::BK, w.nb * BN);
                if (p.has_bias) ptx::tma_load_2d(bres + kblocks * C::B_BYTES, &p.tma_bias, bres_bar, 0, w.nb * BN);
            }
            int stage = 0;
            uint32_t phase = 0;
            uint32_t it = 0;  // stage iterations (producer prod issues it % 2 == prod)
            gemm_detail::TileSeq seq(args, s_tile_start, s_tiles_n);
            int pi, mb, nb;
            while (seq.next(pi, mb, nb)) {
                const GemmProblem& p = args.p[pi];
                const int kblocks = s_kblocks[pi];
                const bool p_bias = s_has_bias[pi];
                for (int kb = 0; kb < kblocks; kb += KS, ++it) {
                    if ((it & 1) != prod) {
                        if (++stage == n_stages) {
                            stage = 0;
                            phase ^= 1;
                        }
                        continue;
                    }
                    ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * stage_bytes;
                    uint8_t* sb = sa + KS * C::A_BYTES;
                    const bool bias_here = !args.b_res && p_bias && kb + KS >= kblocks;  // streaming: bias tile with the last stage
                    const int bytes = KS * C::A_BYTES + (args.b_res ? 0 : KS * C::B_BYTES) + (bias_here ? BN * 32 : 0);
                    ptx::mbar_arrive_expect_tx(&full_bar[stage], bytes);
                    // one TMA instruction per operand and stage (each costs ~150 clk of issue)
                    if (KS > 1) ptx::tma_load_3d(sa, &p.tma_a, &full_bar[stage], 0, mb * C::BM, kb);
                    else ptx::tma_load_2d(sa, &p.tma_a, &full_bar[stage], kb * C::BK, mb * C::BM);
                    if (args.cl > 1) {
                        // this CTA's half of the B k-block (BN / 2 rows, box {64, BN / 2}) to both CTAs
                        ptx::tma_load_2d_mc(sb + cl_rank * (BN / 2) * 128, &p.tma_b, &full_bar[stage], kb * C::BK,
                                            nb * BN + static_cast<int>(cl_rank) * (BN / 2), 0x3);
                    } else if (!args.b_res) {
                        if (KS > 1) ptx::tma_load_3d(sb, &p.tma_b, &full_bar[stage], 0, nb * BN, kb);
                        else ptx::tma_load_2d(sb, &p.tma_b, &full_bar[stage], kb * C::BK, nb * BN);
                    }
                    if (bias_here) ptx::tma_load_2d(sb + KS * C::B_BYTES, &p.tma_bias, &full_bar[stage], 0, nb * BN);
                    if (++stage == n_stages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == kWarpMma) {
        // ------------------------------------------------ MMA issuer (one elected lane per stage)
        const uint32_t idesc = ptx::instr_desc_bf16(128, BN, false, false);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        bool bres_ready = false;
        gemm_detail::TileSeq seq(args, s_tile_start, s_tiles_n);
        int pi, mb, nb;
        while (seq.next(pi, mb, nb)) {
            const int kblocks = s_kblocks[pi];
            if (args.b_res && !bres_ready) {
                ptx::mbar_wait(bres_bar, 0);
                bres_ready = true;
            }
            // the epilogue hands every accumulator back, including before its first use
            ptx::mbar_wait(&tempty_bar[acc], acc_phase);
            ptx::tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * BN;
            const bool has_bias = s_has_bias[pi];
            for (int kb0 = 0; kb0 < kblocks; kb0 += KS) {
                // TMA -> MMA is async-proxy to async-proxy through the mbarrier
                ptx::mbar_wait(&full_bar[stage], phase);
                const int nk = min(KS, kblocks - kb0);
                const bool last = kb0 + KS >= kblocks;
                if (ptx::elect_one()) {
                    const uint32_t sa0 = ptx::smem_u32(smem + stage * stage_bytes);
                    const uint32_t sb0 = args.b_res ? ptx::smem_u32(bres + kb0 * C::B_BYTES) : sa0 + KS * C::A_BYTES;
                    for (int kbi = 0; kbi < nk; ++kbi) {
                        const uint32_t sa = sa0 + kbi * C::A_BYTES, sb = sb0 + kbi * C::B_BYTES;
#pragma unroll
                        for (int k = 0; k < C::BK / 16; ++k) {
                            const uint64_t da = ptx::smem_desc(sa + k * 32, 16, 1024, 2);
                            const uint64_t db = ptx::smem_desc(sb + k * 32, 16, 1024, 2);
                            ptx::umma_bf16(d_tmem, da, db, idesc, ((kb0 | kbi | k) != 0) ? 1u : 0u);
                        }
                    }
                    if (has_bias && last) {
                        // D += ones(128 x 16) * bias_t(BN x 16)^T: the bias, exact to ~2^-17 (hi + lo)
                        const uint32_t sbias = args.b_res ? ptx::smem_u32(bres + kblocks * C::B_BYTES)
                                                          : sb0 + KS * C::B_BYTES;
                        ptx::umma_bf16(d_tmem, ptx::smem_desc(ptx::smem_u32(ones), 16, 256, 6),
                                       ptx::smem_desc(sbias, 16, 256, 6), idesc, 1u);
                    }
                    if (args.cl > 1) ptx::umma_commit_mc(&empty_bar[stage], 0x3);
                    else ptx::umma_commit(&empty_bar[stage]);
                    if (last) ptx::umma_commit(&tfull_bar[acc]);
                }
                __syncwarp();
                if (++stage == n_stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (++acc == C::kAcc) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else if (warp < static_cast<uint32_t>(args.n_epi)) {
        // ------------------------------------------------ epilogue
        // TMEM -> registers (SiLU) -> swizzled SMEM staging (double buffered
        // per warp) -> TMA bulk-tensor store, or for row-mapped outputs
        // coalesced 16-byte row-segment stores. The bias is already in the
        // accumulator (added by the MMA warp).
        const uint32_t q = warp & 3;                    // TMEM lane quarter
        const int group = warp >> 2;                    // epilogue group: tiles j = group (mod n_groups)
        const int n_groups = args.n_epi >> 2;
        float* stg_base = stg_all + warp * (args.stg_warp / 4);
        const bool stg_single = args.stg_warp < C::STG_WARP;  // one 4 KB buffer (bf16 bulk-store launches)
        const int sub = lane >> 3;                      // row within a 4-row group
        const int ch = lane & 7;                        // 16-byte chunk within a 32-column row slice
        const uint32_t lane_base = tmem_base + ((q * 32u) << 16);
        constexpr int kChunks = BN / 32;                // 32-column chunks per tile row quarter
        int acc = 0;
        uint32_t acc_phase = 0;
        uint32_t nstore = 0;                            // staging buffers used by this warp
        uint32_t res_phase = 0;                         // parity bit per staging buffer
        uint64_t* my_res = res_bar + warp * 2;
        // column unit per warp: 64 for bf16 bulk-stored outputs (128-byte rows), else 32
        auto unit_of = [&](const GemmProblem& pp) {
            return ((pp.epi == EPI_SILU_BF16 || pp.epi == EPI_BIAS_BF16) && (pp.use_tma_c || pp.use_scatter_c) &&
                    BN >= 64)
                       ? 64
                       : 32;
        };
        auto release = [&](int b) {
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty_bar[b]);
        };
        // residual prefetch of one 32 x 32 fp32 block into staging buffer b
        auto res_load = [&](const GemmProblem& pp, int b, int col, int row) {
            if (lane == 0) {
                ptx::bulk_wait_read<1>();  // the store that last used buffer b has read it
                ptx::mbar_arrive_expect_tx(&my_res[b], 32 * 32 * 4);
                ptx::tma_load_2d(stg_base + b * 32 * 32, &pp.tma_c, &my_res[b], col, row);
            }
        };
        // Group g owns the CTA's tiles j = g, g + n_groups, ...; tile j uses
        // accumulator j % kAcc, so n_groups tiles are drained concurrently while
        // the MMA warp runs up to kAcc tiles ahead.
        gemm_detail::TileSeq seq(args, s_tile_start, s_tiles_n);
        // hand out the accumulators of the first kAcc tiles (each by the group that drains it)
        for (int b = 0; b < C::kAcc; ++b)
            if (b % n_groups == group) release(b);
        int pi, mb, nb;
        // this group's tiles are j = group, group + n_groups, ... (the others only skipped)
        bool more = true;
        for (int g = 0; g < group && more; ++g) more = seq.skip();
        for (int j = group; more && seq.next(pi, mb, nb); j += n_groups) {
            for (int g = 1; g < n_groups && more; ++g) more = seq.skip();
            acc = j % C::kAcc;
            acc_phase = (j / C::kAcc) & 1;
            const GemmProblem& p = args.p[pi];
            const int row0 = mb * C::BM + q * 32;
            const bool bf16_out = p.epi == EPI_SILU_BF16 || p.epi == EPI_BIAS_BF16;
            const int unit = unit_of(p);
            const int step = unit / 32;  // in 32-column chunks
            int ci = 0;
            if (p.use_tma_r && ci < kChunks && nb * BN + ci * 32 < p.N) res_load(p, nstore & 1, nb * BN + ci * 32, row0);
            // scattered bf16 rows: lane i holds the output row of tile row row0 + i
            const int my_orow = (p.use_scatter_c && row0 + static_cast<int>(lane) < p.M) ? __ldg(p.row_map + row0 + lane) : -1;
            ptx::mbar_wait(&tfull_bar[acc], acc_phase);
            ptx::tc_fence_after();
#pragma unroll 1
            for (; ci < kChunks; ci += step) {
                const int c = ci * 32;
                const int n0 = nb * BN + c;
                if (bf16_out && (p.use_tma_c || p.use_scatter_c) && unit == 64) {
                    // ---- fast path: 64 columns -> bf16 (SiLU) -> one 32 x 128 B SW128 box
                    if (n0 >= p.N) continue;  // warp-uniform (TMEM reads below are all-or-nothing)
                    float* stg = stg_base + (stg_single ? 0 : (nstore & 1) * 32 * 32);
                    uint8_t* sb = reinterpret_cast<uint8_t*>(stg) + lane * 128;
                    uint32_t w[2][16];
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        // 32 columns at a time: TMEM -> SiLU (batched MUFU) -> bf16 -> staging
                        float v[32];
                        ptx::tmem_ld16(lane_base + acc * BN + c + 32 * hh, *reinterpret_cast<float(*)[16]>(v));
                        ptx::tmem_ld16(lane_base + acc * BN + c + 32 * hh + 16, *reinterpret_cast<float(*)[16]>(v + 16));
                        ptx::tmem_ld_wait();
                        if (p.epi == EPI_SILU_BF16) {
                            ptx::silu_bf16_batch<16>(v, w[hh]);
                        } else {
#pragma unroll
                            for (int e = 0; e < 32; e += 2) w[hh][e / 2] = pack_bf16(v[e], v[e + 1]);
                        }
                    }
                    // the bulk store that last read this staging buffer must be done with it
                    if (lane == 0) {
                        if (stg_single) ptx::bulk_wait_read<0>();
                        else ptx::bulk_wait_read<1>();
                    }
                    __syncwarp();
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        *reinterpret_cast<uint4*>(sb + ((k ^ (lane & 7)) << 4)) =
                            make_uint4(w[k >> 2][4 * (k & 3)], w[k >> 2][4 * (k & 3) + 1], w[k >> 2][4 * (k & 3) + 2],
                                       w[k >> 2][4 * (k & 3) + 3]);
                    if (p.use_scatter_c) {
                        // row-mapped rows: 8 lanes per 128-byte row segment, 4 rows per pass
                        __syncwarp();
                        // all eight shared loads and row shuffles first: the global stores may
                        // alias the generic staging pointer, so interleaving them would serialise
                        // every load behind the previous store
                        const uint8_t* s0 = reinterpret_cast<const uint8_t*>(stg);
                        uint4 vals[8];
                        int orows[8];
#pragma unroll
                        for (int it = 0; it < 8; ++it) {
                            const int r = it * 4 + sub;
                            vals[it] = *reinterpret_cast<const uint4*>(s0 + r * 128 + ((ch ^ (r & 7)) << 4));
                            orows[it] = __shfl_sync(0xffffffffu, my_orow, r);
                        }
#pragma unroll
                        for (int it = 0; it < 8; ++it)
                            if (orows[it] >= 0)
                                *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) +
                                                          static_cast<long long>(orows[it]) * p.ldo + n0 + ch * 8) =
                                    vals[it];
                        ++nstore;
                        continue;
                    }
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::tma_store_2d(&p.tma_c, stg, n0, row0);
                        ptx::bulk_commit();
                    }
                    ++nstore;
                    continue;
                }
                float v[32];
                ptx::tmem_ld16(lane_base + acc * BN + c, *reinterpret_cast<float(*)[16]>(v));
                ptx::tmem_ld16(lane_base + acc * BN + c + 16, *reinterpret_cast<float(*)[16]>(v + 16));
                ptx::tmem_ld_wait();
                if (n0 >= p.N) continue;  // warp-uniform
                float* stg = stg_base + (nstore & 1) * 32 * 32;
                if (p.use_tma_r) {
                    const int b = nstore & 1;
                    ptx::mbar_wait(&my_res[b], (res_phase >> b) & 1);
                    res_phase ^= 1u << b;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        float4* cell = reinterpret_cast<float4*>(stg + lane * 32 + ((k ^ (lane & 7)) << 2));
                        const float4 r4 = *cell;
                        *cell = make_float4(v[4 * k] + r4.x, v[4 * k + 1] + r4.y, v[4 * k + 2] + r4.z,
                                            v[4 * k + 3] + r4.w);
                    }
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::tma_store_2d(&p.tma_c, stg, n0, row0);
                        ptx::bulk_commit();
                    }
                    ++nstore;
                    // prefetch the next chunk's residual into the other buffer
                    const int cn = ci + step;
                    if (cn < kChunks && nb * BN + cn * 32 < p.N) res_load(p, nstore & 1, nb * BN + cn * 32, row0);
                    continue;
                }
                if (p.use_tma_c) {
                    if (lane == 0) ptx::bulk_wait_read<1>();
                    __syncwarp();
                    if (bf16_out) {
                        // 64-column unit: this chunk and the next (loaded below) -> one
                        // 32 rows x 128 B SW128 box (chunk k of row r at (k ^ (r & 7)))
                        uint8_t* sb = reinterpret_cast<uint8_t*>(stg);
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            if (hh == 1) {
                                ptx::tmem_ld16(lane_base + acc * BN + c + 32, *reinterpret_cast<float(*)[16]>(v));
                                ptx::tmem_ld16(lane_base + acc * BN + c + 48, *reinterpret_cast<float(*)[16]>(v + 16));
                                ptx::tmem_ld_wait();
                            }
                            uint32_t w[16];
                            if (p.epi == EPI_SILU_BF16) {
#pragma unroll
                                for (int e = 0; e < 32; e += 2) w[e / 2] = ptx::silu2_bf16(v[e], v[e + 1]);
                            } else {
#pragma unroll
                                for (int e = 0; e < 32; e += 2) w[e / 2] = pack_bf16(v[e], v[e + 1]);
                            }
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const int kk = hh * 4 + k;
                                *reinterpret_cast<uint4*>(sb + lane * 128 + ((kk ^ (lane & 7)) << 4)) =
                                    make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
                            }
                        }
                    } else {
                        // 32 rows x 128 B, SWIZZLE_128B: chunk k of row r at (k ^ (r & 7))
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            *reinterpret_cast<float4*>(stg + lane * 32 + ((k ^ (lane & 7)) << 2)) =
                                make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
                    }
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::tma_store_2d(&p.tma_c, stg, n0, row0);
                        ptx::bulk_commit();
                    }
                    ++nstore;
                    continue;
                }
                // ---- manual path (row-mapped scatter / residual without TMA)
                if (p.epi == EPI_SILU_BF16) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = ptx::silu_fast(v[i]);
                }
                if (lane == 0) ptx::bulk_wait_read<1>();
                __syncwarp();
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    *reinterpret_cast<float4*>(stg + lane * 32 + ((k ^ (lane & 7)) << 2)) =
                        make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
                __syncwarp();
                const int col = n0 + 4 * ch;
                const int nval = min(4, p.N - col);
                long long orow[8];
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    const int m = row0 + 4 * g + sub;
                    orow[g] = (m < p.M && nval > 0)
                                  ? (p.row_map ? static_cast<long long>(__ldg(p.row_map + m)) : p.row_offset + m)
                                  : -1;
                }
                if (bf16_out) {
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        const int r = 4 * g + sub;
                        const float4 w = *reinterpret_cast<const float4*>(stg + r * 32 + ((ch ^ (r & 7)) << 2));
                        if (orow[g] < 0) continue;
                        __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out) + orow[g] * p.ldo + col;
                        if (nval == 4) {
                            *reinterpret_cast<uint2*>(o) = make_uint2(pack_bf16(w.x, w.y), pack_bf16(w.z, w.w));
                        } else {
                            const float ww[4] = {w.x, w.y, w.z, w.w};
                            for (int i = 0; i < nval; ++i) o[i] = __float2bfloat16_rn(ww[i]);
                        }
                    }
                } else {
                    // f32 outputs: load every residual first (resid may alias out), then store
                    float4 rr[8];
                    if (p.epi == EPI_RESID_F32) {
#pragma unroll
                        for (int g = 0; g < 8; ++g) {
                            rr[g] = make_float4(0.f, 0.f, 0.f, 0.f);
                            if (orow[g] >= 0 && nval == 4) {
                                rr[g] = *reinterpret_cast<const float4*>(p.resid + orow[g] * p.ldo + col);
                            } else if (orow[g] >= 0) {
                                float t4[4] = {0.f, 0.f, 0.f, 0.f};
                                for (int i = 0; i < nval; ++i) t4[i] = p.resid[orow[g] * p.ldo + col + i];
                                rr[g] = make_float4(t4[0], t4[1], t4[2], t4[3]);
                            }
                        }
                    }
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        const int r = 4 * g + sub;
                        float4 w = *reinterpret_cast<const float4*>(stg + r * 32 + ((ch ^ (r & 7)) << 2));
                        if (orow[g] < 0) continue;
                        if (p.epi == EPI_RESID_F32) {
                            w.x += rr[g].x;
                            w.y += rr[g].y;
                            w.z += rr[g].z;
                            w.w += rr[g].w;
                        }
                        float* o = static_cast<float*>(p.out) + orow[g] * p.ldo + col;
                        if (nval == 4) {
                            *reinterpret_cast<float4*>(o) = w;
                        } else {
                            const float ww[4] = {w.x, w.y, w.z, w.w};
                            for (int i = 0; i < nval; ++i) o[i] = ww[i];
                        }
                    }
                }
                __syncwarp();
                ++nstore;
            }
            release(acc);  // hand the accumulator back to the MMA warp (tile j + kAcc)
        }
        if (lane == 0) ptx::bulk_wait<0>();  // all bulk stores complete before exit
        __syncwarp();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (args.cl > 1) ptx::cluster_sync();  // no CTA leaves while its peer may still multicast or arrive
    if (warp == kWarpAlloc) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<C::TMEM_COLS>(tmem_base);
    }
}

}  // namespace mtfm
