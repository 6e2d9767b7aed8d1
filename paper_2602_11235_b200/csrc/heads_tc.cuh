// heads_tc.cuh — MMoE heads fused with their GEMM on tcgen05 (sm_100a), K5 of the
// bf16 forward (heads.hpp:47-99, records as model.hpp:244-312):
//
//   per T row x:  gate_k = softmax_e(x Wg_k + bg_k)             (task k of the row's scenario)
//                 act_e  = silu(x We + be)                       (expert e, d_expert wide)
//                 z_k    = sum_e gate_k[e] (act_e . tw_k) + tb_k ;  p_k = sigmoid(z_k)
//
// One 128-row tile of T rows per CTA at a time. Its gate columns (all tasks of all
// scenarios, n_tasks * E) and then every expert in 128-column chunks are produced
// by tcgen05 MMAs into TMEM (the gate block once, the expert chunks through two
// buffers) and consumed straight from TMEM by 16 epilogue warps (lane = row, four
// groups of 32 columns whose partial logits are summed through SMEM): the
// expert activations are never stored — each chunk is reduced into the row's
// per-task dots act_e . tw_k on the fly. This replaces the head GEMM's
// [T][E*de + n_tasks*E] fp32 round trip through HBM and the separate heads pass.
//
// Roles (608 threads): warps 0..15 epilogue (which also convert the tile's fp32 X rows
// to the bf16 A operand in SMEM), warp 16 TMEM allocator, warp 17 TMA producer (the
// chunks' weight k-blocks), warp 18 MMA issuer.
#pragma once

#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace mtfm {

constexpr int kHeadsMaxTasks = 4;   // tasks per scenario
constexpr int kHeadsMaxE = 4;       // experts (E <= 4: the gate weights live in registers)

struct HeadsTcArgs {
    const float* x;         // X_T [n_t][ldx] fp32 (the residual stream's T rows), converted to bf16 in SMEM
    long long ldx;
    CUtensorMap tma_w;      // head weights K-major [head_n][d] bf16, box {64, 128}, SW128
    int n_t, d, E, de;
    int n_gate;             // n_tasks_total * E gate columns, after the E * de expert columns
    int n_tasks_total;
    int n_wstages;          // weight k-block stages (SMEM left after the resident X tile)
    const float* exp_bias;  // [E * de]
    const float* gate_bias; // [n_tasks_total * E]
    const float* tower_w;   // [n_tasks_total][de]
    const float* tower_b;   // [n_tasks_total]
    const SourceInfo* src;
    int n_src;
    const int* t_scen;
    const int* t_user;
    const int* t_exp_ref;
    const long long* t_rec0;
    const int* t_rec_stride;
    const long long* user_id;
    long long* rec_user;
    int* rec_scen;
    int* rec_exp;
    int* rec_task;
    float* rec_logit;
    double* rec_prob;
};

namespace heads_detail {
constexpr int BM = 128, BK = 64, CH = 128;        // rows, k-block, expert chunk columns
constexpr int A_BYTES = BM * BK * 2;              // 16 KB per k-block of the resident X tile
constexpr int W_BYTES = CH * BK * 2;              // 16 KB: 128 weight rows (a chunk, or the gate block) x 64 k
constexpr int kMaxWStages = 12;
constexpr int kEpiGroups = 4;                     // epilogue groups: each takes 32 columns of every chunk
constexpr int kEpiWarps = 4 * kEpiGroups;
constexpr int kThreads = 32 * (kEpiWarps + 3);
constexpr int XZ_BYTES = 2 * kEpiGroups * BM * 4 * 4;  // per-group partial logits, double-buffered by tile
constexpr uint32_t ACC_COL = 0, GATE_COL = 2 * CH;  // two expert-chunk buffers, then the gate block
}  // namespace heads_detail

// SMEM: the X tile (d/64 k-blocks, loaded once per tile), n_wstages weight k-blocks,
// exp_bias [E*de] and tower_w [n_tasks_total][de + 4] (fp32), partial logits, barriers
__global__ void __launch_bounds__(heads_detail::kThreads, 1) heads_tc_kernel(const __grid_constant__ HeadsTcArgs a) {
    using namespace heads_detail;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int n_kb = a.d / BK;
    const int n_ws = a.n_wstages;
    uint8_t* sA = base;
    uint8_t* sW = base + n_kb * A_BYTES;
    float* s_eb = reinterpret_cast<float*>(sW + n_ws * W_BYTES);
    float* s_tw = s_eb + a.E * a.de;               // rows padded to de + 4 (rows of different tasks in other banks)
    const int tw_ld = a.de + 4;
    float* s_xz = s_tw + a.n_tasks_total * tw_ld;  // [2][group][row][task] partial logits
    float* s_gate = s_xz + XZ_BYTES / 4;          // [BM][ng_pad + 1] gate logits of the tile
    uint64_t* bars = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(s_gate + BM * (((a.n_gate + 15) & ~15) + 1)) + 15) & ~uintptr_t(15));
    uint64_t* full = bars;                   // [kMaxWStages]
    uint64_t* empty = bars + kMaxWStages;    // [kMaxWStages]
    uint64_t* acc_full = bars + 2 * kMaxWStages;  // [3]: expert buffers 0, 1, gate block
    uint64_t* acc_empty = acc_full + 3;           // [3]
    uint64_t* a_full = acc_empty + 3;
    uint64_t* a_empty = a_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_empty + 1);

    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    constexpr uint32_t kWarpAlloc = kEpiWarps, kWarpTma = kEpiWarps + 1, kWarpMma = kEpiWarps + 2;
    const int sub = a.de / CH;                         // chunks per expert
    const int n_chunks = 1 + a.E * sub;                // gate block first
    const int ng_pad = (a.n_gate + 15) & ~15;
    const int n_tiles = (a.n_t + BM - 1) / BM;

    for (int i = threadIdx.x; i < a.E * a.de; i += blockDim.x) s_eb[i] = a.exp_bias[i];
    for (int i = threadIdx.x; i < a.n_tasks_total * a.de; i += blockDim.x)
        s_tw[(i / a.de) * tw_ld + i % a.de] = a.tower_w[i];
    if (warp == kWarpTma && lane == 0) {
        for (int i = 0; i < n_ws; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], 1);
        }
        ptx::mbar_init(a_full, kEpiWarps);  // the epilogue warps convert the X tile
        ptx::mbar_init(a_empty, 1);
        for (int i = 0; i < 3; ++i) {
            ptx::mbar_init(&acc_full[i], 1);
            ptx::mbar_init(&acc_empty[i], i == 2 ? 4 : kEpiWarps);  // the gate block is read by group 0
        }
        ptx::fence_mbar_init();
        ptx::tma_prefetch(&a.tma_w);
    }
    if (warp == kWarpAlloc) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    MTFM_PDL_ENTRY();

    if (warp == kWarpTma) {
        if (ptx::elect_one()) {
            uint32_t it = 0, n_t = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++n_t) {
                for (int c = 0; c < n_chunks; ++c) {
                    // chunk c: weight rows [r0, r0 + 128) (the gate block: E*de .. + ng_pad)
                    const int r0 = c == 0 ? a.E * a.de : (c - 1) * CH;
                    for (int kb = 0; kb < n_kb; ++kb, ++it) {
                        const uint32_t s = it % n_ws;
                        ptx::mbar_wait(&empty[s], ((it / n_ws) & 1) ^ 1);
                        ptx::mbar_arrive_expect_tx(&full[s], W_BYTES);
                        ptx::tma_load_2d(sW + s * W_BYTES, &a.tma_w, &full[s], kb * BK, r0);
                    }
                }
            }
        }
    } else if (warp == kWarpMma) {
        uint32_t it = 0, n_exp = 0, n_gate = 0, n_t = 0;
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++n_t) {
            ptx::mbar_wait(a_full, n_t & 1);
            for (int c = 0; c < n_chunks; ++c) {
                const bool gate = c == 0;
                const int nw = gate ? ng_pad : CH;
                const uint32_t ab = gate ? 2u : (n_exp & 1);
                const uint32_t use = gate ? n_gate : (n_exp >> 1);
                ptx::mbar_wait(&acc_empty[ab], (use & 1) ^ 1);
                ptx::tc_fence_after();
                const uint32_t idesc = ptx::instr_desc_bf16(BM, nw, false, false);
                const uint32_t d_col = gate ? GATE_COL : ACC_COL + ab * CH;
                for (int kb = 0; kb < n_kb; ++kb, ++it) {
                    const uint32_t s = it % n_ws;
                    ptx::mbar_wait(&full[s], (it / n_ws) & 1);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        const uint32_t sa = ptx::smem_u32(sA + kb * A_BYTES);
                        const uint32_t sw = ptx::smem_u32(sW + s * W_BYTES);
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k)
                            ptx::umma_bf16(tmem + d_col, ptx::smem_desc(sa + k * 32, 16, 1024, 2),
                                           ptx::smem_desc(sw + k * 32, 16, 1024, 2), idesc, (kb > 0 || k > 0) ? 1u : 0u);
                        ptx::umma_commit(&empty[s]);
                        if (kb == n_kb - 1) ptx::umma_commit(&acc_full[ab]);
                        if (kb == n_kb - 1 && c == n_chunks - 1) ptx::umma_commit(a_empty);
                    }
                    __syncwarp();
                }
                if (gate) ++n_gate;
                else ++n_exp;
            }
        }
    } else if (warp < kEpiWarps) {
        // epilogue: lane = row of the tile; group gq reduces columns [32 gq, 32 gq + 32) of
        // every expert chunk, the groups' partial logits are summed through SMEM
        const uint32_t q = warp & 3, gq = warp >> 2;
        uint32_t n_xt = 0;
        const uint32_t lane_addr = (q * 32u) << 16;
        uint32_t n_exp = 0, n_gate = 0;
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
            const long long row = static_cast<long long>(t) * BM + q * 32 + lane;
            const bool valid = row < a.n_t;
            // the tile's X rows (fp32 residual stream) -> bf16 in the K-major SW128 layout of the
            // MMA's A operand: 16-byte chunk c of row r of k-block kb at kb*16K + r*128 + ((c ^ r%8) << 4)
            {
                ptx::mbar_wait(a_empty, (n_xt & 1) ^ 1);  // the previous tile's MMAs are done with it
                const int cpr = a.d / 8;                   // 8-element chunks per row
                for (int i = static_cast<int>(threadIdx.x); i < BM * cpr; i += kEpiWarps * 32) {
                    const int r = i / cpr, cc = i - r * cpr;
                    const long long xr = static_cast<long long>(t) * BM + r;
                    float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
                    if (xr < a.n_t) {
                        const float4* src = reinterpret_cast<const float4*>(a.x + xr * a.ldx + cc * 8);
                        lo = __ldg(src);
                        hi = __ldg(src + 1);
                    }
                    const int kb = cc >> 3, c = cc & 7;
                    ptx::sts128(ptx::smem_u32(sA) + kb * A_BYTES + r * 128 + ((c ^ (r & 7)) << 4),
                                __uint_as_float(pack_bf16(lo.x, lo.y)), __uint_as_float(pack_bf16(lo.z, lo.w)),
                                __uint_as_float(pack_bf16(hi.x, hi.y)), __uint_as_float(pack_bf16(hi.z, hi.w)));
                }
                ptx::fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(a_full);
                ++n_xt;
            }
            // the row's scenario: task window [task0, task0 + ntasks)
            int task0 = 0, ntasks = 0, scen = 0;
            if (valid) {
                scen = __ldg(a.t_scen + row);
                for (int i = 0; i < a.n_src; ++i) {
                    const SourceInfo si = a.src[i];
                    if (si.kind == 2 && si.id == scen) {
                        task0 = si.task0;
                        ntasks = si.ntasks;
                    }
                }
            }
            // ---- gate block: softmax over E per task of the row (sequential sum, as softmax_rows)
            float g[kHeadsMaxTasks][kHeadsMaxE];
#pragma unroll
            for (int k = 0; k < kHeadsMaxTasks; ++k)
#pragma unroll
                for (int e = 0; e < kHeadsMaxE; ++e) g[k][e] = 0.f;
            // group 0 stages the tile's gate block (+ bias) in SMEM ([row][ng_pad + 1]); every
            // thread then reads its row's task window by index
            const int gl = ng_pad + 1;
            const int rl = static_cast<int>(q * 32 + lane);
            if (gq == 0) {
                ptx::mbar_wait(&acc_full[2], n_gate & 1);
                ptx::tc_fence_after();
                for (int c0 = 0; c0 < ng_pad; c0 += 16) {
                    float v[16];
                    ptx::tmem_ld16(tmem + lane_addr + GATE_COL + c0, v);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        s_gate[rl * gl + c0 + i] = c0 + i < a.n_gate ? v[i] + __ldg(a.gate_bias + c0 + i) : 0.f;
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&acc_empty[2]);
            }
            ++n_gate;
            ptx::named_bar_sync(2, kEpiWarps * 32);
#pragma unroll
            for (int k = 0; k < kHeadsMaxTasks; ++k)
#pragma unroll
                for (int e = 0; e < kHeadsMaxE; ++e)
                    g[k][e] = (k < ntasks && e < a.E) ? s_gate[rl * gl + (task0 + k) * a.E + e] : 0.f;
#pragma unroll
            for (int k = 0; k < kHeadsMaxTasks; ++k) {
                float mx = -INFINITY;
#pragma unroll
                for (int e = 0; e < kHeadsMaxE; ++e)
                    if (e < a.E) mx = fmaxf(mx, g[k][e]);
                float sum = 0.f;
#pragma unroll
                for (int e = 0; e < kHeadsMaxE; ++e) {
                    const float x = e < a.E ? expf(g[k][e] - mx) : 0.f;
                    g[k][e] = x;
                    sum += x;
                }
                const float inv = __fdiv_rn(1.f, sum);
#pragma unroll
                for (int e = 0; e < kHeadsMaxE; ++e) g[k][e] *= inv;
            }
            // ---- experts: per task, sum_e gate[e] * (silu(x We + be) . tw_k)
            float z[kHeadsMaxTasks] = {0.f, 0.f, 0.f, 0.f};
            uint32_t tw[kHeadsMaxTasks];  // shared-window addresses of the row's tower weights
#pragma unroll
            for (int k = 0; k < kHeadsMaxTasks; ++k)
                tw[k] = ptx::smem_u32(s_tw) + static_cast<uint32_t>((task0 + (k < ntasks ? k : 0)) * tw_ld) * 4u;
            const uint32_t eb_base = ptx::smem_u32(s_eb);
            for (int e = 0; e < a.E; ++e) {
                float dot[kHeadsMaxTasks] = {0.f, 0.f, 0.f, 0.f};
                for (int sc = 0; sc < sub; ++sc, ++n_exp) {
                    const uint32_t ab = n_exp & 1;
                    ptx::mbar_wait(&acc_full[ab], (n_exp >> 1) & 1);
                    ptx::tc_fence_after();
                    const int j0 = sc * CH;
                    float v[32];
                    const uint32_t ta = tmem + lane_addr + ACC_COL + ab * CH + gq * 32;
                    ptx::tmem_ld16(ta, *reinterpret_cast<float(*)[16]>(v));
                    ptx::tmem_ld16(ta + 16, *reinterpret_cast<float(*)[16]>(v + 16));
                    ptx::tmem_ld_wait();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&acc_empty[ab]);
#pragma unroll
                    for (int p8 = 0; p8 < 4; ++p8) {
                        const int j = j0 + static_cast<int>(gq) * 32 + 8 * p8;
                        const float4 b0 = ptx::lds128(eb_base + static_cast<uint32_t>(e * a.de + j) * 4u);
                        const float4 b1 = ptx::lds128(eb_base + static_cast<uint32_t>(e * a.de + j + 4) * 4u);
                        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                        float act[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) act[i] = ptx::silu_fast(v[8 * p8 + i] + bv[i]);
#pragma unroll
                        for (int k = 0; k < kHeadsMaxTasks; ++k) {
                            if (k >= ntasks) break;  // the row's scenario has fewer towers
                            const float4 w0 = ptx::lds128(tw[k] + static_cast<uint32_t>(j) * 4u);
                            const float4 w1 = ptx::lds128(tw[k] + static_cast<uint32_t>(j + 4) * 4u);
                            const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
                            for (int i = 0; i < 8; ++i) dot[k] = fmaf(act[i], wv[i], dot[k]);
                        }
                    }
                }
                float ge[kHeadsMaxTasks];
#pragma unroll
                for (int k = 0; k < kHeadsMaxTasks; ++k) {
                    ge[k] = 0.f;
#pragma unroll
                    for (int ee = 0; ee < kHeadsMaxE; ++ee)
                        if (ee == e) ge[k] = g[k][ee];
                    z[k] = fmaf(ge[k], dot[k], z[k]);
                }
            }
            // ---- the groups' partial logits -> group 0 (fixed order g0 + g1 + g2 + g3)
            float* xz = s_xz + (n_gate & 1) * (kEpiGroups * BM * 4);
#pragma unroll
            for (int k = 0; k < kHeadsMaxTasks; ++k) xz[(gq * BM + rl) * 4 + k] = z[k];
            ptx::named_bar_sync(1, kEpiWarps * 32);
            if (gq != 0) continue;
#pragma unroll
            for (int k = 0; k < kHeadsMaxTasks; ++k) {
                float zs = xz[rl * 4 + k];
                for (int gg = 1; gg < kEpiGroups; ++gg) zs += xz[(gg * BM + rl) * 4 + k];
                z[k] = zs;
            }
            // ---- records (heads.hpp:93-99, model.hpp:296-306): logit, clamped probability
            if (valid) {
#pragma unroll
                for (int k = 0; k < kHeadsMaxTasks; ++k) {
                    if (k >= ntasks) break;
                    const float zz = z[k] + __ldg(a.tower_b + task0 + k);
                    const long long r = __ldg(a.t_rec0 + row) + static_cast<long long>(k) * __ldg(a.t_rec_stride + row);
                    double pr = static_cast<double>(sigmoid_precise(zz));
                    pr = pr < 1e-12 ? 1e-12 : (pr > 1.0 - 1e-12 ? 1.0 - 1e-12 : pr);
                    a.rec_user[r] = a.user_id[__ldg(a.t_user + row)];
                    a.rec_scen[r] = scen;
                    a.rec_exp[r] = __ldg(a.t_exp_ref + row);
                    a.rec_task[r] = k;
                    if (a.rec_logit) a.rec_logit[r] = zz;
                    a.rec_prob[r] = pr;
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

}  // namespace mtfm
