// attn_tc.cuh — Hybrid Target Attention on tcgen05 (sm_100a).
//
// Computes, for every query row i of a tile and every head h of one KV group g
// (hta.hpp:115-134 with the mask of mask.cpp:5-29 in closed form):
//
//   A_h[i] = s_i * ( sum_{j < prefix_i} silu(Q_h[i] . K_g[j]) V_g[j]
//                    + [i is T] silu(Q_h[i] . K_g[self_i]) V_g[self_i] )
//
// The dense N x N mask never exists: row i sees the first prefix_i context
// keys of its user (H tokens plus R tokens strictly older than i) and, when it
// is a T token, itself. There is no softmax: weights are pointwise SiLU, so
// no running max / rescale; O simply accumulates in TMEM across key tiles.
//
// Tile = 128 MMA rows = HS heads of one GQA group x RT query rows (HS*RT=128),
// so every K/V tile TMA-loaded into SMEM is shared by the HS query heads that
// read it. Per key tile j (three S/P TMEM buffers, b = j % 3):
//   S warp       : S[b] = Q K_j^T              (TMEM, fp32, 128 x BKV)
//   16 SiLU warps: each takes a quarter of every key tile's columns: S -> regs,
//                  silu = h + h*tanh(h) (h = s/2: FMUL2, MUFU.TANH, FFMA2), mask
//                  only on the boundary key tile, packed bf16 P written over the
//                  first half of the warp's own S columns (tcgen05.st), arrive.
//   PV warp      : O[t%2] += P[b] V_j (P from TMEM, V MN-major SMEM); its commit
//                  hands S/P buffer b back to the S warp.
//   4 epilogue warps: O[t%2] -> regs, x s_i, + self term for T rows, bf16 out
//                  (overlaps the next tile's key loop).
// Q and O are double-buffered, so consecutive tiles of a CTA pipeline.
#pragma once

#include "common.cuh"
#include "ptx.cuh"

namespace mtfm {

struct AttnTile {
    int q_row0;    // first query row (row index of the Q matrix)
    int n_rows;    // valid query rows in this tile (<= RT)
    int key_base;  // KV-matrix row of the user's first context key
    int head0;     // first query head of the tile (HS consecutive heads, one group)
    int kmax;      // max prefix over the tile's rows (filled on device)
    int pad[3];
};

struct AttnParams {
    CUtensorMap tma_q;   // Q matrix, box {chunk, RT}
    CUtensorMap tma_kv;  // KV matrix, box {chunk, BKV}
    const AttnTile* tiles;
    int n_tiles;
    int q_col0, k_col0, v_col0;  // column offsets of head/group 0
    int heads, kv_heads, hs, rt;
    const int* q_prefix;         // per Q row
    const float* q_scale;        // per Q row
    const int* q_self;           // per Q row: KV row of the self key, or -1
    const __nv_bfloat16* q_ptr;  // Q matrix (self term)
    long long ldq;
    const __nv_bfloat16* kv_ptr;
    long long ldkv;
    __nv_bfloat16* out;          // A rows indexed like Q rows
    long long ldo;
    int tma_box_kv, tma_chunk;   // host check: the boxes tma_q / tma_kv were built with
};

namespace attn_detail {

template <int D>
struct Cfg {
    static constexpr int BKV = D <= 64 ? 128 : 64;
    static constexpr int CHUNK = D < 64 ? D : 64;          // elements per swizzle row
    static constexpr int SLABS = D / CHUNK;
    static constexpr int ROWB = CHUNK * 2;                  // bytes per swizzled row
    static constexpr uint32_t LAYOUT = ROWB == 128 ? 2 : (ROWB == 64 ? 4 : 6);
    static constexpr int Q_BYTES = 128 * D * 2;
    static constexpr int KV_TILE_BYTES = BKV * D * 2;       // one of K or V
    static constexpr int P_BYTES = 128 * BKV * 2;
    static constexpr int QB = D <= 64 ? 2 : 1;              // Q buffers
    // separate K and V rings, as deep as SMEM allows (~200 KB for d_h <= 64, everything
    // for the wide heads): a K slot is refilled as soon as its S = QK^T completed, not
    // after the P.V of the same key tile, so the S warp's K loads run further ahead
    static constexpr int BAR_BYTES = 1024;
    static constexpr int kRingBudget = (D <= 64 ? 200 * 1024 : 227 * 1024 - 1024 - BAR_BYTES) - QB * Q_BYTES;
    static constexpr int kSlots = kRingBudget / KV_TILE_BYTES;
    static constexpr int KS = (kSlots + 1) / 2 > 12 ? 12 : (kSlots + 1) / 2;  // K slots
    static constexpr int VS = kSlots / 2 > 12 ? 12 : kSlots / 2;              // V slots
    static constexpr int SMEM = QB * Q_BYTES + (KS + VS) * KV_TILE_BYTES + 1024 + BAR_BYTES;
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr int NB = 3;                            // S/P TMEM buffers (P aliases S)
    static constexpr uint32_t O_COL = NB * BKV;
    static constexpr int OB = (NB * BKV + 2 * D <= 512) ? 2 : 1;  // O buffers
    static constexpr int kSilu = 16;                        // SiLU warps (4 per TMEM lane quarter)
    // two groups of 8 SiLU warps take alternate key tiles (a group's warps split a tile's
    // columns in halves), so one group's SiLUs run while the other's loads, stores and
    // barrier hand-offs are in flight
    static constexpr int kSiluGroups = 2;
    static constexpr int CW = BKV / (kSilu / kSiluGroups / 4);  // key columns per SiLU warp and key tile
    static constexpr int kThreads = (4 + kSilu + 4) * 32;   // + TMA/MMA/alloc/spare + 4 epilogue warps
    static_assert(O_COL + OB * D <= 512, "TMEM budget");
    static_assert(SMEM <= 227 * 1024, "SMEM budget");
};

// Byte offset of 16-byte chunk `chunk16` of row `row` in a K-major SW128 slab.
__device__ __forceinline__ uint32_t sw128_off(uint32_t row, uint32_t chunk16) {
    return (row >> 3) * 1024 + (row & 7) * 128 + ((chunk16 ^ (row & 7)) << 4);
}

using ptx::silu2_bf16;

// 16 keys (columns base .. base + 15 of the warp's chunk) -> 8 packed bf16 P words, keys at
// or past nvalid masked to 0
__device__ __forceinline__ void silu_half(const float (&v)[16], uint32_t (&p)[8], int nvalid, int base) {
    if (__all_sync(0xffffffffu, nvalid >= base + 16)) {
#pragma unroll
        for (int e = 0; e < 16; e += 2) p[e / 2] = silu2_bf16(v[e], v[e + 1]);
    } else {
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
            const uint32_t w = silu2_bf16(v[e], v[e + 1]);
            const int k = base + e;
            const uint32_t keep = (k + 1 < nvalid) ? 0xffffffffu : (k < nvalid ? 0x0000ffffu : 0u);
            p[e / 2] = w & keep;
        }
    }
}

}  // namespace attn_detail

// P aliases S: each SiLU warp overwrites the first half of its own S columns
// with packed bf16 P and every one of the 16 SiLU warps works on every key tile
// (a quarter of its columns); a buffer is released to the S issuer only after
// the P.V that reads it completed.
template <int D>
__global__ void __launch_bounds__(768, 1) attn_tc_kernel(const __grid_constant__ AttnParams prm) {
    using C = attn_detail::Cfg<D>;
    constexpr int BKV = C::BKV;
    constexpr int NB = C::NB;
    constexpr uint32_t kOCol = C::O_COL;
    constexpr int kOB = C::OB;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + C::QB * C::Q_BYTES;
    uint8_t* sV = sK + C::KS * C::KV_TILE_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + C::VS * C::KV_TILE_BYTES);
    uint64_t* q_full = bars + 0;   // [2]
    uint64_t* q_empty = bars + 2;  // [2]
    uint64_t* o_full = bars + 4;   // [2]
    uint64_t* o_empty = bars + 6;  // [2]
    uint64_t* s_full = bars + 8;            // [NB]
    uint64_t* s_empty = bars + 8 + NB;      // [NB] released by the P.V commit
    uint64_t* p_full = bars + 8 + 2 * NB;   // [NB]
    uint64_t* k_full = bars + 8 + 3 * NB;   // [KS]
    uint64_t* k_empty = k_full + C::KS;     // [KS] released by the S commit
    uint64_t* v_full = k_empty + C::KS;     // [VS]
    uint64_t* v_empty = v_full + C::VS;     // [VS] released by the P.V commit
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_empty + C::VS);
    static_assert((8 + 3 * NB + 2 * C::KS + 2 * C::VS) * 8 + 4 <= C::BAR_BYTES, "barrier area");

    const uint32_t warp = ptx::warp_id();
    const uint32_t lane = ptx::lane_id();
    const int r_per_g = prm.heads / prm.kv_heads;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&q_full[i], 1);
            ptx::mbar_init(&q_empty[i], 1);
            ptx::mbar_init(&o_full[i], 1);
            ptx::mbar_init(&o_empty[i], 4);
        }
        for (int i = 0; i < NB; ++i) {
            ptx::mbar_init(&s_full[i], 1);
            ptx::mbar_init(&s_empty[i], 1);
            ptx::mbar_init(&p_full[i], C::kSilu / C::kSiluGroups);
        }
        for (int i = 0; i < C::KS; ++i) {
            ptx::mbar_init(&k_full[i], 1);
            ptx::mbar_init(&k_empty[i], 1);
        }
        for (int i = 0; i < C::VS; ++i) {
            ptx::mbar_init(&v_full[i], 1);
            ptx::mbar_init(&v_empty[i], 1);
        }
        ptx::fence_mbar_init();
        ptx::tma_prefetch(&prm.tma_q);
        ptx::tma_prefetch(&prm.tma_kv);
    }
    if (warp == 2) ptx::tmem_alloc<C::TMEM_COLS>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // prologue done (barriers, TMEM, SMEM tables): wait for the producer of our inputs
    MTFM_PDL_ENTRY();

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (ptx::elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int t = blockIdx.x; t < prm.n_tiles; t += gridDim.x, ++it) {
                const AttnTile tile = prm.tiles[t];
                const int g = tile.head0 / r_per_g;
                const int n_kv = (tile.kmax + BKV - 1) / BKV;
                const int qb = it % C::QB;
                const uint32_t qpar = (it / C::QB) & 1;
                ptx::mbar_wait(&q_empty[qb], qpar ^ 1);
                ptx::mbar_arrive_expect_tx(&q_full[qb], C::Q_BYTES);
                uint8_t* q_dst = sQ + qb * C::Q_BYTES;
                for (int hs = 0; hs < prm.hs; ++hs)
                    for (int sl = 0; sl < C::SLABS; ++sl)
                        ptx::tma_load_2d(q_dst + sl * (128 * C::ROWB) + hs * prm.rt * C::ROWB, &prm.tma_q, &q_full[qb],
                                         prm.q_col0 + (tile.head0 + hs) * D + sl * C::CHUNK, tile.q_row0);
                for (int j = 0; j < n_kv; ++j) {
                    ptx::mbar_wait(&k_empty[stage], phase ^ 1);
                    uint8_t* sk = sK + stage * C::KV_TILE_BYTES;
                    ptx::mbar_arrive_expect_tx(&k_full[stage], C::KV_TILE_BYTES);
                    const int row = tile.key_base + j * BKV;
                    for (int sl = 0; sl < C::SLABS; ++sl)
                        ptx::tma_load_2d(sk + sl * (BKV * C::ROWB), &prm.tma_kv, &k_full[stage],
                                         prm.k_col0 + g * D + sl * C::CHUNK, row);
                    if (++stage == C::KS) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 2) {
        // ------------------------------------------------ V producer (the TMEM allocator warp)
        if (ptx::elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < prm.n_tiles; t += gridDim.x) {
                const AttnTile tile = prm.tiles[t];
                const int g = tile.head0 / r_per_g;
                const int n_kv = (tile.kmax + BKV - 1) / BKV;
                for (int j = 0; j < n_kv; ++j) {
                    ptx::mbar_wait(&v_empty[stage], phase ^ 1);
                    uint8_t* sv = sV + stage * C::KV_TILE_BYTES;
                    ptx::mbar_arrive_expect_tx(&v_full[stage], C::KV_TILE_BYTES);
                    const int row = tile.key_base + j * BKV;
                    for (int sl = 0; sl < C::SLABS; ++sl)
                        ptx::tma_load_2d(sv + sl * (BKV * C::ROWB), &prm.tma_kv, &v_full[stage],
                                         prm.v_col0 + g * D + sl * C::CHUNK, row);
                    if (++stage == C::VS) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ S issuer: S[buf] = Q K_j^T
        // Runs ahead of the SiLU warps, bounded only by free S buffers and K tiles.
        const uint32_t idesc_s = ptx::instr_desc_bf16(128, BKV, false, false);
        int stage = 0;
        uint32_t phase = 0;
        uint32_t s_cnt = 0;
        int it = 0;
        for (int t = blockIdx.x; t < prm.n_tiles; t += gridDim.x, ++it) {
            const AttnTile tile = prm.tiles[t];
            const int n_kv = (tile.kmax + BKV - 1) / BKV;
            const int qb = it % C::QB;
            ptx::mbar_wait(&q_full[qb], (it / C::QB) & 1);
            ptx::tc_fence_after();
            if (n_kv == 0) {
                if (ptx::elect_one()) ptx::umma_commit(&q_empty[qb]);
                __syncwarp();
                continue;
            }
            const uint32_t sq = ptx::smem_u32(sQ + qb * C::Q_BYTES);
            for (int j = 0; j < n_kv; ++j) {
                const uint32_t buf = s_cnt % NB;
                ptx::mbar_wait(&k_full[stage], phase);
                ptx::mbar_wait(&s_empty[buf], ((s_cnt / NB) & 1) ^ 1);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    const uint32_t sk = ptx::smem_u32(sK + stage * C::KV_TILE_BYTES);
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t sl = (kk * 16) / C::CHUNK;
                        const uint32_t in = ((kk * 16) % C::CHUNK) * 2;
                        const uint64_t da = ptx::smem_desc(sq + sl * (128 * C::ROWB) + in, 16, 8 * C::ROWB, C::LAYOUT);
                        const uint64_t db = ptx::smem_desc(sk + sl * (BKV * C::ROWB) + in, 16, 8 * C::ROWB, C::LAYOUT);
                        ptx::umma_bf16(tmem + buf * BKV, da, db, idesc_s, kk > 0);
                    }
                    if (j == n_kv - 1) ptx::umma_commit(&q_empty[qb]);
                    ptx::umma_commit(&s_full[buf]);
                    ptx::umma_commit(&k_empty[stage]);  // K consumed
                }
                __syncwarp();
                ++s_cnt;
                if (++stage == C::KS) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 3) {
        // ------------------------------------------------ PV issuer: O[ob] += P[buf] V_j
        // A second MMA-issuing warp: the eight K=16 steps of every P.V do not
        // delay the next S, and vice versa.
        const uint32_t idesc_o = ptx::instr_desc_bf16(128, D, false, true);
        int stage = 0;
        uint32_t phase = 0;
        uint32_t cnt = 0;
        int it = 0;
        for (int t = blockIdx.x; t < prm.n_tiles; t += gridDim.x, ++it) {
            const AttnTile tile = prm.tiles[t];
            const int n_kv = (tile.kmax + BKV - 1) / BKV;
            const int ob = it % kOB;
            ptx::mbar_wait(&o_empty[ob], ((it / kOB) & 1) ^ 1);
            ptx::tc_fence_after();
            if (n_kv == 0) {
                if (ptx::elect_one()) ptx::umma_commit(&o_full[ob]);
                __syncwarp();
                continue;
            }
            for (int j = 0; j < n_kv; ++j, ++cnt) {
                const uint32_t buf = cnt % NB;
                ptx::mbar_wait(&p_full[buf], (cnt / NB) & 1);
                ptx::mbar_wait(&v_full[stage], phase);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    const uint32_t sv = ptx::smem_u32(sV + stage * C::KV_TILE_BYTES);
                    const uint32_t o_tmem = tmem + kOCol + ob * D;
#pragma unroll
                    for (int kk = 0; kk < BKV / 16; ++kk) {
                        // keys [16kk, 16kk+16) were packed by the SiLU warp owning
                        // S columns [CW*c, CW*(c+1)), c = 16kk / CW, into its first CW/2
                        constexpr int CW = C::CW;
                        const uint32_t p_col = buf * BKV + ((16 * kk) / CW) * CW + ((16 * kk) % CW) / 2;
                        const uint64_t db = ptx::smem_desc(sv + kk * 16 * C::ROWB, BKV * C::ROWB, 8 * C::ROWB, C::LAYOUT);
                        ptx::umma_bf16_ts(o_tmem, tmem + p_col, db, idesc_o, (j > 0 || kk > 0));
                    }
                    ptx::umma_commit(&v_empty[stage]);
                    ptx::umma_commit(&s_empty[buf]);
                    if (j == n_kv - 1) ptx::umma_commit(&o_full[ob]);
                }
                __syncwarp();
                if (++stage == C::VS) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp >= 4 && warp < 4 + C::kSilu) {
        // ------------------------------------------------ SiLU warps, P aliasing S
        constexpr int CW = C::CW;                 // key columns per warp and key tile
        constexpr int NQ = CW / 16;               // 16-key chunks per warp
        const uint32_t q = warp & 3;              // TMEM lane quarter
        const uint32_t grp = (warp - 4) / (C::kSilu / C::kSiluGroups);  // key tiles s_cnt % 2 == grp
        const uint32_t cq = ((warp - 4) >> 2) % (BKV / CW);             // column part
        const uint32_t m = q * 32 + lane;         // MMA row == TMEM lane
        const uint32_t lane_addr = (q * 32u) << 16;
        // (announcing P(j) only after issuing the S load of tile j+1 measured 3-5% slower)
        uint32_t s_base = 0;  // key tiles of the CTA's earlier tiles (the S/P ring position)
        const int hs = m / prm.rt;
        const int i = m - hs * prm.rt;
        // the row's mask prefix of the next tile is loaded while this tile's keys are processed
        auto prefix_of = [&](int tt) -> int {
            if (tt >= prm.n_tiles) return 0;
            const AttnTile tl = prm.tiles[tt];
            return i < tl.n_rows ? __ldg(prm.q_prefix + tl.q_row0 + i) : 0;
        };
        int prefix_next = prefix_of(blockIdx.x);
        for (int t = blockIdx.x; t < prm.n_tiles; t += gridDim.x) {
            const AttnTile tile = prm.tiles[t];
            const int n_kv = (tile.kmax + BKV - 1) / BKV;
            const int prefix = prefix_next;
            prefix_next = prefix_of(t + gridDim.x);
            // this group's key tiles: s_cnt = s_base + j with s_cnt % kSiluGroups == grp
            const int j0 = static_cast<int>((grp + C::kSiluGroups - s_base % C::kSiluGroups) % C::kSiluGroups);
            const uint32_t s_next = s_base + n_kv;
            for (int j = j0; j < n_kv; j += C::kSiluGroups) {
                const uint32_t s_cnt = s_base + j;
                const uint32_t buf = s_cnt % NB;
                ptx::mbar_wait(&s_full[buf], (s_cnt / NB) & 1);
                ptx::tc_fence_after();
                const uint32_t col = buf * BKV + cq * CW;
                const int nvalid = prefix - (j * BKV + static_cast<int>(cq) * CW);  // >= CW: no masking
                // 16-key chunks: the next chunk's TMEM load and this chunk's P store are in
                // flight while its SiLUs run; P (packed bf16) overwrites the S columns already read
                if (__all_sync(0xffffffffu, nvalid <= 0)) {
                    const uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
                    for (int c = 0; c < NQ; ++c) ptx::tmem_st8(tmem + lane_addr + col + 8 * c, z);
                } else {
                    float v[2][16];
                    ptx::tmem_ld16(tmem + lane_addr + col, v[0]);
                    ptx::tmem_ld_wait_dep(v[0]);
#pragma unroll
                    for (int c = 0; c < NQ; ++c) {
                        if (c + 1 < NQ) ptx::tmem_ld16(tmem + lane_addr + col + 16 * (c + 1), v[(c + 1) & 1]);
                        uint32_t pk[8];
                        attn_detail::silu_half(v[c & 1], pk, nvalid, 16 * c);
                        ptx::tmem_st8(tmem + lane_addr + col + 8 * c, pk);
                        if (c + 1 < NQ) ptx::tmem_ld_wait_dep(v[(c + 1) & 1]);
                    }
                }
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&p_full[buf]);
            }
            s_base = s_next;
        }
    } else if (warp >= 4 + C::kSilu) {
        // ------------------------------------------------ epilogue warps
        // The row's scale / self index of the next tile are fetched a tile ahead, and the
        // self term's Q, K (and for D <= 32 V) rows are loaded together before the O wait:
        // one global round trip per tile on the epilogue's critical path instead of three.
        constexpr bool kVpre = D <= 32;
        const uint32_t q = warp & 3;
        const uint32_t m = q * 32 + lane;
        const uint32_t lane_addr = (q * 32u) << 16;
        const int hs = m / prm.rt;
        const int i = m - hs * prm.rt;
        auto meta_of = [&](int tt, float& sc, int& sr) {
            sc = 0.f;
            sr = -1;
            if (tt < prm.n_tiles) {
                const AttnTile tl = prm.tiles[tt];
                if (i < tl.n_rows) {
                    sc = __ldg(prm.q_scale + tl.q_row0 + i);
                    sr = __ldg(prm.q_self + tl.q_row0 + i);
                }
            }
        };
        float scale_next;
        int self_next;
        meta_of(blockIdx.x, scale_next, self_next);
        int it = 0;
        for (int t = blockIdx.x; t < prm.n_tiles; t += gridDim.x, ++it) {
            const AttnTile tile = prm.tiles[t];
            const int n_kv = (tile.kmax + BKV - 1) / BKV;
            const int ob = it % kOB;
            const bool valid = i < tile.n_rows;
            const int qrow = tile.q_row0 + i;
            const int head = tile.head0 + hs;
            const int g = tile.head0 / r_per_g;
            const float scale = scale_next;
            const int self_row = self_next;
            meta_of(t + gridDim.x, scale_next, self_next);
            // self term inputs (T rows) are independent of O: fetch before waiting
            float wself = 0.f;
            uint4 vpre[kVpre ? D / 8 : 1];
            if (valid && self_row >= 0) {
                const __nv_bfloat16* qp = prm.q_ptr + (long long)qrow * prm.ldq + prm.q_col0 + head * D;
                const __nv_bfloat16* kp = prm.kv_ptr + (long long)self_row * prm.ldkv + prm.k_col0 + g * D;
                if constexpr (kVpre) {
                    const __nv_bfloat16* vp = prm.kv_ptr + (long long)self_row * prm.ldkv + prm.v_col0 + g * D;
#pragma unroll
                    for (int e = 0; e < D / 8; ++e) vpre[e] = *reinterpret_cast<const uint4*>(vp + 8 * e);
                }
                float dot = 0.f;
#pragma unroll 4
                for (int e = 0; e < D; e += 8) {
                    const uint4 a = *reinterpret_cast<const uint4*>(qp + e);
                    const uint4 b = *reinterpret_cast<const uint4*>(kp + e);
                    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
                    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const float2 fa = __bfloat1622float2(a2[k]), fb = __bfloat1622float2(b2[k]);
                        dot = fmaf(fa.x, fb.x, dot);
                        dot = fmaf(fa.y, fb.y, dot);
                    }
                }
                wself = silu_precise(dot);
            }
            // one 16-column chunk of O: x scale (+ the self term), bf16, stored
            auto emit = [&](float (&v)[16], const int c, const uint4 a, const uint4 b) {
                if (n_kv == 0) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = 0.f;
                }
                if (valid) {
                    if (self_row >= 0) {
                        const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
                        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const float2 fa = __bfloat1622float2(a2[k]), fb = __bfloat1622float2(b2[k]);
                            v[2 * k] += wself * fa.x;
                            v[2 * k + 1] += wself * fa.y;
                            v[8 + 2 * k] += wself * fb.x;
                            v[8 + 2 * k + 1] += wself * fb.y;
                        }
                    }
                    __nv_bfloat16* o = prm.out + (long long)qrow * prm.ldo + head * D + c;
                    uint4 w0, w1;
                    w0.x = pack_bf16(v[0] * scale, v[1] * scale);
                    w0.y = pack_bf16(v[2] * scale, v[3] * scale);
                    w0.z = pack_bf16(v[4] * scale, v[5] * scale);
                    w0.w = pack_bf16(v[6] * scale, v[7] * scale);
                    w1.x = pack_bf16(v[8] * scale, v[9] * scale);
                    w1.y = pack_bf16(v[10] * scale, v[11] * scale);
                    w1.z = pack_bf16(v[12] * scale, v[13] * scale);
                    w1.w = pack_bf16(v[14] * scale, v[15] * scale);
                    reinterpret_cast<uint4*>(o)[0] = w0;
                    reinterpret_cast<uint4*>(o)[1] = w1;
                }
            };
            // O is read out two chunks at a time: the next chunk's TMEM load is in flight while
            // this one is scaled and stored, and O goes back to the PV warp right after the last
            // load (before the last chunk's stores)
            auto release = [&]() {
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&o_empty[ob]);
            };
            // the self row's V columns of a chunk (T rows), fetched with the chunk's TMEM load
            auto vload = [&](const int c, uint4& a, uint4& b) {
                if constexpr (kVpre) {
                    a = vpre[c / 8];
                    b = vpre[c / 8 + 1];
                } else if (valid && self_row >= 0) {
                    const __nv_bfloat16* vp = prm.kv_ptr + (long long)self_row * prm.ldkv + prm.v_col0 + g * D + c;
                    a = *reinterpret_cast<const uint4*>(vp);
                    b = *reinterpret_cast<const uint4*>(vp + 8);
                }
            };
            uint4 a0 = make_uint4(0, 0, 0, 0), b0 = a0, a1 = a0, b1 = a0;
            vload(0, a0, b0);
            ptx::mbar_wait(&o_full[ob], (it / kOB) & 1);
            ptx::tc_fence_after();
            float v0[16], v1[16];
            ptx::tmem_ld16(tmem + lane_addr + kOCol + ob * D, v0);
            // fully unrolled when V was preloaded (register-array indices must be constant)
#pragma unroll(kVpre ? (D + 31) / 32 : 1)
            for (int c = 0; c < D; c += 32) {
                ptx::tmem_ld_wait_dep(v0);
                const bool two = c + 16 < D;
                if (two) {
                    ptx::tmem_ld16(tmem + lane_addr + kOCol + ob * D + c + 16, v1);
                    vload(c + 16, a1, b1);
                } else {
                    release();
                }
                emit(v0, c, a0, b0);
                if (two) {
                    ptx::tmem_ld_wait_dep(v1);
                    if (c + 32 < D) {
                        ptx::tmem_ld16(tmem + lane_addr + kOCol + ob * D + c + 32, v0);
                        vload(c + 32, a0, b0);
                    } else {
                        release();
                    }
                    emit(v1, c + 16, a1, b1);
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<C::TMEM_COLS>(tmem);
    }
}

}  // namespace mtfm
