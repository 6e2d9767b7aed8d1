// kernels.cu — planning (K0), tokenizer gather (K1 prologue), group LayerNorm,
// gate, heads (K5 epilogue) and the fp32 SIMT check-mode GEMM / attention.
#include <type_traits>
#include <climits>

#include "common.cuh"
#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace mtfm {

// Error keys: atomicMin over (user, piece, stage, row, code) so the batch
// reports the exception the reference would throw first (users in order;
// within a user: pieces in pile order (tokenizer.hpp:244-264); within a piece
// slot-major, dimension check of a slot before its range check
// (tokenizer.hpp:193-207, eval_ctx.hpp:190-198)).
__device__ __forceinline__ unsigned long long err_key(long long u, long long piece, long long stage, long long row,
                                                      int code) {
    u = u < (1ll << 22) - 1 ? u : (1ll << 22) - 1;
    piece = piece < 2047 ? piece : 2047;
    stage = stage < 2047 ? stage : 2047;
    row = row < (1ll << 17) - 1 ? row : (1ll << 17) - 1;
    return (static_cast<unsigned long long>(u) << 42) | (static_cast<unsigned long long>(piece) << 31) |
           (static_cast<unsigned long long>(stage) << 20) | (static_cast<unsigned long long>(row) << 3) |
           static_cast<unsigned long long>(code);
}
enum { ERR_META = 1, ERR_INTEGRITY = 2, ERR_DIMENSION = 3, ERR_LOOKUP = 5, ERR_CONTRACT = 6 };

__device__ __forceinline__ int find_source(const SourceInfo* src, int n_src, int kind, int id, int only_scenario) {
    for (int s = 0; s < n_src; ++s)
        if (src[s].kind == kind && src[s].id == id) {
            if (kind == 2 && only_scenario >= 0 && id != only_scenario) return -1;
            return s;
        }
    return -1;
}

// Sequence of global event e among the user's sequences [s0, s1).
__device__ __forceinline__ int find_seq(const int* ev_off, int s0, int s1, int e) {
    int lo = s0, hi = s1 - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (ev_off[mid] <= e)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

struct CtxLess {  // (kind, ts, pile index) — std::stable_sort by ts per kind (tokenizer.hpp:117-123)
    __device__ bool operator()(long long ta, long long sa, long long tb, long long sb) const {
        const long long ka = sa >> 32, kb = sb >> 32;
        if (ka != kb) return ka < kb;
        if (ta != tb) return ta < tb;
        return sa < sb;
    }
};
struct TLess {  // (ts, scenario, index) — canonical exposure order (tokenizer.hpp:82-90)
    __device__ bool operator()(long long ta, long long sa, long long tb, long long sb) const {
        if (ta != tb) return ta < tb;
        return sa < sb;
    }
};

template <typename Less>
__device__ void bitonic_sort(long long* ts, long long* sec, int npad, Less less) {
    for (int k = 2; k <= npad; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            // one compare-exchange pair per thread and pass (no idle half):
            // pair t -> lower index i (bit j clear), partner i + j
            for (int t = threadIdx.x; t < (npad >> 1); t += blockDim.x) {
                const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
                const int ixj = i + j;
                {
                    const bool up = (i & k) == 0;
                    const long long ta = ts[i], sa = sec[i], tb = ts[ixj], sb = sec[ixj];
                    const bool swap = up ? less(tb, sb, ta, sa) : less(ta, sa, tb, sb);
                    if (swap) {
                        ts[i] = tb;
                        sec[i] = sb;
                        ts[ixj] = ta;
                        sec[ixj] = sa;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// number of entries of sorted a[0, n) strictly below v
// number of a[0..n) <= v (a sorted)
__device__ __forceinline__ int count_le(const long long* a, int n, long long v) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] <= v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int count_below(const long long* a, int n, long long v) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__device__ __forceinline__ float row_scale_of(int norm, int c, int n_tokens) {
    if (norm == 0) return __fdiv_rn(1.f, static_cast<float>(c > 1 ? c : 1));
    if (norm == 1) return __fdiv_rn(1.f, static_cast<float>(n_tokens));
    return 1.f;
}

// One CTA per user: plan_tokens (tokenizer.hpp:53-134) + make_stack_geom
// (hta.hpp:40-71) in prefix form + record slots + input validation.
__global__ void __launch_bounds__(256, 8) plan_kernel(PlanArgs a) {
    MTFM_PDL_ENTRY();
    extern __shared__ long long sm_sort[];
    // sort area: SMEM, or a per-user global scratch slice for users above the SMEM
    // capacity (same algorithm; __syncthreads orders the CTA's global accesses too)
    long long cap = a.max_sort;
    long long* s_ts = sm_sort;
    if (a.sort_off && a.sort_off[blockIdx.x + 1] > a.sort_off[blockIdx.x]) {
        s_ts = a.sort_scratch + a.sort_off[blockIdx.x];
        cap = (a.sort_off[blockIdx.x + 1] - a.sort_off[blockIdx.x]) / 2;
    }
    long long* s_sec = s_ts + cap;
    __shared__ unsigned long long s_err;
    __shared__ int s_lh;
    // per-CTA copies: the source table (find_source from SMEM) and, for the T
    // tokens, a per-source histogram (records / pieces before a scenario)
    constexpr int kMaxSrcSm = 32;
    __shared__ SourceInfo s_srcs[kMaxSrcSm];
    __shared__ int s_tcnt[kMaxSrcSm];
    __shared__ int s_t_unknown;  // a T token without a source: exact slow path (error ordering)
    const bool src_sm = a.n_src <= kMaxSrcSm;
    for (int i = threadIdx.x; i < a.n_src && i < kMaxSrcSm; i += blockDim.x) {
        s_srcs[i] = a.src[i];
        s_tcnt[i] = 0;
    }
    if (threadIdx.x == 0) s_t_unknown = 0;
    const SourceInfo* srcs = src_sm ? s_srcs : a.src;
    const DevBatch& b = a.b;
    const int u = blockIdx.x;
    const int tid = threadIdx.x;
    const int s0 = b.seq_off[u], s1 = b.seq_off[u + 1];
    const int ev0 = b.ev_off[s0], ev1 = b.ev_off[s1];
    const int n_ev = ev1 - ev0;
    const int x0 = b.exp_off[u], x1 = b.exp_off[u + 1];
    const int n_t = x1 - x0;
    const int n_tok = n_ev + n_t;
    if (tid == 0) {
        s_err = ~0ull;
        s_lh = 0;
        if (n_tok == 0) s_err = err_key(u, 0, 0, 0, ERR_CONTRACT);
    }
    int npad = 1;
    while (npad < n_ev) npad <<= 1;
    int tpad = 1;
    while (tpad < n_t) tpad <<= 1;
    if (npad > cap || tpad + n_ev > cap) {
        if (tid == 0) atomicMin(a.err, err_key(u, 0, 0, 0, ERR_CONTRACT) | 7ull);  // capacity
        return;
    }

    // ---------------- context tokens: (kind, ts, pile order)
    // When every sequence is in time order (the usual input) that order is a stable merge
    // of the sequences of each kind: an event's rank is its index in its sequence plus, per
    // other sequence of its kind, the events before it (binary search; the earlier sequence
    // wins ties, as the pile index does). Otherwise, or with many sequences: bitonic sort.
    constexpr int kMergeSeqs = 16;
    int unsorted = s1 - s0 > kMergeSeqs;
    if (!unsorted)
        for (int q = s0; q < s1; ++q)
            for (int e = b.ev_off[q] + tid; e + 1 < b.ev_off[q + 1]; e += blockDim.x)
                unsorted |= b.ev_ts[e + 1] < b.ev_ts[e];
    const bool merge = !__syncthreads_or(unsorted);
    if (merge) {
        int n_k0 = 0;  // H events precede every R event
        for (int q = s0; q < s1; ++q)
            if (!b.seq_kind[q]) n_k0 += b.ev_off[q + 1] - b.ev_off[q];
        for (int i = tid; i < n_ev; i += blockDim.x) {
            const int e = ev0 + i;
            const int sq = find_seq(b.ev_off, s0, s1, e);
            const int kind = b.seq_kind[sq] ? 1 : 0;
            const long long ts = b.ev_ts[e];
            int rank = (kind ? n_k0 : 0) + (e - b.ev_off[sq]);
            for (int q = s0; q < s1; ++q) {
                if (q == sq || (b.seq_kind[q] ? 1 : 0) != kind) continue;
                const int a0 = b.ev_off[q], n = b.ev_off[q + 1] - a0;
                rank += q < sq ? count_le(b.ev_ts + a0, n, ts) : count_below(b.ev_ts + a0, n, ts);
            }
            s_ts[rank] = ts;
            s_sec[rank] = (static_cast<long long>(kind) << 32) | i;
        }
    } else {
        for (int i = tid; i < npad; i += blockDim.x) {
            if (i < n_ev) {
                const int e = ev0 + i;
                const int sq = find_seq(b.ev_off, s0, s1, e);
                s_ts[i] = b.ev_ts[e];
                s_sec[i] = (static_cast<long long>(b.seq_kind[sq] ? 1 : 0) << 32) | i;
            } else {
                s_ts[i] = LLONG_MAX;
                s_sec[i] = 3ll << 32;
            }
        }
    }
    __syncthreads();
    // check_meta_order (token_types.hpp:53-72, run by plan_tokens before any tokenizer
    // check): the first H / R token of each block is compared with -1, so a context
    // timestamp below -1 is a dimension_error that precedes every other error of the user
    for (int i = tid; i < n_ev; i += blockDim.x)
        if (b.ev_ts[ev0 + i] < -1) atomicMin(&s_err, err_key(u, 0, 0, 0, ERR_META));
    if (!merge && n_ev > 1) bitonic_sort(s_ts, s_sec, npad, CtxLess{});
    for (int i = tid; i < n_ev; i += blockDim.x)
        if ((s_sec[i] >> 32) == 0 && (i + 1 == n_ev || (s_sec[i + 1] >> 32) != 0)) s_lh = i + 1;
    __syncthreads();
    const int l_h = s_lh;
    const int l_r = n_ev - l_h;
    const long long* r_ts = s_ts + l_h;  // sorted R timestamps

    // per-row outputs for context rows + tokenizer grouping
    for (int i = tid; i < n_ev; i += blockDim.x) {
        const int local = static_cast<int>(s_sec[i] & 0xffffffffll);
        const int kind = static_cast<int>(s_sec[i] >> 32);
        const int e = ev0 + local;
        const int sq = find_seq(b.ev_off, s0, s1, e);
        const int src = find_source(srcs, a.n_src, kind, b.seq_schema[sq], -1);
        const int row = e - local + i;  // == ev0 + i
        const int prefix = l_h + count_below(r_ts, l_r, s_ts[i]);
        a.rm.src[row] = src;
        a.rm.item[row] = e;
        a.rm.prefix[row] = prefix;
        a.rm.scale[row] = row_scale_of(a.norm, prefix, n_tok);
        a.rm.self[row] = -1;
        a.rm.keybase[row] = ev0;
        if (src >= 0) {
            long long rank = e - b.ev_off[sq];
            for (int q = s0; q < sq; ++q)
                if (b.seq_kind[q] == b.seq_kind[sq] && b.seq_schema[q] == b.seq_schema[sq])
                    rank += b.ev_off[q + 1] - b.ev_off[q];
            a.rm.src_rows[a.src_base[src] + a.us_off[(long long)u * a.n_src + src] + rank] = row;
        }
    }
    // validation of sequence pieces (pile order = non-empty sequences in list order),
    // one (event, slot) check per thread: the smallest error key wins, which is
    // each event's first failing slot as in the sequential rule
    int cslots = 1;
    for (int sc = 0; sc < a.n_src; ++sc)
        if (srcs[sc].kind < 2) cslots = max(cslots, srcs[sc].nslot[0]);
    for (int idx = tid; idx < n_ev * cslots; idx += blockDim.x) {
        const int e = ev0 + idx / cslots;
        const int s = idx - (e - ev0) * cslots;
        const int sq = find_seq(b.ev_off, s0, s1, e);
        int piece = 0;
        for (int q = s0; q < sq; ++q) piece += b.ev_off[q + 1] > b.ev_off[q];
        const int src = find_source(srcs, a.n_src, b.seq_kind[sq] ? 1 : 0, b.seq_schema[sq], -1);
        const int r = e - b.ev_off[sq];
        unsigned long long k = ~0ull;
        if (src < 0) {
            if (s == 0) k = err_key(u, piece, 0, 0, ERR_INTEGRITY);
        } else if (s < srcs[src].nslot[0]) {
            const int cnt = b.ev_feat_off[e + 1] - b.ev_feat_off[e];
            if (cnt <= s) {
                k = err_key(u, piece, 1 + 2 * s, r, ERR_DIMENSION);
            } else {
                const int id = b.ev_feats[b.ev_feat_off[e] + s];
                if (id < 0 || id >= a.slots[srcs[src].slot0 + s].vocab) k = err_key(u, piece, 2 + 2 * s, r, ERR_LOOKUP);
            }
        }
        if (k != ~0ull) atomicMin(&s_err, k);
    }
    int n_pieces_seq = 0;
    for (int q = s0; q < s1; ++q) n_pieces_seq += b.ev_off[q + 1] > b.ev_off[q];
    __syncthreads();

    // ---------------- target tokens: canonical (ts, scenario, index)
    // The sorted R timestamps are needed after the T sort: stash them right
    // behind the T sort area (the host sizes the buffer for tpad + n_ev).
    long long* r_stash = s_ts + tpad;
    for (int i = tid; i < l_r; i += blockDim.x) s_sec[i] = s_ts[l_h + i];
    __syncthreads();
    for (int i = tid; i < l_r; i += blockDim.x) r_stash[i] = s_sec[i];
    __syncthreads();
    for (int i = tid; i < tpad; i += blockDim.x) {
        if (i < n_t) {
            s_ts[i] = b.exp_ts[x0 + i];
            s_sec[i] = (static_cast<long long>(b.exp_scenario[x0 + i]) << 32) | i;
        } else {
            s_ts[i] = LLONG_MAX;
            s_sec[i] = LLONG_MAX;
        }
    }
    __syncthreads();
    if (n_t > 1) bitonic_sort(s_ts, s_sec, tpad, TLess{});
    if (src_sm) {
        for (int p = tid; p < n_t; p += blockDim.x) {
            const int sc = find_source(srcs, a.n_src, 2, static_cast<int>(s_sec[p] >> 32), -1);
            if (sc >= 0) atomicAdd(&s_tcnt[sc], 1);
            else s_t_unknown = 1;
        }
        __syncthreads();
    }
    const bool t_fast = src_sm && !s_t_unknown;
    for (int p = tid; p < n_t; p += blockDim.x) {
        const int local = static_cast<int>(s_sec[p] & 0xffffffffll);
        const int scen = static_cast<int>(s_sec[p] >> 32);
        const int x = x0 + local;
        const long long row = static_cast<long long>(b.n_events) + x0 + p;
        const long long t = x0 + p;
        const int prefix = l_h + count_below(r_stash, l_r, s_ts[p]);
        int rho = 0, n_s = 0, distinct_below = 0;
        long long rec_before = 0;
        if (t_fast) {
            // every T scenario has a source: counts per scenario from the SMEM histogram
            // (sources are distinct scenario ids), rank within the scenario by a scan
            for (int sc = 0; sc < a.n_src; ++sc) {
                const SourceInfo& si2 = srcs[sc];
                if (si2.kind != 2 || s_tcnt[sc] == 0) continue;
                if (si2.id == scen) {
                    n_s = s_tcnt[sc];
                } else if (si2.id < scen) {
                    const bool kept = a.only_scenario < 0 || si2.id == a.only_scenario;
                    rec_before += kept ? static_cast<long long>(s_tcnt[sc]) * si2.ntasks : 0;
                    ++distinct_below;
                }
            }
            for (int q = 0; q < p; ++q) rho += static_cast<int>(s_sec[q] >> 32) == scen;
        }
        for (int q = 0; q < n_t && !t_fast; ++q) {
            const int sq = static_cast<int>(s_sec[q] >> 32);
            if (sq == scen) {
                ++n_s;
                if (q < p) ++rho;
            } else if (sq < scen) {
                const int ss = find_source(srcs, a.n_src, 2, sq, a.only_scenario);
                rec_before += ss >= 0 ? a.src[ss].ntasks : 0;
                // first occurrence of each smaller scenario counts as a piece
                bool first = true;
                for (int q2 = 0; q2 < q; ++q2)
                    if (static_cast<int>(s_sec[q2] >> 32) == sq) {
                        first = false;
                        break;
                    }
                distinct_below += first;
            }
        }
        const int src = find_source(srcs, a.n_src, 2, scen, a.only_scenario);
        a.rm.src[row] = src;
        a.rm.item[row] = x;
        a.rm.prefix[row] = prefix;
        a.rm.scale[row] = row_scale_of(a.norm, prefix + 1, n_tok);
        a.rm.self[row] = static_cast<int>(row);
        a.rm.keybase[row] = ev0;
        a.rm.t_user[t] = u;
        a.rm.t_exp_ref[t] = local;
        a.rm.t_scen[t] = scen;
        a.rm.t_rec0[t] = a.rec_off[u] + rec_before + rho;
        a.rm.t_rec_stride[t] = n_s;
        const int piece = n_pieces_seq + distinct_below;
        if (src >= 0)
            a.rm.src_rows[a.src_base[src] + a.us_off[(long long)u * a.n_src + src] + rho] = static_cast<int>(row);
        // s_ts[p] is only read by this iteration: stash what the slot checks need
        s_ts[p] = (static_cast<long long>(piece) << 40) | (static_cast<long long>(rho) << 16) | (src + 1);
    }
    __syncthreads();
    // one (exposure, slot) check per thread (smallest key = first failing slot)
    int tslots = 1;
    for (int sc = 0; sc < a.n_src; ++sc)
        if (srcs[sc].kind == 2) tslots = max(tslots, srcs[sc].nslot[0] + srcs[sc].nslot[1] + srcs[sc].nslot[2]);
    for (int idx = tid; idx < n_t * tslots; idx += blockDim.x) {
        const int p = idx / tslots;
        const int gs = idx - p * tslots;
        const long long pk = s_ts[p];
        const int src = static_cast<int>(pk & 0xffff) - 1;
        const int rho = static_cast<int>((pk >> 16) & 0xffffff);
        const int piece = static_cast<int>(pk >> 40);
        unsigned long long k = ~0ull;
        if (src < 0) {
            if (gs == 0) k = err_key(u, piece, 0, 0, ERR_INTEGRITY);
        } else {
            const SourceInfo& si = srcs[src];
            if (gs < si.nslot[0] + si.nslot[1] + si.nslot[2]) {
                const int x = x0 + static_cast<int>(s_sec[p] & 0xffffffffll);
                int blk = 0, base = 0, blk_off = 0;
                while (gs >= base + si.nslot[blk]) {
                    base += si.nslot[blk];
                    blk_off += b.exp_blk[3 * x + blk];
                    ++blk;
                }
                const int sl = gs - base;
                const int cnt = b.exp_blk[3 * x + blk];
                if (cnt <= sl) {
                    k = err_key(u, piece, 1 + 2 * gs, rho, ERR_DIMENSION);
                } else {
                    const int id = b.exp_feats[b.exp_feat_off[x] + blk_off + sl];
                    if (id < 0 || id >= a.slots[si.slot0 + gs].vocab) k = err_key(u, piece, 2 + 2 * gs, rho, ERR_LOOKUP);
                }
            }
        }
        if (k != ~0ull) atomicMin(&s_err, k);
    }
    __syncthreads();
    if (tid == 0 && s_err != ~0ull) atomicMin(a.err, s_err);
}

void launch_plan(const PlanArgs& a, int smem_elems, cudaStream_t st) {
    if (a.b.n_users == 0) return;
    const size_t smem = static_cast<size_t>(smem_elems) * 16;
    cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    launch_k(plan_kernel, dim3(a.b.n_users), dim3(256), smem, st, a);
}

// ---------------------------------------------------------------- gather
template <typename T>
__global__ void gather_kernel(DevBatch b, const SourceInfo* __restrict__ srcs, const SlotInfo* __restrict__ slots,
                              const int* __restrict__ src_rows, const int* __restrict__ row_item,
                              const long long* __restrict__ src_base, const long long* __restrict__ src_cnt,
                              const long long* __restrict__ emb_base, const T* __restrict__ tables, int d_emb,
                              int n_src, long long total_rows, int max_slots, T* __restrict__ out) {
    // source and slot tables in SMEM (n_src <= 32, slots <= kGatherSlots or read from global)
    constexpr int kGatherSlots = 128;
    __shared__ long long s_base[33], s_cnt[32], s_emb[32];
    __shared__ SourceInfo s_src[32];
    __shared__ SlotInfo s_slot[kGatherSlots];
    int n_slots = 0;
    for (int i = 0; i < n_src; ++i) n_slots = max(n_slots, srcs[i].slot0 + srcs[i].nslot[0] + srcs[i].nslot[1] + srcs[i].nslot[2]);
    for (int i = threadIdx.x; i < n_src; i += blockDim.x) {
        s_base[i] = src_base[i];
        s_cnt[i] = src_cnt[i];
        s_emb[i] = emb_base[i];
        s_src[i] = srcs[i];
    }
    for (int i = threadIdx.x; i < n_slots && i < kGatherSlots; i += blockDim.x) s_slot[i] = slots[i];
    const SlotInfo* sl_tab = n_slots <= kGatherSlots ? s_slot : slots;
    if (threadIdx.x == 0) s_base[n_src] = total_rows;
    MTFM_PDL_ENTRY();
    __syncthreads();
    // one source row per thread: its (row -> item -> feature offset) chain is loaded once,
    // then every slot's id and table row are independent loads
    for (long long P = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; P < total_rows;
         P += static_cast<long long>(gridDim.x) * blockDim.x) {
        int s = 0;
        while (s + 1 < n_src && P >= s_base[s + 1]) ++s;
        const long long p = P - s_base[s];
        if (p >= s_cnt[s]) continue;
        const SourceInfo& si = s_src[s];
        const int nslots = si.nslot[0] + si.nslot[1] + si.nslot[2];
        T* orow = out + s_emb[s] + p * si.k_pad;
        for (int c = si.k_in; c < si.k_pad; ++c) orow[c] = from_f32<T>(0.f);  // zero padding columns
        const int item = __ldg(row_item + __ldg(src_rows + P));
        const int* fb;
        int nu = 0, nc = 0;
        if (si.kind < 2) {
            fb = b.ev_feats + __ldg(b.ev_feat_off + item);
        } else {
            nu = __ldg(b.exp_blk + 3 * item);
            nc = __ldg(b.exp_blk + 3 * item + 1);
            fb = b.exp_feats + __ldg(b.exp_feat_off + item);
        }
#pragma unroll 4
        for (int k = 0; k < nslots; ++k) {
            const int off = si.kind < 2 || k < si.nslot[0]
                                ? k
                                : (k < si.nslot[0] + si.nslot[1] ? nu + (k - si.nslot[0])
                                                                 : nu + nc + (k - si.nslot[0] - si.nslot[1]));
            int id = __ldg(fb + off);
            const SlotInfo sl = sl_tab[si.slot0 + k];
            id = id < 0 ? 0 : (id >= sl.vocab ? sl.vocab - 1 : id);  // invalid ids were reported by the plan
            const T* trow = tables + sl.emb_off + static_cast<long long>(id) * d_emb;
            T* dst = orow + k * d_emb;
            if (sizeof(T) * d_emb % 16 == 0) {
                const uint4* s4 = reinterpret_cast<const uint4*>(trow);
                uint4* d4 = reinterpret_cast<uint4*>(dst);
                for (int c = 0; c < static_cast<int>(sizeof(T) * d_emb / 16); ++c) d4[c] = __ldg(s4 + c);
            } else {
                for (int c = 0; c < d_emb; ++c) dst[c] = trow[c];
            }
        }
    }
}

template <typename T>
bool launch_gather(const DevBatch& b, const SourceInfo* src_dev, const SlotInfo* slots_dev, const RowMeta& rm,
                   const long long* src_base_dev, const long long* src_cnt_dev, const long long* emb_base_dev,
                   const T* tables, int d_emb, int n_src, long long total_rows, int max_slots, T* out,
                   cudaStream_t st) {
    if (total_rows == 0) return true;
    if (n_src > 32) return false;
    // one source row per thread (the dependent load chain row -> item -> feature
    // offset -> ids -> table rows is latency-bound): every row in flight at once
    const int blocks = static_cast<int>(std::min<long long>(cdiv(total_rows, 256), 148ll * 64));
    launch_k(gather_kernel<T>, dim3(blocks), dim3(256), 0, st, b, src_dev, slots_dev, rm.src_rows, rm.item, src_base_dev, src_cnt_dev,
                                             emb_base_dev, tables, d_emb, n_src, total_rows, max_slots, out);
    return true;
}
template bool launch_gather<float>(const DevBatch&, const SourceInfo*, const SlotInfo*, const RowMeta&,
                                   const long long*, const long long*, const long long*, const float*, int, int,
                                   long long, int, float*, cudaStream_t);
template bool launch_gather<__nv_bfloat16>(const DevBatch&, const SourceInfo*, const SlotInfo*, const RowMeta&,
                                           const long long*, const long long*, const long long*,
                                           const __nv_bfloat16*, int, int, long long, int, __nv_bfloat16*,
                                           cudaStream_t);

// ---------------------------------------------------------------- GLN
// row_normalize (kernels.hpp:132-153) + group_affine (eval_ctx.hpp:130-143).
// One warp per row, 4 consecutive columns per lane per 128-column slice,
// vectorised loads/stores (memory-bound: one read + one write of the row).

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ld4(const __nv_bfloat16* p) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
    const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
    const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
    return make_float4(fa.x, fa.y, fb.x, fb.y);
}
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ void st4(__nv_bfloat16* p, float4 v) {
    uint2 u;
    u.x = pack_bf16(v.x, v.y);
    u.y = pack_bf16(v.z, v.w);
    *reinterpret_cast<uint2*>(p) = u;
}

// Normalises the row held as float4 slices (c = 128*i + 4*lane) in place.
template <int NS, bool kFast = false>
__device__ __forceinline__ void normalize_slices(float4 (&v)[NS], int d, int lane, float eps) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NS; ++i)
        if (128 * i + 4 * lane < d) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    s = warp_sum(s);
    // kFast (bf16 outputs): multiply by the rounded reciprocal (exact for power-of-two d)
    const float rd = kFast ? 1.f / static_cast<float>(d) : 0.f;
    const float mean = kFast ? s * rd : __fdiv_rn(s, static_cast<float>(d));
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < NS; ++i)
        if (128 * i + 4 * lane < d) {
            v[i].x -= mean;
            v[i].y -= mean;
            v[i].z -= mean;
            v[i].w -= mean;
            q += (v[i].x * v[i].x + v[i].y * v[i].y) + (v[i].z * v[i].z + v[i].w * v[i].w);
        }
    q = warp_sum(q);
    const float var = kFast ? q * rd : __fdiv_rn(q, static_cast<float>(d));
    const float inv = kFast ? rsqrtf(var + eps) : __fdiv_rn(1.f, sqrtf(var + eps));
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        v[i].x *= inv;
        v[i].y *= inv;
        v[i].z *= inv;
        v[i].w *= inv;
    }
}

template <typename T, int NS>
__global__ void __launch_bounds__(256) gln_kernel(const float* __restrict__ x, long long ldx, long long r0,
                                                  long long n_rows, int d, const int* __restrict__ row_src,
                                                  const float* __restrict__ gain, const float* __restrict__ bias,
                                                  float eps, T* __restrict__ out, long long ldo) {
    MTFM_PDL_ENTRY();
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long i = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n_rows; i += warps) {
        const long long r = r0 + i;
        const float* xr = x + r * ldx;
        int g = row_src[r];
        float4 v[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const int c = 128 * k + 4 * lane;
            v[k] = c < d ? __ldcs(reinterpret_cast<const float4*>(xr + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        normalize_slices<NS, std::is_same_v<T, __nv_bfloat16>>(v, d, lane, eps);
        g = g < 0 ? 0 : g;
        const float* gg = gain + (long long)g * d;
        const float* bb = bias + (long long)g * d;
        T* o = out + i * ldo;
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const int c = 128 * k + 4 * lane;
            if (c < d) {
                const float4 ga = __ldg(reinterpret_cast<const float4*>(gg + c));
                const float4 be = __ldg(reinterpret_cast<const float4*>(bb + c));
                st4(o + c, make_float4(v[k].x * ga.x + be.x, v[k].y * ga.y + be.y, v[k].z * ga.z + be.z,
                                       v[k].w * ga.w + be.w));
            }
        }
    }
}

template <typename T>
void launch_gln(const float* x, long long ldx, long long r0, long long n_rows, int d, const int* row_src,
                const float* gain, const float* bias, float eps, T* out, long long ldo, cudaStream_t st) {
    if (n_rows == 0) return;
    const int blocks = static_cast<int>(std::min<long long>(cdiv(n_rows, 8), 148ll * 16));
    const int ns = static_cast<int>(cdiv(d, 128));
    if (ns <= 1) launch_k(gln_kernel<T, 1>, dim3(blocks), dim3(256), 0, st, x, ldx, r0, n_rows, d, row_src, gain, bias, eps, out, ldo);
    else if (ns == 2) launch_k(gln_kernel<T, 2>, dim3(blocks), dim3(256), 0, st, x, ldx, r0, n_rows, d, row_src, gain, bias, eps, out, ldo);
    else if (ns <= 4) launch_k(gln_kernel<T, 4>, dim3(blocks), dim3(256), 0, st, x, ldx, r0, n_rows, d, row_src, gain, bias, eps, out, ldo);
    else launch_k(gln_kernel<T, 8>, dim3(blocks), dim3(256), 0, st, x, ldx, r0, n_rows, d, row_src, gain, bias, eps, out, ldo);
}
template void launch_gln<float>(const float*, long long, long long, long long, int, const int*, const float*,
                                const float*, float, float*, long long, cudaStream_t);
template void launch_gln<__nv_bfloat16>(const float*, long long, long long, long long, int, const int*,
                                        const float*, const float*, float, __nv_bfloat16*, long long,
                                        cudaStream_t);

template <int NS>
__global__ void __launch_bounds__(256) gln_multi_kernel(const float* __restrict__ x, long long ldx, long long n_rows,
                                                        int d, const int* __restrict__ row_src,
                                                        const __grid_constant__ GlnCopies c, float eps, long long ldo) {
    // two rows per warp iteration: twice the loads in flight, and one gain/bias
    // fetch serves both rows when they share a group (the common case)
    MTFM_PDL_ENTRY();
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long r0 = 2 * (blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5)); r0 < n_rows;
         r0 += 2 * warps) {
        const bool two = r0 + 1 < n_rows;
        const long long x0 = c.in_rows ? static_cast<long long>(__ldg(c.in_rows + r0)) : r0;
        const long long x1 = two ? (c.in_rows ? static_cast<long long>(__ldg(c.in_rows + r0 + 1)) : r0 + 1) : x0;
        float4 v[NS], w[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const int col = 128 * k + 4 * lane;
            v[k] = col < d ? __ldcs(reinterpret_cast<const float4*>(x + x0 * ldx + col)) : make_float4(0.f, 0.f, 0.f, 0.f);
            w[k] = (two && col < d) ? __ldcs(reinterpret_cast<const float4*>(x + x1 * ldx + col))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        int g0 = row_src[x0], g1 = two ? row_src[x1] : g0;
        normalize_slices<NS, true>(v, d, lane, eps);
        normalize_slices<NS, true>(w, d, lane, eps);
        g0 = g0 < 0 ? 0 : g0;
        g1 = g1 < 0 ? 0 : g1;
        for (int l = 0; l < c.n; ++l) {
            __nv_bfloat16* o = static_cast<__nv_bfloat16*>(c.out[l]) + r0 * ldo;
            if (c.gain[l] == nullptr) {  // the normalised rows themselves (xhat)
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                    const int col = 128 * k + 4 * lane;
                    if (col < d) {
                        st4(o + col, v[k]);
                        if (two) st4(o + ldo + col, w[k]);
                    }
                }
                continue;
            }
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                const int col = 128 * k + 4 * lane;
                if (col < d) {
                    float4 ga = __ldg(reinterpret_cast<const float4*>(c.gain[l] + (long long)g0 * d + col));
                    float4 be = __ldg(reinterpret_cast<const float4*>(c.bias[l] + (long long)g0 * d + col));
                    st4(o + col, make_float4(v[k].x * ga.x + be.x, v[k].y * ga.y + be.y, v[k].z * ga.z + be.z,
                                             v[k].w * ga.w + be.w));
                    if (two) {
                        if (g1 != g0) {
                            ga = __ldg(reinterpret_cast<const float4*>(c.gain[l] + (long long)g1 * d + col));
                            be = __ldg(reinterpret_cast<const float4*>(c.bias[l] + (long long)g1 * d + col));
                        }
                        st4(o + ldo + col, make_float4(w[k].x * ga.x + be.x, w[k].y * ga.y + be.y,
                                                       w[k].z * ga.z + be.z, w[k].w * ga.w + be.w));
                    }
                }
            }
        }
    }
}

void launch_gln_multi_bf16(const float* x, long long ldx, long long n_rows, int d, const int* row_src,
                           const GlnCopies& c, float eps, long long ldo, cudaStream_t st) {
    if (n_rows == 0 || c.n == 0) return;
    const int blocks = static_cast<int>(std::min<long long>(cdiv(n_rows, 16), 148ll * 16));
    const int ns = static_cast<int>(cdiv(d, 128));
    if (ns <= 1) launch_k(gln_multi_kernel<1>, dim3(blocks), dim3(256), 0, st, x, ldx, n_rows, d, row_src, c, eps, ldo);
    else if (ns == 2) launch_k(gln_multi_kernel<2>, dim3(blocks), dim3(256), 0, st, x, ldx, n_rows, d, row_src, c, eps, ldo);
    else if (ns <= 4) launch_k(gln_multi_kernel<4>, dim3(blocks), dim3(256), 0, st, x, ldx, n_rows, d, row_src, c, eps, ldo);
    else if (ns <= 6) launch_k(gln_multi_kernel<6>, dim3(blocks), dim3(256), 0, st, x, ldx, n_rows, d, row_src, c, eps, ldo);
    else launch_k(gln_multi_kernel<8>, dim3(blocks), dim3(256), 0, st, x, ldx, n_rows, d, row_src, c, eps, ldo);
}

template <typename T, int NS>
__global__ void __launch_bounds__(256) gate_kernel(const T* __restrict__ a, long long lda, const T* __restrict__ u,
                                                   long long ldu, long long n_rows, int d,
                                                   const int* __restrict__ row_src, const float* __restrict__ gain,
                                                   const float* __restrict__ bias, float eps, T* __restrict__ out,
                                                   long long ldo) {
    MTFM_PDL_ENTRY();
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long i = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n_rows; i += warps) {
        const T* ar = a + i * lda;
        const T* ur = u + i * ldu;
        int g = row_src[i];
        float4 v[NS], uu[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const int c = 128 * k + 4 * lane;
            const bool ok = c < d;
            v[k] = ok ? ld4(ar + c) : make_float4(0.f, 0.f, 0.f, 0.f);
            uu[k] = ok ? ld4(ur + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        normalize_slices<NS, std::is_same_v<T, __nv_bfloat16>>(v, d, lane, eps);
        g = g < 0 ? 0 : g;
        const float* gg = gain + (long long)g * d;
        const float* bb = bias + (long long)g * d;
        T* o = out + i * ldo;
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const int c = 128 * k + 4 * lane;
            if (c < d) {
                const float4 ga = __ldg(reinterpret_cast<const float4*>(gg + c));
                const float4 be = __ldg(reinterpret_cast<const float4*>(bb + c));
                st4(o + c, make_float4((v[k].x * ga.x + be.x) * uu[k].x, (v[k].y * ga.y + be.y) * uu[k].y,
                                       (v[k].z * ga.z + be.z) * uu[k].z, (v[k].w * ga.w + be.w) * uu[k].w));
            }
        }
    }
}

// bf16, d = 256*NS8: lane owns 8 consecutive columns per 256-column slice (one
// 16-byte load per tensor, slice and row) and each warp carries RPW rows at
// once, so 2*RPW*NS8 independent loads are in flight per warp.
template <int RPW, int NS8>
__global__ void __launch_bounds__(256, NS8 * RPW <= 2 ? 4 : 2) gate_bf16_kernel(const __nv_bfloat16* __restrict__ a, long long lda,
                                                        const __nv_bfloat16* __restrict__ u, long long ldu,
                                                        long long n_rows, const int* __restrict__ row_src,
                                                        const float* __restrict__ gain,
                                                        const float* __restrict__ bias, float eps,
                                                        __nv_bfloat16* __restrict__ out, long long ldo) {
    MTFM_PDL_ENTRY();
    constexpr int d = 256 * NS8;
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long i0 = (blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5)) * RPW; i0 < n_rows;
         i0 += warps * RPW) {
        uint4 av[RPW][NS8], uv[RPW][NS8];
        int g[RPW];
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const long long i = i0 + r;
#pragma unroll
            for (int k = 0; k < NS8; ++k) {
                const int c = 256 * k + 8 * lane;
                av[r][k] = i < n_rows ? __ldcs(reinterpret_cast<const uint4*>(a + i * lda + c)) : make_uint4(0, 0, 0, 0);
                uv[r][k] = i < n_rows ? __ldcs(reinterpret_cast<const uint4*>(u + i * ldu + c)) : make_uint4(0, 0, 0, 0);
            }
            g[r] = i < n_rows ? row_src[i] : 0;
        }
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const long long i = i0 + r;
            // two passes over the packed row (sum, then centred squares): no unpacked copy
            float sum = 0.f;
#pragma unroll
            for (int k = 0; k < NS8; ++k) {
                const __nv_bfloat162* ah = reinterpret_cast<const __nv_bfloat162*>(&av[r][k]);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float2 fa = __bfloat1622float2(ah[j]);
                    sum += fa.x + fa.y;
                }
            }
            sum = warp_sum(sum);
            // multiply by the rounded reciprocal (exact for power-of-two d), as normalize_slices<kFast>
            const float mean = sum * (1.f / static_cast<float>(d));
            float q = 0.f;
#pragma unroll
            for (int k = 0; k < NS8; ++k) {
                const __nv_bfloat162* ah = reinterpret_cast<const __nv_bfloat162*>(&av[r][k]);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float2 fa = __bfloat1622float2(ah[j]);
                    const float dx = fa.x - mean, dy = fa.y - mean;
                    q += dx * dx + dy * dy;
                }
            }
            q = warp_sum(q);
            // bf16 output: MUFU.RSQ (~2 ulp) instead of the IEEE sqrt + divide sequence
            const float inv = rsqrtf(q * (1.f / static_cast<float>(d)) + eps);
            if (i >= n_rows) continue;
            const int gg = g[r] < 0 ? 0 : g[r];
#pragma unroll
            for (int k = 0; k < NS8; ++k) {
                const int c = 256 * k + 8 * lane;
                const float4 g0 = __ldg(reinterpret_cast<const float4*>(gain + gg * d + c));
                const float4 g1 = __ldg(reinterpret_cast<const float4*>(gain + gg * d + c + 4));
                const float4 b0 = __ldg(reinterpret_cast<const float4*>(bias + gg * d + c));
                const float4 b1 = __ldg(reinterpret_cast<const float4*>(bias + gg * d + c + 4));
                const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
                const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                const __nv_bfloat162* ah = reinterpret_cast<const __nv_bfloat162*>(&av[r][k]);
                const __nv_bfloat162* uh = reinterpret_cast<const __nv_bfloat162*>(&uv[r][k]);
                uint32_t o[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float2 fa = __bfloat1622float2(ah[j]);
                    const float2 fu = __bfloat1622float2(uh[j]);
                    const float lo = (((fa.x - mean) * inv) * gv[2 * j] + bv[2 * j]) * fu.x;
                    const float hi = (((fa.y - mean) * inv) * gv[2 * j + 1] + bv[2 * j + 1]) * fu.y;
                    const __nv_bfloat162 h2 = __floats2bfloat162_rn(lo, hi);
                    o[j] = *reinterpret_cast<const uint32_t*>(&h2);
                }
                *reinterpret_cast<uint4*>(out + i * ldo + c) = make_uint4(o[0], o[1], o[2], o[3]);
            }
        }
    }
}

template <typename T>
void launch_gate(const T* a, long long lda, const T* u, long long ldu, long long n_rows, int d,
                 const int* row_src_of_rows, const float* gain, const float* bias, float eps, T* out,
                 long long ldo, cudaStream_t st) {
    if (n_rows == 0) return;
    if constexpr (std::is_same_v<T, __nv_bfloat16>) {
        const bool al = lda % 8 == 0 && ldu % 8 == 0 && ldo % 8 == 0;
#define MTFM_GATE16(RPW, NS8)                                                                                     \
    launch_k(gate_bf16_kernel<RPW, NS8>, dim3(static_cast<int>(std::min<long long>(cdiv(n_rows, 8 * RPW), 148ll * 16))), \
             dim3(256), 0, st, a, lda, u, ldu, n_rows, row_src_of_rows, gain, bias, eps, out, ldo)
        if (al && d == 256) { MTFM_GATE16(2, 1); return; }
        if (al && d == 512) { MTFM_GATE16(2, 2); return; }
        if (al && d == 768) { MTFM_GATE16(2, 3); return; }
        if (al && d == 1024) { MTFM_GATE16(2, 4); return; }
#undef MTFM_GATE16
    }
    const int blocks = static_cast<int>(std::min<long long>(cdiv(n_rows, 8), 148ll * 16));
    const int ns = static_cast<int>(cdiv(d, 128));
#define MTFM_GATE(NS) launch_k(gate_kernel<T, NS>, dim3(blocks), dim3(256), 0, st, a, lda, u, ldu, n_rows, d, row_src_of_rows, gain, bias, eps, out, ldo)
    if (ns <= 1) MTFM_GATE(1);
    else if (ns == 2) MTFM_GATE(2);
    else if (ns <= 4) MTFM_GATE(4);
    else MTFM_GATE(8);
#undef MTFM_GATE
}
template void launch_gate<float>(const float*, long long, const float*, long long, long long, int, const int*,
                                 const float*, const float*, float, float*, long long, cudaStream_t);
template void launch_gate<__nv_bfloat16>(const __nv_bfloat16*, long long, const __nv_bfloat16*, long long,
                                         long long, int, const int*, const float*, const float*, float,
                                         __nv_bfloat16*, long long, cudaStream_t);

__global__ void to_bf16_kernel(const float* __restrict__ x, long long n_rows, int d, __nv_bfloat16* __restrict__ out,
                               long long ldo) {
    MTFM_PDL_ENTRY();
    const long long n = n_rows * d;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / d;
        const int c = static_cast<int>(i - r * d);
        out[r * ldo + c] = __float2bfloat16_rn(x[i]);
    }
}
void launch_to_bf16(const float* x, long long n_rows, int d, __nv_bfloat16* out, long long ldo, cudaStream_t st) {
    if (n_rows == 0) return;
    const int blocks = static_cast<int>(std::min<long long>(cdiv(n_rows * d, 256), 148ll * 16));
    launch_k(to_bf16_kernel, dim3(blocks), dim3(256), 0, st, x, n_rows, d, out, ldo);
}

// ---------------------------------------------------------------- heads
// mmoe_forward (heads.hpp:47-99) for one T row per warp, then the record of
// model.hpp:284-311: probability = clamp(sigmoid(z), 1e-12, 1 - 1e-12).
// The task gates (softmax over E, kernels.hpp:155-173) are computed first,
// then every expert activation silu(x W_e + b_e) once, shared by all tasks.
constexpr int kMaxTasks = 8;

__global__ void __launch_bounds__(256) heads_kernel(HeadArgs a) {
    MTFM_PDL_ENTRY();
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    __shared__ float s_gate[8][kMaxTasks][32];
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long t = blockIdx.x * (long long)(blockDim.x >> 5) + wib; t < a.n_t; t += warps) {
        const int scen = a.t_scen[t];
        int s = -1;
        for (int i = 0; i < a.n_src; ++i)
            if (a.src[i].kind == 2 && a.src[i].id == scen) s = i;
        if (s < 0) continue;  // reported by the plan
        const SourceInfo si = a.src[s];
        const float* y = a.y + t * a.ldy;
        for (int k0 = 0; k0 < si.ntasks; k0 += kMaxTasks) {
            const int nk = min(kMaxTasks, si.ntasks - k0);
            // gates: lane e holds logit e of each task
            for (int k = 0; k < nk; ++k) {
                const int task = si.task0 + k0 + k;
                const float g = lane < a.E ? y[a.E * a.de + task * a.E + lane] + a.gate_bias[task * a.E + lane]
                                           : -INFINITY;
                float mx = g;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                const float e = lane < a.E ? expf(g - mx) : 0.f;
                // sequential sum over e, as softmax_rows does
                float sum = 0.f;
                for (int i = 0; i < a.E; ++i) sum += __shfl_sync(0xffffffffu, e, i);
                s_gate[wib][k][lane] = e * __fdiv_rn(1.f, sum);
            }
            __syncwarp();
            float z[kMaxTasks];
#pragma unroll
            for (int k = 0; k < kMaxTasks; ++k) z[k] = 0.f;
            for (int c = lane; c < a.de; c += 32) {
                float m[kMaxTasks];
#pragma unroll
                for (int k = 0; k < kMaxTasks; ++k) m[k] = 0.f;
                for (int e = 0; e < a.E; ++e) {
                    const float pre = y[e * a.de + c] + a.exp_bias[e * a.de + c];
                    float act;
                    if (a.precise) {
                        act = silu_precise(pre);
                    } else {
                        const float h = 0.5f * pre;
                        float th;
                        asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(h));
                        act = fmaf(h, th, h);
                    }
#pragma unroll
                    for (int k = 0; k < kMaxTasks; ++k)
                        if (k < nk) m[k] += act * s_gate[wib][k][e];
                }
#pragma unroll
                for (int k = 0; k < kMaxTasks; ++k)
                    if (k < nk) z[k] += m[k] * a.tower_w[(long long)(si.task0 + k0 + k) * a.de + c];
            }
#pragma unroll
            for (int k = 0; k < kMaxTasks; ++k) {
                if (k >= nk) break;
                const float zz = warp_sum(z[k]) + a.tower_b[si.task0 + k0 + k];
                if (lane == 0) {
                    const long long r = a.t_rec0[t] + (long long)(k0 + k) * a.t_rec_stride[t];
                    double p = static_cast<double>(sigmoid_precise(zz));
                    p = p < 1e-12 ? 1e-12 : (p > 1.0 - 1e-12 ? 1.0 - 1e-12 : p);
                    a.rec_user[r] = a.user_id[a.t_user[t]];
                    a.rec_scen[r] = scen;
                    a.rec_exp[r] = a.t_exp_ref[t];
                    a.rec_task[r] = k0 + k;
                    if (a.rec_logit) a.rec_logit[r] = zz;
                    a.rec_prob[r] = p;
                }
            }
            __syncwarp();
        }
    }
}
// Fast path: one warp per target with everything per-target in registers and
// the small per-model tables (expert bias, gate bias, tower weights) in SMEM.
// Lane l owns columns 4l + 128j (j < NJ) of every expert: the expert
// pre-activations are read as coalesced float4 rows, SiLU'd once, and every
// task's gate mix and tower dot product reuse them.
template <int E, int NJ>
__global__ void __launch_bounds__(256) heads_fast_kernel(HeadArgs a, int n_tasks_total) {
    MTFM_PDL_ENTRY();
    extern __shared__ float hsm[];
    const int de = NJ * 128;
    float* s_eb = hsm;                          // [E*de]
    float* s_tw = s_eb + E * de;                // [n_tasks_total*de]
    float* s_gb = s_tw + n_tasks_total * de;    // [n_tasks_total*E]
    float* s_tb = s_gb + n_tasks_total * E;     // [n_tasks_total]
    for (int i = threadIdx.x; i < E * de; i += blockDim.x) s_eb[i] = a.exp_bias[i];
    for (int i = threadIdx.x; i < n_tasks_total * de; i += blockDim.x) s_tw[i] = a.tower_w[i];
    for (int i = threadIdx.x; i < n_tasks_total * E; i += blockDim.x) s_gb[i] = a.gate_bias[i];
    for (int i = threadIdx.x; i < n_tasks_total; i += blockDim.x) s_tb[i] = a.tower_b[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long t = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); t < a.n_t; t += warps) {
        const int scen = a.t_scen[t];
        int s = -1;
        for (int i = 0; i < a.n_src; ++i)
            if (a.src[i].kind == 2 && a.src[i].id == scen) s = i;
        if (s < 0) continue;  // reported by the plan
        const int task0 = a.src[s].task0, ntasks = a.src[s].ntasks;
        const float* y = a.y + t * a.ldy;
        float act[E][NJ][4];
#pragma unroll
        for (int e = 0; e < E; ++e)
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int c = 4 * lane + 128 * j;
                const float4 v = __ldcs(reinterpret_cast<const float4*>(y + e * de + c));
                const float4 b = *reinterpret_cast<const float4*>(s_eb + e * de + c);
                const float pre[4] = {v.x + b.x, v.y + b.y, v.z + b.z, v.w + b.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (a.precise) {
                        act[e][j][i] = silu_precise(pre[i]);
                    } else {
                        const float h = 0.5f * pre[i];
                        float th;
                        asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(h));
                        act[e][j][i] = fmaf(h, th, h);
                    }
                }
            }
        for (int k = 0; k < ntasks; ++k) {
            const int task = task0 + k;
            // softmax over the E gate logits (every lane; sequential sum as softmax_rows)
            float g[E], mx = -INFINITY;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                g[e] = y[E * de + task * E + e] + s_gb[task * E + e];
                mx = fmaxf(mx, g[e]);
            }
            float sum = 0.f;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                g[e] = expf(g[e] - mx);
                sum += g[e];
            }
            const float inv = __fdiv_rn(1.f, sum);
            float z = 0.f;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const float4 w = *reinterpret_cast<const float4*>(s_tw + task * de + 4 * lane + 128 * j);
                const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    float m = 0.f;
#pragma unroll
                    for (int e = 0; e < E; ++e) m += act[e][j][i] * (g[e] * inv);
                    z += m * wv[i];
                }
            }
            const float zz = warp_sum(z) + s_tb[task];
            if (lane == 0) {
                const long long r = a.t_rec0[t] + (long long)k * a.t_rec_stride[t];
                double p = static_cast<double>(sigmoid_precise(zz));
                p = p < 1e-12 ? 1e-12 : (p > 1.0 - 1e-12 ? 1.0 - 1e-12 : p);
                a.rec_user[r] = a.user_id[a.t_user[t]];
                a.rec_scen[r] = scen;
                a.rec_exp[r] = a.t_exp_ref[t];
                a.rec_task[r] = k;
                if (a.rec_logit) a.rec_logit[r] = zz;
                a.rec_prob[r] = p;
            }
        }
    }
}

template <int E, int NJ>
bool try_heads_fast(const HeadArgs& a, int n_tasks_total, cudaStream_t st) {
    if (a.E != E || a.de != NJ * 128) return false;
    const size_t smem = sizeof(float) * (static_cast<size_t>(E) * a.de + static_cast<size_t>(n_tasks_total) * a.de +
                                         static_cast<size_t>(n_tasks_total) * E + n_tasks_total);
    if (smem > 160 * 1024) return false;
    static int attr_set = 0;
    if (static_cast<int>(smem) > attr_set) {
        cudaFuncSetAttribute(heads_fast_kernel<E, NJ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        attr_set = static_cast<int>(smem);
    }
    const int blocks = static_cast<int>(std::min<long long>(cdiv(a.n_t, 8), 148ll * 4));
    launch_k(heads_fast_kernel<E, NJ>, dim3(blocks), dim3(256), smem, st, a, n_tasks_total);
    return true;
}

void launch_heads(const HeadArgs& a, cudaStream_t st, int n_tasks_total) {
    if (a.n_t == 0) return;
    if (n_tasks_total > 0 &&
        (try_heads_fast<4, 1>(a, n_tasks_total, st) || try_heads_fast<4, 2>(a, n_tasks_total, st) ||
         try_heads_fast<4, 4>(a, n_tasks_total, st) || try_heads_fast<2, 2>(a, n_tasks_total, st) ||
         try_heads_fast<8, 2>(a, n_tasks_total, st) || try_heads_fast<3, 1>(a, n_tasks_total, st) ||
         try_heads_fast<3, 2>(a, n_tasks_total, st)))
        return;
    const int blocks = static_cast<int>(std::min<long long>(cdiv(a.n_t, 8), 148ll * 32));
    launch_k(heads_kernel, dim3(blocks), dim3(256), 0, st, a);
}

// ---------------------------------------------------------------- SIMT GEMM (check mode)
struct SimtGemmBatch {
    SimtGemm p[kMaxProblems];
    int n;
};

__global__ void __launch_bounds__(256) gemm_simt_kernel(const __grid_constant__ SimtGemmBatch bt) {
    MTFM_PDL_ENTRY();
    const SimtGemm& p = bt.p[blockIdx.z];
    const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
    if (m0 >= p.M || n0 >= p.N) return;
    __shared__ float As[16][65];
    __shared__ float Ws[16][64];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < p.K; k0 += 16) {
        for (int i = threadIdx.x; i < 64 * 16; i += 256) {
            const int r = i >> 4, c = i & 15;
            const int m = m0 + r, k = k0 + c;
            As[c][r] = (m < p.M && k < p.K) ? p.A[(long long)m * p.lda + k] : 0.f;
            const int kr = i >> 6, nc = i & 63;
            const int kk = k0 + kr, n = n0 + nc;
            Ws[kr][nc] = (kk < p.K && n < p.N) ? p.W[(long long)kk * p.N + n] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            float a[4], w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) w[j] = Ws[k][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty * 4 + i;
        if (m >= p.M) continue;
        const long long orow = p.row_map ? static_cast<long long>(p.row_map[m]) : p.row_offset + m;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n >= p.N) continue;
            float v = acc[i][j] + (p.bias ? p.bias[n] : 0.f);
            if (p.epi == EPI_SILU_BF16) v = silu_precise(v);
            if (p.epi == EPI_RESID_F32) v += p.resid[orow * p.ldo + n];
            static_cast<float*>(p.out)[orow * p.ldo + n] = v;
        }
    }
}

void launch_gemm_simt(const SimtGemm* probs, int n, cudaStream_t st) {
    SimtGemmBatch bt{};
    int gm = 0, gn = 0;
    for (int i = 0; i < n; ++i) {
        bt.p[i] = probs[i];
        gm = std::max<int>(gm, static_cast<int>(cdiv(probs[i].M, 64)));
        gn = std::max<int>(gn, static_cast<int>(cdiv(probs[i].N, 64)));
    }
    bt.n = n;
    if (gm == 0 || gn == 0) return;
    launch_k(gemm_simt_kernel, dim3(dim3(gn, gm, n)), dim3(256), 0, st, bt);
}

// ---------------------------------------------------------------- SIMT attention (check mode)
// One warp per (query row, head); keys in order j = 0.. prefix-1 (gemm_nn
// accumulation order of hta.hpp:128-131), then the T self key.
__global__ void attn_simt_kernel(SimtAttn a) {
    MTFM_PDL_ENTRY();
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    extern __shared__ float q_sm[];
    float* qv = q_sm + wib * a.dh;
    const long long total = a.n_q * a.heads;
    const int r = a.heads / a.kv_heads;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long w = blockIdx.x * (long long)(blockDim.x >> 5) + wib; w < total; w += warps) {
        const long long i = w / a.heads;
        const int h = static_cast<int>(w - i * a.heads);
        const int g = h / r;
        const int p = a.prefix[i];
        const long long base = a.keybase[i];
        const int self = a.self[i];
        const float* qrow = a.q + i * a.ldq + a.q_col0 + h * a.dh;
        for (int c = lane; c < a.dh; c += 32) qv[c] = qrow[c];
        __syncwarp();
        float acc[8] = {};
        for (int j0 = 0; j0 < p; j0 += 32) {
            const int j = j0 + lane;
            float wgt = 0.f;
            if (j < p) {
                const float* kr = a.kv + (base + j) * a.ldkv + a.k_col0 + g * a.dh;
                float dot = 0.f;
                for (int c = 0; c < a.dh; ++c) dot = fmaf(qv[c], kr[c], dot);
                wgt = silu_precise(dot);
            }
            const int n = min(32, p - j0);
            for (int jj = 0; jj < n; ++jj) {
                const float wj = __shfl_sync(0xffffffffu, wgt, jj);
                const float* vr = a.kv + (base + j0 + jj) * a.ldkv + a.v_col0 + g * a.dh;
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    const int c = lane + 32 * m;
                    if (c < a.dh) acc[m] = fmaf(wj, vr[c], acc[m]);
                }
            }
        }
        if (self >= 0) {
            const float* kr = a.kv + (long long)self * a.ldkv + a.k_col0 + g * a.dh;
            const float* vr = a.kv + (long long)self * a.ldkv + a.v_col0 + g * a.dh;
            float dot = 0.f;
            for (int c = 0; c < a.dh; ++c) dot = fmaf(qv[c], kr[c], dot);
            const float ws = silu_precise(dot);
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int c = lane + 32 * m;
                if (c < a.dh) acc[m] = fmaf(ws, vr[c], acc[m]);
            }
        }
        const float s = a.scale[i];
        float* orow = a.out + i * a.ldo + h * a.dh;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int c = lane + 32 * m;
            if (c < a.dh) orow[c] = acc[m] * s;
        }
        __syncwarp();
    }
}

void launch_attn_simt(const SimtAttn& a, cudaStream_t st) {
    if (a.n_q == 0) return;
    const int wpb = 8;
    const int blocks = static_cast<int>(std::min<long long>(cdiv(a.n_q * a.heads, wpb), 148ll * 64));
    launch_k(attn_simt_kernel, dim3(blocks), dim3(wpb * 32), wpb * a.dh * sizeof(float), st, a);
}

}  // namespace mtfm
