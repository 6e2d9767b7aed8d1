// aggregate.cu — aggregate_users (proj/src/datagen.cpp:171-216) on the GPU.
//
// The reference groups a (user_id, Exposure) stream in two std::map stages:
// per scenario then per user, exposures in stream order; scenario groups are
// merged per user in ascending scenario id, users come out in ascending id and
// are joined with their shared historical/realtime sequences. An unknown
// scenario or user raises integrity_error at the first offending stream
// element (scenario checked before user, datagen.cpp:177-183).
//
// Device formulation (all integer work, bit-exact):
//   classify   x -> (store rank r of its user, scenario index s): bucket r*S + s;
//              first failing x by atomicMin; bucket counts by atomicAdd
//   scan       bucket offsets (bucket order = users ascending, scenarios ascending)
//   scatter    x into its bucket through an atomic cursor (arbitrary order)...
//   sort       ...then each bucket sorted by x (stream order restored: stable)
//   users      users with >= 1 exposure, compacted by a scan; per user the
//              sequence / event / feature spans of the store are contiguous and
//              map to contiguous output spans (output users are a subsequence
//              of the ascending store), so the join is a rebased segmented copy
//   exposures  gathered in bucket order with their feature ids
// The store must list users in ascending id (the iteration order of the
// reference's std::map<int64_t, UserContext>); this is checked.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mtfm_cuda.h"
#include "common.cuh"

namespace mtfm {
namespace agg {

constexpr int kMaxScen = 1024;

// ---------------------------------------------------------------- scans
// Exclusive scan of n int64 values (in may alias out): per-block sums, one block
// scans the block sums, then every block scans its tile with its carry-in.
constexpr int kScanThreads = 512, kScanItems = 4, kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ long long block_exclusive_scan(long long v, long long* sh, long long& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        long long s = lane < (blockDim.x >> 5) ? sh[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        sh[lane] = s;  // inclusive warp totals
    }
    __syncthreads();
    total = sh[(blockDim.x >> 5) - 1];
    const long long before = w ? sh[w - 1] : 0;
    __syncthreads();
    return before + x - v;
}

template <typename T>
__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const T* __restrict__ in, long long n,
                                                                   long long* __restrict__ block_sums) {
    __shared__ long long sh[32];
    const long long base = static_cast<long long>(blockIdx.x) * kScanTile;
    long long s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const long long i = base + threadIdx.x * kScanItems + k;
        if (i < n) s += static_cast<long long>(in[i]);
    }
    long long total;
    block_exclusive_scan(s, sh, total);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads) scan_sums_kernel(long long* __restrict__ sums, long long nb,
                                                                 long long* __restrict__ grand) {
    __shared__ long long sh[32];
    long long carry = 0;
    for (long long b0 = 0; b0 < nb; b0 += kScanThreads) {
        const long long i = b0 + threadIdx.x;
        const long long v = i < nb ? sums[i] : 0;
        long long total;
        const long long ex = block_exclusive_scan(v, sh, total);
        if (i < nb) sums[i] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0) *grand = carry;
}

template <typename T, typename O>
__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(const T* in, long long n,
                                                                  const long long* __restrict__ block_off,
                                                                  long long add, O* out) {
    __shared__ long long sh[32];
    const long long base = static_cast<long long>(blockIdx.x) * kScanTile;
    long long v[kScanItems];
    long long s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const long long i = base + threadIdx.x * kScanItems + k;
        v[k] = i < n ? static_cast<long long>(in[i]) : 0;
        s += v[k];
    }
    long long total;
    long long run = block_exclusive_scan(s, sh, total) + block_off[blockIdx.x] + add;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const long long i = base + threadIdx.x * kScanItems + k;
        if (i < n) out[i] = static_cast<O>(run);
        run += v[k];
    }
}

// ---------------------------------------------------------------- kernels
// err: (stream index << 2) | code, code 1 unknown scenario, 2 unknown user; ~0 = none
__global__ void classify_kernel(const long long* __restrict__ uid, const int* __restrict__ scen, long long n,
                                const long long* __restrict__ store_uid, int n_store,
                                const int* __restrict__ scen_ids, int n_scen, int* __restrict__ bucket,
                                int* __restrict__ counts, unsigned long long* __restrict__ err) {
    __shared__ int s_ids[kMaxScen];
    for (int i = threadIdx.x; i < n_scen; i += blockDim.x) s_ids[i] = scen_ids[i];
    __syncthreads();
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n; x += (long long)gridDim.x * blockDim.x) {
        const int sc = scen[x];
        // scenario ids ascending (std::map order of the reference's per_scenario stage)
        int lo = 0, hi = n_scen;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (s_ids[mid] < sc) lo = mid + 1;
            else hi = mid;
        }
        if (lo >= n_scen || s_ids[lo] != sc) {
            atomicMin(err, (static_cast<unsigned long long>(x) << 2) | 1ull);
            bucket[x] = -1;
            continue;
        }
        const long long u = uid[x];
        int a = 0, b = n_store;
        while (a < b) {
            const int mid = (a + b) >> 1;
            if (store_uid[mid] < u) a = mid + 1;
            else b = mid;
        }
        if (a >= n_store || store_uid[a] != u) {
            atomicMin(err, (static_cast<unsigned long long>(x) << 2) | 2ull);
            bucket[x] = -1;
            continue;
        }
        const int bk = a * n_scen + lo;
        bucket[x] = bk;
        atomicAdd(counts + bk, 1);
    }
}

__global__ void store_order_kernel(const long long* __restrict__ store_uid, int n_store, int* __restrict__ bad) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x + 1; i < n_store; i += gridDim.x * blockDim.x)
        if (store_uid[i - 1] >= store_uid[i]) atomicMin(bad, i);
}

__global__ void scatter_kernel(const int* __restrict__ bucket, long long n, const long long* __restrict__ bucket_off,
                               int* __restrict__ cursor, int* __restrict__ slot) {
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n; x += (long long)gridDim.x * blockDim.x) {
        const int bk = bucket[x];
        slot[bucket_off[bk] + atomicAdd(cursor + bk, 1)] = static_cast<int>(x);
    }
}

// Ascending bitonic sort of a[0, n) by one thread block in the all-ascending
// formulation (per merge stage: a flip step i <-> i ^ (k - 1), then half-cleaners
// i <-> i ^ j): every compare-exchange puts the minimum at the lower index, so
// the virtual +inf padding past n never moves and pairs reaching past n are skipped.
__device__ void block_bitonic(int* a, int n) {
    int cap = 1;
    while (cap < n) cap <<= 1;
    for (int k = 2; k <= cap; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            const int mask = j == (k >> 1) ? k - 1 : j;  // flip at the stage's first step
            for (int i = threadIdx.x; i < cap; i += blockDim.x) {
                const int p = i ^ mask;
                if (p > i && p < n) {
                    const int ai = a[i], ap = a[p];
                    if (ai > ap) {
                        a[i] = ap;
                        a[p] = ai;
                    }
                }
            }
            __syncthreads();
        }
}

constexpr int kSmemSort = 4096;

// One block per bucket with > 1 element: restore stream order inside the bucket
// (in shared memory up to kSmemSort elements, else in place in global memory).
__global__ void bucket_sort_kernel(const long long* __restrict__ bucket_off, const int* __restrict__ counts,
                                   long long n_buckets, int* __restrict__ slot) {
    __shared__ int sh[kSmemSort];
    for (long long bk = blockIdx.x; bk < n_buckets; bk += gridDim.x) {
        const int n = counts[bk];
        if (n <= 1) continue;
        int* seg = slot + bucket_off[bk];
        if (n <= kSmemSort) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) sh[i] = seg[i];
            __syncthreads();
            block_bitonic(sh, n);
            for (int i = threadIdx.x; i < n; i += blockDim.x) seg[i] = sh[i];
            __syncthreads();
        } else {
            block_bitonic(seg, n);
        }
    }
}

// users: present[r] = store user r has >= 1 exposure
__global__ void present_kernel(const long long* __restrict__ bucket_off, int n_store, int n_scen,
                               int* __restrict__ present) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_store; r += gridDim.x * blockDim.x)
        present[r] = bucket_off[static_cast<long long>(r + 1) * n_scen] > bucket_off[static_cast<long long>(r) * n_scen];
}

struct StoreView {
    const long long* user_id;
    const int* seq_off;
    const uint8_t* seq_kind;
    const int* seq_schema;
    const int* ev_off;
    const long long* ev_ts;
    const int* ev_feat_off;
    const int* ev_feats;
};

// per output user: counts of sequences / events / event features / exposures
__global__ void user_counts_kernel(StoreView st, const int* __restrict__ present, const long long* __restrict__ uidx,
                                   int n_store, const long long* __restrict__ bucket_off, int n_scen,
                                   int* __restrict__ u_rank, long long* __restrict__ c_seq,
                                   long long* __restrict__ c_ev, long long* __restrict__ c_evf) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_store; r += gridDim.x * blockDim.x) {
        if (!present[r]) continue;
        const long long u = uidx[r];
        u_rank[u] = r;
        const int s0 = st.seq_off[r], s1 = st.seq_off[r + 1];
        c_seq[u] = s1 - s0;
        const int e0 = st.ev_off[s0], e1 = st.ev_off[s1];
        c_ev[u] = e1 - e0;
        c_evf[u] = st.ev_feat_off[e1] - st.ev_feat_off[e0];
    }
}

struct OutView {
    long long* user_id;
    int* seq_off;
    uint8_t* seq_kind;
    int* seq_schema;
    int* ev_off;
    long long* ev_ts;
    int* ev_feat_off;
    int* ev_feats;
    int* exp_off;
    int* exp_scenario;
    long long* exp_ts;
    int* exp_feat_off;
    int* exp_blk;
    int* exp_feats;
    int* exp_src;
};

// one block per output user: the user's store spans copied with rebased offsets
__global__ void join_kernel(StoreView st, OutView out, long long n_users, const int* __restrict__ u_rank,
                            const long long* __restrict__ o_seq, const long long* __restrict__ o_ev,
                            const long long* __restrict__ o_evf, const long long* __restrict__ bucket_off,
                            int n_scen) {
    for (long long u = blockIdx.x; u < n_users; u += gridDim.x) {
        const int r = u_rank[u];
        const int s0 = st.seq_off[r], s1 = st.seq_off[r + 1];
        const int e0 = st.ev_off[s0], e1 = st.ev_off[s1];
        const int f0 = st.ev_feat_off[e0], f1 = st.ev_feat_off[e1];
        const long long os = o_seq[u], oe = o_ev[u], of = o_evf[u];
        if (threadIdx.x == 0) {
            out.user_id[u] = st.user_id[r];
            out.exp_off[u] = static_cast<int>(bucket_off[static_cast<long long>(r) * n_scen]);
            out.seq_off[u] = static_cast<int>(os);
        }
        for (int q = threadIdx.x; q < s1 - s0; q += blockDim.x) {
            out.seq_kind[os + q] = st.seq_kind[s0 + q];
            out.seq_schema[os + q] = st.seq_schema[s0 + q];
            out.ev_off[os + q] = static_cast<int>(st.ev_off[s0 + q] - e0 + oe);
        }
        for (int e = threadIdx.x; e < e1 - e0; e += blockDim.x) {
            out.ev_ts[oe + e] = st.ev_ts[e0 + e];
            out.ev_feat_off[oe + e] = static_cast<int>(st.ev_feat_off[e0 + e] - f0 + of);
        }
        for (int f = threadIdx.x; f < f1 - f0; f += blockDim.x) out.ev_feats[of + f] = st.ev_feats[f0 + f];
    }
}

struct StreamView {
    const long long* uid;
    const int* scen;
    const long long* ts;
    const int* feat_off;
    const int* blk;
    const int* feats;
};

__global__ void exp_counts_kernel(StreamView sv, const int* __restrict__ slot, long long n, int* __restrict__ nfeat) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
        const int x = slot[j];
        nfeat[j] = sv.feat_off[x + 1] - sv.feat_off[x];
    }
}

// one warp per output exposure
__global__ void exp_gather_kernel(StreamView sv, OutView out, const int* __restrict__ slot, long long n) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long j = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); j < n; j += warps) {
        const int x = slot[j];
        if (lane == 0) {
            out.exp_src[j] = x;
            out.exp_scenario[j] = sv.scen[x];
            out.exp_ts[j] = sv.ts[x];
        }
        if (lane < 3) out.exp_blk[3 * j + lane] = sv.blk[3 * x + lane];
        const int f0 = sv.feat_off[x], nf = sv.feat_off[x + 1] - f0;
        const int o = out.exp_feat_off[j];
        for (int f = lane; f < nf; f += 32) out.exp_feats[o + f] = sv.feats[f0 + f];
    }
}

}  // namespace agg
}  // namespace mtfm

// ---------------------------------------------------------------- host
namespace {


}  // namespace
namespace mtfm {
void set_last_error(const std::string& what);  // model.cu (mtfm_cuda_last_error)
}
namespace {

struct AggFail : std::runtime_error {
    mtfm_status st;
    AggFail(mtfm_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw AggFail(MTFM_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DBuf {
    void* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    void alloc(size_t bytes) {
        if (p) cudaFree(p);
        p = nullptr;
        n = bytes;
        ck(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "cudaMalloc");
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

template <typename T>
void up(DBuf& d, const T* h, size_t n, cudaStream_t st) {
    d.alloc(n * sizeof(T));
    if (n) ck(cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice, st), "H2D");
}

// exclusive scan in[0, n) -> out[0, n] (out[n] = total); returns total
template <typename T, typename O>
long long exclusive_scan(const T* in, long long n, O* out, cudaStream_t st, DBuf& tmp) {
    using namespace mtfm::agg;
    const long long nb = std::max<long long>(1, mtfm::cdiv(n, kScanTile));
    tmp.alloc(static_cast<size_t>(nb + 1) * 8);
    long long* sums = tmp.as<long long>();
    if (n > 0) scan_reduce_kernel<T><<<static_cast<int>(nb), kScanThreads, 0, st>>>(in, n, sums);
    else ck(cudaMemsetAsync(sums, 0, 8, st), "memset");
    scan_sums_kernel<<<1, kScanThreads, 0, st>>>(sums, n > 0 ? nb : 0, sums + nb);
    if (n > 0) scan_apply_kernel<T, O><<<static_cast<int>(nb), kScanThreads, 0, st>>>(in, n, sums, 0, out);
    ck(cudaGetLastError(), "scan");
    long long total = 0;
    ck(cudaMemcpyAsync(&total, sums + nb, 8, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "scan sync");
    const O t = static_cast<O>(total);
    ck(cudaMemcpyAsync(out + n, &t, sizeof(O), cudaMemcpyHostToDevice, st), "H2D");
    ck(cudaStreamSynchronize(st), "scan sync");
    return total;
}

}  // namespace

struct mtfm_cuda_aggregate {
    int device = 0;
    long long n_users = 0, n_seqs = 0, n_events = 0, n_ev_feats = 0, n_exp = 0, n_exp_feats = 0;
    DBuf user_id, seq_off, seq_kind, seq_schema, ev_off, ev_ts, ev_feat_off, ev_feats, exp_off, exp_scenario, exp_ts,
        exp_feat_off, exp_blk, exp_feats, exp_src;
};

extern "C" {

mtfm_status mtfm_cuda_aggregate_users(int device, const int32_t* scenario_ids, int32_t n_scenarios,
                                      const mtfm_exposure_stream* sv, const mtfm_packed_batch* store,
                                      mtfm_cuda_aggregate** out, mtfm_aggregation_report* rep) {
    using namespace mtfm::agg;
    try {
        if (!sv || !store || !out || (n_scenarios > 0 && !scenario_ids)) throw AggFail(MTFM_CONTRACT_ERROR, "null argument");
        if (n_scenarios < 0 || n_scenarios > kMaxScen) throw AggFail(MTFM_CONFIG_ERROR, "aggregate: at most 1024 scenarios");
        for (int i = 1; i < n_scenarios; ++i)
            if (scenario_ids[i - 1] >= scenario_ids[i])
                throw AggFail(MTFM_CONTRACT_ERROR, "aggregate: scenario ids must be strictly ascending");
        if (sv->n_exposures < 0 || store->n_users < 0) throw AggFail(MTFM_DIMENSION_ERROR, "negative sizes");
        if (store->n_exposures != 0) throw AggFail(MTFM_CONTRACT_ERROR, "aggregate: the user store carries no exposures");
        ck(cudaSetDevice(device), "cudaSetDevice");
        cudaStream_t st;
        ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
        struct StreamGuard {
            cudaStream_t s;
            ~StreamGuard() { cudaStreamDestroy(s); }
        } sg{st};
        const long long n = sv->n_exposures;
        const int U = store->n_users, S = n_scenarios;
        // uploads: the stream and the store (store arrays keep their own offsets)
        DBuf s_uid, s_scen, s_ts, s_foff, s_blk, s_feats, scen_ids;
        up(s_uid, sv->user_id, n, st);
        up(s_scen, sv->scenario, n, st);
        up(s_ts, sv->ts, n, st);
        up(s_foff, sv->feat_off, n + 1, st);
        up(s_blk, sv->blk, 3 * n, st);
        up(s_feats, sv->feats, sv->n_feats, st);
        up(scen_ids, scenario_ids, S, st);
        DBuf t_uid, t_soff, t_kind, t_schema, t_eoff, t_ets, t_efoff, t_efeats;
        const int n_seqs = store->n_seqs;
        up(t_uid, store->user_id, U, st);
        up(t_soff, store->seq_off, U + 1, st);
        up(t_kind, store->seq_kind, n_seqs, st);
        up(t_schema, store->seq_schema, n_seqs, st);
        const int zero = 0;
        up(t_eoff, n_seqs ? store->ev_off : &zero, n_seqs ? n_seqs + 1 : 1, st);
        up(t_ets, store->ev_ts, store->n_events, st);
        up(t_efoff, store->ev_feat_off, store->n_events + 1, st);
        up(t_efeats, store->ev_feats, store->n_ev_feats, st);
        const int grid = 148 * 8;
        // store order (std::map iteration order)
        DBuf bad;
        bad.alloc(4);
        const int big = 0x7fffffff;
        ck(cudaMemcpyAsync(bad.p, &big, 4, cudaMemcpyHostToDevice, st), "H2D");
        if (U > 1) store_order_kernel<<<grid, 256, 0, st>>>(t_uid.as<long long>(), U, bad.as<int>());
        // classify
        const long long nbk = static_cast<long long>(U) * S;
        if (nbk >= (1ll << 31)) throw AggFail(MTFM_CONTRACT_ERROR, "aggregate: users x scenarios must stay below 2^31");
        DBuf bucket, counts, err;
        bucket.alloc(n * 4);
        counts.alloc(static_cast<size_t>(nbk + 1) * 4);
        ck(cudaMemsetAsync(counts.p, 0, static_cast<size_t>(nbk + 1) * 4, st), "memset");
        err.alloc(8);
        ck(cudaMemsetAsync(err.p, 0xff, 8, st), "memset");
        if (n > 0)
            classify_kernel<<<grid, 256, 0, st>>>(s_uid.as<long long>(), s_scen.as<int>(), n, t_uid.as<long long>(), U,
                                                  scen_ids.as<int>(), S, bucket.as<int>(), counts.as<int>(),
                                                  err.as<unsigned long long>());
        ck(cudaGetLastError(), "classify");
        int h_bad = 0;
        unsigned long long h_err = 0;
        ck(cudaMemcpyAsync(&h_bad, bad.p, 4, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(&h_err, err.p, 8, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "classify sync");
        if (h_bad != big)
            throw AggFail(MTFM_CONTRACT_ERROR, "aggregate: store users must be in strictly ascending user_id order (at index " +
                                                   std::to_string(h_bad) + ")");
        if (h_err != ~0ull) {
            const long long x = static_cast<long long>(h_err >> 2);
            if ((h_err & 3) == 1)
                throw AggFail(MTFM_INTEGRITY_ERROR,
                              "aggregate: exposure references unknown scenario " + std::to_string(sv->scenario[x]));
            throw AggFail(MTFM_INTEGRITY_ERROR, "aggregate: exposure references unknown user " + std::to_string(sv->user_id[x]));
        }
        // bucket offsets (users ascending, scenarios ascending), scatter, per-bucket stream order
        DBuf boff, tmp, cursor, slot;
        boff.alloc(static_cast<size_t>(nbk + 1) * 8);
        exclusive_scan(counts.as<int>(), nbk, boff.as<long long>(), st, tmp);
        cursor.alloc(static_cast<size_t>(std::max<long long>(nbk, 1)) * 4);
        ck(cudaMemsetAsync(cursor.p, 0, static_cast<size_t>(std::max<long long>(nbk, 1)) * 4, st), "memset");
        slot.alloc(n * 4);
        if (n > 0) {
            scatter_kernel<<<grid, 256, 0, st>>>(bucket.as<int>(), n, boff.as<long long>(), cursor.as<int>(), slot.as<int>());
            bucket_sort_kernel<<<grid, 256, 0, st>>>(boff.as<long long>(), counts.as<int>(), nbk, slot.as<int>());
        }
        ck(cudaGetLastError(), "scatter/sort");
        // users with exposures
        DBuf present, uidx;
        present.alloc(static_cast<size_t>(U) * 4);
        uidx.alloc(static_cast<size_t>(U + 1) * 8);
        if (U > 0) present_kernel<<<grid, 256, 0, st>>>(boff.as<long long>(), U, S, present.as<int>());
        const long long n_out = exclusive_scan(present.as<int>(), U, uidx.as<long long>(), st, tmp);
        auto A = std::make_unique<mtfm_cuda_aggregate>();
        A->device = device;
        A->n_users = n_out;
        A->n_exp = n;
        DBuf u_rank, c_seq, c_ev, c_evf, o_seq, o_ev, o_evf;
        u_rank.alloc(static_cast<size_t>(n_out) * 4);
        c_seq.alloc(static_cast<size_t>(n_out) * 8);
        c_ev.alloc(static_cast<size_t>(n_out) * 8);
        c_evf.alloc(static_cast<size_t>(n_out) * 8);
        StoreView sview{t_uid.as<long long>(), t_soff.as<int>(), t_kind.as<uint8_t>(), t_schema.as<int>(),
                        t_eoff.as<int>(), t_ets.as<long long>(), t_efoff.as<int>(), t_efeats.as<int>()};
        if (U > 0)
            user_counts_kernel<<<grid, 256, 0, st>>>(sview, present.as<int>(), uidx.as<long long>(), U,
                                                     boff.as<long long>(), S, u_rank.as<int>(), c_seq.as<long long>(),
                                                     c_ev.as<long long>(), c_evf.as<long long>());
        o_seq.alloc(static_cast<size_t>(n_out + 1) * 8);
        o_ev.alloc(static_cast<size_t>(n_out + 1) * 8);
        o_evf.alloc(static_cast<size_t>(n_out + 1) * 8);
        A->n_seqs = exclusive_scan(c_seq.as<long long>(), n_out, o_seq.as<long long>(), st, tmp);
        A->n_events = exclusive_scan(c_ev.as<long long>(), n_out, o_ev.as<long long>(), st, tmp);
        A->n_ev_feats = exclusive_scan(c_evf.as<long long>(), n_out, o_evf.as<long long>(), st, tmp);
        if (A->n_events >= (1ll << 31) || A->n_ev_feats >= (1ll << 31) || sv->n_feats >= (1ll << 31))
            throw AggFail(MTFM_CONTRACT_ERROR, "aggregate: a batch holds < 2^31 events / feature ids");
        // outputs
        A->user_id.alloc(n_out * 8);
        A->seq_off.alloc((n_out + 1) * 4);
        A->seq_kind.alloc(A->n_seqs);
        A->seq_schema.alloc(A->n_seqs * 4);
        A->ev_off.alloc((A->n_seqs + 1) * 4);
        A->ev_ts.alloc(A->n_events * 8);
        A->ev_feat_off.alloc((A->n_events + 1) * 4);
        A->ev_feats.alloc(A->n_ev_feats * 4);
        A->exp_off.alloc((n_out + 1) * 4);
        A->exp_scenario.alloc(n * 4);
        A->exp_ts.alloc(n * 8);
        A->exp_feat_off.alloc((n + 1) * 4);
        A->exp_blk.alloc(3 * n * 4);
        A->exp_src.alloc(n * 4);
        OutView ov{A->user_id.as<long long>(), A->seq_off.as<int>(), A->seq_kind.as<uint8_t>(), A->seq_schema.as<int>(),
                   A->ev_off.as<int>(), A->ev_ts.as<long long>(), A->ev_feat_off.as<int>(), A->ev_feats.as<int>(),
                   A->exp_off.as<int>(), A->exp_scenario.as<int>(), A->exp_ts.as<long long>(),
                   A->exp_feat_off.as<int>(), A->exp_blk.as<int>(), nullptr, A->exp_src.as<int>()};
        if (n_out > 0)
            join_kernel<<<static_cast<int>(std::min<long long>(n_out, 148 * 16)), 128, 0, st>>>(
                sview, ov, n_out, u_rank.as<int>(), o_seq.as<long long>(), o_ev.as<long long>(), o_evf.as<long long>(),
                boff.as<long long>(), S);
        ck(cudaGetLastError(), "join");
        // closing offsets
        const int iS = static_cast<int>(A->n_seqs), iE = static_cast<int>(A->n_events), iF = static_cast<int>(A->n_ev_feats),
                  iX = static_cast<int>(n);
        ck(cudaMemcpyAsync(A->seq_off.as<int>() + n_out, &iS, 4, cudaMemcpyHostToDevice, st), "H2D");
        ck(cudaMemcpyAsync(A->ev_off.as<int>() + A->n_seqs, &iE, 4, cudaMemcpyHostToDevice, st), "H2D");
        ck(cudaMemcpyAsync(A->ev_feat_off.as<int>() + A->n_events, &iF, 4, cudaMemcpyHostToDevice, st), "H2D");
        ck(cudaMemcpyAsync(A->exp_off.as<int>() + n_out, &iX, 4, cudaMemcpyHostToDevice, st), "H2D");
        // exposures in bucket order
        StreamView sw{s_uid.as<long long>(), s_scen.as<int>(), s_ts.as<long long>(), s_foff.as<int>(), s_blk.as<int>(),
                      s_feats.as<int>()};
        DBuf nfeat;
        nfeat.alloc(n * 4);
        if (n > 0) exp_counts_kernel<<<grid, 256, 0, st>>>(sw, slot.as<int>(), n, nfeat.as<int>());
        A->n_exp_feats = exclusive_scan(nfeat.as<int>(), n, A->exp_feat_off.as<int>(), st, tmp);
        A->exp_feats.alloc(A->n_exp_feats * 4);
        ov.exp_feats = A->exp_feats.as<int>();
        if (n > 0) exp_gather_kernel<<<grid, 256, 0, st>>>(sw, ov, slot.as<int>(), n);
        ck(cudaGetLastError(), "exposures");
        ck(cudaStreamSynchronize(st), "aggregate");
        if (rep) {
            rep->n_exposure_records = n;
            rep->n_user_samples = n_out;
            rep->compression_ratio = n_out ? static_cast<double>(n) / static_cast<double>(n_out) : 0.0;
        }
        *out = A.release();
        return MTFM_OK;
    } catch (const AggFail& e) {
        mtfm::set_last_error(e.what());
        return e.st;
    } catch (const std::exception& e) {
        mtfm::set_last_error(e.what());
        return MTFM_CONTRACT_ERROR;
    }
}

mtfm_status mtfm_cuda_aggregate_sizes(const mtfm_cuda_aggregate* a, mtfm_packed_sizes* s) {
    if (!a || !s) return MTFM_CONTRACT_ERROR;
    s->n_users = a->n_users;
    s->n_seqs = a->n_seqs;
    s->n_events = a->n_events;
    s->n_exposures = a->n_exp;
    s->n_ev_feats = a->n_ev_feats;
    s->n_exp_feats = a->n_exp_feats;
    return MTFM_OK;
}

mtfm_status mtfm_cuda_aggregate_fetch(mtfm_cuda_aggregate* a, const mtfm_packed_buffers* o) {
    try {
        if (!a || !o) throw AggFail(MTFM_CONTRACT_ERROR, "null argument");
        ck(cudaSetDevice(a->device), "cudaSetDevice");
        auto cp = [&](void* dst, const DBuf& src, long long bytes) {
            if (bytes > 0) {
                if (!dst) throw AggFail(MTFM_CONTRACT_ERROR, "null output array");
                ck(cudaMemcpy(dst, src.p, static_cast<size_t>(bytes), cudaMemcpyDeviceToHost), "D2H");
            }
        };
        cp(o->user_id, a->user_id, a->n_users * 8);
        cp(o->seq_off, a->seq_off, (a->n_users + 1) * 4);
        cp(o->seq_kind, a->seq_kind, a->n_seqs);
        cp(o->seq_schema, a->seq_schema, a->n_seqs * 4);
        cp(o->ev_off, a->ev_off, (a->n_seqs + 1) * 4);
        cp(o->ev_ts, a->ev_ts, a->n_events * 8);
        cp(o->ev_feat_off, a->ev_feat_off, (a->n_events + 1) * 4);
        cp(o->ev_feats, a->ev_feats, a->n_ev_feats * 4);
        cp(o->exp_off, a->exp_off, (a->n_users + 1) * 4);
        cp(o->exp_scenario, a->exp_scenario, a->n_exp * 4);
        cp(o->exp_ts, a->exp_ts, a->n_exp * 8);
        cp(o->exp_feat_off, a->exp_feat_off, (a->n_exp + 1) * 4);
        cp(o->exp_blk, a->exp_blk, a->n_exp * 12);
        cp(o->exp_feats, a->exp_feats, a->n_exp_feats * 4);
        if (o->exp_src) cp(o->exp_src, a->exp_src, a->n_exp * 4);
        return MTFM_OK;
    } catch (const AggFail& e) {
        mtfm::set_last_error(e.what());
        return e.st;
    }
}

mtfm_status mtfm_cuda_aggregate_free(mtfm_cuda_aggregate* a) {
    delete a;
    return MTFM_OK;
}

}  // extern "C"
