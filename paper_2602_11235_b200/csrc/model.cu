// model.cu — host side of libmtfm_cuda.so: the C ABI of include/mtfm_cuda.h.
//
// Owns the device weights (fp32 originals for the check mode, bf16 K-major
// copies for the tensor-core path), lays out each packed batch (row space =
// all context tokens of all users, then all T tokens; per-source tokenizer
// regions; attention tile tables), encodes the TMA descriptors and enqueues
// the forward (model.hpp:265-312 for every user at once):
//
//   plan -> gather -> tokenizer MLP (2 grouped GEMMs) -> per layer
//   [GLN1 -> projection GEMM(s) -> attention -> gate -> f2 GEMM (+residual)]
//   -> heads GEMM -> heads/records.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <tuple>
#include <string>
#include <vector>

#include "../../include/mtfm_cuda.h"
#include "attn_tc.cuh"
#include "common.cuh"
#include "gemm_sp.cuh"
#include "gemm_tc.cuh"
#include "heads_tc.cuh"
#include "kernels.cuh"
#include "tok_tc.cuh"
#include "train_kernels.cuh"

namespace mtfm {

// ---------------------------------------------------------------- errors
namespace {
thread_local std::string g_last_error;

struct Error : std::runtime_error {
    mtfm_status status;
    Error(mtfm_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] void fail(mtfm_status s, const std::string& m) { throw Error(s, m); }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(MTFM_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
mtfm_status guard(F&& f) {
    try {
        f();
        return MTFM_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return MTFM_CONTRACT_ERROR;
    }
}

// ---------------------------------------------------------------- TMA
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        ck(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q), "driver entry point");
        if (!p || q != cudaDriverEntryPointSuccess) fail(MTFM_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

// 2-D tensor map over a row-major [rows][cols] matrix with row stride ld (elements).
CUtensorMap tma_2d(const void* ptr, long long rows, long long cols, long long ld, int box_cols, int box_rows,
                   int swizzle_bytes, int elem_bytes = 2) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof(m));
    if (rows == 0) return m;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * elem_bytes)};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t es[2] = {1, 1};
    CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                            : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                            : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                  : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = encode_fn()(&m, elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                             2, const_cast<void*>(ptr), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(MTFM_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return m;
}

// k-block view of a row-major bf16 matrix with K % 64 == 0: dims {64, rows, K/64},
// box {64, box_rows, box_kb} -> box_kb SW128 [box_rows][64] tiles back to back in SMEM.
CUtensorMap tma_3d_kb(const void* ptr, long long rows, long long cols, long long ld, int box_rows, int box_kb) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof(m));
    if (rows == 0) return m;
    cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols / 64)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld * 2), 128};
    cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(box_kb)};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(MTFM_CUDA_ERROR, "cuTensorMapEncodeTiled (3D) failed (" + std::to_string(int(r)) + ")");
    return m;
}

// ---------------------------------------------------------------- device buffers
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void alloc(size_t n) {
        if (n <= bytes && p) return;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        if (n == 0) return;
        ck(cudaMalloc(&p, n), "cudaMalloc");
        bytes = n;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Forward activations live in one model-level arena shared by every prepared
// batch: forwards are serialised on the model stream, so only the inputs, the
// layout tables and the records are per batch (two batches in flight cost one
// set of activations). A batch records the bytes it needs; run_forward grows
// the arena (after draining the stream) when a bigger batch arrives.
enum ActId { ACT_X, ACT_XN, ACT_P, ACT_KV, ACT_UQ, ACT_A, ACT_GT, ACT_E, ACT_HID, ACT_Y, ACT_N };

// Page-locked host staging (grows, never shrinks): host-computed layout tables
// are written here and copied with truly asynchronous H2D transfers.
struct PinnedBuf {
    void* p = nullptr;
    size_t bytes = 0, used = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
    void reserve(size_t n) {
        if (n <= bytes) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
        ck(cudaMallocHost(&p, n), "cudaMallocHost");
        bytes = n;
    }
    // copy h into the staging area (16-byte aligned slot) and enqueue H2D into d
    template <typename T>
    void upload(DevBuf& d, const std::vector<T>& h, cudaStream_t st) {
        d.alloc(std::max<size_t>(h.size() * sizeof(T), 16));
        if (h.empty()) return;
        const size_t nb = h.size() * sizeof(T);
        if (used + nb > bytes) fail(MTFM_CONTRACT_ERROR, "pinned staging overflow");
        void* dst = static_cast<char*>(p) + used;
        std::memcpy(dst, h.data(), nb);
        used += (nb + 15) & ~size_t(15);
        ck(cudaMemcpyAsync(d.p, dst, nb, cudaMemcpyHostToDevice, st), "H2D");
    }
};

// Bias tiles for the tensor-core GEMM: bias_t[n] = (hi, lo, 0 x 14) in bf16 with
// hi + lo = bias[n] to ~2^-17, added by one K=16 MMA against a ones tile.
__global__ void bias_tile_kernel(const float* __restrict__ bias, int N, __nv_bfloat16* __restrict__ t) {
    MTFM_PDL_ENTRY();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N * 16) return;
    const int n = i >> 4, c = i & 15;
    const float b = bias[n];
    const __nv_bfloat16 hi = __float2bfloat16_rn(b);
    float v = 0.f;
    if (c == 0) v = __bfloat162float(hi);
    if (c == 1) v = b - __bfloat162float(hi);
    t[i] = c == 0 ? hi : __float2bfloat16_rn(v);
}

// 2:4-compressed forms of the pruned projection weights for gemm_sp.cuh, keyed by
// the K-major bf16 weight slice they are derived from (built on first use).
struct SparseForms {
    struct Form {
        DevBuf comp, meta;
        int Np = 0, KB = 0;
    };
    bool active = false;  // every projection weight is 2:4 along K: f1 / fuq / fkv / f2 run gemm_sp
    std::vector<std::pair<const char*, const char*>> ranges;  // the eligible bf16 weight buffers
    std::map<std::tuple<const void*, int, int>, std::unique_ptr<Form>> forms;
    void clear() {
        active = false;
        ranges.clear();
        forms.clear();
    }
    bool eligible(const void* w) const {
        const char* c = static_cast<const char*>(w);
        for (const auto& r : ranges)
            if (c >= r.first && c < r.second) return true;
        return false;
    }
    const Form& get(const __nv_bfloat16* w, long long ldw, int N, int K, cudaStream_t st) {
        auto& slot = forms[{w, N, K}];
        if (!slot) {
            slot = std::make_unique<Form>();
            slot->Np = static_cast<int>(round_up(N, 128));
            slot->KB = static_cast<int>(cdiv(K, 128));
            slot->comp.alloc(static_cast<size_t>(slot->Np) * slot->KB * 64 * 2);
            slot->meta.alloc(static_cast<size_t>(slot->Np / 128) * slot->KB * 512 * 4);
            DevBuf bad;
            bad.alloc(8);
            ck(cudaMemsetAsync(bad.p, 0, 8, st), "memset");
            const long long words = static_cast<long long>(slot->Np / 128) * slot->KB * 512;
            sp_compress_kernel<<<static_cast<int>(std::min<long long>(cdiv(words, 256), 4 * kNumSMs)), 256, 0, st>>>(
                w, ldw, N, K, slot->Np, slot->KB, slot->comp.as<__nv_bfloat16>(), slot->meta.as<uint32_t>(),
                bad.as<unsigned long long>());
            ck(cudaGetLastError(), "sparse compress");
            unsigned long long nb = 0;
            ck(cudaMemcpyAsync(&nb, bad.p, 8, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaStreamSynchronize(st), "sparse compress");
            if (nb) fail(MTFM_CONTRACT_ERROR, "projection weight is not 2:4 sparse along K");
        }
        return *slot;
    }
};

struct BiasTiles {
    std::map<std::pair<const float*, int>, std::unique_ptr<DevBuf>> tiles;
    SparseForms sparse;    // compressed projection weights (pruned models)
    bool rebuild = false;  // re-derive on every use (debug entry: caller-owned bias buffers)
    const __nv_bfloat16* get(const float* bias, int N, cudaStream_t st) {
        auto& slot = tiles[{bias, N}];
        if (!slot || rebuild) {
            if (!slot) slot = std::make_unique<DevBuf>();
            slot->alloc(static_cast<size_t>(N) * 16 * 2);
            bias_tile_kernel<<<static_cast<int>(cdiv(N * 16, 256)), 256, 0, st>>>(bias, N, slot->as<__nv_bfloat16>());
            ck(cudaGetLastError(), "bias tile");
        }
        return slot->as<__nv_bfloat16>();
    }
};

template <typename T>
void upload(DevBuf& d, const std::vector<T>& h, cudaStream_t st) {
    d.alloc(std::max<size_t>(h.size() * sizeof(T), 16));
    if (!h.empty()) ck(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st), "H2D");
}

template <typename T>
void upload_raw(DevBuf& d, const T* h, size_t n, cudaStream_t st) {
    d.alloc(std::max<size_t>(n * sizeof(T), 16));
    if (n) ck(cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice, st), "H2D");
}

uint16_t f2bf(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return static_cast<uint16_t>(u >> 16);
}

}  // namespace

// ---------------------------------------------------------------- model
struct ParamSpec {
    std::string name;
    long long rows, cols;
    std::vector<float> host;
    bool set = false;
    int owner = -1;  // names::owner_scenario (model.hpp:71-87): scenario owning it, -1 shared
};

// model.hpp:71-87: the first path component "s<digits>" or "t<digits>" names the
// owning scenario; everything else is shared (the subgraph extraction rule).
int owner_scenario(const std::string& name) {
    size_t pos = 0;
    while (pos < name.size()) {
        size_t end = name.find('/', pos);
        if (end == std::string::npos) end = name.size();
        if (end > pos + 1 && (name[pos] == 's' || name[pos] == 't')) {
            bool digits = true;
            for (size_t i = pos + 1; i < end; ++i) digits = digits && name[i] >= '0' && name[i] <= '9';
            if (digits) return std::stoi(name.substr(pos + 1, end - pos - 1));
        }
        pos = end + 1;
    }
    return -1;
}

struct LayerW {
    bool target;
    // fp32 originals ([in][out]) for check mode
    DevBuf w1, w2, b1, b2, wkv, bkv;  // full: w1=f1, b1=f1_b ; target: w1=fuq, wkv=fkv
    DevBuf f2, f2b;
    DevBuf g1g, g1b, g2g, g2b;        // [n_groups][d] / [n_groups][hd]
    // bf16 K-major ([out][in]) for the tensor-core path
    DevBuf t1, tkv, tf2;
    // GLN1 affine of each context source folded into the context-row projection
    // (bf16 [n_ctx][N][d] K-major, fp32 [n_ctx][N]): x~W + b = xhat (gain (.) W) + (bias W + b)
    // target: fkv (N = 2gd), full: f1 (N = 2hd + 2gd)
    DevBuf tfold, bfold;
};

struct SourceW {
    DevBuf w1, b1, w2, b2;  // fp32 [k_pad][2d] (zero rows past k_in), [2d][d]
    DevBuf t1, t2;          // bf16 [2d][k_pad], [d][2d]
};

// Where a registered parameter lives among the fp32 device weights:
// rows x cols at element `off` of `buf`, row stride `ld` (mtfm_cuda_get_param).
struct ParamView {
    DevBuf* buf = nullptr;
    long long off = 0, ld = 0;
};

// Training state (train_step.inc): one flat gradient buffer (one NCCL all-reduce),
// Adam moments in the same layout, saved activations of the last step.
struct TrainState {
    struct Seg {
        DevBuf* w;        // fp32 device weights
        long long n;      // elements
        long long off;    // offset in the flat gradient / moment buffers
    };
    std::vector<Seg> segs;
    long long n_total = 0;
    DevBuf grad, adam_m, adam_v, scratch;
    int64_t t = 0;        // Adam step count (params.hpp:87-119)
    std::vector<std::unique_ptr<DevBuf>> act;  // activation / gradient buffers, grown on demand
    size_t act_used = 0;
    float* grad_of(const DevBuf& w) const {
        for (const auto& s : segs)
            if (s.w == &w) return const_cast<float*>(grad.as<float>()) + s.off;
        return nullptr;
    }
};

}  // namespace mtfm

struct mtfm_cuda_model {
    int device = 0;
    int precision = 0;
    mtfm_model_desc cfg{};
    int d = 0, H = 0, G = 0, dh = 0, hd = 0, gd = 0, n_layers = 0;
    std::vector<mtfm::SourceInfo> sources;
    std::vector<mtfm::SlotInfo> slots;
    std::vector<std::string> slot_param;  // embedding param name per slot
    std::vector<std::vector<std::string>> tasks;  // per scenario source
    int n_hist = 0, n_rt = 0, n_scen = 0, n_tasks_total = 0;
    std::vector<mtfm::ParamSpec> params;
    std::map<std::string, size_t> by_name;
    // scenario subgraph (subgraph.hpp:25-42): >= 0 -> only the shared parameters and this
    // scenario's are registered; every forward is scoped to it
    int subgraph = -1;
    // 2:4 sparse tensor-core projections: 0 off, 1 required, 2 when the weights are 2:4
    int sparse_mode = 2;
    int max_run = 1;  // longest run of consecutive target layers (sizes the K|V buffer)
    std::vector<size_t> visible;  // registered parameters in registration order
    bool finalized = false;
    int n_ctx_src = 0;  // leading sources of kind hist/rt (context rows) when they precede every scenario source
    cudaStream_t stream = nullptr;       // kernels
    cudaStream_t copy_stream = nullptr;  // batch uploads (overlap the previous batch's kernels)
    cudaStream_t d2h_stream = nullptr;   // record read-back (does not queue behind the next batch)
    // device weights
    mtfm::DevBuf d_src, d_slots;
    mtfm::BiasTiles bias_tiles;  // GEMM bias tiles, built on first use
    std::vector<int> src_lookup;  // [kind][id < 4096] -> source, built on first prepare
    mtfm::DevBuf emb_f32, emb_bf16;
    std::vector<std::unique_ptr<mtfm::SourceW>> srcw;
    std::vector<std::unique_ptr<mtfm::LayerW>> layers;
    mtfm::DevBuf head_w, head_t, head_eb, head_gb, tower_w, tower_b;
    mtfm::DevBuf act[mtfm::ACT_N];  // forward activation arena shared by all batches
    int head_n = 0;
    int head_ld = 0;  // head_n rounded up to 8 (16-byte rows)
    mtfm_run_stats stats{};
    // per-stage profiling (CUDA events around every launch) — off by default
    bool profiling = false;
    struct Prof {
        std::string name;
        cudaEvent_t a = nullptr, b = nullptr;
        double flops = 0, bytes = 0, ms = 0;
    };
    std::vector<Prof> prof;
    size_t prof_n = 0;
    std::unique_ptr<mtfm_cuda_batch> ws;  // reusable workspace of mtfm_cuda_forward
    std::vector<mtfm::ParamView> views;    // per registered parameter (finalize)
    std::unique_ptr<mtfm::TrainState> train;  // reset when parameters are set again (weights re-uploaded)
    bool device_ahead = false;             // training updated the device weights past the host copies
    void* nccl = nullptr;                  // ncclComm_t of the data-parallel group (owned)
    int dp_ranks = 1, dp_rank = 0;
    ~mtfm_cuda_model();
};

struct mtfm_cuda_batch {
    mtfm_cuda_model* m = nullptr;
    int only_scenario = -1;
    long long n_users = 0, n_events = 0, n_exp = 0, rows = 0, n_records = 0;
    // batch arrays
    mtfm::DevBuf user_id, seq_off, seq_kind, seq_schema, ev_off, ev_ts, ev_feat_off, ev_feats, exp_off, exp_scen,
        exp_ts, exp_feat_off, exp_blk, exp_feats;
    // layout
    std::vector<long long> src_cnt, src_base, emb_base, hid_base;
    mtfm::DevBuf d_us_off, d_src_base, d_src_cnt, d_emb_base, d_rec_off;
    int sort_cap = 0;
    // plan sort areas of users above the SMEM capacity (global scratch); empty when none
    std::vector<long long> sort_off;
    mtfm::DevBuf d_sort_off, d_sort_scratch;
    // row meta
    mtfm::DevBuf r_src, r_item, r_prefix, r_scale, r_self, r_keybase, r_src_rows, t_user, t_exp_ref, t_scen, t_rec0,
        t_rec_stride, err;
    // activation bytes this batch needs in the model arena (mtfm_cuda_model::act)
    size_t act_bytes[mtfm::ACT_N] = {};
    // attention tiles
    long long n_tiles_full = 0, n_tiles_tgt = 0;
    mtfm::DevBuf d_tile_off;  // per-user first tile, full then target tables
    mtfm::DevBuf tiles_full, tiles_tgt;
    // records
    mtfm::DevBuf rec_user, rec_scen, rec_exp, rec_task, rec_logit, rec_prob;
    mtfm::DevBuf stat_buf;
    mtfm::PinnedBuf pin;  // staging of the host-computed layout tables + stats read-back
    cudaEvent_t ev_h2d = nullptr;   // uploads of the current contents done (copy stream)
    cudaEvent_t ev_done = nullptr;  // forward of the current contents done (kernel stream)
    bool ran = false;
    ~mtfm_cuda_batch() {
        if (ev_h2d) cudaEventDestroy(ev_h2d);
        if (ev_done) cudaEventDestroy(ev_done);
    }
    long long launches = 0;
    unsigned long long sum_c_ctx = 0, sum_c_t = 0;  // sum of visible keys (stats)
};

namespace mtfm {
namespace {

void register_params(mtfm_cuda_model& m) {
    auto add = [&](const std::string& n, long long r, long long c) {
        if (m.by_name.count(n)) fail(MTFM_CONFIG_ERROR, "duplicate parameter name: " + n);
        m.by_name[n] = m.params.size();
        m.params.push_back({n, r, c, {}, false, owner_scenario(n)});
    };
    const int d = m.d, hd = m.hd, gd = m.gd, de = m.cfg.d_emb;
    // model.hpp:377-463 registration order
    for (const auto& s : m.sources) {
        std::string base;
        if (s.kind == 0) base = "tok/h" + std::to_string(s.id);
        if (s.kind == 1) base = "tok/r" + std::to_string(s.id);
        if (s.kind == 2) base = "tok/s" + std::to_string(s.id);
        int slot = s.slot0;
        if (s.kind < 2) {
            for (int k = 0; k < s.nslot[0]; ++k, ++slot) {
                add(base + "/emb" + std::to_string(k), m.slots[slot].vocab, de);
                m.slot_param[slot] = base + "/emb" + std::to_string(k);
            }
        } else {
            const char* pre[3] = {"/emb_u", "/emb_c", "/emb_i"};
            for (int blk = 0; blk < 3; ++blk)
                for (int k = 0; k < s.nslot[blk]; ++k, ++slot) {
                    add(base + pre[blk] + std::to_string(k), m.slots[slot].vocab, de);
                    m.slot_param[slot] = base + pre[blk] + std::to_string(k);
                }
        }
        add(base + "/mlp_w1", s.k_in, 2 * d);
        add(base + "/mlp_b1", 1, 2 * d);
        add(base + "/mlp_w2", 2 * d, d);
        add(base + "/mlp_b2", 1, d);
    }
    const int n_groups = static_cast<int>(m.sources.size());
    for (int b = 0; b < m.cfg.blocks; ++b)
        for (int l = 0; l < m.cfg.target_layers + m.cfg.full_layers; ++l) {
            const bool tgt = l < m.cfg.target_layers;
            const std::string base = "hta/b" + std::to_string(b) + "/l" + std::to_string(l);
            if (tgt) {
                add(base + "/fuq_w", d, 2 * hd);
                add(base + "/fuq_b", 1, 2 * hd);
                add(base + "/fkv_w", d, 2 * gd);
                add(base + "/fkv_b", 1, 2 * gd);
            } else {
                add(base + "/f1_w", d, 2 * hd + 2 * gd);
                add(base + "/f1_b", 1, 2 * hd + 2 * gd);
            }
            add(base + "/f2_w", hd, d);
            add(base + "/f2_b", 1, d);
            for (int g = 0; g < n_groups; ++g) {
                const auto& s = m.sources[g];
                const std::string key = std::string(s.kind == 0 ? "h" : (s.kind == 1 ? "r" : "t")) + std::to_string(s.id);
                add(base + "/gln1/" + key + "/gain", 1, d);
                add(base + "/gln1/" + key + "/bias", 1, d);
                if (!tgt || s.kind == 2) {
                    add(base + "/gln2/" + key + "/gain", 1, hd);
                    add(base + "/gln2/" + key + "/bias", 1, hd);
                }
            }
        }
    for (int e = 0; e < m.cfg.experts; ++e) {
        add("head/expert" + std::to_string(e) + "_w", d, m.cfg.d_expert);
        add("head/expert" + std::to_string(e) + "_b", 1, m.cfg.d_expert);
    }
    for (const auto& s : m.sources) {
        if (s.kind != 2) continue;
        for (const auto& t : m.tasks[&s - m.sources.data()]) {
            const std::string base = "head/s" + std::to_string(s.id) + "/" + t;
            add(base + "/gate_w", d, m.cfg.experts);
            add(base + "/gate_b", 1, m.cfg.experts);
            add(base + "/tower_w", m.cfg.d_expert, 1);
            add(base + "/tower_b", 1, 1);
        }
    }
}

const std::vector<float>& P(mtfm_cuda_model& m, const std::string& n) {
    auto it = m.by_name.find(n);
    if (it == m.by_name.end()) fail(MTFM_CONFIG_ERROR, "unknown parameter: " + n);
    return m.params[it->second].host;
}

// [rows][cols] f32 -> bf16 [cols][kpad] (transposed, zero padded along k)
std::vector<uint16_t> to_kmajor_bf16(const std::vector<float>& w, long long rows, long long cols, long long kpad) {
    std::vector<uint16_t> t(static_cast<size_t>(cols * kpad), 0);
    for (long long r = 0; r < rows; ++r)
        for (long long c = 0; c < cols; ++c) t[c * kpad + r] = f2bf(w[r * cols + c]);
    return t;
}

// every hta/.../{f1_w, fuq_w, fkv_w, f2_w} ([K][N], K a multiple of 64) keeps at most two
// non-zeros in each group of 4 consecutive rows: the 2:4 pattern prune_2_4 leaves
bool projections_2_4(const mtfm_cuda_model& m) {
    bool any = false;
    for (const auto& p : m.params) {
        const std::string& n = p.name;
        if (n.rfind("hta/", 0) != 0) continue;
        const size_t sl = n.rfind('/');
        const std::string leaf = n.substr(sl + 1);
        if (leaf != "f1_w" && leaf != "fuq_w" && leaf != "fkv_w" && leaf != "f2_w") continue;
        any = true;
        const long long K = p.rows, N = p.cols;
        if (K % 64 != 0) return false;
        for (long long r0 = 0; r0 < K; r0 += 4)
            for (long long c = 0; c < N; ++c) {
                int nz = 0;
                for (int e = 0; e < 4; ++e) nz += p.host[(r0 + e) * N + c] != 0.f;
                if (nz > 2) return false;
            }
    }
    return any;
}

void finalize(mtfm_cuda_model& m) {
    if (m.finalized) return;
    // bias tiles are keyed by device pointer: rebuilt weights may reuse freed addresses
    m.bias_tiles.tiles.clear();
    m.bias_tiles.sparse.clear();
    for (auto& p : m.params) {
        if (m.subgraph >= 0 && p.owner >= 0 && p.owner != m.subgraph) {
            // not part of the subgraph: never bound (forwards are scoped to the subgraph scenario)
            p.host.assign(static_cast<size_t>(p.rows * p.cols), 0.f);
            p.set = true;
        }
        if (!p.set) fail(MTFM_CONFIG_ERROR, "parameter not set: " + p.name);
    }
    cudaStream_t st = m.stream;
    const int d = m.d, hd = m.hd, gd = m.gd;
    // embeddings: one flat table buffer
    std::vector<float> emb;
    for (size_t s = 0; s < m.slots.size(); ++s) {
        m.slots[s].emb_off = static_cast<long long>(emb.size());
        const auto& w = P(m, m.slot_param[s]);
        emb.insert(emb.end(), w.begin(), w.end());
        while (emb.size() % 8) emb.push_back(0.f);
    }
    upload(m.emb_f32, emb, st);
    std::vector<uint16_t> embh(emb.size());
    for (size_t i = 0; i < emb.size(); ++i) embh[i] = f2bf(emb[i]);
    upload(m.emb_bf16, embh, st);
    upload(m.d_slots, m.slots, st);
    // tokenizer MLPs
    for (const auto& s : m.sources) {
        auto w = std::make_unique<SourceW>();
        std::string base = s.kind == 0 ? "tok/h" : (s.kind == 1 ? "tok/r" : "tok/s");
        base += std::to_string(s.id);
        std::vector<float> w1 = P(m, base + "/mlp_w1");
        w1.resize(static_cast<size_t>(s.k_pad) * 2 * d, 0.f);  // zero rows past k_in
        upload(w->w1, w1, st);
        upload(w->b1, P(m, base + "/mlp_b1"), st);
        upload(w->w2, P(m, base + "/mlp_w2"), st);
        upload(w->b2, P(m, base + "/mlp_b2"), st);
        upload(w->t1, to_kmajor_bf16(P(m, base + "/mlp_w1"), s.k_in, 2 * d, s.k_pad), st);
        upload(w->t2, to_kmajor_bf16(P(m, base + "/mlp_w2"), 2 * d, d, 2 * d), st);
        m.srcw.push_back(std::move(w));
    }
    // stack
    const int n_groups = static_cast<int>(m.sources.size());
    for (int b = 0; b < m.cfg.blocks; ++b)
        for (int l = 0; l < m.cfg.target_layers + m.cfg.full_layers; ++l) {
            auto L = std::make_unique<LayerW>();
            L->target = l < m.cfg.target_layers;
            const std::string base = "hta/b" + std::to_string(b) + "/l" + std::to_string(l);
            if (L->target) {
                upload(L->w1, P(m, base + "/fuq_w"), st);
                upload(L->b1, P(m, base + "/fuq_b"), st);
                upload(L->wkv, P(m, base + "/fkv_w"), st);
                upload(L->bkv, P(m, base + "/fkv_b"), st);
                upload(L->t1, to_kmajor_bf16(P(m, base + "/fuq_w"), d, 2 * hd, d), st);
                upload(L->tkv, to_kmajor_bf16(P(m, base + "/fkv_w"), d, 2 * gd, d), st);
            } else {
                upload(L->w1, P(m, base + "/f1_w"), st);
                upload(L->b1, P(m, base + "/f1_b"), st);
                upload(L->t1, to_kmajor_bf16(P(m, base + "/f1_w"), d, 2 * hd + 2 * gd, d), st);
            }
            upload(L->f2, P(m, base + "/f2_w"), st);
            upload(L->f2b, P(m, base + "/f2_b"), st);
            upload(L->tf2, to_kmajor_bf16(P(m, base + "/f2_w"), hd, d, hd), st);
            std::vector<float> g1g, g1b, g2g, g2b;
            for (int g = 0; g < n_groups; ++g) {
                const auto& s = m.sources[g];
                const std::string key = std::string(s.kind == 0 ? "h" : (s.kind == 1 ? "r" : "t")) + std::to_string(s.id);
                const auto& a = P(m, base + "/gln1/" + key + "/gain");
                const auto& c = P(m, base + "/gln1/" + key + "/bias");
                g1g.insert(g1g.end(), a.begin(), a.end());
                g1b.insert(g1b.end(), c.begin(), c.end());
                if (!L->target || s.kind == 2) {
                    const auto& e = P(m, base + "/gln2/" + key + "/gain");
                    const auto& f = P(m, base + "/gln2/" + key + "/bias");
                    g2g.insert(g2g.end(), e.begin(), e.end());
                    g2b.insert(g2b.end(), f.begin(), f.end());
                } else {  // never read: target layers gate-normalise T rows only
                    g2g.insert(g2g.end(), hd, 1.f);
                    g2b.insert(g2b.end(), hd, 0.f);
                }
            }
            upload(L->g1g, g1g, st);
            upload(L->g1b, g1b, st);
            if (m.n_ctx_src > 0) {
                const auto& wf = P(m, base + (L->target ? "/fkv_w" : "/f1_w"));
                const auto& bf = P(m, base + (L->target ? "/fkv_b" : "/f1_b"));
                const int N = L->target ? 2 * gd : 2 * hd + 2 * gd;
                std::vector<uint16_t> tf(static_cast<size_t>(m.n_ctx_src) * N * d);
                std::vector<float> bb(static_cast<size_t>(m.n_ctx_src) * N);
                std::vector<double> acc(N);
                for (int g = 0; g < m.n_ctx_src; ++g) {
                    const float* ga = g1g.data() + static_cast<size_t>(g) * d;
                    const float* be = g1b.data() + static_cast<size_t>(g) * d;
                    for (int n = 0; n < N; ++n) acc[n] = bf[n];
                    for (int k = 0; k < d; ++k) {
                        const float* wr = wf.data() + static_cast<size_t>(k) * N;
                        uint16_t* tc = tf.data() + static_cast<size_t>(g) * N * d + k;
                        for (int n = 0; n < N; ++n) {
                            acc[n] += static_cast<double>(be[k]) * wr[n];
                            tc[static_cast<size_t>(n) * d] = f2bf(ga[k] * wr[n]);
                        }
                    }
                    for (int n = 0; n < N; ++n) bb[static_cast<size_t>(g) * N + n] = static_cast<float>(acc[n]);
                }
                upload(L->tfold, tf, st);
                upload(L->bfold, bb, st);
            }
            upload(L->g2g, g2g, st);
            upload(L->g2b, g2b, st);
            m.layers.push_back(std::move(L));
        }
    // longest run of consecutive target layers: the K|V buffer holds one layer of each
    // (with no full layers a run spans blocks)
    m.max_run = 1;
    for (size_t li = 0; li < m.layers.size();) {
        size_t lj = li;
        while (lj < m.layers.size() && m.layers[lj]->target) ++lj;
        m.max_run = std::max(m.max_run, static_cast<int>(lj - li));
        li = lj == li ? li + 1 : lj;
    }
    // pruned projections (prune.hpp:83-90) run on the sparse tensor cores
    if (m.sparse_mode != 0) {
        const bool ok = projections_2_4(m);
        if (!ok && m.sparse_mode == 1)
            fail(MTFM_CONTRACT_ERROR, "sparse MMA requested but the projection weights are not 2:4 along K");
        if (ok) {
            auto& sf = m.bias_tiles.sparse;
            sf.active = true;
            for (const auto& L : m.layers)
                for (const DevBuf* b : {&L->t1, &L->tkv, &L->tf2, &L->tfold})
                    if (b->p) sf.ranges.push_back({static_cast<const char*>(b->p), static_cast<const char*>(b->p) + b->bytes});
        }
    }
    // heads: [d][E*de | n_tasks*E]
    const int E = m.cfg.experts, dx = m.cfg.d_expert;
    m.head_n = E * dx + m.n_tasks_total * E;
    m.head_ld = static_cast<int>(round_up(m.head_n, 8));
    std::vector<float> hw(static_cast<size_t>(d) * m.head_n, 0.f), eb, gb, tw, tb;
    for (int e = 0; e < E; ++e) {
        const auto& w = P(m, "head/expert" + std::to_string(e) + "_w");
        for (int r = 0; r < d; ++r)
            for (int c = 0; c < dx; ++c) hw[static_cast<size_t>(r) * m.head_n + e * dx + c] = w[r * dx + c];
        const auto& b = P(m, "head/expert" + std::to_string(e) + "_b");
        eb.insert(eb.end(), b.begin(), b.end());
    }
    int task = 0;
    for (size_t si = 0; si < m.sources.size(); ++si) {
        const auto& s = m.sources[si];
        if (s.kind != 2) continue;
        for (const auto& t : m.tasks[si]) {
            const std::string base = "head/s" + std::to_string(s.id) + "/" + t;
            const auto& w = P(m, base + "/gate_w");
            for (int r = 0; r < d; ++r)
                for (int c = 0; c < E; ++c) hw[static_cast<size_t>(r) * m.head_n + E * dx + task * E + c] = w[r * E + c];
            const auto& b = P(m, base + "/gate_b");
            gb.insert(gb.end(), b.begin(), b.end());
            const auto& tw1 = P(m, base + "/tower_w");
            tw.insert(tw.end(), tw1.begin(), tw1.end());
            tb.push_back(P(m, base + "/tower_b")[0]);
            ++task;
        }
    }
    upload(m.head_w, hw, st);
    upload(m.head_t, to_kmajor_bf16(hw, d, m.head_n, d), st);
    upload(m.head_eb, eb, st);
    upload(m.head_gb, gb, st);
    upload(m.tower_w, tw, st);
    upload(m.tower_b, tb, st);
    upload(m.d_src, m.sources, st);
    ck(cudaStreamSynchronize(st), "weight upload");
    // parameter views into the fp32 device weights (registration order)
    m.views.assign(m.params.size(), ParamView{});
    auto view = [&](const std::string& n, DevBuf& b, long long off, long long ld) {
        auto it = m.by_name.find(n);
        if (it != m.by_name.end()) m.views[it->second] = ParamView{&b, off, ld};
    };
    for (size_t sl = 0; sl < m.slots.size(); ++sl) view(m.slot_param[sl], m.emb_f32, m.slots[sl].emb_off, m.cfg.d_emb);
    for (size_t si = 0; si < m.sources.size(); ++si) {
        const auto& src = m.sources[si];
        std::string base = src.kind == 0 ? "tok/h" : (src.kind == 1 ? "tok/r" : "tok/s");
        base += std::to_string(src.id);
        auto& w = *m.srcw[si];
        view(base + "/mlp_w1", w.w1, 0, 2 * d);
        view(base + "/mlp_b1", w.b1, 0, 2 * d);
        view(base + "/mlp_w2", w.w2, 0, d);
        view(base + "/mlp_b2", w.b2, 0, d);
    }
    for (int b = 0, li = 0; b < m.cfg.blocks; ++b)
        for (int l = 0; l < m.cfg.target_layers + m.cfg.full_layers; ++l, ++li) {
            auto& L = *m.layers[static_cast<size_t>(li)];
            const std::string base = "hta/b" + std::to_string(b) + "/l" + std::to_string(l);
            if (L.target) {
                view(base + "/fuq_w", L.w1, 0, 2 * hd);
                view(base + "/fuq_b", L.b1, 0, 2 * hd);
                view(base + "/fkv_w", L.wkv, 0, 2 * gd);
                view(base + "/fkv_b", L.bkv, 0, 2 * gd);
            } else {
                view(base + "/f1_w", L.w1, 0, 2 * hd + 2 * gd);
                view(base + "/f1_b", L.b1, 0, 2 * hd + 2 * gd);
            }
            view(base + "/f2_w", L.f2, 0, d);
            view(base + "/f2_b", L.f2b, 0, d);
            for (int g = 0; g < n_groups; ++g) {
                const auto& src = m.sources[static_cast<size_t>(g)];
                const std::string key = std::string(src.kind == 0 ? "h" : (src.kind == 1 ? "r" : "t")) + std::to_string(src.id);
                view(base + "/gln1/" + key + "/gain", L.g1g, static_cast<long long>(g) * d, d);
                view(base + "/gln1/" + key + "/bias", L.g1b, static_cast<long long>(g) * d, d);
                view(base + "/gln2/" + key + "/gain", L.g2g, static_cast<long long>(g) * hd, hd);
                view(base + "/gln2/" + key + "/bias", L.g2b, static_cast<long long>(g) * hd, hd);
            }
        }
    for (int e = 0; e < E; ++e) {
        view("head/expert" + std::to_string(e) + "_w", m.head_w, static_cast<long long>(e) * dx, m.head_n);
        view("head/expert" + std::to_string(e) + "_b", m.head_eb, static_cast<long long>(e) * dx, dx);
    }
    for (size_t si = 0, tg = 0; si < m.sources.size(); ++si) {
        const auto& src = m.sources[si];
        if (src.kind != 2) continue;
        for (const auto& t : m.tasks[si]) {
            const std::string base = "head/s" + std::to_string(src.id) + "/" + t;
            view(base + "/gate_w", m.head_w, static_cast<long long>(E) * dx + static_cast<long long>(tg) * E, m.head_n);
            view(base + "/gate_b", m.head_gb, static_cast<long long>(tg) * E, E);
            view(base + "/tower_w", m.tower_w, static_cast<long long>(tg) * dx, 1);
            view(base + "/tower_b", m.tower_b, static_cast<long long>(tg), 1);
            ++tg;
        }
    }
    m.finalized = true;
}

// ---------------------------------------------------------------- GEMM launch helpers

template <int BN>
int gemm_smem_bytes(const GemmArgs& a) {
    return 1024 + a.bres_bytes + 4096 + a.n_stages * a.stage_bytes + a.n_epi * a.stg_warp +
           gemm_detail::Cfg<BN>::BAR_BYTES;
}

template <int BN>
cudaLaunchConfig_t gemm_cluster_cfg(const GemmArgs& a, int grid, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(gemm_detail::Cfg<BN>::kThreads);
    cfg.dynamicSmemBytes = static_cast<size_t>(gemm_smem_bytes<BN>(a));
    cfg.stream = st;
    return cfg;
}

bool gemm_pairs_enabled() {
    static const bool on = std::getenv("MTFM_GEMM_PAIRS") == nullptr || std::atoi(std::getenv("MTFM_GEMM_PAIRS")) != 0;
    return on;
}

// co-resident CTAs of a pair launch (clusters of two never straddle a GPC)
template <int BN>
int gemm_pair_slots(const GemmArgs& a) {
    using C = gemm_detail::Cfg<BN>;
    static std::map<int, int> by_smem;  // occupancy depends only on the SMEM size
    const auto hit = by_smem.find(gemm_smem_bytes<BN>(a));
    if (hit != by_smem.end()) return hit->second;
    static bool attr = false;
    if (!attr) {
        ck(cudaFuncSetAttribute(gemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kMaxSmem),
           "gemm smem attr");
        attr = true;
    }
    cudaLaunchConfig_t cfg = gemm_cluster_cfg<BN>(a, kNumSMs, nullptr);
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeClusterDimension;
    la[0].val.clusterDim.x = 2;
    la[0].val.clusterDim.y = 1;
    la[0].val.clusterDim.z = 1;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    int n = 0;
    ck(cudaOccupancyMaxActiveClusters(&n, gemm_tc_kernel<BN>, &cfg), "gemm cluster occupancy");
    if (n < 1) fail(MTFM_CUDA_ERROR, "gemm clusters cannot be scheduled");
    by_smem[gemm_smem_bytes<BN>(a)] = 2 * n;
    return 2 * n;
}

template <int BN>
void launch_gemm_tc_bn(GemmArgs& a, int grid, cudaStream_t st) {
    using C = gemm_detail::Cfg<BN>;
    static bool attr = false;
    if (!attr) {
        ck(cudaFuncSetAttribute(gemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kMaxSmem),
           "gemm smem attr");
        attr = true;
    }
    const int smem = gemm_smem_bytes<BN>(a);
    if (smem > C::kMaxSmem) fail(MTFM_CONTRACT_ERROR, "gemm smem plan exceeds 227 KB");
    if (a.cl > 1) {
        cudaLaunchConfig_t cfg = gemm_cluster_cfg<BN>(a, grid, st);
        cudaLaunchAttribute la[2];
        la[0].id = cudaLaunchAttributeClusterDimension;
        la[0].val.clusterDim.x = static_cast<unsigned>(a.cl);
        la[0].val.clusterDim.y = 1;
        la[0].val.clusterDim.z = 1;
        la[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        la[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = la;
        cfg.numAttrs = 2;
        ck(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN>, a), "gemm_tc cluster launch");
        return;
    }
    launch_k(gemm_tc_kernel<BN>, dim3(grid), dim3(C::kThreads), smem, st, a);
    ck(cudaGetLastError(), "gemm_tc launch");
}

void launch_tok_fused(const TokArgs& a, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        ck(cudaFuncSetAttribute(tok_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tok_detail::SMEM),
           "tok smem attr");
        attr = true;
    }
    launch_k(tok_fused_kernel, dim3(std::min(a.n_tiles, kNumSMs)), dim3(kTokThreads), tok_detail::SMEM, st, a);
    ck(cudaGetLastError(), "tok_fused launch");
}

struct TcProblem {
    const __nv_bfloat16* A;
    long long lda;
    const __nv_bfloat16* Bt;  // [N][K]
    long long ldb;
    int M, N, K;
    int epi;
    const float* bias;
    void* out;
    long long ldo;
    const int* row_map;
    long long row_offset;
    const float* resid;
};

int pick_bn(const std::vector<TcProblem>& ps) {
    int best = 256;
    double best_eff = -1;
    for (int bn : {256, 128, 64}) {
        double used = 0, padded = 0;
        for (const auto& p : ps) {
            used += p.N;
            padded += static_cast<double>(cdiv(p.N, bn) * bn);
        }
        const double eff = used / std::max(padded, 1.0);
        if (eff > best_eff + 0.02) {
            best_eff = eff;
            best = bn;
        }
    }
    return best;
}

// B-resident plan (weights slice kept in SMEM, A streamed once per CTA group)
// when every problem's slice fits; otherwise the streaming schedule.
constexpr int kBresMax = 96 * 1024;

int pick_bn_resident(const std::vector<TcProblem>& ps) {
    int best = 0;
    double best_eff = -1;
    // a resident slice narrower than 128 columns makes N=64 MMAs (half the work per
    // instruction) and re-reads A per slice: measured 2-3x slower than streaming
    // B at BN=256 for K >= 512 (paper config projections), so it is not offered
    for (int bn : {256, 128}) {
        bool fits = true;
        double used = 0, padded = 0;
        for (const auto& p : ps) {
            fits = fits && round_up(p.K, 64) * bn * 2 <= kBresMax;
            used += p.N;
            padded += static_cast<double>(cdiv(p.N, bn) * bn);
        }
        if (!fits) continue;
        const double eff = used / std::max(padded, 1.0);
        if (eff > best_eff + 0.02) {
            best_eff = eff;
            best = bn;
        }
    }
    return best;
}

// Pruned projections on the sparse tensor cores (gemm_sp.cuh): same problems, the
// weight slice replaced by its compressed 2:4 form.
void run_gemm_sp(const std::vector<TcProblem>& ps, cudaStream_t st, long long& launches, SparseForms& sf) {
    static bool attr = false;
    if (!attr) {
        ck(cudaFuncSetAttribute(gemm_sp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sp_detail::SMEM),
           "sparse gemm smem attr");
        attr = true;
    }
    for (size_t i0 = 0; i0 < ps.size(); i0 += kMaxProblems) {
        const size_t i1 = std::min(ps.size(), i0 + kMaxProblems);
        SpArgs a;
        std::memset(&a, 0, sizeof(a));
        int tiles = 0;
        for (size_t i = i0; i < i1; ++i) {
            const TcProblem& s = ps[i];
            const SparseForms::Form& f = sf.get(s.Bt, s.ldb, s.N, s.K, st);
            SpProblem& p = a.p[a.n_problems++];
            p.tma_w = tma_2d(f.comp.p, f.Np, static_cast<long long>(f.KB) * 64, static_cast<long long>(f.KB) * 64, 64,
                             128, 128);
            p.tma_x = tma_2d(s.A, s.M, s.K, s.lda, 64, 128, 128);
            p.meta = f.meta.as<uint32_t>();
            p.M = s.M;
            p.N = s.N;
            p.K = s.K;
            p.kb = f.KB;
            p.tile_start = tiles;
            p.tiles_f = f.Np / 128;
            p.epi = s.epi;
            p.bias = s.bias;
            p.out = s.out;
            p.ldo = s.ldo;
            p.row_map = s.row_map;
            p.row_offset = s.row_offset;
            tiles += static_cast<int>(cdiv(s.M, 128)) * p.tiles_f;
        }
        a.n_tiles = tiles;
        launch_k(gemm_sp_kernel, dim3(std::min(tiles, kNumSMs)), dim3(sp_detail::kThreads), sp_detail::SMEM, st, a);
        ck(cudaGetLastError(), "gemm_sp launch");
        ++launches;
    }
}

void run_gemm_tc(std::vector<TcProblem> ps, cudaStream_t st, long long& launches, BiasTiles& bias_tiles) {
    ps.erase(std::remove_if(ps.begin(), ps.end(), [](const TcProblem& p) { return p.M == 0 || p.N == 0; }),
             ps.end());
    if (ps.empty()) return;
    if (bias_tiles.sparse.active &&
        std::all_of(ps.begin(), ps.end(), [&](const TcProblem& p) {
            // 16 B output vectors: N, ldo multiples of 8 and a 16 B aligned output
            return bias_tiles.sparse.eligible(p.Bt) && p.K % 64 == 0 && p.lda % 8 == 0 && p.N % 8 == 0 &&
                   p.ldo % 8 == 0 && reinterpret_cast<uintptr_t>(p.out) % 16 == 0 &&
                   (p.epi == EPI_SILU_BF16 || (p.epi == EPI_RESID_F32 && p.resid == p.out && !p.row_map));
        })) {
        run_gemm_sp(ps, st, launches, bias_tiles.sparse);
        return;
    }
    const int bn_res = pick_bn_resident(ps);
    for (size_t i0 = 0; i0 < ps.size(); i0 += kMaxProblems) {
        const size_t i1 = std::min(ps.size(), i0 + kMaxProblems);
        GemmArgs a;
        std::memset(&a, 0, sizeof(a));
        a.cl = 1;
        // ---- schedule
        int bn = bn_res;
        int grid = 0;
        if (bn) {
            // CTA rows per problem (a row = one CTA per n-slice, lockstep on an m-block so
            // A is read from HBM once): start at one row each, then repeatedly give a row to
            // the problem whose CTAs walk the most m-blocks while the SMs last (min-makespan
            // greedy; a proportional share rounded down leaves small problems' CTAs with ~2x
            // the m-blocks)
            std::vector<int> cpsv(i1 - i0, 1);
            int used = 0;
            for (size_t i = i0; i < i1; ++i) used += static_cast<int>(cdiv(ps[i].N, bn));
            for (;;) {
                int best = -1;
                long long best_load = 0;
                for (size_t i = i0; i < i1; ++i) {
                    const long long load = cdiv(cdiv(ps[i].M, 128), cpsv[i - i0]);
                    if (load > best_load) {
                        best_load = load;
                        best = static_cast<int>(i - i0);
                    }
                }
                const int ns = best < 0 ? 0 : static_cast<int>(cdiv(ps[i0 + best].N, bn));
                if (best < 0 || best_load <= 1 || used + ns > kNumSMs) break;
                ++cpsv[best];
                used += ns;
            }
            int n = 0;
            bool ok = true;
            for (size_t i = i0; i < i1 && ok; ++i) {
                const int ns = static_cast<int>(cdiv(ps[i].N, bn));
                const int mb = static_cast<int>(cdiv(ps[i].M, 128));
                const int cps = cpsv[i - i0];
                for (int j = 0; j < cps && ok; ++j)
                    for (int nb = 0; nb < ns; ++nb) {
                        if (n >= kNumSMs) {
                            ok = false;
                            break;
                        }
                        CtaWork& w = a.cta[n++];
                        w.pi = static_cast<short>(i - i0);
                        w.nb = static_cast<short>(nb);
                        w.m0 = j;
                        w.mstep = cps;
                        w.mcount = static_cast<int>(cdiv(mb - j, cps));
                    }
            }
            if (ok) {
                grid = n;
                a.b_res = 1;
            } else {
                std::memset(a.cta, 0, sizeof(a.cta));
                bn = 0;
            }
        }
        if (!bn) bn = pick_bn(std::vector<TcProblem>(ps.begin() + i0, ps.begin() + i1));
        int tiles = 0;
        int kmax = 0;
        // k-blocks per pipeline stage: 2 (one 3D TMA per operand per 2 k-blocks) when
        // every K is a multiple of 64, else 1
        int ks = 2;
        for (size_t i = i0; i < i1; ++i)
            if (ps[i].K % 64 != 0 || ps[i].K < 128) ks = 1;
        a.stage_kb = ks;
        for (size_t i = i0; i < i1; ++i) {
            const auto& s = ps[i];
            GemmProblem& p = a.p[a.n_problems++];
            p.tma_a = ks > 1 ? tma_3d_kb(s.A, s.M, s.K, s.lda, 128, ks) : tma_2d(s.A, s.M, s.K, s.lda, 64, 128, 128);
            // B: 2D boxes for the resident slice (loaded once per CTA), 3D per stage when streaming
            p.tma_b = (ks > 1 && !a.b_res) ? tma_3d_kb(s.Bt, s.N, s.K, s.ldb, bn, ks) : tma_2d(s.Bt, s.N, s.K, s.ldb, 64, bn, 128);
            p.M = s.M;
            p.N = s.N;
            p.K = static_cast<int>(round_up(s.K, 64));
            kmax = std::max(kmax, p.K);
            p.tile_start = tiles;
            p.tiles_n = static_cast<int>(cdiv(s.N, bn));
            p.epi = s.epi;
            p.has_bias = s.bias != nullptr;
            if (p.has_bias) p.tma_bias = tma_2d(bias_tiles.get(s.bias, s.N, st), s.N, 16, 16, 16, bn, 32);
            p.out = s.out;
            p.ldo = s.ldo;
            p.row_map = s.row_map;
            p.row_offset = s.row_offset;
            p.resid = s.resid;
            // bulk-tensor stores for plain row-major outputs (rows [row_offset, row_offset + M))
            const bool bf16_out = s.epi == EPI_SILU_BF16 || s.epi == EPI_BIAS_BF16;
            const int eb = bf16_out ? 2 : 4;
            const bool tma_ok = !s.row_map && (s.ldo * eb) % 16 == 0 && (reinterpret_cast<uintptr_t>(s.out) % 16) == 0;
            p.use_tma_c = tma_ok && (s.epi != EPI_RESID_F32 || s.resid == s.out);
            p.use_tma_r = p.use_tma_c && s.epi == EPI_RESID_F32;
            p.use_scatter_c = bf16_out && s.row_map && bn >= 64 && s.N % 64 == 0 && (s.ldo * 2) % 16 == 0 &&
                              (reinterpret_cast<uintptr_t>(s.out) % 16) == 0;
            if (p.use_tma_c) {
                // 32 rows x 128 B boxes: 64 bf16 columns or 32 fp32 columns (SW128)
                const char* base = static_cast<const char*>(s.out) + s.row_offset * s.ldo * eb;
                const bool wide = bf16_out && bn >= 64;
                p.tma_c = tma_2d(base, s.M, s.N, s.ldo, wide ? 64 : 32, 32, wide ? 128 : (bf16_out ? 64 : 128), eb);
            }
            tiles += static_cast<int>(cdiv(s.M, 128)) * p.tiles_n;
        }
        a.n_tiles = tiles;
        const int a_bytes = 128 * 64 * 2;
        const int b_bytes = bn * 64 * 2;
        // bf16 bulk-store epilogues (64-column units) need one 4 KB staging buffer per warp
        bool all_fast = true;
        for (int i = 0; i < a.n_problems; ++i) {
            const GemmProblem& p = a.p[i];
            all_fast = all_fast && (p.use_tma_c || p.use_scatter_c) && bn >= 64 &&
                       (p.epi == EPI_SILU_BF16 || p.epi == EPI_BIAS_BF16);
        }
        const int stg_warp = all_fast ? 4096 : 8192;
        a.stg_warp = stg_warp;
        if (!a.b_res) grid = std::min(tiles, kNumSMs);
        bool any_bias = false;
        for (int i = 0; i < a.n_problems; ++i) any_bias = any_bias || a.p[i].has_bias;
        a.bias_bytes = any_bias ? bn * 32 : 0;
        a.bres_bytes = a.b_res ? (kmax / 64) * b_bytes + a.bias_bytes : 0;
        a.stage_bytes = a.b_res ? ks * a_bytes : ks * (a_bytes + b_bytes) + a.bias_bytes;
        // 12 epilogue warps when >= 3 stages still fit (and there are 4 accumulators), else 8
        for (int ne : {12, 8, 0}) {
            if (ne == 0) {
                // nothing fits with multi-k-block stages: fall back to one k-block per stage
                if (a.stage_kb == 1) break;
                a.stage_kb = 1;
                for (int i = 0; i < a.n_problems; ++i) {
                    const auto& s = ps[i0 + i];
                    a.p[i].tma_a = tma_2d(s.A, s.M, s.K, s.lda, 64, 128, 128);
                    if (!a.b_res) a.p[i].tma_b = tma_2d(s.Bt, s.N, s.K, s.ldb, 64, bn, 128);
                }
                a.stage_bytes = a.b_res ? a_bytes : a_bytes + b_bytes + a.bias_bytes;
                ne = 8;
            }
            if (ne == 12 && bn >= 256) continue;  // epilogue groups <= accumulator buffers
            const int avail = 227 * 1024 - 1024 - gemm_detail::Cfg<128>::BAR_BYTES - 4096 - ne * stg_warp - a.bres_bytes;
            a.n_epi = ne;
            a.n_stages = std::min(8, avail / a.stage_bytes);
            if (a.n_stages >= 3) break;
        }
        if (a.n_stages < 2) fail(MTFM_CONTRACT_ERROR, "gemm pipeline does not fit in SMEM");
        // streamed BN = 256 GEMMs with more tiles than SMs: CTA pairs on m-block pairs load
        // half of each B k-block each and multicast it (L2 -> SMEM bytes per k-block 48 -> 32 KB)
        if (!a.b_res && bn == 256 && a.stage_kb == 1 && tiles > 2 * kNumSMs && gemm_pairs_enabled()) {
            int pt = 0;
            for (int i = 0; i < a.n_problems; ++i) {
                GemmProblem& p = a.p[i];
                const auto& s = ps[i0 + i];
                p.tile_start = pt;
                pt += static_cast<int>(cdiv(cdiv(p.M, 128), 2)) * p.tiles_n;
                p.tma_b = tma_2d(s.Bt, s.N, s.K, s.ldb, 64, bn / 2, 128);
            }
            a.n_tiles = pt;
            a.cl = 2;
            grid = std::min(2 * pt, gemm_pair_slots<256>(a));
        }
        if (bn == 256) launch_gemm_tc_bn<256>(a, grid, st);
        else if (bn == 128) launch_gemm_tc_bn<128>(a, grid, st);
        else launch_gemm_tc_bn<64>(a, grid, st);
        ++launches;
    }
}

void run_gemm_simt(std::vector<SimtGemm> ps, cudaStream_t st, long long& launches) {
    ps.erase(std::remove_if(ps.begin(), ps.end(), [](const SimtGemm& p) { return p.M == 0 || p.N == 0; }),
             ps.end());
    for (size_t i0 = 0; i0 < ps.size(); i0 += kMaxProblems) {
        launch_gemm_simt(ps.data() + i0, static_cast<int>(std::min<size_t>(kMaxProblems, ps.size() - i0)), st);
        ck(cudaGetLastError(), "gemm_simt launch");
        ++launches;
    }
}

// ---------------------------------------------------------------- attention helpers
// max mask prefix over each tile's rows, for the full-layer table (tiles [0, na)) and the
// target-layer table (tiles [na, na + nb)) in one launch
__global__ void tile_kmax_kernel(AttnTile* ta, int na, const int* pa, AttnTile* tb, int nb, const int* pb) {
    MTFM_PDL_ENTRY();
    int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (t >= na + nb) return;
    AttnTile* tiles = t < na ? ta : tb;
    const int* prefix = t < na ? pa : pb;
    if (t >= na) t -= na;
    AttnTile tl = tiles[t];
    int mx = 0;
    for (int i = lane; i < tl.n_rows; i += 32) mx = max(mx, prefix[tl.q_row0 + i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) tiles[t].kmax = mx;
}

struct AttnGeom {
    int hs, rt;
};

AttnGeom attn_geom(const mtfm_cuda_model& m) {
    const int r = m.H / m.G;
    if (r <= 128 && 128 % r == 0 && 128 / r >= 8) return {r, 128 / r};
    return {1, 128};
}

template <int D>
void launch_attn_tc_d(const AttnParams& p, cudaStream_t st) {
    using C = attn_detail::Cfg<D>;
    // the tensor maps' boxes must be the kernel's K/V tile and swizzle row
    if (p.tma_box_kv != C::BKV || p.tma_chunk != C::CHUNK) fail(MTFM_CONTRACT_ERROR, "attention tile config mismatch");
    static bool attr = false;
    if (!attr) {
        ck(cudaFuncSetAttribute(attn_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM),
           "attn smem attr");
        attr = true;
    }
    const int grid = std::min(p.n_tiles, kNumSMs);
    launch_k(attn_tc_kernel<D>, dim3(grid), dim3(C::kThreads), C::SMEM, st, p);
    ck(cudaGetLastError(), "attn_tc launch");
}

void run_attn_tc(const mtfm_cuda_model& m, AttnParams p, const __nv_bfloat16* q, long long n_q, long long q_cols,
                 long long kv_rows, long long kv_cols, cudaStream_t st) {
    if (p.n_tiles == 0) return;
    const int D = m.dh;
    const int chunk = std::min(D, 64);
    const int bkv = D <= 64 ? 128 : 64;  // attn_detail::Cfg<D>::BKV
    p.tma_box_kv = bkv;
    p.tma_chunk = chunk;
    p.tma_q = tma_2d(q, n_q, q_cols, p.ldq, chunk, p.rt, chunk * 2);
    p.tma_kv = tma_2d(p.kv_ptr, kv_rows, kv_cols, p.ldkv, chunk, bkv, chunk * 2);
    switch (D) {
        case 16: launch_attn_tc_d<16>(p, st); break;
        case 32: launch_attn_tc_d<32>(p, st); break;
        case 64: launch_attn_tc_d<64>(p, st); break;
        case 128: launch_attn_tc_d<128>(p, st); break;
        case 256: launch_attn_tc_d<256>(p, st); break;
        default: fail(MTFM_CONFIG_ERROR, "bf16 attention supports head_dim in {16,32,64,128,256}");
    }
}

// ---------------------------------------------------------------- batch layout
long long next_pow2(long long n) {
    long long p = 1;
    while (p < n) p <<= 1;
    return p;
}

int source_of_slow(const mtfm_cuda_model& m, int kind, int id, int only_scenario) {
    for (size_t s = 0; s < m.sources.size(); ++s)
        if (m.sources[s].kind == kind && m.sources[s].id == id) {
            if (kind == 2 && only_scenario >= 0 && id != only_scenario) return -1;
            return static_cast<int>(s);
        }
    return -1;
}

// Attention tile tables on the device: user u owns tiles [off[u], off[u+1]) of the
// full table (per head group: context query tiles then T query tiles) and the
// matching T tiles of the target table (same order as the host layout had).
__global__ void tile_expand_kernel(const long long* __restrict__ toff, const int* __restrict__ seq_off,
                                   const int* __restrict__ ev_off, const int* __restrict__ exp_off, int n_users,
                                   int n_seqs, long long n_events, int rt, int hs, int r, int G,
                                   AttnTile* __restrict__ tf, AttnTile* __restrict__ tt) {
    MTFM_PDL_ENTRY();
    const int u = blockIdx.x;
    if (u >= n_users) return;
    const long long ev0 = n_seqs ? ev_off[seq_off[u]] : 0, ev1 = n_seqs ? ev_off[seq_off[u + 1]] : 0;
    const long long x0 = exp_off[u], x1 = exp_off[u + 1];
    const int qc = static_cast<int>((ev1 - ev0 + rt - 1) / rt), qt = static_cast<int>((x1 - x0 + rt - 1) / rt);
    const int per_group = qc + qt;
    const int hpg = (r + hs - 1) / hs;
    const long long f0 = toff[u], t0 = toff[n_users + 1 + u];
    for (int i = threadIdx.x; i < G * hpg * per_group; i += blockDim.x) {
        const int grp = i / per_group, k = i - grp * per_group;
        const int g = grp / hpg, hb0 = (grp - g * hpg) * hs;
        const int head0 = g * r + hb0;
        if (k < qc) {
            const long long q = ev0 + static_cast<long long>(k) * rt;
            tf[f0 + i] = {static_cast<int>(q), static_cast<int>(min(static_cast<long long>(rt), ev1 - q)),
                          static_cast<int>(ev0), head0, 0, {0, 0, 0}};
        } else {
            const long long q = x0 + static_cast<long long>(k - qc) * rt;
            const int n = static_cast<int>(min(static_cast<long long>(rt), x1 - q));
            tf[f0 + i] = {static_cast<int>(n_events + q), n, static_cast<int>(ev0), head0, 0, {0, 0, 0}};
            tt[t0 + grp * qt + (k - qc)] = {static_cast<int>(q), n, static_cast<int>(ev0), head0, 0, {0, 0, 0}};
        }
    }
}

void launch_tile_expand(mtfm_cuda_batch& B, int rt, int hs, int r, int G, cudaStream_t st) {
    tile_expand_kernel<<<static_cast<int>(B.n_users), 128, 0, st>>>(
        B.d_tile_off.as<long long>(), B.seq_off.as<int>(), B.ev_off.as<int>(), B.exp_off.as<int>(),
        static_cast<int>(B.n_users), 1 /* ev_off always holds >= 1 entry */, B.n_events, rt, hs, r, G,
        B.tiles_full.as<AttnTile>(), B.tiles_tgt.as<AttnTile>());
    ck(cudaGetLastError(), "tile_expand launch");
}

// (kind, id) -> source through direct tables for ids in [0, 4096) (model-owned)
void build_source_lookup(mtfm_cuda_model& m) {
    m.src_lookup.assign(3 * 4096, -1);
    for (size_t s = 0; s < m.sources.size(); ++s) {
        const auto& si = m.sources[s];
        if (si.kind >= 0 && si.kind < 3 && si.id >= 0 && si.id < 4096 && m.src_lookup[si.kind * 4096 + si.id] < 0)
            m.src_lookup[si.kind * 4096 + si.id] = static_cast<int>(s);
    }
}
inline int source_of_fast(const mtfm_cuda_model& m, int kind, int id, int only_scenario) {
    if (id >= 0 && id < 4096) {
        if (kind == 2 && only_scenario >= 0 && id != only_scenario) return -1;
        return m.src_lookup[kind * 4096 + id];
    }
    return source_of_slow(m, kind, id, only_scenario);
}
int source_of(const mtfm_cuda_model& m, int kind, int id, int only_scenario) {
    return source_of_slow(m, kind, id, only_scenario);
}

void check_batch(const mtfm_packed_batch* b) {
    if (!b) fail(MTFM_CONTRACT_ERROR, "null batch");
    if (b->n_users < 0 || b->n_seqs < 0 || b->n_events < 0 || b->n_exposures < 0)
        fail(MTFM_DIMENSION_ERROR, "negative batch sizes");
    if (b->n_users > 0 && (!b->seq_off || !b->exp_off || !b->user_id)) fail(MTFM_CONTRACT_ERROR, "null batch arrays");
    if (b->seq_off && b->seq_off[b->n_users] != b->n_seqs) fail(MTFM_DIMENSION_ERROR, "seq_off does not end at n_seqs");
    if (b->exp_off && b->exp_off[b->n_users] != b->n_exposures)
        fail(MTFM_DIMENSION_ERROR, "exp_off does not end at n_exposures");
    if (b->n_seqs && b->ev_off[b->n_seqs] != b->n_events) fail(MTFM_DIMENSION_ERROR, "ev_off does not end at n_events");
    for (int u = 0; u < b->n_users; ++u)
        if (b->seq_off[u + 1] < b->seq_off[u] || b->exp_off[u + 1] < b->exp_off[u])
            fail(MTFM_DIMENSION_ERROR, "batch offsets not monotone");
}

void prepare(mtfm_cuda_model& m, const mtfm_packed_batch* hb, int only_scenario, mtfm_cuda_batch& B) {
    check_batch(hb);
    if (m.subgraph >= 0) {
        // infer_request (subgraph.hpp:51-55): a subgraph only scores its own scenario
        if (only_scenario >= 0 && only_scenario != m.subgraph)
            fail(MTFM_INTEGRITY_ERROR, "request scenario " + std::to_string(only_scenario) +
                                           " does not match subgraph scenario " + std::to_string(m.subgraph));
        only_scenario = m.subgraph;
    }
    finalize(m);
    // uploads go on the copy stream, after the previous forward of this batch object
    // (its device buffers are overwritten) and after the weights
    cudaStream_t st = m.copy_stream;
    if (!B.ev_h2d) ck(cudaEventCreateWithFlags(&B.ev_h2d, cudaEventDisableTiming), "event");
    if (!B.ev_done) ck(cudaEventCreateWithFlags(&B.ev_done, cudaEventDisableTiming), "event");
    if (B.ran) ck(cudaStreamWaitEvent(st, B.ev_done, 0), "wait previous forward");
    B.m = &m;
    B.only_scenario = only_scenario;
    B.n_users = hb->n_users;
    B.n_events = hb->n_events;
    B.n_exp = hb->n_exposures;
    B.rows = B.n_events + B.n_exp;
    const int n_src = static_cast<int>(m.sources.size());
    // upload the batch
    upload_raw(B.user_id, hb->user_id, hb->n_users, st);
    upload_raw(B.seq_off, hb->seq_off, hb->n_users + 1, st);
    upload_raw(B.seq_kind, hb->seq_kind, hb->n_seqs, st);
    upload_raw(B.seq_schema, hb->seq_schema, hb->n_seqs, st);
    upload_raw(B.ev_off, hb->n_seqs ? hb->ev_off : nullptr, hb->n_seqs ? hb->n_seqs + 1 : 0, st);
    if (!hb->n_seqs) {
        const int zero = 0;
        upload_raw(B.ev_off, &zero, 1, st);
    }
    upload_raw(B.ev_ts, hb->ev_ts, hb->n_events, st);
    upload_raw(B.ev_feat_off, hb->ev_feat_off, hb->n_events + 1, st);
    upload_raw(B.ev_feats, hb->ev_feats, hb->n_ev_feats, st);
    upload_raw(B.exp_off, hb->exp_off, hb->n_users + 1, st);
    upload_raw(B.exp_scen, hb->exp_scenario, hb->n_exposures, st);
    upload_raw(B.exp_ts, hb->exp_ts, hb->n_exposures, st);
    upload_raw(B.exp_feat_off, hb->exp_feat_off, hb->n_exposures + 1, st);
    upload_raw(B.exp_blk, hb->exp_blk, 3ll * hb->n_exposures, st);
    upload_raw(B.exp_feats, hb->exp_feats, hb->n_exp_feats, st);

    // host layout: per (user, source) counts -> source regions, record offsets
    std::vector<long long> us(static_cast<size_t>(B.n_users) * n_src, 0);
    std::vector<long long> rec_off(B.n_users + 1, 0);
    // plan sort area per user: max(pow2(n_ev), pow2(n_t) + n_ev) elements of (key, payload);
    // SMEM up to kPlanSmemCap, larger users sort in a global scratch slice
    constexpr long long kPlanSmemCap = 12288;
    long long max_sort = 1;
    std::vector<long long> sort_need(hb->n_users, 1);
    if (m.src_lookup.empty()) build_source_lookup(m);
    for (int u = 0; u < hb->n_users; ++u) {
        long long n_ev = 0;
        for (int s = hb->seq_off[u]; s < hb->seq_off[u + 1]; ++s) {
            const int src = source_of_fast(m, hb->seq_kind[s] ? 1 : 0, hb->seq_schema[s], -1);
            const long long len = hb->ev_off[s + 1] - hb->ev_off[s];
            n_ev += len;
            if (src >= 0) us[static_cast<size_t>(u) * n_src + src] += len;
        }
        long long recs = 0;
        for (int x = hb->exp_off[u]; x < hb->exp_off[u + 1]; ++x) {
            const int src = source_of_fast(m, 2, hb->exp_scenario[x], only_scenario);
            if (src >= 0) {
                us[static_cast<size_t>(u) * n_src + src] += 1;
                recs += m.sources[src].ntasks;
            }
        }
        rec_off[u + 1] = rec_off[u] + recs;
        const long long n_t = hb->exp_off[u + 1] - hb->exp_off[u];
        sort_need[u] = std::max(next_pow2(n_ev), next_pow2(n_t) + n_ev);
        if (sort_need[u] <= kPlanSmemCap) max_sort = std::max(max_sort, sort_need[u]);
    }
    B.n_records = rec_off[B.n_users];
    B.sort_cap = static_cast<int>(max_sort);
    B.sort_off.clear();
    for (int u = 0; u < hb->n_users; ++u)
        if (sort_need[u] > kPlanSmemCap) {
            B.sort_off.assign(hb->n_users + 1, 0);
            for (int v = 0; v < hb->n_users; ++v)
                B.sort_off[v + 1] = B.sort_off[v] + (sort_need[v] > kPlanSmemCap ? 2 * sort_need[v] : 0);
            B.d_sort_scratch.alloc(static_cast<size_t>(B.sort_off.back()) * sizeof(long long));
            break;
        }
    B.src_cnt.assign(n_src, 0);
    B.src_base.assign(n_src, 0);
    B.emb_base.assign(n_src, 0);
    B.hid_base.assign(n_src, 0);
    std::vector<long long> us_off(us.size(), 0);
    for (int s = 0; s < n_src; ++s)
        for (int u = 0; u < hb->n_users; ++u) {
            us_off[static_cast<size_t>(u) * n_src + s] = B.src_cnt[s];
            B.src_cnt[s] += us[static_cast<size_t>(u) * n_src + s];
        }
    long long pos = 0, eb = 0, hbse = 0;
    for (int s = 0; s < n_src; ++s) {
        B.src_base[s] = pos;
        B.emb_base[s] = eb;
        B.hid_base[s] = hbse;
        pos += B.src_cnt[s];
        eb += B.src_cnt[s] * m.sources[s].k_pad;
        hbse += B.src_cnt[s] * 2 * m.d;
    }
    // (the previous forward on this batch has completed: results() synchronised)
    // tile tables: per user and head group ceil(n/rt) query tiles, at most (n + rt - 1) / rt each
    const AttnGeom ag0 = attn_geom(m);
    const size_t hg0 = static_cast<size_t>(m.G) * ((m.H / m.G + ag0.hs - 1) / ag0.hs);
    const size_t tiles_est = hg0 * (static_cast<size_t>(B.n_events + 2 * B.n_exp) / ag0.rt + 3 * B.n_users) + 64;
    B.pin.reserve((us_off.size() + 4 * static_cast<size_t>(n_src) + rec_off.size() + B.sort_off.size()) * 8 +
                  tiles_est * sizeof(AttnTile) + 4096);
    B.pin.used = 64;  // first 64 bytes: stats read-back
    B.pin.upload(B.d_us_off, us_off, st);
    B.pin.upload(B.d_src_base, B.src_base, st);
    B.pin.upload(B.d_src_cnt, B.src_cnt, st);
    B.pin.upload(B.d_emb_base, B.emb_base, st);
    B.pin.upload(B.d_rec_off, rec_off, st);
    if (!B.sort_off.empty()) B.pin.upload(B.d_sort_off, B.sort_off, st);

    // attention tiles
    const AttnGeom ag = attn_geom(m);
    const int r = m.H / m.G;
    // count, then write straight into the pinned staging area (one H2D per table)
    const int hgroups = m.G * ((r + ag.hs - 1) / ag.hs);
    long long nf = 0, nt = 0;
    for (int u = 0; u < hb->n_users; ++u) {
        const long long ev0 = hb->n_seqs ? hb->ev_off[hb->seq_off[u]] : 0;
        const long long ev1 = hb->n_seqs ? hb->ev_off[hb->seq_off[u + 1]] : 0;
        const long long tq = cdiv(hb->exp_off[u + 1] - hb->exp_off[u], ag.rt);
        nf += hgroups * (cdiv(ev1 - ev0, ag.rt) + tq);
        nt += hgroups * tq;
    }
    B.n_tiles_full = nf;
    B.n_tiles_tgt = nt;
    // per-user tile offsets go to the device; tile_expand_kernel writes the tables
    std::vector<long long> toff(static_cast<size_t>(2 * (B.n_users + 1)), 0);  // [full offsets | target offsets]
    for (int u = 0; u < hb->n_users; ++u) {
        const long long ev0 = hb->n_seqs ? hb->ev_off[hb->seq_off[u]] : 0;
        const long long ev1 = hb->n_seqs ? hb->ev_off[hb->seq_off[u + 1]] : 0;
        const long long tq = cdiv(hb->exp_off[u + 1] - hb->exp_off[u], ag.rt);
        toff[u + 1] = toff[u] + hgroups * (cdiv(ev1 - ev0, ag.rt) + tq);
        toff[B.n_users + 1 + u + 1] = toff[B.n_users + 1 + u] + hgroups * tq;
    }
    B.pin.upload(B.d_tile_off, toff, st);
    B.tiles_full.alloc(std::max<size_t>(static_cast<size_t>(nf) * sizeof(AttnTile), 16));
    B.tiles_tgt.alloc(std::max<size_t>(static_cast<size_t>(nt) * sizeof(AttnTile), 16));
    if (B.n_users > 0)
        launch_tile_expand(B, ag.rt, ag.hs, r, m.G, st);
    // row meta + activations
    const long long R = B.rows, T = B.n_exp;
    auto ia = [&](DevBuf& b, long long n, size_t el) { b.alloc(std::max<size_t>(static_cast<size_t>(n) * el, 16)); };
    ia(B.r_src, R, 4);
    ia(B.r_item, R, 4);
    ia(B.r_prefix, R, 4);
    ia(B.r_scale, R, 4);
    ia(B.r_self, R, 4);
    ia(B.r_keybase, R, 4);
    ia(B.r_src_rows, R, 4);
    ia(B.t_user, T, 4);
    ia(B.t_exp_ref, T, 4);
    ia(B.t_scen, T, 4);
    ia(B.t_rec0, T, 8);
    ia(B.t_rec_stride, T, 4);
    ia(B.err, 1, 8);
    const size_t el = m.precision == MTFM_PRECISION_BF16 ? 2 : 4;
    const int pw = 2 * m.hd + 2 * m.gd;
    auto need = [&](int id, long long n, size_t e) { B.act_bytes[id] = std::max<size_t>(static_cast<size_t>(n) * e, 16); };
    need(ACT_X, R * m.d, 4);
    // bf16 path: [0, R) xhat of the context rows (source order) then the T rows' GLN1,
    // [R, 2R) a full layer's GLN1 rows; K|V rows per target layer of a run
    const long long kt = std::max(1, m.max_run);
    need(ACT_XN, 2 * R * m.d, el);
    need(ACT_P, R * pw, el);
    need(ACT_KV, kt * R * 2 * m.gd, el);
    need(ACT_UQ, T * 2 * m.hd, el);
    need(ACT_A, R * m.hd, el);
    need(ACT_GT, R * m.hd, el);
    need(ACT_E, eb, el);
    need(ACT_HID, hbse, el);
    need(ACT_Y, T * m.head_ld, 4);
    const long long nr = B.n_records;
    ia(B.rec_user, nr, 8);
    ia(B.rec_scen, nr, 4);
    ia(B.rec_exp, nr, 4);
    ia(B.rec_task, nr, 4);
    ia(B.rec_logit, nr, 4);
    ia(B.rec_prob, nr, 8);
    // every upload of this batch is enqueued: the host arrays may be released once they
    // have been read (the kernels of the previous batch keep running meanwhile)
    ck(cudaEventRecord(B.ev_h2d, st), "record h2d");
    ck(cudaEventSynchronize(B.ev_h2d), "h2d");
}

DevBatch dev_batch(const mtfm_cuda_batch& B) {
    DevBatch b;
    b.n_users = static_cast<int>(B.n_users);
    b.n_seqs = 0;
    b.n_events = static_cast<int>(B.n_events);
    b.n_exposures = static_cast<int>(B.n_exp);
    b.user_id = B.user_id.as<long long>();
    b.seq_off = B.seq_off.as<int>();
    b.seq_kind = B.seq_kind.as<uint8_t>();
    b.seq_schema = B.seq_schema.as<int>();
    b.ev_off = B.ev_off.as<int>();
    b.ev_ts = B.ev_ts.as<long long>();
    b.ev_feat_off = B.ev_feat_off.as<int>();
    b.ev_feats = B.ev_feats.as<int>();
    b.exp_off = B.exp_off.as<int>();
    b.exp_scenario = B.exp_scen.as<int>();
    b.exp_ts = B.exp_ts.as<long long>();
    b.exp_feat_off = B.exp_feat_off.as<int>();
    b.exp_blk = B.exp_blk.as<int>();
    b.exp_feats = B.exp_feats.as<int>();
    return b;
}

RowMeta row_meta(const mtfm_cuda_batch& B) {
    RowMeta r;
    r.src = B.r_src.as<int>();
    r.item = B.r_item.as<int>();
    r.prefix = B.r_prefix.as<int>();
    r.scale = B.r_scale.as<float>();
    r.self = B.r_self.as<int>();
    r.keybase = B.r_keybase.as<int>();
    r.src_rows = B.r_src_rows.as<int>();
    r.t_user = B.t_user.as<int>();
    r.t_exp_ref = B.t_exp_ref.as<int>();
    r.t_scen = B.t_scen.as<int>();
    r.t_rec0 = B.t_rec0.as<long long>();
    r.t_rec_stride = B.t_rec_stride.as<int>();
    return r;
}

// ---------------------------------------------------------------- profiling
struct StageScope {
    mtfm_cuda_model& m;
    bool on;
    size_t idx = 0;
    StageScope(mtfm_cuda_model& mm, const char* name, double flops, double bytes) : m(mm), on(mm.profiling) {
        if (!on) return;
        if (m.prof_n == m.prof.size()) {
            m.prof.emplace_back();
            ck(cudaEventCreate(&m.prof.back().a), "event");
            ck(cudaEventCreate(&m.prof.back().b), "event");
        }
        idx = m.prof_n++;
        auto& e = m.prof[idx];
        e.name = name;
        e.flops = flops;
        e.bytes = bytes;
        ck(cudaEventRecord(e.a, m.stream), "event record");
    }
    ~StageScope() {
        if (on) cudaEventRecord(m.prof[idx].b, m.stream);
    }
};

// ---------------------------------------------------------------- the forward
template <typename T>
void run_forward(mtfm_cuda_model& m, mtfm_cuda_batch& B) {
    BiasTiles& BT = m.bias_tiles;
    constexpr bool kTc = std::is_same<T, __nv_bfloat16>::value;
    constexpr double el = sizeof(T);
    cudaStream_t st = m.stream;
    long long& L = B.launches;
    L = 0;
    m.prof_n = 0;
    const int n_src = static_cast<int>(m.sources.size());
    const int d = m.d, hd = m.hd, gd = m.gd, dh = m.dh;
    const int pw = 2 * hd + 2 * gd;
    const long long R = B.rows, NE = B.n_events, NT = B.n_exp;
    const double Rd = static_cast<double>(R), Td = static_cast<double>(NT);
    const float eps = static_cast<float>(m.cfg.eps);
    if (B.n_users == 0) return;
    {
        bool grow = false;
        for (int i = 0; i < ACT_N; ++i) grow |= B.act_bytes[i] > m.act[i].bytes;
        if (grow) {  // earlier forwards may still read the arena
            ck(cudaStreamSynchronize(st), "arena sync");
            for (int i = 0; i < ACT_N; ++i) m.act[i].alloc(B.act_bytes[i]);
        }
    }
    RowMeta rm = row_meta(B);
    ck(cudaMemsetAsync(B.err.p, 0xff, 8, st), "memset err");

    // ---- K0: plan (tokenizer.hpp:53-134 + make_stack_geom in prefix form)
    PlanArgs pa{};
    pa.b = dev_batch(B);
    pa.src = m.d_src.as<SourceInfo>();
    pa.slots = m.d_slots.as<SlotInfo>();
    pa.n_src = n_src;
    pa.n_hist = m.n_hist;
    pa.n_rt = m.n_rt;
    pa.norm = m.cfg.norm;
    pa.only_scenario = B.only_scenario;
    pa.us_off = B.d_us_off.as<long long>();
    pa.src_base = B.d_src_base.as<long long>();
    pa.rec_off = B.d_rec_off.as<long long>();
    pa.rm = rm;
    pa.err = B.err.as<unsigned long long>();
    pa.max_sort = B.sort_cap;
    pa.sort_off = B.sort_off.empty() ? nullptr : B.d_sort_off.as<long long>();
    pa.sort_scratch = B.sort_off.empty() ? nullptr : B.d_sort_scratch.as<long long>();
    {
        StageScope sc(m, "plan", 0, Rd * 8 * 4 + Rd * 7 * 4);
        launch_plan(pa, B.sort_cap, st);
        ck(cudaGetLastError(), "plan launch");
        ++L;
    }

    // ---- K1: tokenizer (embedding gather + 2-layer SiLU MLP per source)
    T* E = m.act[ACT_E].as<T>();
    T* HID = m.act[ACT_HID].as<T>();
    int max_slots = 0;
    for (const auto& s : m.sources) max_slots = std::max(max_slots, s.nslot[0] + s.nslot[1] + s.nslot[2]);
    long long tok_rows = 0;
    double tok_f1 = 0, tok_f2 = 0, tok_in = 0;
    for (int s = 0; s < n_src; ++s) {
        tok_rows += B.src_cnt[s];
        tok_f1 += 2.0 * B.src_cnt[s] * m.sources[s].k_in * 2 * d;
        tok_f2 += 2.0 * B.src_cnt[s] * 2 * d * d;
        tok_in += static_cast<double>(B.src_cnt[s]) * m.sources[s].k_pad;
    }
    {
        if (tok_rows >= (1ll << 31) || n_src > 32)
            fail(MTFM_CONTRACT_ERROR, "batch too large for one forward (tokens >= 2^31 or > 32 token sources)");
        StageScope sc(m, "gather", 0, tok_in * el * 2);
        if (!launch_gather<T>(pa.b, pa.src, pa.slots, rm, B.d_src_base.as<long long>(), B.d_src_cnt.as<long long>(),
                              B.d_emb_base.as<long long>(),
                              kTc ? static_cast<const T*>(m.emb_bf16.p) : static_cast<const T*>(m.emb_f32.p),
                              m.cfg.d_emb, n_src, tok_rows, max_slots, E, st))
            fail(MTFM_CONTRACT_ERROR, "more than 32 token sources");
        ck(cudaGetLastError(), "gather launch");
        ++L;
    }
    float* X = m.act[ACT_X].as<float>();
    // the first target run's xhat (normalised context rows, source order) straight from the
    // fused tokenizer's Y tiles when every context source goes through it (MTFM_TOK_XHAT=0:
    // separate GLN pass, kept selectable for the parity test of the two)
    bool xhat_from_tok = false;
    if constexpr (kTc) {
        std::vector<TcProblem> p1, p2;
        static const bool tok_xhat = std::getenv("MTFM_TOK_XHAT") == nullptr || std::atoi(std::getenv("MTFM_TOK_XHAT")) != 0;
        long long ctx_rows0 = 0;
        for (int s = 0; s < m.n_ctx_src; ++s) ctx_rows0 += B.src_cnt[s];
        xhat_from_tok = tok_xhat && m.n_ctx_src > 0 && ctx_rows0 == NE && !m.layers.empty() && m.layers[0]->target;
        // sequence sources with one k-block of embeddings: fused MLP (tok_tc.cuh)
        TokArgs ta{};
        std::vector<int> fused_src;
        double fused_f = 0, fused_in = 0, p_f1 = 0, p_f2 = 0, p_in = 0, p_rows = 0;
        if (d % 256 == 0) {
            ta.n_pass = d / 256;
            ta.nch = 2 * d / 64;
            ta.ldx = d;
            for (int s = 0; s < n_src && ta.n_src < kTokMaxSrc; ++s) {
                const auto& si = m.sources[s];
                const int M = static_cast<int>(B.src_cnt[s]);
                if (si.k_pad > 64 || M == 0) continue;
                const auto& w = *m.srcw[s];
                TokSource& ts = ta.s[ta.n_src++];
                ts.tma_e = tma_2d(E + B.emb_base[s], M, si.k_pad, si.k_pad, 64, 128, 128);
                ts.tma_w1 = tma_2d(w.t1.p, 2 * d, si.k_pad, si.k_pad, 64, 64, 128);
                ts.tma_w2 = tma_2d(w.t2.p, d, 2 * d, 2 * d, 64, 256, 128);
                ts.tma_b1 = tma_2d(BT.get(w.b1.as<float>(), 2 * d, st), 2 * d, 16, 16, 16, 64, 32);
                ts.tma_b2 = tma_2d(BT.get(w.b2.as<float>(), d, st), d, 16, 16, 16, 256, 32);
                ts.row_map = rm.src_rows + B.src_base[s];
                ts.M = M;
                ts.k_steps = static_cast<int>(cdiv(si.k_pad, 16));
                ts.tile_start = ta.n_tiles / ta.n_pass;  // in tiles (work items are tiles x passes)
                ts.xhat_row0 = s < m.n_ctx_src && d == 256 ? B.src_base[s] : -1;  // x̂ needs whole rows: one pass
                ta.n_tiles += static_cast<int>(cdiv(M, 128)) * ta.n_pass;
                fused_src.push_back(s);
                fused_f += 2.0 * M * (si.k_in * 2.0 * d + 2.0 * d * d);
                fused_in += static_cast<double>(M) * si.k_pad;
            }
            ta.X = X;
            ta.xhat = m.act[ACT_XN].as<__nv_bfloat16>();
            ta.eps = static_cast<float>(m.cfg.eps);
        }
        for (int s = 0; s < m.n_ctx_src; ++s)
            if (B.src_cnt[s] > 0 && std::find(fused_src.begin(), fused_src.end(), s) == fused_src.end())
                xhat_from_tok = false;
        if (d != 256) xhat_from_tok = false;
        if (!xhat_from_tok)
            for (int i = 0; i < ta.n_src; ++i) ta.s[i].xhat_row0 = -1;
        for (int s = 0; s < n_src; ++s) {
            if (std::find(fused_src.begin(), fused_src.end(), s) != fused_src.end()) continue;
            const auto& si = m.sources[s];
            const auto& w = *m.srcw[s];
            const int M = static_cast<int>(B.src_cnt[s]);
            p1.push_back({E + B.emb_base[s], si.k_pad, w.t1.as<__nv_bfloat16>(), si.k_pad, M, 2 * d, si.k_pad,
                          EPI_SILU_BF16, w.b1.as<float>(), HID + B.hid_base[s], 2 * d, nullptr, 0, nullptr});
            p2.push_back({HID + B.hid_base[s], 2 * d, w.t2.as<__nv_bfloat16>(), 2 * d, M, d, 2 * d, EPI_BIAS_F32,
                          w.b2.as<float>(), X, d, rm.src_rows + B.src_base[s], 0, nullptr});
            p_f1 += 2.0 * M * si.k_in * 2 * d;
            p_f2 += 2.0 * M * 2 * d * d;
            p_in += static_cast<double>(M) * si.k_pad;
            p_rows += M;
        }
        if (ta.n_tiles > 0) {
            StageScope sc(m, "tok_fused", fused_f, fused_in * el + (Rd - p_rows) * d * 4);
            launch_tok_fused(ta, st);
            ++L;
        }
        {
            StageScope sc(m, "tok_mlp1", p_f1, p_in * el + p_rows * 2 * d * el);
            run_gemm_tc(p1, st, L, BT);
        }
        {
            StageScope sc(m, "tok_mlp2", p_f2, p_rows * 2 * d * el + p_rows * d * 4);
            run_gemm_tc(p2, st, L, BT);
        }
    } else {
        std::vector<SimtGemm> p1, p2;
        for (int s = 0; s < n_src; ++s) {
            const auto& si = m.sources[s];
            const auto& w = *m.srcw[s];
            const int M = static_cast<int>(B.src_cnt[s]);
            p1.push_back({reinterpret_cast<const float*>(E) + B.emb_base[s], si.k_pad, w.w1.as<float>(), M, 2 * d,
                          si.k_pad, w.b1.as<float>(), EPI_SILU_BF16, reinterpret_cast<float*>(HID) + B.hid_base[s],
                          2 * d, nullptr, 0, nullptr});
            p2.push_back({reinterpret_cast<const float*>(HID) + B.hid_base[s], 2 * d, w.w2.as<float>(), M, d, 2 * d,
                          w.b2.as<float>(), EPI_BIAS_F32, X, d, rm.src_rows + B.src_base[s], 0, nullptr});
        }
        {
            StageScope sc(m, "tok_mlp1", tok_f1, tok_in * el + Rd * 2 * d * el);
            run_gemm_simt(p1, st, L);
        }
        {
            StageScope sc(m, "tok_mlp2", tok_f2, Rd * 2 * d * el + Rd * d * 4);
            run_gemm_simt(p2, st, L);
        }
    }

    // ---- attention tile extents (max visible prefix per tile)
    const AttnGeom ag = attn_geom(m);
    const int n_full = static_cast<int>(B.n_tiles_full);
    const int n_tgt = static_cast<int>(B.n_tiles_tgt);
    if (kTc && (n_full || n_tgt)) {
        StageScope sc(m, "tile_kmax", 0, (n_full + n_tgt) * 32.0);
        launch_k(tile_kmax_kernel, dim3(static_cast<unsigned>(cdiv(n_full + n_tgt, 8))), dim3(256), 0, st,
                 B.tiles_full.as<AttnTile>(), n_full, static_cast<const int*>(rm.prefix), B.tiles_tgt.as<AttnTile>(),
                 n_tgt, static_cast<const int*>(rm.prefix + NE));
        ck(cudaGetLastError(), "tile_kmax launch");
        ++L;
    }

    // ---- K2..K4: the HTA stack (hta.hpp:188-212)
    T* XN = m.act[ACT_XN].as<T>();
    T* Pm = m.act[ACT_P].as<T>();
    T* KV = m.act[ACT_KV].as<T>();
    T* UQ = m.act[ACT_UQ].as<T>();
    T* A = m.act[ACT_A].as<T>();
    T* G = m.act[ACT_GT].as<T>();
    // attention FLOPs need sum(c_i): known after the plan; use the value of
    // the previous results() (same batch) for the profile annotation
    const double sc_full = static_cast<double>(B.sum_c_ctx + B.sum_c_t), sc_t = static_cast<double>(B.sum_c_t);
    if constexpr (kTc) {
        // Context rows X[0, NE) are the same for every target layer of a run and for the
        // full layer right after it (target layers only update T rows, hta.hpp:158-184).
        // At the start of a run they are normalised once, without the affine, into
        // source order (xhat = XN[0, NE)); every context source's GLN1 affine is folded
        // into its own copy of the K|V (target) / f1 (full) weights (LayerW::tfold), and
        // the GEMM outputs are scattered back to X-row order.
        size_t full_ctx_from_run = static_cast<size_t>(-1);  // full layer whose context rows come from xhat
        T* XNT = XN + NE * d;                                 // T rows' GLN1 of the current target layer
        T* XNF = XN + R * d;                                  // GLN1 of a full layer's rows (T rows only after a run)
        int tl = 0;                                           // index of the current target layer within its run
        for (size_t li = 0; li < m.layers.size(); ++li) {
            const auto& Lw = m.layers[li];
            if (!Lw->target) {
                // full layer (hta.hpp:138-155)
                const bool from_run = full_ctx_from_run == li;
                if (from_run) {
                    StageScope sc(m, "gln1", 0, Td * d * (4 + el));
                    launch_gln<T>(X, d, NE, NT, d, rm.src, Lw->g1g.as<float>(), Lw->g1b.as<float>(), eps,
                                  XNF + NE * d, d, st);
                    ++L;
                } else {
                    StageScope sc(m, "gln1", 0, Rd * d * (4 + el));
                    launch_gln<T>(X, d, 0, R, d, rm.src, Lw->g1g.as<float>(), Lw->g1b.as<float>(), eps, XNF, d, st);
                    ++L;
                }
                // U and Q|K|V as two contiguous matrices (one grouped launch): the gate
                // then streams U rows and the attention Q|K|V rows without gaps
                T* U = Pm;
                T* QKV = Pm + R * hd;
                const long long ldqkv = hd + 2 * gd;
                {
                    StageScope sc(m, "proj_full", 2.0 * Rd * d * pw, Rd * d * el + Rd * pw * el);
                    std::vector<TcProblem> pp;
                    const long long r0 = from_run ? NE : 0;  // rows taken from XNF
                    if (from_run) {
                        // context rows: per source, xhat rows x folded f1, scattered to X-row order
                        for (int s = 0; s < m.n_ctx_src; ++s) {
                            const __nv_bfloat16* wf = Lw->tfold.as<__nv_bfloat16>() + static_cast<long long>(s) * pw * d;
                            const float* bfo = Lw->bfold.as<float>() + static_cast<long long>(s) * pw;
                            const int Ms = static_cast<int>(B.src_cnt[s]);
                            const int* rmap = rm.src_rows + B.src_base[s];
                            pp.push_back({XN + B.src_base[s] * d, d, wf, d, Ms, hd, d, EPI_SILU_BF16, bfo, U, hd, rmap, 0,
                                          nullptr});
                            pp.push_back({XN + B.src_base[s] * d, d, wf + static_cast<long long>(hd) * d, d, Ms,
                                          hd + 2 * gd, d, EPI_SILU_BF16, bfo + hd, QKV, ldqkv, rmap, 0, nullptr});
                        }
                    }
                    const int Mr = static_cast<int>(R - r0);
                    pp.push_back({XNF + r0 * d, d, Lw->t1.as<__nv_bfloat16>(), d, Mr, hd, d, EPI_SILU_BF16,
                                  Lw->b1.as<float>(), U, hd, nullptr, r0, nullptr});
                    pp.push_back({XNF + r0 * d, d, Lw->t1.as<__nv_bfloat16>() + static_cast<long long>(hd) * d, d, Mr,
                                  hd + 2 * gd, d, EPI_SILU_BF16, Lw->b1.as<float>() + hd, QKV, ldqkv, nullptr, r0,
                                  nullptr});
                    run_gemm_tc(pp, st, L, BT);
                }
                {
                    StageScope sc(m, "attn_full", 4.0 * hd * sc_full, Rd * (hd + 2 * gd) * el + Rd * hd * el);
                    AttnParams ap{};
                    ap.tiles = B.tiles_full.as<AttnTile>();
                    ap.n_tiles = n_full;
                    ap.q_col0 = 0;
                    ap.k_col0 = hd;
                    ap.v_col0 = hd + gd;
                    ap.heads = m.H;
                    ap.kv_heads = m.G;
                    ap.hs = ag.hs;
                    ap.rt = ag.rt;
                    ap.q_prefix = rm.prefix;
                    ap.q_scale = rm.scale;
                    ap.q_self = rm.self;
                    ap.q_ptr = QKV;
                    ap.ldq = ldqkv;
                    ap.kv_ptr = QKV;
                    ap.ldkv = ldqkv;
                    ap.out = A;
                    ap.ldo = hd;
                    run_attn_tc(m, ap, QKV, R, ldqkv, R, ldqkv, st);
                    ++L;
                }
                {
                    StageScope sc(m, "gate", 0, Rd * hd * el * 3);
                    launch_gate<T>(A, hd, U, hd, R, hd, rm.src, Lw->g2g.as<float>(), Lw->g2b.as<float>(), eps, G, hd, st);
                    ++L;
                }
                StageScope sc(m, "f2_full", 2.0 * Rd * hd * d, Rd * hd * el + Rd * d * 8);
                run_gemm_tc({{G, hd, Lw->tf2.as<__nv_bfloat16>(), hd, static_cast<int>(R), d, hd, EPI_RESID_F32,
                              Lw->f2b.as<float>(), X, d, nullptr, 0, X}},
                            st, L, BT);
            } else {
                // target layer (hta.hpp:158-184): T rows only; H/R rows untouched
                if (li == 0 || !m.layers[li - 1]->target) {
                    // start of a target run: xhat of the context rows, then every layer's
                    // context K|V from it in one grouped GEMM (per source and layer)
                    size_t lj = li;
                    while (lj < m.layers.size() && m.layers[lj]->target) ++lj;
                    const int kt = static_cast<int>(lj - li);
                    if (NE > 0) {
                        if (!(li == 0 && xhat_from_tok)) {
                            GlnCopies gc{};
                            gc.n = 1;
                            gc.out[0] = XN;
                            gc.in_rows = rm.src_rows;
                            StageScope sc(m, "gln1", 0, NE * d * (4.0 + el));
                            launch_gln_multi_bf16(X, d, NE, d, rm.src, gc, eps, d, st);
                            ++L;
                        }
                        std::vector<TcProblem> kvp;
                        for (int s = 0; s < m.n_ctx_src; ++s)
                            for (int c = 0; c < kt; ++c) {
                                const auto& Lc = m.layers[li + c];
                                kvp.push_back({XN + B.src_base[s] * d, d,
                                               Lc->tfold.as<__nv_bfloat16>() + static_cast<long long>(s) * 2 * gd * d, d,
                                               static_cast<int>(B.src_cnt[s]), 2 * gd, d, EPI_SILU_BF16,
                                               Lc->bfold.as<float>() + s * 2 * gd,
                                               KV + static_cast<long long>(c) * R * 2 * gd, 2 * gd,
                                               rm.src_rows + B.src_base[s], 0, nullptr});
                            }
                        StageScope sc(m, "proj_ctx_kv", 2.0 * kt * NE * d * 2 * gd, NE * d * el + kt * NE * 2.0 * gd * el);
                        run_gemm_tc(kvp, st, L, BT);
                    }
                    if (lj < m.layers.size()) full_ctx_from_run = lj;
                    tl = 0;
                }
                T* KVl = KV + static_cast<long long>(tl) * R * 2 * gd;  // this layer's K|V rows (context, then T)
                {
                    StageScope sc(m, "gln1", 0, Td * d * (4 + el));
                    launch_gln<T>(X, d, NE, NT, d, rm.src, Lw->g1g.as<float>(), Lw->g1b.as<float>(), eps, XNT, d, st);
                    ++L;
                }
                {
                    StageScope sc(m, "proj_target", 2.0 * Td * d * (2 * gd + 2 * hd), Td * d * el + Td * (2 * gd + 2 * hd) * el);
                    run_gemm_tc({{XNT, d, Lw->tkv.as<__nv_bfloat16>(), d, static_cast<int>(NT), 2 * gd, d, EPI_SILU_BF16,
                                  Lw->bkv.as<float>(), KVl + NE * 2 * gd, 2 * gd, nullptr, 0, nullptr},
                                 {XNT, d, Lw->t1.as<__nv_bfloat16>(), d, static_cast<int>(NT), 2 * hd, d,
                                  EPI_SILU_BF16, Lw->b1.as<float>(), UQ, 2 * hd, nullptr, 0, nullptr}},
                                st, L, BT);
                }
                ++tl;
                {
                    StageScope sc(m, "attn_target", 4.0 * hd * sc_t, Rd * 2 * gd * el + Td * 2 * hd * el);
                    AttnParams ap{};
                    ap.tiles = B.tiles_tgt.as<AttnTile>();
                    ap.n_tiles = n_tgt;
                    ap.q_col0 = hd;
                    ap.k_col0 = 0;
                    ap.v_col0 = gd;
                    ap.heads = m.H;
                    ap.kv_heads = m.G;
                    ap.hs = ag.hs;
                    ap.rt = ag.rt;
                    ap.q_prefix = rm.prefix + NE;
                    ap.q_scale = rm.scale + NE;
                    ap.q_self = rm.self + NE;
                    ap.q_ptr = UQ;
                    ap.ldq = 2 * hd;
                    ap.kv_ptr = KVl;
                    ap.ldkv = 2 * gd;
                    ap.out = A;
                    ap.ldo = hd;
                    run_attn_tc(m, ap, UQ, NT, 2 * hd, R, 2 * gd, st);
                    ++L;
                }
                {
                    StageScope sc(m, "gate", 0, Td * hd * el * 3);
                    launch_gate<T>(A, hd, UQ, 2 * hd, NT, hd, rm.src + NE, Lw->g2g.as<float>(), Lw->g2b.as<float>(),
                                   eps, G, hd, st);
                    ++L;
                }
                StageScope sc(m, "f2_target", 2.0 * Td * hd * d, Td * hd * el + Td * d * 8);
                run_gemm_tc({{G, hd, Lw->tf2.as<__nv_bfloat16>(), hd, static_cast<int>(NT), d, hd, EPI_RESID_F32,
                              Lw->f2b.as<float>(), X, d, nullptr, NE, X}},
                            st, L, BT);
            }
        }
    } else {
    for (const auto& Lw : m.layers) {
        {
            StageScope sc(m, "gln1", 0, Rd * d * (4 + el));
            launch_gln<T>(X, d, 0, R, d, rm.src, Lw->g1g.as<float>(), Lw->g1b.as<float>(), eps, XN, d, st);
            ++L;
        }
        if (!Lw->target) {
            // full layer (hta.hpp:138-155)
            {
                StageScope sc(m, "proj_full", 2.0 * Rd * d * pw, Rd * d * el + Rd * pw * el);
                if constexpr (kTc)
                    run_gemm_tc({{XN, d, Lw->t1.as<__nv_bfloat16>(), d, static_cast<int>(R), pw, d, EPI_SILU_BF16,
                                  Lw->b1.as<float>(), Pm, pw, nullptr, 0, nullptr}},
                                st, L, BT);
                else
                    run_gemm_simt({{reinterpret_cast<const float*>(XN), d, Lw->w1.as<float>(), static_cast<int>(R), pw,
                                    d, Lw->b1.as<float>(), EPI_SILU_BF16, Pm, pw, nullptr, 0, nullptr}},
                                  st, L);
            }
            {
                StageScope sc(m, "attn_full", 4.0 * hd * sc_full, Rd * (hd + 2 * gd) * el + Rd * hd * el);
                if constexpr (kTc) {
                    AttnParams ap{};
                    ap.tiles = B.tiles_full.as<AttnTile>();
                    ap.n_tiles = n_full;
                    ap.q_col0 = hd;
                    ap.k_col0 = 2 * hd;
                    ap.v_col0 = 2 * hd + gd;
                    ap.heads = m.H;
                    ap.kv_heads = m.G;
                    ap.hs = ag.hs;
                    ap.rt = ag.rt;
                    ap.q_prefix = rm.prefix;
                    ap.q_scale = rm.scale;
                    ap.q_self = rm.self;
                    ap.q_ptr = Pm;
                    ap.ldq = pw;
                    ap.kv_ptr = Pm;
                    ap.ldkv = pw;
                    ap.out = A;
                    ap.ldo = hd;
                    run_attn_tc(m, ap, Pm, R, pw, R, pw, st);
                } else {
                    SimtAttn sa{reinterpret_cast<const float*>(Pm), pw, hd, reinterpret_cast<const float*>(Pm), pw,
                                2 * hd, 2 * hd + gd, R, rm.prefix, rm.scale, rm.self, rm.keybase, m.H, m.G, dh,
                                reinterpret_cast<float*>(A), hd};
                    launch_attn_simt(sa, st);
                    ck(cudaGetLastError(), "attn_simt launch");
                }
                ++L;
            }
            {
                StageScope sc(m, "gate", 0, Rd * hd * el * 3);
                launch_gate<T>(A, hd, Pm, pw, R, hd, rm.src, Lw->g2g.as<float>(), Lw->g2b.as<float>(), eps, G, hd, st);
                ++L;
            }
            {
                StageScope sc(m, "f2_full", 2.0 * Rd * hd * d, Rd * hd * el + Rd * d * 8);
                if constexpr (kTc)
                    run_gemm_tc({{G, hd, Lw->tf2.as<__nv_bfloat16>(), hd, static_cast<int>(R), d, hd, EPI_RESID_F32,
                                  Lw->f2b.as<float>(), X, d, nullptr, 0, X}},
                                st, L, BT);
                else
                    run_gemm_simt({{reinterpret_cast<const float*>(G), hd, Lw->f2.as<float>(), static_cast<int>(R), d,
                                    hd, Lw->f2b.as<float>(), EPI_RESID_F32, X, d, nullptr, 0, X}},
                                  st, L);
            }
        } else {
            // target layer (hta.hpp:158-184): T rows only; H/R rows untouched
            {
                StageScope sc(m, "proj_target", 2.0 * (Rd * d * 2 * gd + Td * d * 2 * hd),
                              Rd * d * el + Rd * 2 * gd * el + Td * 2 * hd * el);
                if constexpr (kTc)
                    run_gemm_tc({{XN, d, Lw->tkv.as<__nv_bfloat16>(), d, static_cast<int>(R), 2 * gd, d, EPI_SILU_BF16,
                                  Lw->bkv.as<float>(), KV, 2 * gd, nullptr, 0, nullptr},
                                 {XN + NE * d, d, Lw->t1.as<__nv_bfloat16>(), d, static_cast<int>(NT), 2 * hd, d,
                                  EPI_SILU_BF16, Lw->b1.as<float>(), UQ, 2 * hd, nullptr, 0, nullptr}},
                                st, L, BT);
                else
                    run_gemm_simt({{reinterpret_cast<const float*>(XN), d, Lw->wkv.as<float>(), static_cast<int>(R),
                                    2 * gd, d, Lw->bkv.as<float>(), EPI_SILU_BF16, KV, 2 * gd, nullptr, 0, nullptr},
                                   {reinterpret_cast<const float*>(XN) + NE * d, d, Lw->w1.as<float>(),
                                    static_cast<int>(NT), 2 * hd, d, Lw->b1.as<float>(), EPI_SILU_BF16, UQ, 2 * hd,
                                    nullptr, 0, nullptr}},
                                  st, L);
            }
            {
                StageScope sc(m, "attn_target", 4.0 * hd * sc_t, Rd * 2 * gd * el + Td * 2 * hd * el);
                if constexpr (kTc) {
                    AttnParams ap{};
                    ap.tiles = B.tiles_tgt.as<AttnTile>();
                    ap.n_tiles = n_tgt;
                    ap.q_col0 = hd;
                    ap.k_col0 = 0;
                    ap.v_col0 = gd;
                    ap.heads = m.H;
                    ap.kv_heads = m.G;
                    ap.hs = ag.hs;
                    ap.rt = ag.rt;
                    ap.q_prefix = rm.prefix + NE;
                    ap.q_scale = rm.scale + NE;
                    ap.q_self = rm.self + NE;
                    ap.q_ptr = UQ;
                    ap.ldq = 2 * hd;
                    ap.kv_ptr = KV;
                    ap.ldkv = 2 * gd;
                    ap.out = A;
                    ap.ldo = hd;
                    run_attn_tc(m, ap, UQ, NT, 2 * hd, R, 2 * gd, st);
                } else {
                    SimtAttn sa{reinterpret_cast<const float*>(UQ), 2 * hd, hd, reinterpret_cast<const float*>(KV),
                                2 * gd, 0, gd, NT, rm.prefix + NE, rm.scale + NE, rm.self + NE, rm.keybase + NE,
                                m.H, m.G, dh, reinterpret_cast<float*>(A), hd};
                    launch_attn_simt(sa, st);
                    ck(cudaGetLastError(), "attn_simt launch");
                }
                ++L;
            }
            {
                StageScope sc(m, "gate", 0, Td * hd * el * 3);
                launch_gate<T>(A, hd, UQ, 2 * hd, NT, hd, rm.src + NE, Lw->g2g.as<float>(), Lw->g2b.as<float>(), eps,
                               G, hd, st);
                ++L;
            }
            {
                StageScope sc(m, "f2_target", 2.0 * Td * hd * d, Td * hd * el + Td * d * 8);
                if constexpr (kTc)
                    run_gemm_tc({{G, hd, Lw->tf2.as<__nv_bfloat16>(), hd, static_cast<int>(NT), d, hd, EPI_RESID_F32,
                                  Lw->f2b.as<float>(), X, d, nullptr, NE, X}},
                                st, L, BT);
                else
                    run_gemm_simt({{reinterpret_cast<const float*>(G), hd, Lw->f2.as<float>(), static_cast<int>(NT), d,
                                    hd, Lw->f2b.as<float>(), EPI_RESID_F32, X, d, nullptr, NE, X}},
                                  st, L);
            }
        }
    }

    }

    // ---- K5: heads (heads.hpp:47-99) + records
    float* Y = m.act[ACT_Y].as<float>();
    // algorithmic head work: every T row's experts, and per record its task's gate;
    // the GEMM also evaluates the other scenarios' gate columns, which are not counted
    const double hflops = 2.0 * (Td * m.cfg.experts * d * m.cfg.d_expert + static_cast<double>(B.n_records) * d * m.cfg.experts);
    if constexpr (kTc) {
        // fused heads (heads_tc.cuh): the head GEMM's expert columns are reduced to the
        // per-task logits in its epilogue instead of round-tripping [T][E*de] through HBM
        int max_nt = 0;
        for (const auto& sc : m.sources)
            if (sc.kind == 2) max_nt = std::max(max_nt, sc.ntasks);
        const int E = m.cfg.experts, dx = m.cfg.d_expert;
        const int ng_pad = static_cast<int>(round_up(static_cast<long long>(m.n_tasks_total) * E, 16));
        // SMEM: resident X tile (d/64 x 16 KB), weight stages, tables, partial logits, barriers
        const size_t fixed = 1024 + static_cast<size_t>(d / 64) * heads_detail::A_BYTES +
                             static_cast<size_t>(E * dx + m.n_tasks_total * (dx + 4)) * 4 + heads_detail::XZ_BYTES +
                             static_cast<size_t>(heads_detail::BM * (ng_pad + 1) + 4) * 4 + 512;
        const int n_ws = fixed < 227 * 1024 ? static_cast<int>(std::min<size_t>(
                                                  (227 * 1024 - fixed) / heads_detail::W_BYTES, heads_detail::kMaxWStages))
                                            : 0;
        const size_t hsmem = fixed + static_cast<size_t>(n_ws) * heads_detail::W_BYTES;
        if (E <= kHeadsMaxE && max_nt <= kHeadsMaxTasks && dx % heads_detail::CH == 0 && d % 64 == 0 &&
            ng_pad <= heads_detail::CH && n_ws >= 3) {
            HeadsTcArgs ha{};
            ha.x = X + NE * d;
            ha.ldx = d;
            ha.tma_w = tma_2d(m.head_t.p, m.head_n, d, d, 64, 128, 128);
            ha.n_t = static_cast<int>(NT);
            ha.d = d;
            ha.E = E;
            ha.de = dx;
            ha.n_gate = m.n_tasks_total * E;
            ha.n_tasks_total = m.n_tasks_total;
            ha.n_wstages = n_ws;
            ha.exp_bias = m.head_eb.as<float>();
            ha.gate_bias = m.head_gb.as<float>();
            ha.tower_w = m.tower_w.as<float>();
            ha.tower_b = m.tower_b.as<float>();
            ha.src = m.d_src.as<SourceInfo>();
            ha.n_src = n_src;
            ha.t_scen = rm.t_scen;
            ha.t_user = rm.t_user;
            ha.t_exp_ref = rm.t_exp_ref;
            ha.t_rec0 = rm.t_rec0;
            ha.t_rec_stride = rm.t_rec_stride;
            ha.user_id = B.user_id.as<long long>();
            ha.rec_user = B.rec_user.as<long long>();
            ha.rec_scen = B.rec_scen.as<int>();
            ha.rec_exp = B.rec_exp.as<int>();
            ha.rec_task = B.rec_task.as<int>();
            ha.rec_logit = B.rec_logit.as<float>();
            ha.rec_prob = B.rec_prob.as<double>();
            StageScope sc(m, "heads", hflops + 2.0 * B.n_records * m.cfg.d_expert, Td * d * 4 + B.n_records * 32.0);
            if (NT > 0) {
                static size_t attr = 0;
                if (hsmem > attr) {
                    ck(cudaFuncSetAttribute(heads_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(hsmem)),
                       "heads smem attr");
                    attr = hsmem;
                }
                launch_k(heads_tc_kernel, dim3(static_cast<int>(std::min<long long>(cdiv(NT, 128), kNumSMs))),
                         dim3(heads_detail::kThreads), hsmem, st, ha);
                ck(cudaGetLastError(), "heads_tc launch");
                ++L;
            }
            return;
        }
        {
            StageScope sc(m, "to_bf16", 0, Td * d * 6);
            launch_to_bf16(X + NE * d, NT, d, XN, d, st);
            ++L;
        }
        StageScope sc(m, "heads_gemm", hflops, Td * d * 2 + Td * m.head_n * 4);
        run_gemm_tc({{XN, d, m.head_t.as<__nv_bfloat16>(), d, static_cast<int>(NT), m.head_n, d, EPI_BIAS_F32, nullptr,
                      Y, m.head_ld, nullptr, 0, nullptr}},
                    st, L, BT);
    } else {
        StageScope sc(m, "heads_gemm", hflops, Td * d * 4 + Td * m.head_n * 4);
        run_gemm_simt({{X + NE * d, d, m.head_w.as<float>(), static_cast<int>(NT), m.head_n, d, nullptr, EPI_BIAS_F32, Y,
                        m.head_ld, nullptr, 0, nullptr}},
                      st, L);
    }
    HeadArgs ha{};
    ha.y = Y;
    ha.ldy = m.head_ld;
    ha.exp_bias = m.head_eb.as<float>();
    ha.gate_bias = m.head_gb.as<float>();
    ha.tower_w = m.tower_w.as<float>();
    ha.tower_b = m.tower_b.as<float>();
    ha.E = m.cfg.experts;
    ha.de = m.cfg.d_expert;
    ha.src = m.d_src.as<SourceInfo>();
    ha.n_src = n_src;
    ha.t_scen = rm.t_scen;
    ha.t_user = rm.t_user;
    ha.t_exp_ref = rm.t_exp_ref;
    ha.t_rec0 = rm.t_rec0;
    ha.t_rec_stride = rm.t_rec_stride;
    ha.user_id = B.user_id.as<long long>();
    ha.n_t = NT;
    ha.precise = !kTc;  // fp32 check mode: expf-based SiLU; bf16 mode: one MUFU.TANH
    ha.rec_user = B.rec_user.as<long long>();
    ha.rec_scen = B.rec_scen.as<int>();
    ha.rec_exp = B.rec_exp.as<int>();
    ha.rec_task = B.rec_task.as<int>();
    ha.rec_logit = B.rec_logit.as<float>();
    ha.rec_prob = B.rec_prob.as<double>();
    {
        StageScope sc(m, "heads", 2.0 * B.n_records * m.cfg.d_expert,
                      Td * m.head_ld * 4 + B.n_records * 32.0);
        launch_heads(ha, st, m.n_tasks_total);
        ck(cudaGetLastError(), "heads launch");
        ++L;
    }
}

void launch_sum_valid(mtfm_cuda_batch& B, cudaStream_t st);

void results(mtfm_cuda_model& m, mtfm_cuda_batch& B, mtfm_records* out) {
    // read-back on its own stream, behind this batch's forward only
    cudaStream_t st = m.d2h_stream;
    if (B.ran) ck(cudaStreamWaitEvent(st, B.ev_done, 0), "wait forward");
    // error key + the visible-key sums of the stats, read back with one synchronisation
    B.pin.reserve(4096);
    auto* hb = static_cast<unsigned long long*>(B.pin.p);
    hb[0] = ~0ull;
    hb[1] = hb[2] = 0;
    if (B.n_users > 0) ck(cudaMemcpyAsync(hb, B.err.p, 8, cudaMemcpyDeviceToHost, st), "D2H err");
    launch_sum_valid(B, st);
    ck(cudaMemcpyAsync(hb + 1, B.stat_buf.p, 16, cudaMemcpyDeviceToHost, st), "D2H stats");
    ck(cudaStreamSynchronize(st), "forward");
    B.sum_c_ctx = hb[1];
    B.sum_c_t = hb[2];
    const unsigned long long err = hb[0];
    if (err != ~0ull) {
        const int code = static_cast<int>(err & 7);
        const long long user = static_cast<long long>(err >> 42);
        std::string what;
        switch (code) {
            case 1: what = "token metas not time-sorted within block"; break;
            case 2: what = "no tokenizer for a sequence schema or scenario of the sample"; break;
            case 3: what = "embed_rows: feature slot missing"; break;
            case 5: what = "gather_rows: feature id out of range"; break;
            case 6: what = "assemble_tokens: sample has no tokens"; break;
            default: what = "planning capacity exceeded";
        }
        const mtfm_status s = code == 2 ? MTFM_INTEGRITY_ERROR
                              : (code == 3 || code == 1) ? MTFM_DIMENSION_ERROR
                              : code == 5 ? MTFM_LOOKUP_ERROR
                                          : MTFM_CONTRACT_ERROR;
        fail(s, what + " (user index " + std::to_string(user) + ")");
    }
    if (!out) return;
    if (out->capacity < B.n_records)
        fail(MTFM_CONTRACT_ERROR, "record buffer too small: need " + std::to_string(B.n_records));
    const size_t n = static_cast<size_t>(B.n_records);
    if (n) {
        ck(cudaMemcpyAsync(out->user_id, B.rec_user.p, n * 8, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(out->scenario_id, B.rec_scen.p, n * 4, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(out->exposure_index, B.rec_exp.p, n * 4, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(out->task_index, B.rec_task.p, n * 4, cudaMemcpyDeviceToHost, st), "D2H");
        if (out->logit) ck(cudaMemcpyAsync(out->logit, B.rec_logit.p, n * 4, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(out->probability, B.rec_prob.p, n * 8, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "D2H records");
    }
    out->n_records = B.n_records;
}

void launch_sum_valid(mtfm_cuda_batch& B, cudaStream_t st);
// Algorithmic FLOPs of the run: projections per complexity.hpp:54-64,
// mask-aware attention 4*d_h*H*sum(c_i) per layer, tokenizer MLPs, heads.
__global__ void sum_valid_kernel(const int* prefix, const int* self, long long n, unsigned long long* out) {
    MTFM_PDL_ENTRY();
    unsigned long long s = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        s += static_cast<unsigned long long>(prefix[i] + (self[i] >= 0 ? 1 : 0));
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

void launch_sum_valid(mtfm_cuda_batch& B, cudaStream_t st) {
    B.stat_buf.alloc(16);
    ck(cudaMemsetAsync(B.stat_buf.p, 0, 16, st), "memset stats");
    auto* a = B.stat_buf.as<unsigned long long>();
    if (B.n_events)
        launch_k(sum_valid_kernel, dim3(64), dim3(256), 0, st, B.r_prefix.as<int>(), B.r_self.as<int>(), B.n_events, a);
    if (B.n_exp)
        launch_k(sum_valid_kernel, dim3(64), dim3(256), 0, st, B.r_prefix.as<int>() + B.n_events, B.r_self.as<int>() + B.n_events,
                                             B.n_exp, a + 1);
}

}  // namespace
}  // namespace mtfm

namespace mtfm {
void set_last_error(const std::string& what) { g_last_error = what; }
}  // namespace mtfm

#include "train_step.inc"

namespace mtfm {
namespace {

// device fp32 weights -> the host parameter copies (after training / pruning on the device)
void sync_host_params(mtfm_cuda_model& m) {
    ck(cudaStreamSynchronize(m.stream), "sync");
    for (size_t i = 0; i < m.params.size(); ++i) {
        auto& q = m.params[i];
        const ParamView& pv = m.views[i];
        if (!pv.buf) continue;
        q.host.resize(static_cast<size_t>(q.rows * q.cols));
        ck(cudaMemcpy2D(q.host.data(), static_cast<size_t>(q.cols) * 4, pv.buf->as<float>() + pv.off,
                        static_cast<size_t>(pv.ld) * 4, static_cast<size_t>(q.cols) * 4, static_cast<size_t>(q.rows),
                        cudaMemcpyDeviceToHost),
           "D2H param");
    }
    m.device_ahead = false;
}

// prune_2_4_inplace (prune.hpp:33-70): per column, every full group of 4 consecutive input
// rows keeps its two largest magnitudes (ties keep the earlier row); one thread per (group, column)
__global__ void prune_2_4_kernel(float* w, int rows, int cols, unsigned long long* zeros) {
    const long long n = static_cast<long long>(rows / 4) * cols;
    unsigned long long z = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long g = i / cols;
        const int j = static_cast<int>(i - g * cols);
        float* c = w + g * 4 * cols + j;
        auto mag = [&](int r) { return fabs(static_cast<double>(c[static_cast<long long>(r) * cols])); };
        int keep0 = 0, keep1 = 1;
        if (mag(keep1) > mag(keep0)) {
            keep0 = 1;
            keep1 = 0;
        }
        for (int r = 2; r < 4; ++r) {
            if (mag(r) > mag(keep0)) {
                keep1 = keep0;
                keep0 = r;
            } else if (mag(r) > mag(keep1)) {
                keep1 = r;
            }
        }
        for (int r = 0; r < 4; ++r)
            if (r != keep0 && r != keep1) {
                c[static_cast<long long>(r) * cols] = 0.f;
                ++z;
            }
    }
    z = static_cast<unsigned long long>(warp_sum(static_cast<double>(z)));
    if ((threadIdx.x & 31) == 0 && z) atomicAdd(zeros, z);
}

}  // namespace
}  // namespace mtfm

mtfm_cuda_model::~mtfm_cuda_model() {
    if (nccl) {
        try {
            mtfm::nccl().destroy(nccl);
        } catch (...) {
        }
    }
}

using namespace mtfm;

extern "C" {

const char* mtfm_cuda_last_error(void) { return g_last_error.c_str(); }
const char* mtfm_cuda_version(void) { return "mtfm-b200 0.1 (sm_100a)"; }

mtfm_status mtfm_cuda_create(int device, const mtfm_model_desc* md, const mtfm_schema_desc* sd, int32_t precision,
                             mtfm_cuda_model** out) {
    return guard([&] {
        if (!md || !sd || !out) fail(MTFM_CONTRACT_ERROR, "null argument");
        // HTAConfig::validate / ModelConfig::validate (model_config.hpp:53-66, 82-87)
        if (md->d_model < 1) fail(MTFM_CONFIG_ERROR, "hta: d_model must be positive");
        if (md->blocks < 1) fail(MTFM_CONFIG_ERROR, "hta: blocks must be >= 1");
        if (md->target_layers < 0 || md->full_layers < 0) fail(MTFM_CONFIG_ERROR, "hta: negative layer counts");
        if (md->target_layers + md->full_layers < 1) fail(MTFM_CONFIG_ERROR, "hta: each block needs at least one layer");
        if (md->heads < 1 || md->kv_heads < 1) fail(MTFM_CONFIG_ERROR, "hta: head counts must be >= 1");
        if (md->heads % md->kv_heads != 0) fail(MTFM_CONFIG_ERROR, "hta: heads must be divisible by kv_heads");
        if (md->d_model % md->heads != 0) fail(MTFM_CONFIG_ERROR, "hta: d_model must be divisible by heads");
        if (!(md->eps > 0)) fail(MTFM_CONFIG_ERROR, "hta: eps must be positive");
        if (md->d_emb < 1) fail(MTFM_CONFIG_ERROR, "model: d_emb must be >= 1");
        if (md->experts < 1) fail(MTFM_CONFIG_ERROR, "model: experts must be >= 1");
        if (md->d_expert < 1) fail(MTFM_CONFIG_ERROR, "model: d_expert must be >= 1");
        if (md->norm < 0 || md->norm > 2) fail(MTFM_CONFIG_ERROR, "unknown attention norm");
        if (precision != MTFM_PRECISION_BF16 && precision != MTFM_PRECISION_FP32_CHECK)
            fail(MTFM_CONFIG_ERROR, "unknown precision");
        // limits of this implementation (documented in DESIGN.md)
        if (md->d_model > 1024 || md->d_model % 8) fail(MTFM_CONFIG_ERROR, "d_model must be a multiple of 8 and <= 1024");
        if (md->experts > 32) fail(MTFM_CONFIG_ERROR, "experts must be <= 32");
        const int dh = md->d_model / md->heads;
        if (dh > 256) fail(MTFM_CONFIG_ERROR, "head_dim must be <= 256");
        if (precision == MTFM_PRECISION_BF16 && (dh % 16 || (dh & (dh - 1))))
            fail(MTFM_CONFIG_ERROR, "bf16 tensor-core path needs head_dim in {16,32,64,128,256}; use the fp32 check mode");
        if ((md->d_emb * 2) % 16 && precision == MTFM_PRECISION_BF16)
            fail(MTFM_CONFIG_ERROR, "bf16 path needs d_emb to be a multiple of 8");
        int cnt = 0;
        ck(cudaGetDeviceCount(&cnt), "cudaGetDeviceCount");
        if (device < 0 || device >= cnt) fail(MTFM_CONFIG_ERROR, "no such CUDA device");
        ck(cudaSetDevice(device), "cudaSetDevice");
        auto m = std::make_unique<mtfm_cuda_model>();
        m->device = device;
        m->precision = precision;
        m->cfg = *md;
        m->d = md->d_model;
        m->H = md->heads;
        m->G = md->kv_heads;
        m->dh = dh;
        m->hd = m->H * dh;
        m->gd = m->G * dh;
        m->n_layers = md->blocks * (md->target_layers + md->full_layers);
        // sources in GroupTable order (groups.hpp:20-35)
        auto add_seq = [&](int kind, int n, const int32_t* ids, const int32_t* ns, const int32_t* voc) {
            int p = 0;
            for (int i = 0; i < n; ++i) {
                SourceInfo s{};
                s.kind = kind;
                s.id = ids[i];
                s.nslot[0] = ns[i];
                s.slot0 = static_cast<int>(m->slots.size());
                for (int k = 0; k < ns[i]; ++k) m->slots.push_back({0, voc[p++], 0});
                s.k_in = ns[i] * md->d_emb;
                s.k_pad = static_cast<int>(round_up(std::max(s.k_in, 1), 8));
                m->sources.push_back(s);
                m->tasks.emplace_back();
            }
        };
        add_seq(0, sd->n_hist, sd->hist_ids, sd->hist_nslots, sd->hist_vocabs);
        add_seq(1, sd->n_rt, sd->rt_ids, sd->rt_nslots, sd->rt_vocabs);
        m->n_hist = sd->n_hist;
        m->n_rt = sd->n_rt;
        // GLN1 folded into the context-row projections (bf16 path)
        if (precision == MTFM_PRECISION_BF16) m->n_ctx_src = sd->n_hist + sd->n_rt;
        int p = 0, tp = 0;
        for (int i = 0; i < sd->n_scen; ++i) {
            SourceInfo s{};
            s.kind = 2;
            s.id = sd->scen_ids[i];
            s.nslot[0] = sd->scen_nu[i];
            s.nslot[1] = sd->scen_nc[i];
            s.nslot[2] = sd->scen_ni[i];
            s.slot0 = static_cast<int>(m->slots.size());
            const int ns = s.nslot[0] + s.nslot[1] + s.nslot[2];
            for (int k = 0; k < ns; ++k) m->slots.push_back({0, sd->scen_vocabs[p++], 0});
            s.k_in = ns * md->d_emb;
            s.k_pad = static_cast<int>(round_up(std::max(s.k_in, 1), 8));
            s.ntasks = sd->scen_ntasks[i];
            s.task0 = m->n_tasks_total;
            std::vector<std::string> names;
            for (int t = 0; t < s.ntasks; ++t) names.push_back(sd->task_names[tp++]);
            m->n_tasks_total += s.ntasks;
            m->sources.push_back(s);
            m->tasks.push_back(names);
        }
        m->n_scen = sd->n_scen;
        if (m->sources.empty()) fail(MTFM_CONFIG_ERROR, "schema set is empty");
        m->slot_param.assign(m->slots.size(), "");
        register_params(*m);
        for (size_t i = 0; i < m->params.size(); ++i) m->visible.push_back(i);
        ck(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking), "stream");
        ck(cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking), "copy stream");
        ck(cudaStreamCreateWithFlags(&m->d2h_stream, cudaStreamNonBlocking), "d2h stream");
        *out = m.release();
    });
}

mtfm_status mtfm_cuda_destroy(mtfm_cuda_model* m) {
    return guard([&] {
        if (!m) return;
        if (m->stream) cudaStreamSynchronize(m->stream);
        if (m->copy_stream) cudaStreamSynchronize(m->copy_stream);
        if (m->d2h_stream) cudaStreamSynchronize(m->d2h_stream);
        cudaStream_t st = m->stream, cs = m->copy_stream, ds = m->d2h_stream;
        for (auto& e : m->prof) {
            if (e.a) cudaEventDestroy(e.a);
            if (e.b) cudaEventDestroy(e.b);
        }
        delete m;
        if (st) cudaStreamDestroy(st);
        if (cs) cudaStreamDestroy(cs);
        if (ds) cudaStreamDestroy(ds);
    });
}

mtfm_status mtfm_cuda_set_param(mtfm_cuda_model* m, const char* name, const float* v, int64_t rows, int64_t cols) {
    return guard([&] {
        if (!m || !name || (!v && rows * cols)) fail(MTFM_CONTRACT_ERROR, "null argument");
        auto it = m->by_name.find(name);
        if (it == m->by_name.end() ||
            (m->subgraph >= 0 && m->params[it->second].owner >= 0 && m->params[it->second].owner != m->subgraph))
            fail(MTFM_CONFIG_ERROR, std::string("unknown parameter: ") + name);
        auto& p = m->params[it->second];
        if (p.rows != rows || p.cols != cols)
            fail(MTFM_DIMENSION_ERROR, std::string("shape mismatch for '") + name + "': expected " +
                                           std::to_string(p.rows) + "x" + std::to_string(p.cols));
        if (m->device_ahead) sync_host_params(*m);  // training moved the device weights past the host copies
        p.host.assign(v, v + rows * cols);
        p.set = true;
        m->finalized = false;
        m->train.reset();  // gradient segments point at the device weights about to be rebuilt
        m->srcw.clear();
        m->layers.clear();
    });
}

int64_t mtfm_cuda_num_params(const mtfm_cuda_model* m) { return m ? static_cast<int64_t>(m->visible.size()) : 0; }

const char* mtfm_cuda_param_name(const mtfm_cuda_model* m, int64_t i, int64_t* rows, int64_t* cols) {
    if (!m || i < 0 || i >= static_cast<int64_t>(m->visible.size())) return nullptr;
    const auto& p = m->params[m->visible[static_cast<size_t>(i)]];
    if (rows) *rows = p.rows;
    if (cols) *cols = p.cols;
    return p.name.c_str();
}

mtfm_status mtfm_cuda_restrict_to_scenario(mtfm_cuda_model* m, int32_t scenario_id) {
    return guard([&] {
        if (!m) fail(MTFM_CONTRACT_ERROR, "null argument");
        bool known = false;
        for (const auto& s : m->sources) known = known || (s.kind == 2 && s.id == scenario_id);
        if (!known) fail(MTFM_CONFIG_ERROR, "extract_subgraph: unknown scenario " + std::to_string(scenario_id));
        if (m->subgraph >= 0 && m->subgraph != scenario_id)
            fail(MTFM_CONTRACT_ERROR, "model is already restricted to scenario " + std::to_string(m->subgraph));
        m->subgraph = scenario_id;
        m->visible.clear();
        for (size_t i = 0; i < m->params.size(); ++i)
            if (m->params[i].owner < 0 || m->params[i].owner == scenario_id) m->visible.push_back(i);
        m->finalized = false;
        m->srcw.clear();
        m->layers.clear();
    });
}

int64_t mtfm_cuda_count_records(const mtfm_cuda_model* m, const mtfm_packed_batch* b) {
    if (!m || !b) return 0;
    int64_t n = 0;
    for (int x = 0; x < b->n_exposures; ++x) {
        const int s = source_of(*m, 2, b->exp_scenario[x], -1);
        if (s >= 0) n += m->sources[s].ntasks;
    }
    return n;
}

mtfm_status mtfm_cuda_batch_prepare(mtfm_cuda_model* m, const mtfm_packed_batch* b, int32_t only_scenario,
                                    mtfm_cuda_batch** out) {
    return guard([&] {
        if (!m || !out) fail(MTFM_CONTRACT_ERROR, "null argument");
        ck(cudaSetDevice(m->device), "cudaSetDevice");
        auto B = std::make_unique<mtfm_cuda_batch>();
        prepare(*m, b, only_scenario, *B);
        *out = B.release();
    });
}

mtfm_status mtfm_cuda_batch_update(mtfm_cuda_model* m, mtfm_cuda_batch* b, const mtfm_packed_batch* pb,
                                   int32_t only_scenario) {
    return guard([&] {
        if (!m || !b || !pb) fail(MTFM_CONTRACT_ERROR, "null argument");
        if (b->m && b->m != m) fail(MTFM_CONTRACT_ERROR, "batch belongs to another model");
        ck(cudaSetDevice(m->device), "cudaSetDevice");
        prepare(*m, pb, only_scenario, *b);
    });
}

mtfm_status mtfm_cuda_batch_run(mtfm_cuda_model* m, mtfm_cuda_batch* b) {
    return guard([&] {
        if (!m || !b) fail(MTFM_CONTRACT_ERROR, "null argument");
        if (!m->finalized) fail(MTFM_CONTRACT_ERROR, "parameters changed after prepare; prepare the batch again");
        ck(cudaSetDevice(m->device), "cudaSetDevice");
        // prepare() returns once its uploads completed: a stream wait is only needed if they
        // have not (the wait would also cut the programmatic launch overlap with the previous forward)
        if (cudaEventQuery(b->ev_h2d) != cudaSuccess) ck(cudaStreamWaitEvent(m->stream, b->ev_h2d, 0), "wait uploads");
        if (m->precision == MTFM_PRECISION_BF16)
            run_forward<__nv_bfloat16>(*m, *b);
        else
            run_forward<float>(*m, *b);
        ck(cudaEventRecord(b->ev_done, m->stream), "record forward");
        b->ran = true;
        m->stats.kernel_launches = b->launches;
        m->stats.tokens = b->rows;
        m->stats.targets = b->n_exp;
        m->stats.records = b->n_records;
    });
}

mtfm_status mtfm_cuda_batch_results(mtfm_cuda_model* m, mtfm_cuda_batch* b, mtfm_records* out) {
    return guard([&] {
        if (!m || !b) fail(MTFM_CONTRACT_ERROR, "null argument");
        results(*m, *b, out);
        // algorithmic FLOPs; visible-key sums read back by results()
        const unsigned long long h[2] = {b->sum_c_ctx, b->sum_c_t};
        if (m->profiling)
            for (size_t i = 0; i < m->prof_n; ++i) {
                float ms = 0;
                ck(cudaEventElapsedTime(&ms, m->prof[i].a, m->prof[i].b), "event time");
                m->prof[i].ms = ms;
            }
        const double d = m->d, hd = m->hd, gd = m->gd, R = static_cast<double>(b->rows), T = static_cast<double>(b->n_exp);
        double proj = 0, attn = 0;
        for (const auto& L : m->layers) {
            if (L->target) {
                proj += T * d * 2 * hd + R * d * 2 * gd + T * hd * d;
                attn += 2.0 * hd * static_cast<double>(h[1]);
            } else {
                proj += R * d * (2 * hd + 2 * gd) + R * hd * d;
                attn += 2.0 * hd * static_cast<double>(h[0] + h[1]);
            }
        }
        double tok = 0;
        for (size_t s = 0; s < m->sources.size(); ++s)
            tok += static_cast<double>(b->src_cnt[s]) * (m->sources[s].k_in * 2.0 * d + 2.0 * d * d);
        const double heads = T * (static_cast<double>(m->cfg.experts) * d * m->cfg.d_expert) +
                             static_cast<double>(b->n_records) * (d * m->cfg.experts + m->cfg.d_expert);
        m->stats.algorithmic_flops = 2.0 * (proj + attn + tok + heads);
        m->stats.attention_flops = 2.0 * attn;
    });
}

mtfm_status mtfm_cuda_batch_free(mtfm_cuda_batch* b) {
    return guard([&] {
        if (!b) return;
        if (b->m && b->m->stream) cudaStreamSynchronize(b->m->stream);
        if (b->m && b->m->copy_stream) cudaStreamSynchronize(b->m->copy_stream);
        if (b->m && b->m->d2h_stream) cudaStreamSynchronize(b->m->d2h_stream);
        delete b;
    });
}

mtfm_status mtfm_cuda_forward(mtfm_cuda_model* m, const mtfm_packed_batch* b, int32_t only_scenario,
                              mtfm_records* out) {
    mtfm_status s = guard([&] {
        if (!m) fail(MTFM_CONTRACT_ERROR, "null argument");
        ck(cudaSetDevice(m->device), "cudaSetDevice");
        if (!m->ws) m->ws = std::make_unique<mtfm_cuda_batch>();  // device buffers only grow
        prepare(*m, b, only_scenario, *m->ws);
    });
    if (s == MTFM_OK) s = mtfm_cuda_batch_run(m, m->ws.get());
    if (s == MTFM_OK) s = mtfm_cuda_batch_results(m, m->ws.get(), out);
    return s;
}

mtfm_status mtfm_cuda_train_step(mtfm_cuda_model* m, mtfm_cuda_batch* b, const int32_t* labels, int32_t max_tasks,
                                 const mtfm_train_config* cfg, mtfm_train_result* out) {
    return guard([&] {
        if (!m || !b || !cfg || (!labels && b->n_exp > 0)) fail(MTFM_CONTRACT_ERROR, "null argument");
        if (b->m != m) fail(MTFM_CONTRACT_ERROR, "batch belongs to another model");
        if (!m->finalized) fail(MTFM_CONTRACT_ERROR, "parameters changed after prepare; prepare the batch again");
        ck(cudaSetDevice(m->device), "cudaSetDevice");
        train_step(*m, *b, labels, max_tasks, *cfg, out);
    });
}

mtfm_status mtfm_cuda_get_param(mtfm_cuda_model* m, const char* name, float* host, int64_t rows, int64_t cols) {
    return guard([&] {
        if (!m || !name || !host) fail(MTFM_CONTRACT_ERROR, "null argument");
        auto it = m->by_name.find(name);
        if (it == m->by_name.end()) fail(MTFM_CONFIG_ERROR, std::string("unknown parameter: ") + name);
        const auto& p = m->params[it->second];
        if (p.rows != rows || p.cols != cols) fail(MTFM_DIMENSION_ERROR, std::string("shape mismatch for '") + name + "'");
        if (!m->finalized || m->views.empty() || !m->views[it->second].buf) {
            if (!p.set) fail(MTFM_CONFIG_ERROR, std::string("parameter not set: ") + name);
            std::memcpy(host, p.host.data(), static_cast<size_t>(rows * cols) * 4);
            return;
        }
        const ParamView& v = m->views[it->second];
        ck(cudaSetDevice(m->device), "cudaSetDevice");
        ck(cudaStreamSynchronize(m->stream), "sync");
        ck(cudaMemcpy2D(host, static_cast<size_t>(cols) * 4, v.buf->as<float>() + v.off, static_cast<size_t>(v.ld) * 4,
                        static_cast<size_t>(cols) * 4, static_cast<size_t>(rows), cudaMemcpyDeviceToHost),
           "D2H param");
    });
}

mtfm_status mtfm_cuda_get_grad(mtfm_cuda_model* m, const char* name, float* host, int64_t rows, int64_t cols) {
    return guard([&] {
        if (!m || !name || !host) fail(MTFM_CONTRACT_ERROR, "null argument");
        if (!m->train) fail(MTFM_CONTRACT_ERROR, "no training step has run");
        auto it = m->by_name.find(name);
        if (it == m->by_name.end()) fail(MTFM_CONFIG_ERROR, std::string("unknown parameter: ") + name);
        const auto& p = m->params[it->second];
        if (p.rows != rows || p.cols != cols) fail(MTFM_DIMENSION_ERROR, std::string("shape mismatch for '") + name + "'");
        const ParamView& v = m->views[it->second];
        const float* g = m->train->grad_of(*v.buf);
        if (!g) fail(MTFM_CONTRACT_ERROR, "parameter has no gradient segment");
        ck(cudaSetDevice(m->device), "cudaSetDevice");
        ck(cudaStreamSynchronize(m->stream), "sync");
        ck(cudaMemcpy2D(host, static_cast<size_t>(cols) * 4, g + v.off, static_cast<size_t>(v.ld) * 4,
                        static_cast<size_t>(cols) * 4, static_cast<size_t>(rows), cudaMemcpyDeviceToHost),
           "D2H grad");
    });
}

mtfm_status mtfm_nccl_unique_id(void* out128) {
    return guard([&] {
        if (!out128) fail(MTFM_CONTRACT_ERROR, "null argument");
        nccl_check(nccl().get_id(out128), "ncclGetUniqueId");
    });
}

mtfm_status mtfm_cuda_dp_init(mtfm_cuda_model* m, int32_t nranks, int32_t rank, const void* unique_id128) {
    return guard([&] {
        if (!m || !unique_id128) fail(MTFM_CONTRACT_ERROR, "null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(MTFM_CONFIG_ERROR, "bad rank / world size");
        ck(cudaSetDevice(m->device), "cudaSetDevice");
        finalize(*m);
        if (m->nccl) fail(MTFM_CONTRACT_ERROR, "data-parallel group already initialised");
        NcclId id;
        std::memcpy(id.b, unique_id128, 128);
        using InitFn = int (*)(void**, int, NcclId, int);
        auto init = reinterpret_cast<InitFn>(nccl().init_rank);
        nccl_check(init(&m->nccl, nranks, id, rank), "ncclCommInitRank");
        m->dp_ranks = nranks;
        m->dp_rank = rank;
    });
}

mtfm_status mtfm_cuda_prune_projections(mtfm_cuda_model* m, mtfm_prune_report* rep) {
    return guard([&] {
        if (!m) fail(MTFM_CONTRACT_ERROR, "null argument");
        ck(cudaSetDevice(m->device), "cudaSetDevice");
        finalize(*m);
        if (m->device_ahead) sync_host_params(*m);
        DevBuf zc;
        zc.alloc(8);
        ck(cudaMemsetAsync(zc.p, 0, 8, m->stream), "memset");
        mtfm_prune_report r{};
        // is_projection_param (prune.hpp:83-90): hta/.../{f1_w, fuq_w, fkv_w, f2_w}, in registration order
        for (auto& Lp : m->layers) {
            auto& L = *Lp;
            std::vector<std::pair<DevBuf*, std::pair<int, int>>> mats;
            const int n1 = L.target ? 2 * m->hd : 2 * m->hd + 2 * m->gd;
            mats.push_back({&L.w1, {m->d, n1}});
            if (L.target) mats.push_back({&L.wkv, {m->d, 2 * m->gd}});
            mats.push_back({&L.f2, {m->hd, m->d}});
            for (auto& [buf, rc] : mats) {
                const int rows = rc.first, cols = rc.second;
                const long long n = static_cast<long long>(rows / 4) * cols;
                if (n > 0)
                    prune_2_4_kernel<<<static_cast<int>(std::min<long long>(cdiv(n, 256), 148 * 8)), 256, 0, m->stream>>>(
                        buf->as<float>(), rows, cols, zc.as<unsigned long long>());
                r.groups_covered += n;
                r.exempt_tail_rows += rows - (rows / 4) * 4;
                ++r.pruned_params;
            }
        }
        ck(cudaGetLastError(), "prune");
        unsigned long long z = 0;
        ck(cudaMemcpyAsync(&z, zc.p, 8, cudaMemcpyDeviceToHost, m->stream), "D2H");
        ck(cudaStreamSynchronize(m->stream), "prune");
        r.zeros_written = static_cast<int64_t>(z);
        // the pruned fp32 weights become the parameters; bf16 / folded copies rebuild on next use
        m->device_ahead = true;
        sync_host_params(*m);
        m->finalized = false;
        m->srcw.clear();
        m->layers.clear();
        m->train.reset();
        if (rep) *rep = r;
    });
}

mtfm_status mtfm_cuda_set_sparse_mma(mtfm_cuda_model* m, int32_t mode, int32_t* active) {
    return guard([&] {
        if (!m) fail(MTFM_CONTRACT_ERROR, "null argument");
        if (mode < 0 || mode > 2) fail(MTFM_CONTRACT_ERROR, "sparse MMA mode must be 0, 1 or 2");
        ck(cudaSetDevice(m->device), "cudaSetDevice");
        if (m->device_ahead) sync_host_params(*m);
        const int old = m->sparse_mode;
        m->sparse_mode = mode;
        m->finalized = false;
        m->srcw.clear();
        m->layers.clear();
        try {
            finalize(*m);
        } catch (...) {
            m->sparse_mode = old;  // the model stays usable in its previous mode
            m->finalized = false;
            m->srcw.clear();
            m->layers.clear();
            throw;
        }
        if (active) *active = m->bias_tiles.sparse.active && m->precision == MTFM_PRECISION_BF16 ? 1 : 0;
    });
}

mtfm_status mtfm_cuda_set_profiling(mtfm_cuda_model* m, int32_t on) {
    return guard([&] {
        if (!m) fail(MTFM_CONTRACT_ERROR, "null argument");
        m->profiling = on != 0;
    });
}

int64_t mtfm_cuda_profile_count(const mtfm_cuda_model* m) { return m ? static_cast<int64_t>(m->prof_n) : 0; }

const char* mtfm_cuda_profile_entry(const mtfm_cuda_model* m, int64_t i, double* ms, double* flops, double* bytes) {
    if (!m || i < 0 || i >= static_cast<int64_t>(m->prof_n)) return nullptr;
    const auto& e = m->prof[static_cast<size_t>(i)];
    if (ms) *ms = e.ms;
    if (flops) *flops = e.flops;
    if (bytes) *bytes = e.bytes;
    return e.name.c_str();
}

void* mtfm_cuda_stream(mtfm_cuda_model* m) { return m ? static_cast<void*>(m->stream) : nullptr; }

mtfm_status mtfm_cuda_last_stats(const mtfm_cuda_model* m, mtfm_run_stats* out) {
    return guard([&] {
        if (!m || !out) fail(MTFM_CONTRACT_ERROR, "null argument");
        *out = m->stats;
    });
}

mtfm_status mtfm_cuda_debug_gemm(const void* A, const void* Bt, const float* bias, void* out, int64_t M, int64_t N,
                                 int64_t K, int32_t epi, void* stream) {
    return guard([&] {
        long long L = 0;
        TcProblem tp{static_cast<const __nv_bfloat16*>(A), K, static_cast<const __nv_bfloat16*>(Bt), K,
                     static_cast<int>(M), static_cast<int>(N), static_cast<int>(K), epi, bias, out, N, nullptr, 0,
                     epi == EPI_RESID_F32 ? static_cast<const float*>(out) : nullptr};
        static BiasTiles BT;
        BT.rebuild = true;
        run_gemm_tc({tp}, static_cast<cudaStream_t>(stream), L, BT);
    });
}

int64_t mtfm_cuda_debug_fetch(mtfm_cuda_model* m, mtfm_cuda_batch* b, const char* which, void* dst, int64_t max_bytes) {
    if (!m || !b || !which || !dst) return -1;
    cudaStreamSynchronize(m->stream);
    const std::string w = which;
    auto cp = [&](const DevBuf& src, size_t bytes) -> int64_t {
        bytes = std::min<size_t>(bytes, static_cast<size_t>(max_bytes));
        if (cudaMemcpy(dst, src.p, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
        return static_cast<int64_t>(bytes);
    };
    const size_t R = static_cast<size_t>(b->rows);
    if (w == "x") return cp(m->act[mtfm::ACT_X], R * m->d * 4);
    if (w == "src") return cp(b->r_src, R * 4);
    if (w == "item") return cp(b->r_item, R * 4);
    if (w == "prefix") return cp(b->r_prefix, R * 4);
    if (w == "self") return cp(b->r_self, R * 4);
    if (w == "scale") return cp(b->r_scale, R * 4);
    if (w == "src_rows") return cp(b->r_src_rows, R * 4);
    if (w == "t_exp_ref") return cp(b->t_exp_ref, static_cast<size_t>(b->n_exp) * 4);
    return -1;
}

}  // extern "C"
