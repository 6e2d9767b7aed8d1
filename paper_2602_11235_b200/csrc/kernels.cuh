// kernels.cuh — device data structures and launchers of the non-tensor-core
// kernels (planning, embedding gather, group LayerNorm, gate, heads) and of
// the fp32 SIMT check-mode GEMM / attention.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace mtfm {

// One tokenizer source == one GLN group (groups.hpp:20-35 registration order:
// historical sequence schemas, realtime schemas, scenarios).
struct SourceInfo {
    int kind;        // 0 historical, 1 realtime, 2 scenario
    int id;          // seq_id or scenario_id
    int nslot[3];    // sequences: {slots,0,0}; scenarios: {user, cross, item}
    int slot0;       // first entry in the flat slot table
    int k_in;        // total slots * d_emb
    int k_pad;       // k_in rounded up to 64 (zero padded)
    int ntasks;      // scenarios only
    int task0;       // first global task index (scenario order)
};

struct SlotInfo {
    long long emb_off;  // element offset of the table in the flat embedding buffer
    int vocab;
    int pad;
};

struct DevBatch {
    int n_users, n_seqs, n_events, n_exposures;
    const long long* user_id;
    const int* seq_off;
    const uint8_t* seq_kind;
    const int* seq_schema;
    const int* ev_off;
    const long long* ev_ts;
    const int* ev_feat_off;
    const int* ev_feats;
    const int* exp_off;
    const int* exp_scenario;
    const long long* exp_ts;
    const int* exp_feat_off;
    const int* exp_blk;
    const int* exp_feats;
};

// Per-row outputs of the plan (rows: [0, n_events) context, then T rows).
struct RowMeta {
    int* src;        // tokenizer source == GLN group
    int* item;       // event index (context rows) / exposure index (T rows)
    int* prefix;     // visible context keys
    float* scale;    // attention row scale (hta.hpp:53-67)
    int* self;       // own row for T rows, -1 otherwise
    int* keybase;    // row of the user's first context key
    int* src_rows;   // rows grouped by source (positions from src_pos)
    // T rows only (indexed t in [0, n_exposures))
    int* t_user;
    int* t_exp_ref;  // index into the user's exposure list
    int* t_scen;     // scenario id
    long long* t_rec0;   // record index of task 0
    int* t_rec_stride;   // rows of the same (user, scenario)
};

struct PlanArgs {
    DevBatch b;
    const SourceInfo* src;
    const SlotInfo* slots;
    int n_src, n_hist, n_rt;
    int norm;                    // mtfm_attn_norm
    int only_scenario;
    const long long* us_off;     // [n_users][n_src] start of user u's rows in source s's list
    const long long* src_base;   // [n_src] start of source s's list in src_rows
    const long long* rec_off;    // [n_users]
    RowMeta rm;
    unsigned long long* err;     // min error key (see plan.cu)
    int max_sort;                // smem capacity (elements, power of two)
    // users whose sort does not fit max_sort: [sort_off[u], sort_off[u+1]) of sort_scratch
    // (2 x capacity elements) is their sort area in global memory; null when none
    const long long* sort_off;   // [n_users + 1] or null
    long long* sort_scratch;
};

void launch_plan(const PlanArgs& a, int smem_elems, cudaStream_t st);

// Embedding gather into the per-source tokenizer input matrices.
// false when there are more than 32 token sources (nothing launched)
template <typename T>
bool launch_gather(const DevBatch& b, const SourceInfo* src_dev, const SlotInfo* slots_dev, const RowMeta& rm,
                   const long long* src_base_dev, const long long* src_cnt_dev, const long long* emb_base_dev,
                   const T* tables, int d_emb, int n_src, long long total_rows, int max_kpad, T* out,
                   cudaStream_t st);

// Group LayerNorm: out[r - r0] = ((x - mu) / sqrt(var + eps)) * gain[g] + bias[g]
template <typename T>
void launch_gln(const float* x, long long ldx, long long r0, long long n_rows, int d, const int* row_src,
                const float* gain, const float* bias, float eps, T* out, long long ldo, cudaStream_t st);

// The same rows normalised once and written with L different (gain, bias)
// pairs: the GLN1 inputs of a block's target layers for the context rows, which
// those layers never modify (hta.hpp:158-184 only update T rows).
constexpr int kMaxGlnCopies = 8;
struct GlnCopies {
    const float* gain[kMaxGlnCopies];
    const float* bias[kMaxGlnCopies];
    void* out[kMaxGlnCopies];
    int n;
    const int* in_rows;  // optional: output row j normalises x row in_rows[j] (source-ordered copies)
};
void launch_gln_multi_bf16(const float* x, long long ldx, long long n_rows, int d, const int* row_src,
                           const GlnCopies& c, float eps, long long ldo, cudaStream_t st);

// Gate: out[r] = gln(a[r]) * u[r]   (hta.hpp:153,179)
template <typename T>
void launch_gate(const T* a, long long lda, const T* u, long long ldu, long long n_rows, int d,
                 const int* row_src_of_rows, const float* gain, const float* bias, float eps, T* out,
                 long long ldo, cudaStream_t st);

// f32 -> bf16 copy of rows (head input in the fast path)
void launch_to_bf16(const float* x, long long n_rows, int d, __nv_bfloat16* out, long long ldo, cudaStream_t st);

struct HeadArgs {
    const float* y;        // [n_t][ldy]: experts (E*de) then gates (n_tasks_total*E), pre-bias
    long long ldy;
    const float* exp_bias; // [E*de]
    const float* gate_bias;// [n_tasks_total*E]
    const float* tower_w;  // [n_tasks_total][de]
    const float* tower_b;  // [n_tasks_total]
    int E, de;
    const SourceInfo* src;
    int n_src;
    const RowMeta* rm_unused;
    const int* t_scen;
    const int* t_user;
    const int* t_exp_ref;
    const long long* t_rec0;
    const int* t_rec_stride;
    const long long* user_id;
    long long n_t;
    bool precise;
    // records
    long long* rec_user;
    int* rec_scen;
    int* rec_exp;
    int* rec_task;
    float* rec_logit;
    double* rec_prob;
};
void launch_heads(const HeadArgs& a, cudaStream_t st, int n_tasks_total);  // n_tasks_total: rows of tower_w

// ---------------------------------------------------------------- SIMT (check mode)
struct SimtGemm {
    const float* A;
    long long lda;
    const float* W;   // [K][N] row-major (reference layout)
    int M, N, K;
    const float* bias;
    int epi;          // GemmEpi
    void* out;
    long long ldo;
    const int* row_map;
    long long row_offset;
    const float* resid;
};
void launch_gemm_simt(const SimtGemm* probs, int n, cudaStream_t st);

struct SimtAttn {
    const float* q;   // Q matrix
    long long ldq;
    int q_col0;
    const float* kv;
    long long ldkv;
    int k_col0, v_col0;
    long long n_q;    // query rows
    const int* prefix;
    const float* scale;
    const int* self;
    const int* keybase;
    int heads, kv_heads, dh;
    float* out;
    long long ldo;
};
void launch_attn_simt(const SimtAttn& a, cudaStream_t st);

}  // namespace mtfm
