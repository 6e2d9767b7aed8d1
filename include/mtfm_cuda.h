/* mtfm_cuda.h — C ABI of the B200-native MTFM forward (libmtfm_cuda.so).
 *
 * Drop-in boundary for the reference's batched scoring path. Every entry point
 * replaces one piece of the reference C++ model API (paths relative to
 * /root/reference/proj):
 *
 *   mtfm_cuda_create        Model<Real>::build with the structs of
 *                           include/mtfm/model_config.hpp:39-88 (HTAConfig,
 *                           ModelConfig) and the SchemaSet of model.hpp:117-136.
 *   mtfm_cuda_set_param     ParamStore<Real>::at(name).value (params.hpp:22-132):
 *                           names and (rows, cols) exactly as registered by
 *                           Model::register_params (model.hpp:371-463).
 *   mtfm_cuda_forward       Model<Real>::forward_sample / forward_with /
 *                           forward_scoped (model.hpp:244-312) applied to every
 *                           UserSample of a packed batch; records come back in
 *                           exactly the order of the concatenated per-sample
 *                           forward_sample results (records.hpp:10-19).
 *   mtfm_cuda_batch_*       the same forward split into prepare / run /
 *                           results so callers can keep batches resident in
 *                           HBM and time the device work alone.
 *   mtfm_cuda_last_error    the what() of the exception the reference throws;
 *                           the status code names its type (errors.hpp:9-40).
 *
 * Input: a packed jagged batch of UserSamples (schema.hpp:72-98) as flat CSR
 * arrays (no sorting is done by the caller; token planning runs on the GPU):
 *   users      user_id[n_users]; seq_off[n_users+1] -> sequences;
 *              exp_off[n_users+1] -> exposures
 *   sequences  seq_kind[s] (0 historical, 1 realtime), seq_schema[s],
 *              ev_off[n_seqs+1] -> events. A user's sequences keep the
 *              sample's list order (historical list, then realtime list).
 *   events     ev_ts[e], ev_feat_off[n_events+1] -> ev_feats (item_features)
 *   exposures  exp_scenario[x], exp_ts[x], exp_blk[3x..3x+2] = number of
 *              user/cross/item ids, exp_feat_off[n_exposures+1] -> exp_feats
 *              (user ids, then cross ids, then item ids)
 * Offsets are int32 (a batch holds < 2^31 events / feature ids).
 *
 * Output: one record per (T token, task of its scenario) in reference order:
 * user-major, then scenario id ascending, then task order, then the T tokens'
 * canonical (timestamp, scenario, index) order (heads.hpp:54-97,
 * model.hpp:284-311). probability = clamp(sigmoid(logit), 1e-12, 1-1e-12).
 * Labels are host-side data and are not part of the device path.
 *
 * Threading: one model handle per device, bound to one CUDA stream, not
 * re-entrant per handle (the reference forward is const and re-entrant; use
 * one handle per host thread / device).
 */
#ifndef MTFM_CUDA_H_
#define MTFM_CUDA_H_

#include <stdint.h>

#if defined(__GNUC__)
#define MTFM_API __attribute__((visibility("default")))
#else
#define MTFM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MTFM_OK = 0,
    MTFM_CONFIG_ERROR = 1,    /* config_error    errors.hpp:10 */
    MTFM_INTEGRITY_ERROR = 2, /* integrity_error errors.hpp:15 */
    MTFM_DIMENSION_ERROR = 3, /* dimension_error errors.hpp:20 */
    MTFM_PARSE_ERROR = 4,     /* parse_error     errors.hpp:25 */
    MTFM_LOOKUP_ERROR = 5,    /* lookup_error    errors.hpp:33 */
    MTFM_CONTRACT_ERROR = 6,  /* contract_error  errors.hpp:38 */
    MTFM_CUDA_ERROR = 7       /* device / driver failure (no reference analogue) */
} mtfm_status;

/* AttnNorm, model_config.hpp:18 */
typedef enum { MTFM_NORM_VALID = 0, MTFM_NORM_SEQLEN = 1, MTFM_NORM_NONE = 2 } mtfm_attn_norm;

typedef enum {
    MTFM_PRECISION_BF16 = 0,      /* tcgen05 bf16 tensor cores, fp32 accumulate / residual */
    MTFM_PRECISION_FP32_CHECK = 1 /* fp32 SIMT everywhere: the <=1e-4 parity mode */
} mtfm_precision;

/* ModelConfig + HTAConfig, model_config.hpp:39-88 */
typedef struct {
    int32_t d_model, blocks, target_layers, full_layers, heads, kv_heads;
    int32_t norm; /* mtfm_attn_norm */
    double eps;
    int32_t d_emb, experts, d_expert;
} mtfm_model_desc;

/* SchemaSet (model.hpp:117-136) flattened: SequenceSchema / ScenarioSchema
 * (schema.hpp:18-41) in registration order. */
typedef struct {
    int32_t n_hist;
    const int32_t* hist_ids;    /* [n_hist] seq_id */
    const int32_t* hist_nslots; /* [n_hist] */
    const int32_t* hist_vocabs; /* concatenated feature_vocabs */
    int32_t n_rt;
    const int32_t* rt_ids;
    const int32_t* rt_nslots;
    const int32_t* rt_vocabs;
    int32_t n_scen;
    const int32_t* scen_ids;    /* [n_scen] scenario_id */
    const int32_t* scen_nu;     /* user / cross / item slot counts */
    const int32_t* scen_nc;
    const int32_t* scen_ni;
    const int32_t* scen_vocabs; /* per scenario: user, cross, item vocabs */
    const int32_t* scen_ntasks; /* [n_scen] */
    const char* const* task_names; /* concatenated task names, scenario order */
} mtfm_schema_desc;

typedef struct {
    int32_t n_users, n_seqs, n_events, n_exposures;
    int64_t n_ev_feats, n_exp_feats;
    const int64_t* user_id;
    const int32_t* seq_off;
    const uint8_t* seq_kind;
    const int32_t* seq_schema;
    const int32_t* ev_off;
    const int64_t* ev_ts;
    const int32_t* ev_feat_off;
    const int32_t* ev_feats;
    const int32_t* exp_off;
    const int32_t* exp_scenario;
    const int64_t* exp_ts;
    const int32_t* exp_feat_off;
    const int32_t* exp_blk;
    const int32_t* exp_feats;
} mtfm_packed_batch;

/* Caller-owned record buffers (capacity >= mtfm_cuda_count_records()). */
typedef struct {
    int64_t capacity;
    int64_t n_records;        /* written */
    int64_t* user_id;         /* PredictionRecord::user_id */
    int32_t* scenario_id;     /* PredictionRecord::scenario_id */
    int32_t* exposure_index;  /* PredictionRecord::exposure_index */
    int32_t* task_index;      /* index into the scenario's task list */
    float* logit;             /* pre-sigmoid head output (may be NULL) */
    double* probability;      /* PredictionRecord::probability */
} mtfm_records;

typedef struct mtfm_cuda_model mtfm_cuda_model;
typedef struct mtfm_cuda_batch mtfm_cuda_batch;

typedef struct {
    int64_t kernel_launches;     /* kernels enqueued by the last run */
    double algorithmic_flops;    /* SURVEY 8(d) FLOP model of the last run */
    double attention_flops;      /* mask-aware attention part of it */
    int64_t tokens, targets, records;
} mtfm_run_stats;

MTFM_API const char* mtfm_cuda_last_error(void);
MTFM_API const char* mtfm_cuda_version(void);

MTFM_API mtfm_status mtfm_cuda_create(int device, const mtfm_model_desc* model, const mtfm_schema_desc* schemas,
                             int32_t precision, mtfm_cuda_model** out);
MTFM_API mtfm_status mtfm_cuda_destroy(mtfm_cuda_model* m);

/* Unknown name -> MTFM_CONFIG_ERROR (ParamStore::index_of, params.hpp:48-52);
 * wrong shape -> MTFM_DIMENSION_ERROR. */
MTFM_API mtfm_status mtfm_cuda_set_param(mtfm_cuda_model* m, const char* name, const float* host_values, int64_t rows,
                                int64_t cols);
/* Number of parameters the model registers and their names (registration order). */
MTFM_API int64_t mtfm_cuda_num_params(const mtfm_cuda_model* m);
MTFM_API const char* mtfm_cuda_param_name(const mtfm_cuda_model* m, int64_t i, int64_t* rows, int64_t* cols);

/* Scenario-subgraph deployment (extract_subgraph, subgraph.hpp:25-42): after
 * this call the handle registers only the shared parameters and scenario_id's
 * own (names::owner_scenario, model.hpp:71-87) — num_params / param_name list
 * exactly the subgraph's ParamStore, set_param on another scenario's parameter
 * is MTFM_CONFIG_ERROR — and every forward is scoped to scenario_id
 * (infer_request, subgraph.hpp:47-62: another only_scenario is
 * MTFM_INTEGRITY_ERROR). Unknown scenario -> MTFM_CONFIG_ERROR. */
MTFM_API mtfm_status mtfm_cuda_restrict_to_scenario(mtfm_cuda_model* m, int32_t scenario_id);

/* Records the batch will produce (host-side count: sum over exposures of the
 * task count of their scenario; exposures of unknown scenarios count 0). */
MTFM_API int64_t mtfm_cuda_count_records(const mtfm_cuda_model* m, const mtfm_packed_batch* b);

/* One-call forward: host batch in, host records out (H2D + device + D2H).
 * only_scenario >= 0 restricts binding to one scenario like forward_scoped
 * (model.hpp:265, subgraph.hpp:47-62); -1 = all scenarios. */
MTFM_API mtfm_status mtfm_cuda_forward(mtfm_cuda_model* m, const mtfm_packed_batch* b, int32_t only_scenario,
                              mtfm_records* out);

/* Split forward. prepare: host layout + H2D of the batch on the model's copy
 * stream (returns once the host arrays have been read: they may be released;
 * the kernels of other batches keep running meanwhile). update: the same into
 * an existing batch object, reusing its device buffers (ordered after that
 * batch's previous forward). run: enqueues every kernel on the model stream
 * behind this batch's uploads, no host synchronisation. results: waits for
 * this batch's forward only, then copies the records (and reports
 * device-detected errors). Two batch objects used alternately pipeline one
 * batch's host work and transfers with the other's kernels. */
MTFM_API mtfm_status mtfm_cuda_batch_prepare(mtfm_cuda_model* m, const mtfm_packed_batch* b, int32_t only_scenario,
                                    mtfm_cuda_batch** out);
MTFM_API mtfm_status mtfm_cuda_batch_update(mtfm_cuda_model* m, mtfm_cuda_batch* batch, const mtfm_packed_batch* b,
                                   int32_t only_scenario);
MTFM_API mtfm_status mtfm_cuda_batch_run(mtfm_cuda_model* m, mtfm_cuda_batch* b);
MTFM_API mtfm_status mtfm_cuda_batch_results(mtfm_cuda_model* m, mtfm_cuda_batch* b, mtfm_records* out);
MTFM_API mtfm_status mtfm_cuda_batch_free(mtfm_cuda_batch* b);

/* The CUDA stream (cudaStream_t) the model enqueues on. */
MTFM_API void* mtfm_cuda_stream(mtfm_cuda_model* m);
MTFM_API mtfm_status mtfm_cuda_last_stats(const mtfm_cuda_model* m, mtfm_run_stats* out);

/* Per-stage profiling: when on, batch_run brackets every kernel stage with
 * CUDA events; after batch_results, entry i reports the stage name, its
 * device time (ms) and its algorithmic FLOPs / bytes. */
MTFM_API mtfm_status mtfm_cuda_set_profiling(mtfm_cuda_model* m, int32_t on);
MTFM_API int64_t mtfm_cuda_profile_count(const mtfm_cuda_model* m);
MTFM_API const char* mtfm_cuda_profile_entry(const mtfm_cuda_model* m, int64_t i, double* ms, double* flops,
                                             double* bytes);

/* Test hook: one plain tensor-core GEMM on device buffers, out = epi(A[M][K] .
 * Bt[N][K]^T + bias) with epi 0 = silu -> bf16, 1 = f32, 2 = f32 += (residual
 * in out), 3 = bf16. A, Bt bf16 row-major; enqueued on `stream`. */
MTFM_API mtfm_status mtfm_cuda_debug_gemm(const void* A, const void* Bt, const float* bias, void* out, int64_t M,
                                          int64_t N, int64_t K, int32_t epi, void* stream);

/* Debug / test hooks over device buffers of the last run (row-major). which:
 * "x" final activations [rows][d] f32, "plan" int32 [rows][4] = (source,
 * item, prefix, self), "scale" f32 [rows]. Returns elements copied. */
MTFM_API int64_t mtfm_cuda_debug_fetch(mtfm_cuda_model* m, mtfm_cuda_batch* b, const char* which, void* host_dst,
                              int64_t max_bytes);

/* ---------------------------------------------------------------- user aggregation
 * aggregate_users (datagen.cpp:171-216, datagen.hpp:55-61) on the device: a
 * (user_id, Exposure) stream is grouped per user with exposures ordered by
 * scenario id ascending and stream order within a scenario, users ascending,
 * joined with each user's shared historical / realtime sequences from the
 * store. Output: the packed jagged batch of the users that have exposures
 * (mtfm_packed_batch layout), bit-exact with the reference's UserSample list.
 * Unknown scenario / user -> MTFM_INTEGRITY_ERROR naming the first offending
 * stream element (scenario checked first, datagen.cpp:177-183). The store is
 * a std::map<int64_t, UserContext> flattened in its iteration order (user ids
 * strictly ascending; violations -> MTFM_CONTRACT_ERROR) as a packed batch
 * with no exposures. Labels are host data: exp_src maps every output
 * exposure back to its stream index. */
typedef struct {
    int32_t n_exposures;
    int64_t n_feats;
    const int64_t* user_id;   /* [n] stream order */
    const int32_t* scenario;  /* [n] Exposure::scenario_id */
    const int64_t* ts;        /* [n] Exposure::timestamp */
    const int32_t* feat_off;  /* [n+1] -> feats (user ids, cross ids, item ids) */
    const int32_t* blk;       /* [3n] user / cross / item id counts */
    const int32_t* feats;
} mtfm_exposure_stream;

typedef struct { /* AggregationReport (datagen.hpp:44-53) */
    int64_t n_exposure_records, n_user_samples;
    double compression_ratio;
} mtfm_aggregation_report;

typedef struct {
    int64_t n_users, n_seqs, n_events, n_exposures, n_ev_feats, n_exp_feats;
} mtfm_packed_sizes;

typedef struct { /* writable mtfm_packed_batch arrays (+ exp_src, may be NULL) */
    int64_t* user_id;
    int32_t* seq_off;
    uint8_t* seq_kind;
    int32_t* seq_schema;
    int32_t* ev_off;
    int64_t* ev_ts;
    int32_t* ev_feat_off;
    int32_t* ev_feats;
    int32_t* exp_off;
    int32_t* exp_scenario;
    int64_t* exp_ts;
    int32_t* exp_feat_off;
    int32_t* exp_blk;
    int32_t* exp_feats;
    int32_t* exp_src;
} mtfm_packed_buffers;

typedef struct mtfm_cuda_aggregate mtfm_cuda_aggregate;

/* scenario_ids: the schema context's scenario ids, strictly ascending
 * (Dataset::has_scenario). The result stays on `device` until freed. */
MTFM_API mtfm_status mtfm_cuda_aggregate_users(int device, const int32_t* scenario_ids, int32_t n_scenarios,
                                               const mtfm_exposure_stream* stream, const mtfm_packed_batch* store,
                                               mtfm_cuda_aggregate** out, mtfm_aggregation_report* report);
MTFM_API mtfm_status mtfm_cuda_aggregate_sizes(const mtfm_cuda_aggregate* a, mtfm_packed_sizes* sizes);
MTFM_API mtfm_status mtfm_cuda_aggregate_fetch(mtfm_cuda_aggregate* a, const mtfm_packed_buffers* out);
MTFM_API mtfm_status mtfm_cuda_aggregate_free(mtfm_cuda_aggregate* a);

/* ---------------------------------------------------------------- 2:4 pruning
 * prune_model_projections (prune.hpp:92-103) on the device: every
 * hta/.../{f1_w, fuq_w, fkv_w, f2_w} keeps, per output column and full group
 * of 4 consecutive input rows, its two largest magnitudes (ties keep the
 * earlier row, prune.hpp:33-70); a partial trailing group is exempt. The
 * pruned weights become the model's parameters (get_param returns them; the
 * bf16 copies are rebuilt). Report as PruneReport (prune.hpp:19-31). */
typedef struct {
    int64_t groups_covered, zeros_written, exempt_tail_rows, pruned_params;
} mtfm_prune_report;
MTFM_API mtfm_status mtfm_cuda_prune_projections(mtfm_cuda_model* m, mtfm_prune_report* report);

/* 2:4 sparse tensor cores for the projections (the sm_100a counterpart of the
 * paper's Ampere sparsity): when every f1_w / fuq_w / fkv_w /
 * f2_w keeps at most two non-zeros per group of 4 input rows (what
 * prune_projections leaves) the bf16 forward runs those GEMMs as
 * tcgen05.mma.sp on the compressed weights. mode 2 (default): whenever the
 * weights are 2:4; 1: required (MTFM_CONTRACT_ERROR if they are not); 0: dense.
 * active (optional) receives whether the bf16 forward now uses it. */
MTFM_API mtfm_status mtfm_cuda_set_sparse_mma(mtfm_cuda_model* m, int32_t mode, int32_t* active);

/* ---------------------------------------------------------------- training
 * Trainer::train_step (train.hpp:111-147) on the GPU over every user of a
 * prepared batch: build_loss (model.hpp:323-358: per sample the mean BCE over
 * its records, tape.hpp:462-486) through the whole model, gradients summed
 * over the batch and scaled by 1/global_batch, then ParamStore::adam_step
 * (params.hpp:87-119: non-finite check, global-norm clip, bias-corrected
 * Adam) on the device weights. fp32 (MTFM_PRECISION_FP32_CHECK handles only).
 * labels: [n_exposures][max_tasks] int32 in batch order, the scenario's task
 * order, -1 absent (a needed absent label -> MTFM_INTEGRITY_ERROR, like
 * build_loss). Data parallel: after mtfm_cuda_dp_init every rank's gradients
 * (and loss) are summed by one NCCL all-reduce before the clip and Adam, so
 * the ranks stay identical; global_batch = users over all ranks. */
typedef struct { /* AdamConfig (params.hpp:14-20) + the global batch */
    double lr, beta1, beta2, eps, clip_norm;
    int64_t global_batch; /* <= 0: this batch's users */
} mtfm_train_config;

typedef struct {
    double loss;      /* mean per-sample loss of the (global) batch, as train_step returns */
    double grad_norm; /* global gradient norm before clipping */
    int64_t step;     /* Adam step count */
    int64_t records;
} mtfm_train_result;

MTFM_API mtfm_status mtfm_cuda_train_step(mtfm_cuda_model* m, mtfm_cuda_batch* b, const int32_t* labels, int32_t max_tasks,
                                          const mtfm_train_config* cfg, mtfm_train_result* out);
/* Current value (device weights after training) / last step's gradient of a parameter. */
MTFM_API mtfm_status mtfm_cuda_get_param(mtfm_cuda_model* m, const char* name, float* host, int64_t rows, int64_t cols);
MTFM_API mtfm_status mtfm_cuda_get_grad(mtfm_cuda_model* m, const char* name, float* host, int64_t rows, int64_t cols);
/* Data parallel over NCCL (NVLink / NVSwitch): rank 0 makes the 128-byte id, every rank
 * passes it with its rank (one model handle per GPU). */
MTFM_API mtfm_status mtfm_nccl_unique_id(void* out128);
MTFM_API mtfm_status mtfm_cuda_dp_init(mtfm_cuda_model* m, int32_t nranks, int32_t rank, const void* unique_id128);

/* ---------------------------------------------------------------- dataset ingestion
 * load_dataset (dataset_io.cpp:110-221: header line with the schemas, one
 * UserSample JSON object per line) straight into packed jagged batches of
 * chunk_users users each, parsed by n_threads worker threads (<= 0: all
 * cores) into page-locked host memory, so every chunk reaches the GPU by an
 * asynchronous H2D (mtfm_cuda_batch_prepare / _update) without per-user
 * re-packing. Errors as the reference: MTFM_PARSE_ERROR "line N: ..." for the
 * first malformed line (exact key sets, require_keys dataset_io.cpp:16-31),
 * then validate_dataset (schema.cpp:45-139) in its order (CONFIG / INTEGRITY /
 * LOOKUP). Host-only: needs no GPU (pageable memory when there is none). */
typedef struct mtfm_dataset mtfm_dataset;
typedef struct {
    int32_t format_version;
    int64_t n_users, n_chunks;
    int32_t max_tasks; /* label columns per exposure */
} mtfm_dataset_info_t;

MTFM_API mtfm_status mtfm_dataset_load(const char* path, int32_t n_threads, int32_t chunk_users, mtfm_dataset** out);
MTFM_API mtfm_status mtfm_dataset_info(const mtfm_dataset* d, mtfm_dataset_info_t* info);
/* Schemas as a mtfm_schema_desc (pointers owned by the dataset) for mtfm_cuda_create. */
MTFM_API mtfm_status mtfm_dataset_schema_desc(const mtfm_dataset* d, mtfm_schema_desc* out);
/* Zero-copy view of chunk i (offsets chunk-local); labels: [n_exposures][max_tasks]
 * in scenario task order, -1 where absent. Valid until mtfm_dataset_free. */
MTFM_API mtfm_status mtfm_dataset_chunk(const mtfm_dataset* d, int64_t i, mtfm_packed_batch* out, const int32_t** labels);
MTFM_API void mtfm_dataset_free(mtfm_dataset* d);

#ifdef __cplusplus
}
#endif

#endif /* MTFM_CUDA_H_ */
