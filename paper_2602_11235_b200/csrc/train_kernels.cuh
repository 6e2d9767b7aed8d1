// train_kernels.cuh — fp32 kernels of the training step: the
// reverse-mode counterparts of the forward (tape.hpp:68-488 restated op by op
// for a whole packed batch) plus Adam (params.hpp:87-119).
//
// Everything is fp32 SIMT: the training path is the check-mode numerics of the
// forward with saved activations, matching the reference's Trainer::train_step
// (train.hpp:111-147) to float rounding.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.cuh"

namespace mtfm {
namespace trn {

// C[crow(m)][n] (+)= sum_k A(m, k) * B(k, n), A(m, k) = A[arow(m) * sam + k * sak],
// B(k, n) = B[k * sbk + n * sbn]; arow / crow optional row indirections.
struct Gemm {
    int M, N, K;
    const float* A;
    long long sam, sak;
    const int* arow;
    const float* B;
    long long sbk, sbn;
    float* C;
    long long ldc;
    const int* crow;
    long long c_row0;  // added to the C row when crow is null
    int accumulate;    // 1: C += product
};
void gemm(const Gemm& g, cudaStream_t st);

// P = silu(Z) (n elements)
void silu_fwd(const float* z, float* p, long long n, cudaStream_t st);
// dZ = dP * silu'(Z), matrices [rows][cols] with leading dims (dP/dZ may alias)
void silu_bwd(const float* dp, long long lddp, const float* z, long long ldz, float* dz, long long lddz, long long rows,
              int cols, cudaStream_t st);
// db[c] += sum_r dY[r][c]
void colsum_add(const float* dy, long long ld, long long rows, int cols, float* db, cudaStream_t st);
// out[r][c] = a[r][c] * b[r][c] (strided)
void mul2(const float* a, long long lda, const float* b, long long ldb, float* out, long long ldo, long long rows, int cols,
          cudaStream_t st);

// GLN forward on rows [0, n): xhat = row_normalize(x), y = xhat * gain[g] + bias[g]; saves rstd
void gln_fwd(const float* x, long long ldx, long long n, int d, const int* group, const float* gain, const float* bias,
             float eps, float* xhat, float* y, float* rstd, cudaStream_t st);
// GLN backward: dgain[g] += dy * xhat, dbias[g] += dy, dx (+)= rstd (dxh - mean(dxh) - xhat mean(dxh xhat)),
// dxh = dy * gain[g]
void gln_bwd(const float* dy, long long lddy, const float* xhat, const float* rstd, long long n, int d,
             const int* group, const float* gain, int n_groups, float* dgain, float* dbias, float* dx, long long lddx,
             int accumulate, cudaStream_t st);

// attention backward (hta.hpp:115-134): A_h[i] = s_i sum_j silu(Q_h[i] K_g[j]) V_g[j] over the
// visible keys (prefix form + self). Given dA: dQ (written), dK and dV (accumulated, atomics).
struct AttnBwd {
    const float* q;
    long long ldq;
    int q_col0;
    const float* kv;
    long long ldkv;
    int k_col0, v_col0;
    long long n_q;
    const int* prefix;
    const float* scale;
    const int* self;
    const int* keybase;
    int heads, kv_heads, dh;
    const float* da;
    long long ldda;
    float* dq;
    long long lddq;
    int dq_col0;
    float* dkv;
    long long lddkv;
    int dk_col0, dv_col0;
};
void attn_bwd(const AttnBwd& a, cudaStream_t st);

// MMoE heads (heads.hpp:47-99) forward + BCE (tape.hpp:462-486) + backward, one warp per T row.
struct HeadsTrain {
    const float* yh;        // [T][ldy] = X_T head_w (experts E*de, then gates n_tasks*E), no biases
    long long ldy;
    const float* exp_bias;  // [E*de]
    const float* gate_bias; // [n_tasks*E]
    const float* tower_w;   // [n_tasks][de]
    const float* tower_b;   // [n_tasks]
    int E, de;
    const SourceInfo* src;
    int n_src;
    const int* t_scen;
    const int* t_user;
    const int* t_exp_ref;
    const int* exp_off;     // per user: first exposure (labels index)
    const long long* rec_off;  // per user: records (loss normaliser)
    const int* labels;      // [n_exposures][max_tasks], -1 missing
    int max_tasks;
    long long n_t;
    double inv_batch;       // 1 / global batch size (users)
    // outputs
    float* dyh;             // [T][ldy] pre-activation gradients
    float* d_exp_bias;
    float* d_gate_bias;
    float* d_tower_w;
    float* d_tower_b;
    double* loss;           // += sum over rows of loss contributions
    unsigned long long* err;  // min T row with a missing label
};
void heads_train(const HeadsTrain& h, cudaStream_t st);

// d(embedding tables) += dE scattered through the gather indexing (tokenizer.hpp:193-207)
void embed_bwd(const DevBatch& b, const SourceInfo* srcs, const SlotInfo* slots, const int* src_rows, const int* row_item,
               const long long* src_base, const long long* src_cnt, const long long* emb_base, const float* de,
               int d_emb, int n_src, long long total_rows, int max_slots, float* dtables, cudaStream_t st);

// sum of squares of g (double) into *out
void sumsq(const float* g, long long n, double* out, cudaStream_t st);
// Adam with bias correction and global-norm clip scale (params.hpp:87-119), double arithmetic
void adam(float* w, const float* g, float* m, float* v, long long n, double scale, double lr, double b1, double b2,
          double eps, double bc1, double bc2, cudaStream_t st);
void scale_inplace(float* g, long long n, float s, cudaStream_t st);

}  // namespace trn
}  // namespace mtfm
