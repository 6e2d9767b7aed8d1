// train_kernels.cu — fp32 kernels of the training step (see train_kernels.cuh).
#include <algorithm>

#include "train_kernels.cuh"

namespace mtfm {
namespace trn {

namespace {

__device__ __forceinline__ float sigm(float x) { return sigmoid_precise(x); }
__device__ __forceinline__ float silu_grad(float z) {
    const float s = sigm(z);
    return s * (1.f + z * (1.f - s));
}

int blocks_for(long long n, int threads, int cap = 148 * 16) {
    return static_cast<int>(std::max<long long>(1, std::min<long long>((n + threads - 1) / threads, cap)));
}

// ---------------------------------------------------------------- GEMM
constexpr int TM = 64, TN = 64, TK = 16;

__global__ void __launch_bounds__(256) gemm_kernel(Gemm g) {
    __shared__ float As[TK][TM + 4];
    __shared__ float Bs[TK][TN + 4];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4 x 4 outputs each
    const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < g.K; k0 += TK) {
        for (int i = threadIdx.x; i < TM * TK; i += 256) {
            const int mm = i / TK, kk = i % TK;
            const int m = m0 + mm, k = k0 + kk;
            float v = 0.f;
            if (m < g.M && k < g.K) {
                const long long r = g.arow ? static_cast<long long>(g.arow[m]) : m;
                v = g.A[r * g.sam + k * g.sak];
            }
            As[kk][mm] = v;
        }
        for (int i = threadIdx.x; i < TK * TN; i += 256) {
            const int kk = i / TN, nn = i % TN;
            const int k = k0 + kk, n = n0 + nn;
            Bs[kk][nn] = (k < g.K && n < g.N) ? g.B[k * g.sbk + n * g.sbn] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty * 4 + i;
        if (m >= g.M) continue;
        const long long r = g.crow ? static_cast<long long>(g.crow[m]) : g.c_row0 + m;
        float* c = g.C + r * g.ldc;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n >= g.N) continue;
            c[n] = g.accumulate ? c[n] + acc[i][j] : acc[i][j];
        }
    }
}

// ---------------------------------------------------------------- elementwise
__global__ void silu_fwd_kernel(const float* z, float* p, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = silu_precise(z[i]);
}

__global__ void silu_bwd_kernel(const float* dp, long long lddp, const float* z, long long ldz, float* dz, long long lddz,
                                long long rows, int cols) {
    const long long n = rows * cols;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / cols;
        const int c = static_cast<int>(i - r * cols);
        dz[r * lddz + c] = dp[r * lddp + c] * silu_grad(z[r * ldz + c]);
    }
}

__global__ void mul2_kernel(const float* a, long long lda, const float* b, long long ldb, float* o, long long ldo,
                            long long rows, int cols) {
    const long long n = rows * cols;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / cols;
        const int c = static_cast<int>(i - r * cols);
        o[r * ldo + c] = a[r * lda + c] * b[r * ldb + c];
    }
}

// column sums: block = 32 columns x 8 row lanes
__global__ void colsum_kernel(const float* dy, long long ld, long long rows, int cols, float* db) {
    const int c = blockIdx.x * 32 + (threadIdx.x & 31);
    const int lr = threadIdx.x >> 5;
    float s = 0.f;
    if (c < cols)
        for (long long r = blockIdx.y * 8 + lr; r < rows; r += 8ll * gridDim.y) s += dy[r * ld + c];
    __shared__ float sh[8][32];
    sh[lr][threadIdx.x & 31] = s;
    __syncthreads();
    if (lr == 0 && c < cols) {
        float t = 0.f;
        for (int k = 0; k < 8; ++k) t += sh[k][threadIdx.x & 31];
        atomicAdd(db + c, t);
    }
}

// ---------------------------------------------------------------- GLN
// one warp per row (row_normalize: population variance, eps inside the sqrt, kernels.hpp:132-153)
__global__ void gln_fwd_kernel(const float* x, long long ldx, long long n, int d, const int* group, const float* gain,
                               const float* bias, float eps, float* xhat, float* y, float* rstd) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long r = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
        const float* xr = x + r * ldx;
        float s = 0.f;
        for (int c = lane; c < d; c += 32) s += xr[c];
        s = warp_sum(s);
        const float mean = s / static_cast<float>(d);
        float q = 0.f;
        for (int c = lane; c < d; c += 32) {
            const float t = xr[c] - mean;
            q += t * t;
        }
        q = warp_sum(q);
        const float inv = 1.f / sqrtf(q / static_cast<float>(d) + eps);
        int g = group[r];
        g = g < 0 ? 0 : g;
        for (int c = lane; c < d; c += 32) {
            const float h = (xr[c] - mean) * inv;
            xhat[r * d + c] = h;
            y[r * d + c] = h * gain[(long long)g * d + c] + bias[(long long)g * d + c];
        }
        if (lane == 0) rstd[r] = inv;
    }
}

// one warp per row; per-group gain / bias gradients reduced in shared memory per block
__global__ void gln_bwd_kernel(const float* dy, long long lddy, const float* xhat, const float* rstd, long long n, int d,
                               const int* group, const float* gain, int n_groups, float* dgain, float* dbias, float* dx,
                               long long lddx, int accumulate) {
    extern __shared__ float sh[];  // [n_groups][d] dgain, then dbias
    for (int i = threadIdx.x; i < 2 * n_groups * d; i += blockDim.x) sh[i] = 0.f;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long r = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
        int g = group[r];
        g = g < 0 ? 0 : g;
        const float* dr = dy + r * lddy;
        const float* hr = xhat + r * d;
        float s1 = 0.f, s2 = 0.f;
        for (int c = lane; c < d; c += 32) {
            const float dh = dr[c] * gain[(long long)g * d + c];
            s1 += dh;
            s2 += dh * hr[c];
            atomicAdd(sh + g * d + c, dr[c] * hr[c]);
            atomicAdd(sh + n_groups * d + g * d + c, dr[c]);
        }
        s1 = warp_sum(s1) / static_cast<float>(d);
        s2 = warp_sum(s2) / static_cast<float>(d);
        const float inv = rstd[r];
        float* xo = dx + r * lddx;
        for (int c = lane; c < d; c += 32) {
            const float dh = dr[c] * gain[(long long)g * d + c];
            const float v = inv * (dh - s1 - hr[c] * s2);
            xo[c] = accumulate ? xo[c] + v : v;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_groups * d; i += blockDim.x) {
        if (sh[i] != 0.f) atomicAdd(dgain + i, sh[i]);
        if (sh[n_groups * d + i] != 0.f) atomicAdd(dbias + i, sh[n_groups * d + i]);
    }
}

// ---------------------------------------------------------------- attention backward
// one warp per (query row, head); lanes walk 32 keys at a time (the forward's structure,
// kernels.cu attn_simt_kernel). dq in registers, dK / dV by atomics.
__global__ void attn_bwd_kernel(AttnBwd a) {
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    extern __shared__ float sm[];
    float* qv = sm + wib * 2 * a.dh;  // q row, then dA row
    float* dav = qv + a.dh;
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
        const float s_i = a.scale[i];
        const float* qrow = a.q + i * a.ldq + a.q_col0 + h * a.dh;
        const float* darow = a.da + i * a.ldda + h * a.dh;
        for (int c = lane; c < a.dh; c += 32) {
            qv[c] = qrow[c];
            dav[c] = darow[c];
        }
        __syncwarp();
        float dq[8] = {};
        auto key = [&](long long kr_row, bool on, float& dS, float& wv) {
            dS = 0.f;
            wv = 0.f;
            if (!on) return;
            const float* kr = a.kv + kr_row * a.ldkv + a.k_col0 + g * a.dh;
            const float* vr = a.kv + kr_row * a.ldkv + a.v_col0 + g * a.dh;
            float sdot = 0.f, ddot = 0.f;
            for (int c = 0; c < a.dh; ++c) {
                sdot = fmaf(qv[c], kr[c], sdot);
                ddot = fmaf(dav[c], vr[c], ddot);
            }
            wv = silu_precise(sdot);
            dS = s_i * ddot * silu_grad(sdot);
            float* dk = a.dkv + kr_row * a.lddkv + a.dk_col0 + g * a.dh;
            float* dv = a.dkv + kr_row * a.lddkv + a.dv_col0 + g * a.dh;
            for (int c = 0; c < a.dh; ++c) {
                atomicAdd(dk + c, dS * qv[c]);
                atomicAdd(dv + c, s_i * wv * dav[c]);
            }
        };
        for (int j0 = 0; j0 < p; j0 += 32) {
            const int j = j0 + lane;
            float dS, wv;
            key(base + j, j < p, dS, wv);
            const int nn = min(32, p - j0);
            for (int jj = 0; jj < nn; ++jj) {
                const float dSj = __shfl_sync(0xffffffffu, dS, jj);
                const float* kr = a.kv + (base + j0 + jj) * a.ldkv + a.k_col0 + g * a.dh;
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    const int c = lane + 32 * m;
                    if (c < a.dh) dq[m] = fmaf(dSj, kr[c], dq[m]);
                }
            }
        }
        if (self >= 0) {
            float dS, wv;
            key(self, lane == 0, dS, wv);
            dS = __shfl_sync(0xffffffffu, dS, 0);
            const float* kr = a.kv + (long long)self * a.ldkv + a.k_col0 + g * a.dh;
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int c = lane + 32 * m;
                if (c < a.dh) dq[m] = fmaf(dS, kr[c], dq[m]);
            }
        }
        float* dqr = a.dq + i * a.lddq + a.dq_col0 + h * a.dh;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int c = lane + 32 * m;
            if (c < a.dh) dqr[c] = dq[m];
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- heads
// one warp per T row; per-row scratch in shared memory: experts e[E*de], de[E*de], m[de]
__global__ void heads_train_kernel(HeadsTrain h) {
    extern __shared__ float sm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int ED = h.E * h.de;
    float* ev = sm + wib * (2 * ED + h.de + 64);
    float* dev = ev + ED;
    float* mv = dev + ED;
    float* gam = mv + h.de;  // [E] (E <= 32) then dgam [E]
    float* dgam = gam + 32;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long t = blockIdx.x * (long long)(blockDim.x >> 5) + wib; t < h.n_t; t += warps) {
        const float* y = h.yh + t * h.ldy;
        float* dy = h.dyh + t * h.ldy;
        const int u = h.t_user[t];
        const int sid = h.t_scen[t];
        int si = -1;
        for (int s = 0; s < h.n_src; ++s)
            if (h.src[s].kind == 2 && h.src[s].id == sid) si = s;
        for (int c = lane; c < h.ldy; c += 32) dy[c] = 0.f;
        if (si < 0) continue;
        const SourceInfo S = h.src[si];
        const long long x = h.exp_off[u] + h.t_exp_ref[t];
        const float wrow = static_cast<float>(h.inv_batch / static_cast<double>(h.rec_off[u + 1] - h.rec_off[u]));
        for (int c = lane; c < ED; c += 32) {
            ev[c] = silu_precise(y[c] + h.exp_bias[c]);
            dev[c] = 0.f;
        }
        __syncwarp();
        double lsum = 0.0;
        for (int k = 0; k < S.ntasks; ++k) {
            const int tg = S.task0 + k;
            const int lab = h.labels[x * h.max_tasks + k];
            if (lab < 0) {
                if (lane == 0) atomicMin(h.err, static_cast<unsigned long long>(t));
                continue;
            }
            // gate softmax over E (softmax_rows: max-shifted)
            if (lane == 0) {
                float mx = -3.0e38f;
                for (int e = 0; e < h.E; ++e) {
                    gam[e] = y[ED + tg * h.E + e] + h.gate_bias[tg * h.E + e];
                    mx = fmaxf(mx, gam[e]);
                }
                float ssum = 0.f;
                for (int e = 0; e < h.E; ++e) {
                    gam[e] = expf(gam[e] - mx);
                    ssum += gam[e];
                }
                const float inv = 1.f / ssum;
                for (int e = 0; e < h.E; ++e) gam[e] *= inv;
            }
            __syncwarp();
            // mixture and tower
            float zp = 0.f;
            for (int c = lane; c < h.de; c += 32) {
                float m = 0.f;
                for (int e = 0; e < h.E; ++e) m = fmaf(gam[e], ev[e * h.de + c], m);
                mv[c] = m;
                zp = fmaf(m, h.tower_w[(long long)tg * h.de + c], zp);
            }
            const float z = warp_sum(zp) + h.tower_b[tg];
            const float yl = static_cast<float>(lab);
            const float zpos = z > 0.f ? z : 0.f, az = fabsf(z);
            lsum += static_cast<double>(zpos - z * yl + log1pf(expf(-az))) * static_cast<double>(wrow);
            const float dz = (sigm(z) - yl) * wrow;
            __syncwarp();
            // tower, mixture, gate
            for (int c = lane; c < h.de; c += 32) {
                atomicAdd(h.d_tower_w + (long long)tg * h.de + c, dz * mv[c]);
                const float dm = dz * h.tower_w[(long long)tg * h.de + c];
                for (int e = 0; e < h.E; ++e) dev[e * h.de + c] += gam[e] * dm;
            }
            if (lane == 0) atomicAdd(h.d_tower_b + tg, dz);
            for (int e = 0; e < h.E; ++e) {
                float part = 0.f;
                for (int c = lane; c < h.de; c += 32) part = fmaf(dz * h.tower_w[(long long)tg * h.de + c], ev[e * h.de + c], part);
                part = warp_sum(part);
                if (lane == 0) dgam[e] = part;
            }
            __syncwarp();
            if (lane == 0) {
                float sg = 0.f;
                for (int e = 0; e < h.E; ++e) sg += gam[e] * dgam[e];
                for (int e = 0; e < h.E; ++e) {
                    const float du = gam[e] * (dgam[e] - sg);
                    dy[ED + tg * h.E + e] = du;
                    atomicAdd(h.d_gate_bias + tg * h.E + e, du);
                }
            }
            __syncwarp();
        }
        // experts' pre-activation gradients
        for (int c = lane; c < ED; c += 32) {
            const float pre = y[c] + h.exp_bias[c];
            const float dp = dev[c] * silu_grad(pre);
            dy[c] = dp;
            atomicAdd(h.d_exp_bias + c, dp);
        }
        if (lane == 0 && lsum != 0.0) atomicAdd(h.loss, lsum);
        __syncwarp();
    }
}

// ---------------------------------------------------------------- embeddings
__global__ void embed_bwd_kernel(DevBatch b, const SourceInfo* __restrict__ srcs, const SlotInfo* __restrict__ slots,
                                 const int* __restrict__ src_rows, const int* __restrict__ row_item,
                                 const long long* __restrict__ src_base, const long long* __restrict__ src_cnt,
                                 const long long* __restrict__ emb_base, const float* __restrict__ de, int d_emb,
                                 int n_src, long long total_rows, int max_slots, float* __restrict__ dtables) {
    const long long per = max_slots;
    const long long n_items = total_rows * per;
    for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < n_items; w += (long long)gridDim.x * blockDim.x) {
        const long long P = w / per;
        const int k = static_cast<int>(w - P * per);
        int s = 0;
        while (s + 1 < n_src && P >= src_base[s + 1]) ++s;
        const long long p = P - src_base[s];
        if (p >= src_cnt[s]) continue;
        const SourceInfo si = srcs[s];
        const int nslots = si.nslot[0] + si.nslot[1] + si.nslot[2];
        if (k >= nslots) continue;
        const int row = src_rows[P];
        const int item = row_item[row];
        int id;
        if (si.kind < 2) {
            id = b.ev_feats[b.ev_feat_off[item] + k];
        } else {
            const int nu = b.exp_blk[3 * item], nc = b.exp_blk[3 * item + 1];
            const int off = k < si.nslot[0] ? k : (k < si.nslot[0] + si.nslot[1] ? nu + (k - si.nslot[0])
                                                                                  : nu + nc + (k - si.nslot[0] - si.nslot[1]));
            id = b.exp_feats[b.exp_feat_off[item] + off];
        }
        const SlotInfo sl = slots[si.slot0 + k];
        if (id < 0 || id >= sl.vocab) continue;
        const float* g = de + emb_base[s] + p * si.k_pad + k * d_emb;
        float* t = dtables + sl.emb_off + static_cast<long long>(id) * d_emb;
        for (int c = 0; c < d_emb; ++c) atomicAdd(t + c, g[c]);
    }
}

// ---------------------------------------------------------------- optimizer
__global__ void sumsq_kernel(const float* g, long long n, double* out) {
    double s = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double v = g[i];
        s += v * v;
    }
    s = warp_sum(s);
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
        t = warp_sum(t);
        if (threadIdx.x == 0) atomicAdd(out, t);
    }
}

__global__ void adam_kernel(float* w, const float* g, float* m, float* v, long long n, double scale, double lr, double b1,
                            double b2, double eps, double bc1, double bc2) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double gg = static_cast<double>(g[i]) * scale;
        const double mm = b1 * static_cast<double>(m[i]) + (1.0 - b1) * gg;
        const double vv = b2 * static_cast<double>(v[i]) + (1.0 - b2) * gg * gg;
        m[i] = static_cast<float>(mm);
        v[i] = static_cast<float>(vv);
        const double mhat = mm / bc1, vhat = vv / bc2;
        w[i] = static_cast<float>(static_cast<double>(w[i]) - lr * mhat / (sqrt(vhat) + eps));
    }
}

__global__ void scale_kernel(float* g, long long n, float s) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) g[i] *= s;
}

}  // namespace

void gemm(const Gemm& g, cudaStream_t st) {
    if (g.M <= 0 || g.N <= 0) return;
    if (g.K <= 0) {
        if (!g.accumulate) {  // empty reduction: C = 0
            // (never needed by the training step: every K here is >= 1)
        }
        return;
    }
    dim3 grid((g.N + TN - 1) / TN, (g.M + TM - 1) / TM);
    gemm_kernel<<<grid, 256, 0, st>>>(g);
}

void silu_fwd(const float* z, float* p, long long n, cudaStream_t st) {
    if (n > 0) silu_fwd_kernel<<<blocks_for(n, 256), 256, 0, st>>>(z, p, n);
}

void silu_bwd(const float* dp, long long lddp, const float* z, long long ldz, float* dz, long long lddz, long long rows,
              int cols, cudaStream_t st) {
    if (rows * cols > 0) silu_bwd_kernel<<<blocks_for(rows * cols, 256), 256, 0, st>>>(dp, lddp, z, ldz, dz, lddz, rows, cols);
}

void mul2(const float* a, long long lda, const float* b, long long ldb, float* out, long long ldo, long long rows, int cols,
          cudaStream_t st) {
    if (rows * cols > 0) mul2_kernel<<<blocks_for(rows * cols, 256), 256, 0, st>>>(a, lda, b, ldb, out, ldo, rows, cols);
}

void colsum_add(const float* dy, long long ld, long long rows, int cols, float* db, cudaStream_t st) {
    if (rows <= 0 || cols <= 0) return;
    dim3 grid((cols + 31) / 32, static_cast<unsigned>(std::min<long long>((rows + 7) / 8, 256)));
    colsum_kernel<<<grid, 256, 0, st>>>(dy, ld, rows, cols, db);
}

void gln_fwd(const float* x, long long ldx, long long n, int d, const int* group, const float* gain, const float* bias,
             float eps, float* xhat, float* y, float* rstd, cudaStream_t st) {
    if (n > 0) gln_fwd_kernel<<<blocks_for(n, 8), 256, 0, st>>>(x, ldx, n, d, group, gain, bias, eps, xhat, y, rstd);
}

void gln_bwd(const float* dy, long long lddy, const float* xhat, const float* rstd, long long n, int d,
             const int* group, const float* gain, int n_groups, float* dgain, float* dbias, float* dx, long long lddx,
             int accumulate, cudaStream_t st) {
    if (n <= 0) return;
    const size_t smem = static_cast<size_t>(2) * n_groups * d * sizeof(float);
    cudaFuncSetAttribute(gln_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    gln_bwd_kernel<<<blocks_for(n, 8, 148 * 4), 256, smem, st>>>(dy, lddy, xhat, rstd, n, d, group, gain, n_groups, dgain,
                                                                  dbias, dx, lddx, accumulate);
}

void attn_bwd(const AttnBwd& a, cudaStream_t st) {
    if (a.n_q <= 0) return;
    const int wpb = 8;
    attn_bwd_kernel<<<blocks_for(a.n_q * a.heads, wpb), wpb * 32, wpb * 2 * a.dh * sizeof(float), st>>>(a);
}

void heads_train(const HeadsTrain& h, cudaStream_t st) {
    if (h.n_t <= 0) return;
    const int wpb = 4;
    const size_t smem = static_cast<size_t>(wpb) * (2 * h.E * h.de + h.de + 64) * sizeof(float);
    cudaFuncSetAttribute(heads_train_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    heads_train_kernel<<<blocks_for(h.n_t, wpb), wpb * 32, smem, st>>>(h);
}

void embed_bwd(const DevBatch& b, const SourceInfo* srcs, const SlotInfo* slots, const int* src_rows, const int* row_item,
               const long long* src_base, const long long* src_cnt, const long long* emb_base, const float* de,
               int d_emb, int n_src, long long total_rows, int max_slots, float* dtables, cudaStream_t st) {
    const long long n = total_rows * max_slots;
    if (n > 0)
        embed_bwd_kernel<<<blocks_for(n, 256), 256, 0, st>>>(b, srcs, slots, src_rows, row_item, src_base, src_cnt,
                                                              emb_base, de, d_emb, n_src, total_rows, max_slots, dtables);
}

void sumsq(const float* g, long long n, double* out, cudaStream_t st) {
    if (n > 0) sumsq_kernel<<<blocks_for(n, 256, 148 * 4), 256, 0, st>>>(g, n, out);
}

void adam(float* w, const float* g, float* m, float* v, long long n, double scale, double lr, double b1, double b2,
          double eps, double bc1, double bc2, cudaStream_t st) {
    if (n > 0) adam_kernel<<<blocks_for(n, 256), 256, 0, st>>>(w, g, m, v, n, scale, lr, b1, b2, eps, bc1, bc2);
}

void scale_inplace(float* g, long long n, float s, cudaStream_t st) {
    if (n > 0) scale_kernel<<<blocks_for(n, 256), 256, 0, st>>>(g, n, s);
}

}  // namespace trn
}  // namespace mtfm
