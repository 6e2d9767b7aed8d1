"""bf16 storage emulation of the GPU fast path — TEST INFRASTRUCTURE ONLY.

Bf16Oracle restates the reference forward (mtfm_oracle.Oracle, itself pinned to
the reference's goldens) in float32 arithmetic, rounding to bf16 at exactly the
points where the CUDA fast path stores bf16 (paper_2602_11235_b200/csrc):

  embeddings, every GEMM weight               bf16 (uploaded once)
  tokenizer hidden silu(E W1 + b1)            bf16 (TMEM / HBM), Y -> X fp32
  GLN1 output of T rows / non-folded rows     bf16(xhat * gain + bias)
  context rows of a target run (+ the full    xhat = bf16(row_normalize(x)) times the
    layer right after it)                     folded bf16(gain (.) W), fp32 (bias W + b)
  projections silu(. W + b)                   bf16 (U, Q, K, V)
  attention weights silu(Q K^T)               bf16 P; the T self term and O stay fp32
  attention output s_i * O                    bf16 A
  gate gln2(A) * U                            bf16
  f2 + residual                               fp32
  head input (final T rows)                   bf16

so GPU-vs-emulation isolates kernel defects from the storage precision, and
emulation-vs-reference shows what bf16 storage alone costs on a given model.
"""
from __future__ import annotations

import numpy as np

import mtfm_oracle as O


def rb(x):
    """float32 -> bf16 (round to nearest even) -> float32."""
    u = np.ascontiguousarray(np.asarray(x, dtype=np.float32)).view(np.uint32)
    u = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return u.view(np.float32)


class Bf16Oracle(O.Oracle):
    def __init__(self, sch, cfg, params):
        super().__init__(sch, cfg, params, np.float32)
        self.W = {}  # bf16-rounded weight cache

    def w(self, name):
        if name not in self.W:
            self.W[name] = rb(self.P[name])
        return self.W[name]

    # tokenizer: bf16 tables, bf16 W1/W2, bf16 hidden layer, fp32 Y
    def embed(self, tables, ids):
        saved = {t: self.P[t] for t in tables}
        for t in tables:
            self.P[t] = self.w(t)
        try:
            return super().embed(tables, ids)
        finally:
            self.P.update(saved)

    def mlp(self, x, base):
        h = rb(O.silu((x @ self.w(base + "/mlp_w1") + self.P[base + "/mlp_b1"][0]).astype(np.float32)))
        return (h @ self.w(base + "/mlp_w2") + self.P[base + "/mlp_b2"][0]).astype(np.float32)

    def gln_affine(self, xn, groups, prefix):
        out = np.empty_like(xn)
        for g in np.unique(groups):
            rows = groups == g
            key = self.gt.keys[g]
            out[rows] = xn[rows] * self.P[f"{prefix}/{key}/gain"][0] + self.P[f"{prefix}/{key}/bias"][0]
        return out

    def folded_proj(self, x, groups, base, wname, bname):
        """context rows: bf16(xhat) @ bf16(gain_g (.) W) + (bias_g W + b), per GLN group (model.cu finalize)."""
        xh = rb(O.row_normalize(x, self.cfg.eps))
        W = self.P[wname].astype(np.float64)
        b = self.P[bname][0].astype(np.float64)
        out = np.empty((x.shape[0], W.shape[1]), np.float32)
        for g in np.unique(groups):
            rows = groups == g
            key = self.gt.keys[g]
            gain = self.P[f"{base}/gln1/{key}/gain"][0].astype(np.float32)
            bias = self.P[f"{base}/gln1/{key}/bias"][0].astype(np.float64)
            wf = rb((gain[:, None] * self.P[wname]).astype(np.float32))
            bf = (bias @ W + b).astype(np.float32)
            out[rows] = xh[rows] @ wf + bf
        return rb(O.silu(out))

    def proj(self, xn_bf16, wname, bname):
        return rb(O.silu((xn_bf16 @ self.w(wname) + self.P[bname][0]).astype(np.float32)))

    def gqa(self, q, k, v, mask, scale, self_col=None):
        cfg = self.cfg
        dh = cfg.head_dim
        r = cfg.heads // cfg.kv_heads
        m = mask.astype(np.float32).copy()
        n_q = q.shape[0]
        if self_col is not None:  # the T self key is a separate fp32 term (attn_tc.cuh epilogue)
            m[np.arange(n_q), self_col] = 0
        outs = []
        for h in range(cfg.heads):
            g = h // r
            kk, vv = k[:, g * dh:(g + 1) * dh], v[:, g * dh:(g + 1) * dh]
            s = (q[:, h * dh:(h + 1) * dh] @ kk.T).astype(np.float32)
            p = rb(O.silu(s)) * m
            o = (p @ vv).astype(np.float32)
            if self_col is not None:
                ws = O.silu(np.einsum("ij,ij->i", q[:, h * dh:(h + 1) * dh], kk[self_col]).astype(np.float32))
                o = o + ws[:, None] * vv[self_col]
            outs.append(o * scale[:, None])
        return rb(np.concatenate(outs, axis=1))

    def gate(self, a, groups, prefix, u):
        return rb(self.gln_affine(O.row_normalize(a, self.cfg.eps), groups, prefix) * u)

    def target_layer(self, x, base, groups, mask, scale, off):
        cfg, P = self.cfg, self.P
        hd = cfg.heads * cfg.head_dim
        gd = cfg.kv_heads * cfg.head_dim
        xn_t = rb(self.gln_affine(O.row_normalize(x[off:], cfg.eps), groups[off:], base + "/gln1"))
        uq = self.proj(xn_t, base + "/fuq_w", base + "/fuq_b")
        kv_t = self.proj(xn_t, base + "/fkv_w", base + "/fkv_b")
        kv_c = self.folded_proj(x[:off], groups[:off], base, base + "/fkv_w", base + "/fkv_b") if off else \
            np.zeros((0, 2 * gd), np.float32)
        kv = np.concatenate([kv_c, kv_t], axis=0)
        n_t = x.shape[0] - off
        a = self.gqa(uq[:, hd:], kv[:, :gd], kv[:, gd:], mask[off:], scale[off:], self_col=off + np.arange(n_t))
        g = self.gate(a, groups[off:], base + "/gln2", uq[:, :hd])
        t_new = (g @ self.w(base + "/f2_w") + P[base + "/f2_b"][0]) + x[off:]
        return np.concatenate([x[:off], t_new.astype(np.float32)], axis=0)

    def full_layer_emu(self, x, base, groups, mask, scale, off, after_run):
        cfg, P = self.cfg, self.P
        hd = cfg.heads * cfg.head_dim
        gd = cfg.kv_heads * cfg.head_dim
        if after_run and off:
            p_c = self.folded_proj(x[:off], groups[:off], base, base + "/f1_w", base + "/f1_b")
            xn_t = rb(self.gln_affine(O.row_normalize(x[off:], cfg.eps), groups[off:], base + "/gln1"))
            proj = np.concatenate([p_c, self.proj(xn_t, base + "/f1_w", base + "/f1_b")], axis=0)
        else:
            xn = rb(self.gln_affine(O.row_normalize(x, cfg.eps), groups, base + "/gln1"))
            proj = self.proj(xn, base + "/f1_w", base + "/f1_b")
        u, q = proj[:, :hd], proj[:, hd:2 * hd]
        k, v = proj[:, 2 * hd:2 * hd + gd], proj[:, 2 * hd + gd:]
        n = x.shape[0]
        self_col = np.full(n, -1)
        t = np.arange(off, n)
        has_t = len(t) > 0
        # context rows have no self key; T rows do (only T columns j == i are visible)
        a = np.empty((n, hd), np.float32)
        if off:
            a[:off] = self.gqa(q[:off], k, v, mask[:off], scale[:off])
        if has_t:
            a[off:] = self.gqa(q[off:], k, v, mask[off:], scale[off:], self_col=t)
        g = self.gate(a, groups, base + "/gln2", u)
        return ((g @ self.w(base + "/f2_w") + P[base + "/f2_b"][0]) + x).astype(np.float32)

    def stack(self, x0, plan, groups, mask, scale, keep_layers=False):
        cfg = self.cfg
        x = x0.astype(np.float32)
        layers = []
        off = plan.bounds[0] + plan.bounds[1]
        prev_target = False
        for b in range(cfg.blocks):
            for l in range(cfg.target_layers + cfg.full_layers):
                base = f"hta/b{b}/l{l}"
                if l < cfg.target_layers:
                    x = self.target_layer(x, base, groups, mask, scale, off)
                    prev_target = True
                else:
                    x = self.full_layer_emu(x, base, groups, mask, scale, off, prev_target)
                    prev_target = False
                if keep_layers:
                    layers.append(x)
        return x, layers

    def heads(self, t_rows, plan):
        cfg, P = self.cfg, self.P
        off = plan.bounds[0] + plan.bounds[1]
        scen_of_row = plan.group_id[off:]
        xs_all = rb(t_rows)
        cols = []
        for sid in sorted(set(int(s) for s in scen_of_row)):
            rows = np.nonzero(scen_of_row == sid)[0]
            tasks = self.sch.scenario(sid)[4]
            xs = xs_all[rows]
            ex = [O.silu((xs @ self.w(f"head/expert{e}_w") + P[f"head/expert{e}_b"][0]).astype(np.float32))
                  for e in range(cfg.experts)]
            for ti, t in enumerate(tasks):
                base = f"head/s{sid}/{t}"
                gate = O.softmax_rows((xs @ self.w(base + "/gate_w") + P[base + "/gate_b"][0]).astype(np.float32))
                mix = ex[0] * gate[:, 0:1]
                for e in range(1, cfg.experts):
                    mix = mix + ex[e] * gate[:, e:e + 1]
                z = (mix @ P[base + "/tower_w"] + P[base + "/tower_b"][0])[:, 0]
                cols.append((sid, ti, t, rows, z))
        return cols
