"""CPU restatement of the MTFM hot path (numpy) — THE ORACLE.

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg may import this module, and only as the checker. The product
(paper_2602_11235_b200/) never imports it and has no CPU fallback.

Parity pinned: tests/test_oracle_golden.py checks every function here against
golden vectors produced by the reference itself (oracle/ref_dump.cpp compiled
from /root/reference/proj by oracle/Makefile, fixtures in tests/golden/ made by
oracle/make_golden.py).

Each function restates one reference routine (paths relative to
/root/reference/proj):
  Rng                       include/mtfm/rng.hpp:13-83
  build_params              include/mtfm/model.hpp:371-463 (registration order)
  plan_user                 include/mtfm/tokenizer.hpp:53-134 (plan_tokens)
  GroupTable                include/mtfm/groups.hpp:20-53
  build_mask                src/mask.cpp:5-29 (+ row_valid_counts mask.hpp:35-40)
  row_scale                 include/mtfm/hta.hpp:53-67 (make_stack_geom)
  tokenize_user             include/mtfm/tokenizer.hpp:184-268
  gln                       include/mtfm/hta.hpp:104-109, kernels.hpp:132-153,
                            eval_ctx.hpp:130-143
  gqa_attention             include/mtfm/hta.hpp:115-134
  full_layer / target_layer include/mtfm/hta.hpp:138-184
  forward_stack             include/mtfm/hta.hpp:188-212
  mmoe_forward              include/mtfm/heads.hpp:47-99
  forward_user              include/mtfm/model.hpp:265-312 (forward_scoped)

Inputs use the packed jagged batch layout of include/mtfm_cuda.h (dict of
numpy arrays: user_id, seq_off, seq_kind, seq_schema, ev_off, ev_ts,
ev_feat_off, ev_feats, exp_off, exp_scenario, exp_ts, exp_feat_off, exp_blk,
exp_feats).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

MASK64 = (1 << 64) - 1


# ----------------------------------------------------------------------------
# Errors: the reference's taxonomy (include/mtfm/errors.hpp:9-40).
# ----------------------------------------------------------------------------
class MtfmError(Exception):
    kind = "error"


class ConfigError(MtfmError):
    kind = "config_error"


class IntegrityError(MtfmError):
    kind = "integrity_error"


class DimensionError(MtfmError):
    kind = "dimension_error"


class LookupError_(MtfmError):
    kind = "lookup_error"


class ContractError(MtfmError):
    kind = "contract_error"


# ----------------------------------------------------------------------------
# RNG (rng.hpp:13-83): splitmix64 + xoshiro256**, used for parameter init.
# ----------------------------------------------------------------------------
def splitmix64(state):
    state = (state + 0x9E3779B97F4A7C15) & MASK64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return state, z ^ (z >> 31)


_RNG_LIB = []


def _rng_lib():
    """oracle/rng_block.c compiled on first use (gcc) into oracle/_ref/; None if unavailable."""
    if _RNG_LIB:
        return _RNG_LIB[0]
    lib = None
    try:
        import ctypes
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        src, so = os.path.join(here, "rng_block.c"), os.path.join(here, "_ref", "librng_block.so")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            os.makedirs(os.path.dirname(so), exist_ok=True)
            tmp = so + f".{os.getpid()}"
            subprocess.run(["gcc", "-O2", "-shared", "-fPIC", src, "-o", tmp], check=True, capture_output=True)
            os.replace(tmp, so)
        lib = ctypes.CDLL(so)
        lib.rng_uniform_block.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_void_p]
        lib.rng_uniform_block.restype = None
    except Exception:
        lib = None
    _RNG_LIB.append(lib)
    return lib


class Rng:
    def __init__(self, seed):
        sm = seed & MASK64
        self.s = []
        for _ in range(4):
            sm, v = splitmix64(sm)
            self.s.append(v)

    def next_u64(self):
        s0, s1, s2, s3 = self.s
        x = (s1 * 5) & MASK64
        result = ((((x << 7) | (x >> 57)) & MASK64) * 9) & MASK64
        t = (s1 << 17) & MASK64
        s2 ^= s0
        s3 ^= s1
        s1 ^= s2
        s0 ^= s3
        s2 ^= t
        s3 = ((s3 << 45) | (s3 >> 19)) & MASK64
        self.s = [s0, s1, s2, s3]
        return result

    def next_double(self):
        return (self.next_u64() >> 11) * (2.0 ** -53)

    def uniform_block(self, n, lo, hi):
        # lo + (hi - lo) * next_double(), element by element (rng.hpp:57)
        fast = _rng_lib()
        if fast is not None and n > 64:
            st = np.array(self.s, dtype=np.uint64)
            out = np.empty(n, dtype=np.float64)
            fast.rng_uniform_block(st.ctypes.data, n, float(lo), float(hi), out.ctypes.data)
            self.s = [int(x) for x in st]
            return out
        return self.uniform_block_py(n, lo, hi)

    def uniform_block_py(self, n, lo, hi):
        s0, s1, s2, s3 = self.s
        out = np.empty(n, dtype=np.float64)
        span = hi - lo
        for i in range(n):
            x = (s1 * 5) & MASK64
            r = ((((x << 7) | (x >> 57)) & MASK64) * 9) & MASK64
            t = (s1 << 17) & MASK64
            s2 ^= s0
            s3 ^= s1
            s1 ^= s2
            s0 ^= s3
            s2 ^= t
            s3 = ((s3 << 45) | (s3 >> 19)) & MASK64
            out[i] = lo + span * ((r >> 11) * (2.0 ** -53))
        self.s = [s0, s1, s2, s3]
        return out


# ----------------------------------------------------------------------------
# Schemas / config
# ----------------------------------------------------------------------------
@dataclass
class Schemas:
    hist: list  # [(seq_id, [vocab per slot])]
    rt: list
    scen: list  # [(scenario_id, [u vocabs], [c vocabs], [i vocabs], [tasks])]

    def scenario(self, sid):
        for s in self.scen:
            if s[0] == sid:
                return s
        raise IntegrityError(f"unknown scenario {sid}")


@dataclass
class Config:
    d_model: int = 64
    blocks: int = 4
    target_layers: int = 3
    full_layers: int = 1
    heads: int = 4
    kv_heads: int = 2
    norm: str = "valid"  # valid | seqlen | none  (model_config.hpp:18)
    eps: float = 1e-6
    d_emb: int = 16
    experts: int = 4
    d_expert: int = 64

    @property
    def head_dim(self):
        return self.d_model // self.heads


class GroupTable:
    """groups.hpp:20-53 — h<seq>, r<seq>, t<scenario> in registration order."""

    def __init__(self, sch: Schemas):
        self.keys = []
        self.h, self.r, self.t = {}, {}, {}
        for sid, _ in sch.hist:
            self.h[sid] = len(self.keys)
            self.keys.append(f"h{sid}")
        for sid, _ in sch.rt:
            self.r[sid] = len(self.keys)
            self.keys.append(f"r{sid}")
        for s in sch.scen:
            self.t[s[0]] = len(self.keys)
            self.keys.append(f"t{s[0]}")
        self.scenario_groups = set(self.t.values())

    def group_of(self, kind, gid):
        table = (self.h, self.r, self.t)[kind]
        if gid not in table:
            raise ConfigError(f"unknown token group {'HRT'[kind]}{gid}")
        return table[gid]


def jitter_params(P: dict, seed: int, tower_scale: float) -> dict:
    """Restates oracle/ref_dump.cpp jitter_params (test fixtures only): the
    reference's Rng (rng.hpp:57) drawn in registration order (model.hpp:371-463)
    over gains (1 + U(-0.2, 0.2)), GLN biases (U(-0.1, 0.1)), biases (+ U(-0.1, 0.1))
    and towers (x tower_scale), each value computed in double then rounded to f32."""
    rng = Rng(seed)
    out = {}
    for n, v in P.items():
        v = v.astype(np.float64)
        if n.endswith("/gain"):
            v = 1.0 + rng.uniform_block(v.size, -0.2, 0.2).reshape(v.shape)
        elif "/gln" in n and n.endswith("/bias"):
            v = rng.uniform_block(v.size, -0.1, 0.1).reshape(v.shape)
        elif n.endswith("_b") or n.endswith("/mlp_b1") or n.endswith("/mlp_b2"):
            v = v + rng.uniform_block(v.size, -0.1, 0.1).reshape(v.shape)
        elif n.endswith("/tower_w"):
            v = v * tower_scale
        out[n] = v.astype(np.float32)
    return out


def build_params(sch: Schemas, cfg: Config, seed: int) -> dict:
    """model.hpp:371-463 registration order with Model::build's Rng
    (model.hpp:126-135). Returns name -> float32 array (rows, cols)."""
    rng = Rng(seed ^ 0xA5A5A5A5DEADBEEF)
    d, de = cfg.d_model, cfg.d_emb
    hd = cfg.heads * cfg.head_dim
    gd = cfg.kv_heads * cfg.head_dim
    P = {}
    gt = GroupTable(sch)

    def weight(name, rows, cols, bound):
        P[name] = rng.uniform_block(rows * cols, -bound, bound).astype(np.float32).reshape(rows, cols)

    def add_weight(name, i, o):
        weight(name, i, o, 1.0 / math.sqrt(i))

    def zeros(name, n):
        P[name] = np.zeros((1, n), np.float32)

    def mlp2(base, i):
        add_weight(base + "/mlp_w1", i, 2 * d)
        zeros(base + "/mlp_b1", 2 * d)
        add_weight(base + "/mlp_w2", 2 * d, d)
        zeros(base + "/mlp_b2", d)

    def emb(name, vocab):
        weight(name, vocab, de, 1.0 / math.sqrt(de))

    for pre, lst in (("h", sch.hist), ("r", sch.rt)):
        for sid, vocabs in lst:
            base = f"tok/{pre}{sid}"
            for slot, v in enumerate(vocabs):
                emb(f"{base}/emb{slot}", v)
            mlp2(base, len(vocabs) * de)
    for sid, uv, cv, iv, _ in sch.scen:
        base = f"tok/s{sid}"
        for i, v in enumerate(uv):
            emb(f"{base}/emb_u{i}", v)
        for i, v in enumerate(cv):
            emb(f"{base}/emb_c{i}", v)
        for i, v in enumerate(iv):
            emb(f"{base}/emb_i{i}", v)
        mlp2(base, (len(uv) + len(cv) + len(iv)) * de)
    for b in range(cfg.blocks):
        for l in range(cfg.target_layers + cfg.full_layers):
            tgt = l < cfg.target_layers
            base = f"hta/b{b}/l{l}"
            if tgt:
                add_weight(base + "/fuq_w", d, 2 * hd)
                zeros(base + "/fuq_b", 2 * hd)
                add_weight(base + "/fkv_w", d, 2 * gd)
                zeros(base + "/fkv_b", 2 * gd)
            else:
                add_weight(base + "/f1_w", d, 2 * hd + 2 * gd)
                zeros(base + "/f1_b", 2 * hd + 2 * gd)
            add_weight(base + "/f2_w", hd, d)
            zeros(base + "/f2_b", d)
            for g, key in enumerate(gt.keys):
                P[f"{base}/gln1/{key}/gain"] = np.ones((1, d), np.float32)
                zeros(f"{base}/gln1/{key}/bias", d)
                if not tgt or g in gt.scenario_groups:
                    P[f"{base}/gln2/{key}/gain"] = np.ones((1, hd), np.float32)
                    zeros(f"{base}/gln2/{key}/bias", hd)
    for e in range(cfg.experts):
        add_weight(f"head/expert{e}_w", d, cfg.d_expert)
        zeros(f"head/expert{e}_b", cfg.d_expert)
    for sid, _, _, _, tasks in sch.scen:
        for t in tasks:
            base = f"head/s{sid}/{t}"
            add_weight(base + "/gate_w", d, cfg.experts)
            zeros(base + "/gate_b", cfg.experts)
            add_weight(base + "/tower_w", cfg.d_expert, 1)
            zeros(base + "/tower_b", 1)
    return P


# ----------------------------------------------------------------------------
# Per-user view of the packed batch
# ----------------------------------------------------------------------------
@dataclass
class UserView:
    user_id: int
    hist: list = field(default_factory=list)  # [(schema_id, ts[int64], feats[list of lists])]
    rt: list = field(default_factory=list)
    exposures: list = field(default_factory=list)  # [(scenario, ts, u, c, i)]


def user_views(batch) -> list:
    out = []
    U = len(batch["user_id"])
    for u in range(U):
        v = UserView(int(batch["user_id"][u]))
        for s in range(batch["seq_off"][u], batch["seq_off"][u + 1]):
            e0, e1 = batch["ev_off"][s], batch["ev_off"][s + 1]
            ts = [int(x) for x in batch["ev_ts"][e0:e1]]
            feats = [
                [int(x) for x in batch["ev_feats"][batch["ev_feat_off"][e]:batch["ev_feat_off"][e + 1]]]
                for e in range(e0, e1)
            ]
            rec = (int(batch["seq_schema"][s]), ts, feats)
            (v.hist if batch["seq_kind"][s] == 0 else v.rt).append(rec)
        for x in range(batch["exp_off"][u], batch["exp_off"][u + 1]):
            f0 = batch["exp_feat_off"][x]
            nu, nc, ni = (int(t) for t in batch["exp_blk"][3 * x:3 * x + 3])
            fe = [int(t) for t in batch["exp_feats"][f0:f0 + nu + nc + ni]]
            v.exposures.append((int(batch["exp_scenario"][x]), int(batch["exp_ts"][x]),
                                fe[:nu], fe[nu:nu + nc], fe[nu + nc:]))
        out.append(v)
    return out


# ----------------------------------------------------------------------------
# Plan (tokenizer.hpp:53-134)
# ----------------------------------------------------------------------------
@dataclass
class Plan:
    kind: np.ndarray          # 0 H, 1 R, 2 T  (final order)
    group_id: np.ndarray      # seq schema id (H/R) or scenario id (T)
    ts: np.ndarray
    exposure_ref: np.ndarray  # -1 for H/R
    final_to_pile: np.ndarray
    bounds: tuple             # (l_h, l_r, l_t)
    seq_pieces: list          # [(historical, list_index, schema_id)]
    scen_pieces: list         # [(scenario_id, [exposure indices])]


def plan_user(v: UserView) -> Plan:
    pile = 0
    h_tok, r_tok = [], []
    seq_pieces = []
    for hist, seqs, sink in ((True, v.hist, h_tok), (False, v.rt, r_tok)):
        for li, (sid, ts, _) in enumerate(seqs):
            if not ts:
                continue
            seq_pieces.append((hist, li, sid))
            for t in ts:
                sink.append((t, 0 if hist else 1, sid, -1, pile))
                pile += 1
    order = sorted(range(len(v.exposures)), key=lambda i: (v.exposures[i][1], v.exposures[i][0], i))
    by_scen = {}
    for e in v.exposures:
        by_scen.setdefault(e[0], [])
    for i in order:
        by_scen[v.exposures[i][0]].append(i)
    pile_of = {}
    scen_pieces = []
    for sid in sorted(by_scen):
        idx = by_scen[sid]
        if not idx:
            continue
        for i in idx:
            pile_of[i] = pile
            pile += 1
        scen_pieces.append((sid, list(idx)))
    t_tok = [(v.exposures[i][1], 2, v.exposures[i][0], i, pile_of[i]) for i in order]
    h_tok.sort(key=lambda p: p[0])  # Python sort is stable == std::stable_sort
    r_tok.sort(key=lambda p: p[0])
    allt = h_tok + r_tok + t_tok
    return Plan(
        kind=np.array([p[1] for p in allt], np.uint8),
        group_id=np.array([p[2] for p in allt], np.int32),
        ts=np.array([p[0] for p in allt], np.int64),
        exposure_ref=np.array([p[3] for p in allt], np.int32),
        final_to_pile=np.array([p[4] for p in allt], np.int32),
        bounds=(len(h_tok), len(r_tok), len(t_tok)),
        seq_pieces=seq_pieces,
        scen_pieces=scen_pieces,
    )


def build_mask(kind, ts):
    """mask.cpp:5-29, column rules."""
    n = len(kind)
    m = np.zeros((n, n), np.uint8)
    for j in range(n):
        if kind[j] == 0:
            m[:, j] = 1
        elif kind[j] == 1:
            m[:, j] = (ts > ts[j]).astype(np.uint8)
        else:
            m[j, j] = 1
    return m


def row_scale(counts, n, norm, dtype):
    if norm == "valid":
        return (dtype(1) / np.maximum(counts, 1).astype(dtype)).astype(dtype)
    if norm == "seqlen":
        return np.full(len(counts), dtype(1) / dtype(n), dtype)
    return np.ones(len(counts), dtype)


# ----------------------------------------------------------------------------
# Numerics (kernels.hpp)
# ----------------------------------------------------------------------------
def sigmoid(x):
    x = np.asarray(x)
    one = x.dtype.type(1)
    pos = x >= 0
    e = np.exp(np.where(pos, -x, x))
    return np.where(pos, one / (one + e), e / (one + e)).astype(x.dtype)


def silu(x):
    return (x * sigmoid(x)).astype(x.dtype)


def row_normalize(x, eps):
    dt = x.dtype.type
    mean = x.sum(axis=1, dtype=x.dtype) / dt(x.shape[1])
    c = x - mean[:, None]
    var = (c * c).sum(axis=1, dtype=x.dtype) / dt(x.shape[1])
    inv = dt(1) / np.sqrt(var + dt(eps))
    return (c * inv[:, None]).astype(x.dtype)


def softmax_rows(x):
    m = x.max(axis=1, keepdims=True)
    y = np.exp(x - m)
    return (y * (x.dtype.type(1) / y.sum(axis=1, keepdims=True))).astype(x.dtype)


# ----------------------------------------------------------------------------
# Model
# ----------------------------------------------------------------------------
class Oracle:
    """forward_scoped restated over one user at a time (model.hpp:265-312)."""

    def __init__(self, sch: Schemas, cfg: Config, params: dict, dtype=np.float64):
        self.sch, self.cfg, self.dtype = sch, cfg, dtype
        self.P = {k: np.asarray(v).astype(dtype) for k, v in params.items()}
        self.gt = GroupTable(sch)
        self.PK = (self.P, self.gt.keys)

    # tokenizer.hpp:184-188
    def mlp(self, x, base):
        P = self.P
        h = silu(x @ P[base + "/mlp_w1"] + P[base + "/mlp_b1"][0])
        return h @ P[base + "/mlp_w2"] + P[base + "/mlp_b2"][0]

    def embed(self, tables, ids):
        # tokenizer.hpp:193-207 + eval_ctx.hpp:190-198
        cols = []
        for slot, tab in enumerate(tables):
            sid = []
            for r in ids:
                if slot >= len(r):
                    raise DimensionError("embed_rows: feature slot missing")
                sid.append(r[slot])
            T = self.P[tab]
            for i in sid:
                if i < 0 or i >= T.shape[0]:
                    raise LookupError_(f"gather_rows: id {i} out of range")
            cols.append(T[np.array(sid, dtype=np.int64)])
        return np.concatenate(cols, axis=1) if cols else np.zeros((len(ids), 0), self.dtype)

    def tokenize(self, v: UserView, plan: Plan, only_scenario=-1):
        """assemble_tokens (tokenizer.hpp:240-268)."""
        piles = []
        hist_ids = {sid: voc for sid, voc in self.sch.hist}
        rt_ids = {sid: voc for sid, voc in self.sch.rt}
        for hist, li, sid in plan.seq_pieces:
            table = hist_ids if hist else rt_ids
            if sid not in table:
                raise IntegrityError(f"no tokenizer for sequence schema {sid}")
            base = f"tok/{'h' if hist else 'r'}{sid}"
            rec = (v.hist if hist else v.rt)[li]
            tabs = [f"{base}/emb{k}" for k in range(len(table[sid]))]
            piles.append(self.mlp(self.embed(tabs, rec[2]), base))
        for sid, idx in plan.scen_pieces:
            sc = None
            for s in self.sch.scen:
                if s[0] == sid and (only_scenario < 0 or sid == only_scenario):
                    sc = s
            if sc is None:
                raise IntegrityError(f"no tokenizer for scenario {sid}")
            base = f"tok/s{sid}"
            blocks = []
            for which, n in ((2, len(sc[1])), (3, len(sc[2])), (4, len(sc[3]))):
                if n == 0:
                    continue
                pre = {2: "emb_u", 3: "emb_c", 4: "emb_i"}[which]
                blocks.append(self.embed([f"{base}/{pre}{k}" for k in range(n)],
                                         [v.exposures[i][which] for i in idx]))
            piles.append(self.mlp(np.concatenate(blocks, axis=1), base))
        if not piles:
            raise ContractError("assemble_tokens: sample has no tokens")
        stacked = np.concatenate(piles, axis=0)
        return stacked[plan.final_to_pile]

    def geometry(self, plan: Plan):
        groups = np.array([self.gt.group_of(k, g) for k, g in zip(plan.kind, plan.group_id)], np.int64)
        mask = build_mask(plan.kind, plan.ts)
        counts = mask.sum(axis=1).astype(np.int64)
        scale = row_scale(counts, len(plan.kind), self.cfg.norm, self.dtype)
        return groups, mask, counts, scale

    def gqa(self, q, k, v, mask, scale):
        """hta.hpp:115-134"""
        cfg = self.cfg
        dh = cfg.head_dim
        r = cfg.heads // cfg.kv_heads
        outs = []
        maskf = mask.astype(self.dtype)
        for h in range(cfg.heads):
            g = h // r
            s = q[:, h * dh:(h + 1) * dh] @ k[:, g * dh:(g + 1) * dh].T
            w = silu(s * maskf) * scale[:, None]
            outs.append(w @ v[:, g * dh:(g + 1) * dh])
        return np.concatenate(outs, axis=1)

    def gln(self, x, groups, prefix):
        xn = row_normalize(x, self.cfg.eps)
        out = np.empty_like(xn)
        for g in np.unique(groups):
            rows = groups == g
            key = self.gt.keys[g]
            out[rows] = xn[rows] * self.P[f"{prefix}/{key}/gain"][0] + self.P[f"{prefix}/{key}/bias"][0]
        return out

    def full_layer(self, x, base, groups, mask, scale):
        """hta.hpp:138-155"""
        cfg, P = self.cfg, self.P
        hd = cfg.heads * cfg.head_dim
        gd = cfg.kv_heads * cfg.head_dim
        xn = self.gln(x, groups, base + "/gln1")
        proj = silu(xn @ P[base + "/f1_w"] + P[base + "/f1_b"][0])
        u, q = proj[:, :hd], proj[:, hd:2 * hd]
        k, v = proj[:, 2 * hd:2 * hd + gd], proj[:, 2 * hd + gd:]
        a = self.gqa(q, k, v, mask, scale)
        gated = self.gln(a, groups, base + "/gln2") * u
        return (gated @ P[base + "/f2_w"] + P[base + "/f2_b"][0]) + x

    def target_layer(self, x, base, groups, mask, scale, off):
        """hta.hpp:158-184"""
        cfg, P = self.cfg, self.P
        hd = cfg.heads * cfg.head_dim
        gd = cfg.kv_heads * cfg.head_dim
        xn = self.gln(x, groups, base + "/gln1")
        uq = silu(xn[off:] @ P[base + "/fuq_w"] + P[base + "/fuq_b"][0])
        kv = silu(xn @ P[base + "/fkv_w"] + P[base + "/fkv_b"][0])
        a = self.gqa(uq[:, hd:], kv[:, :gd], kv[:, gd:], mask[off:], scale[off:])
        gated = self.gln(a, groups[off:], base + "/gln2") * uq[:, :hd]
        t_new = (gated @ P[base + "/f2_w"] + P[base + "/f2_b"][0]) + x[off:]
        return np.concatenate([x[:off], t_new], axis=0)

    def stack(self, x0, plan, groups, mask, scale, keep_layers=False):
        """hta.hpp:188-212"""
        cfg = self.cfg
        x = x0
        layers = []
        off = plan.bounds[0] + plan.bounds[1]
        for b in range(cfg.blocks):
            for l in range(cfg.target_layers + cfg.full_layers):
                base = f"hta/b{b}/l{l}"
                if l < cfg.target_layers:
                    x = self.target_layer(x, base, groups, mask, scale, off)
                else:
                    x = self.full_layer(x, base, groups, mask, scale)
                if keep_layers:
                    layers.append(x)
        return x, layers

    def heads(self, t_rows, plan):
        """heads.hpp:47-99 -> list of (scenario, task_idx, task, rows, logits)."""
        cfg, P = self.cfg, self.P
        off = plan.bounds[0] + plan.bounds[1]
        scen_of_row = plan.group_id[off:]
        cols = []
        for sid in sorted(set(int(s) for s in scen_of_row)):
            rows = np.nonzero(scen_of_row == sid)[0]
            try:
                tasks = self.sch.scenario(sid)[4]
            except IntegrityError:
                raise ConfigError(f"mmoe_forward: no tasks registered for scenario {sid}")
            xs = t_rows[rows]
            ex = [silu(xs @ P[f"head/expert{e}_w"] + P[f"head/expert{e}_b"][0]) for e in range(cfg.experts)]
            for ti, t in enumerate(tasks):
                base = f"head/s{sid}/{t}"
                gate = softmax_rows(xs @ P[base + "/gate_w"] + P[base + "/gate_b"][0])
                mix = ex[0] * gate[:, 0:1]
                for e in range(1, cfg.experts):
                    mix = mix + ex[e] * gate[:, e:e + 1]
                z = (mix @ P[base + "/tower_w"] + P[base + "/tower_b"][0])[:, 0]
                cols.append((sid, ti, t, rows, z))
        return cols

    def forward_user(self, v: UserView, keep_layers=False):
        plan = plan_user(v)
        x0 = self.tokenize(v, plan)
        groups, mask, counts, scale = self.geometry(plan)
        xf, layers = self.stack(x0, plan, groups, mask, scale, keep_layers)
        off = plan.bounds[0] + plan.bounds[1]
        cols = self.heads(xf[off:], plan)
        recs = []
        for sid, ti, t, rows, z in cols:
            p = sigmoid(z.astype(self.dtype)).astype(np.float64)
            p = np.minimum(1.0 - 1e-12, np.maximum(1e-12, p))
            for r, zz, pp in zip(rows, z, p):
                recs.append((v.user_id, sid, int(plan.exposure_ref[off + r]), ti, float(zz), float(pp)))
        return dict(plan=plan, x0=x0, layers=layers, xf=xf, records=recs, counts=counts, groups=groups)

    def forward_batch(self, batch):
        """Concatenated forward_sample records over every user of the batch."""
        out = []
        for v in user_views(batch):
            out.extend(self.forward_user(v)["records"])
        return out


# ----------------------------------------------------------------------------
# 2:4 pruning (prune.hpp)
# ----------------------------------------------------------------------------
def prune_2_4(w):
    """prune_2_4_inplace (prune.hpp:33-70) on a copy: per column, each full group of
    4 consecutive rows keeps its two largest |w| (ties keep the earlier row); a
    partial trailing group is exempt. Returns (pruned, zeros_written, groups, tail)."""
    w = np.array(w, dtype=np.float32, copy=True)
    rows, cols = w.shape
    full = rows // 4
    zeros = 0
    for j in range(cols):
        for g in range(full):
            mag = [abs(float(w[4 * g + i, j])) for i in range(4)]
            k0, k1 = 0, 1
            if mag[k1] > mag[k0]:
                k0, k1 = k1, k0
            for i in (2, 3):
                if mag[i] > mag[k0]:
                    k1, k0 = k0, i
                elif mag[i] > mag[k1]:
                    k1 = i
            for i in range(4):
                if i not in (k0, k1):
                    w[4 * g + i, j] = 0.0
                    zeros += 1
    return w, zeros, full * cols, rows - full * 4


def is_projection_param(name):
    """prune.hpp:83-90."""
    return name.startswith("hta/") and name.endswith(("/f1_w", "/fuq_w", "/fkv_w", "/f2_w"))


# ----------------------------------------------------------------------------
# User-level aggregation (datagen.cpp:171-216)
# ----------------------------------------------------------------------------
def aggregate_users(scenario_ids, stream, store):
    """Restates aggregate_users over packed arrays. stream: user_id, scenario, ts,
    feat_off, blk, feats (arrival order); store: packed batch of the users' H/R
    sequences (std::map iteration order). Returns (packed batch, exp_src)."""
    known = set(int(x) for x in scenario_ids)
    store_users = [int(u) for u in store["user_id"]]
    pos = {u: i for i, u in enumerate(store_users)}
    per_scenario = {}  # scenario -> user -> [stream index], each in stream order
    for x in range(len(stream["user_id"])):
        sc, u = int(stream["scenario"][x]), int(stream["user_id"][x])
        if sc not in known:  # datagen.cpp:178-180
            raise IntegrityError(f"aggregate: exposure references unknown scenario {sc}")
        if u not in pos:  # datagen.cpp:181-183
            raise IntegrityError(f"aggregate: exposure references unknown user {u}")
        per_scenario.setdefault(sc, {}).setdefault(u, []).append(x)
    merged = {}  # user -> [stream index]: scenarios ascending, stream order within
    for sc in sorted(per_scenario):
        for u in sorted(per_scenario[sc]):
            merged.setdefault(u, []).extend(per_scenario[sc][u])
    out = {k: [] for k in BATCH_KEYS}
    for k in ("seq_off", "ev_off", "ev_feat_off", "exp_off", "exp_feat_off"):
        out[k].append(0)
    src = []
    for u in sorted(merged):
        r = pos[u]
        out["user_id"].append(u)
        for q in range(store["seq_off"][r], store["seq_off"][r + 1]):
            out["seq_kind"].append(int(store["seq_kind"][q]))
            out["seq_schema"].append(int(store["seq_schema"][q]))
            for e in range(store["ev_off"][q], store["ev_off"][q + 1]):
                out["ev_ts"].append(int(store["ev_ts"][e]))
                out["ev_feats"].extend(int(f) for f in store["ev_feats"][store["ev_feat_off"][e]:store["ev_feat_off"][e + 1]])
                out["ev_feat_off"].append(len(out["ev_feats"]))
            out["ev_off"].append(len(out["ev_ts"]))
        out["seq_off"].append(len(out["seq_kind"]))
        for x in merged[u]:
            src.append(x)
            out["exp_scenario"].append(int(stream["scenario"][x]))
            out["exp_ts"].append(int(stream["ts"][x]))
            out["exp_blk"].extend(int(b) for b in stream["blk"][3 * x:3 * x + 3])
            out["exp_feats"].extend(int(f) for f in stream["feats"][stream["feat_off"][x]:stream["feat_off"][x + 1]])
            out["exp_feat_off"].append(len(out["exp_feats"]))
        out["exp_off"].append(len(out["exp_scenario"]))
    return out, src


# ----------------------------------------------------------------------------
# Fixture helpers
# ----------------------------------------------------------------------------
BATCH_KEYS = ("user_id", "seq_off", "seq_kind", "seq_schema", "ev_off", "ev_ts", "ev_feat_off",
              "ev_feats", "exp_off", "exp_scenario", "exp_ts", "exp_feat_off", "exp_blk", "exp_feats")

NORMS = {0: "valid", 1: "seqlen", 2: "none"}


def schemas_from_arrays(a) -> Schemas:
    def seqs(key):
        ids, ns, voc = a[f"schema/{key}/ids"], a[f"schema/{key}/nslots"], a[f"schema/{key}/vocabs"]
        out, p = [], 0
        for i, n in zip(ids, ns):
            out.append((int(i), [int(x) for x in voc[p:p + n]]))
            p += n
        return out

    tasks = bytes(a["schema/scen/tasks"]).decode().split(";")
    scen, p = [], 0
    voc = a["schema/scen/vocabs"]
    for k, sid in enumerate(a["schema/scen/ids"]):
        nu, nc, ni = int(a["schema/scen/nu"][k]), int(a["schema/scen/nc"][k]), int(a["schema/scen/ni"][k])
        u = [int(x) for x in voc[p:p + nu]]
        c = [int(x) for x in voc[p + nu:p + nu + nc]]
        i = [int(x) for x in voc[p + nu + nc:p + nu + nc + ni]]
        p += nu + nc + ni
        scen.append((int(sid), u, c, i, tasks[k].split(",") if tasks[k] else []))
    return Schemas(seqs("hist"), seqs("rt"), scen)


def config_from_arrays(a) -> Config:
    d, blocks, K, P, H, G, norm, demb, E, dexp = (int(x) for x in a["config/ints"])
    return Config(d_model=d, blocks=blocks, target_layers=K, full_layers=P, heads=H, kv_heads=G,
                  norm=NORMS[norm], eps=float(a["config/eps"][0]), d_emb=demb, experts=E, d_expert=dexp)


def batch_from_arrays(a) -> dict:
    return {k: a[f"batch/{k}"] for k in BATCH_KEYS}
