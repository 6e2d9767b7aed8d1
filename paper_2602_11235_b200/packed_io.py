"""Packed jagged batch files (MTFMPB1) and parameter files (MTFMPF1).

The packed batch of include/mtfm_cuda.h is the unit the device pipeline
consumes; these files let a batch be produced once (ingestion, benchmarking,
sharding) and read back without re-packing per-user objects:

    MTFMPB1\\n
    model <d> <blocks> <K> <P> <H> <G> <norm> <eps> <d_emb> <experts> <d_expert>\\n   ("model -" if absent)
    hist <n>\\n  n x "<seq_id> <n_slots> <vocab>..."
    rt <n>\\n    n x "<seq_id> <n_slots> <vocab>..."
    scen <n>\\n  n x "<scenario_id> <nu> <nc> <ni> <vocab>... <n_tasks> <task>..."
    arrays <k>\\n
    k x ("<key> <i1|u1|i4|i8> <count>\\n" + raw little-endian bytes)
    end\\n

Parameter file: "MTFMPF1\\n<n>\\n" then n x ("<name> <rows> <cols>\\n" + rows*cols
f32), in registration order (model.hpp:371-463). The same layout is read by
oracle/packed_io.hpp (test / baseline infrastructure) so the reference CPU
path and the GPU path can score byte-identical inputs.
"""
from __future__ import annotations

import numpy as np

from .schema import (BATCH_DTYPES, BATCH_KEYS, HTAConfig, ModelConfig, ScenarioSchema, SchemaSet, SequenceSchema,
                     normalize_batch)

_CODES = {np.dtype(np.uint8): "u1", np.dtype(np.int32): "i4", np.dtype(np.int64): "i8", np.dtype(np.int8): "i1"}
_DTYPES = {v: k for k, v in _CODES.items()}
_NORMS = {"valid": 0, "seqlen": 1, "none": 2}


def save_packed(path, batch: dict, schemas: SchemaSet | None = None, cfg: ModelConfig | None = None):
    b = normalize_batch(batch)
    lines = ["MTFMPB1"]
    if cfg is None:
        lines.append("model -")
    else:
        h = cfg.hta
        norm = _NORMS[h.norm] if isinstance(h.norm, str) else int(h.norm)
        lines.append(f"model {h.d_model} {h.blocks} {h.target_layers} {h.full_layers} {h.heads} {h.kv_heads} "
                     f"{norm} {h.eps!r} {cfg.d_emb} {cfg.experts} {cfg.d_expert}")
    hist = schemas.hist if schemas else []
    rt = schemas.rt if schemas else []
    sc = schemas.scenarios if schemas else []
    for tag, seqs in (("hist", hist), ("rt", rt)):
        lines.append(f"{tag} {len(seqs)}")
        for s in seqs:
            lines.append(" ".join(map(str, [s.seq_id, len(s.feature_vocabs), *s.feature_vocabs])))
    lines.append(f"scen {len(sc)}")
    for s in sc:
        for t in s.tasks:
            if not t or any(c.isspace() for c in t):
                raise ValueError(f"task name {t!r} cannot be stored")
        lines.append(" ".join(map(str, [s.scenario_id, len(s.user_feature_vocabs), len(s.cross_feature_vocabs),
                                        len(s.item_feature_vocabs), *s.user_feature_vocabs,
                                        *s.cross_feature_vocabs, *s.item_feature_vocabs, len(s.tasks),
                                        *s.tasks])))
    lines.append(f"arrays {len(BATCH_KEYS)}")
    with open(path, "wb") as f:
        f.write(("\n".join(lines) + "\n").encode())
        for k in BATCH_KEYS:
            a = b[k]
            f.write(f"{k} {_CODES[a.dtype]} {a.size}\n".encode())
            f.write(a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes())
        f.write(b"end\n")


def _line(f):
    s = f.readline()
    if not s:
        raise ValueError("truncated packed file")
    return s.decode().split()


def load_packed(path):
    """-> (batch dict, SchemaSet or None, ModelConfig or None)."""
    with open(path, "rb") as f:
        if f.readline().strip() != b"MTFMPB1":
            raise ValueError(f"{path}: not an MTFMPB1 file")
        m = _line(f)
        cfg = None
        if m[1] != "-":
            d, bl, K, P, H, G, norm = (int(x) for x in m[1:8])
            cfg = ModelConfig(HTAConfig(d_model=d, blocks=bl, target_layers=K, full_layers=P, heads=H, kv_heads=G,
                                        norm={v: k for k, v in _NORMS.items()}[norm], eps=float(m[8])),
                              d_emb=int(m[9]), experts=int(m[10]), d_expert=int(m[11]))
        seqs = {}
        for tag in ("hist", "rt"):
            t, n = _line(f)
            assert t == tag
            out = []
            for _ in range(int(n)):
                v = [int(x) for x in _line(f)]
                out.append(SequenceSchema(v[0], v[2:2 + v[1]]))
            seqs[tag] = out
        t, n = _line(f)
        assert t == "scen"
        sc = []
        for _ in range(int(n)):
            v = _line(f)
            sid, nu, nc, ni = (int(x) for x in v[:4])
            voc = [int(x) for x in v[4:4 + nu + nc + ni]]
            nt = int(v[4 + nu + nc + ni])
            tasks = v[5 + nu + nc + ni:5 + nu + nc + ni + nt]
            sc.append(ScenarioSchema(sid, voc[:nu], voc[nu:nu + nc], voc[nu + nc:], tasks))
        t, n = _line(f)
        assert t == "arrays"
        batch = {}
        for _ in range(int(n)):
            key, code, cnt = _line(f)
            dt = _DTYPES[code].newbyteorder("<")
            raw = f.read(int(cnt) * dt.itemsize)
            if len(raw) != int(cnt) * dt.itemsize:
                raise ValueError("truncated packed file")
            batch[key] = np.frombuffer(raw, dtype=dt).astype(BATCH_DTYPES[key])
        if f.readline().strip() != b"end":
            raise ValueError("missing end marker")
    schemas = SchemaSet(seqs["hist"], seqs["rt"], sc) if (seqs["hist"] or seqs["rt"] or sc) else None
    return normalize_batch(batch), schemas, cfg


def save_params(path, params: dict, order=None):
    names = list(order) if order is not None else list(params)
    with open(path, "wb") as f:
        f.write(f"MTFMPF1\n{len(names)}\n".encode())
        for n in names:
            a = np.ascontiguousarray(np.asarray(params[n], dtype="<f4"))
            a2 = a.reshape(a.shape[0] if a.ndim == 2 else 1, -1)
            f.write(f"{n} {a2.shape[0]} {a2.shape[1]}\n".encode())
            f.write(a2.tobytes())


def load_params(path):
    P = {}
    with open(path, "rb") as f:
        if f.readline().strip() != b"MTFMPF1":
            raise ValueError(f"{path}: not an MTFMPF1 file")
        n = int(f.readline())
        for _ in range(n):
            name, r, c = _line(f)
            r, c = int(r), int(c)
            P[name] = np.frombuffer(f.read(r * c * 4), dtype="<f4").astype(np.float32).reshape(r, c)
    return P
