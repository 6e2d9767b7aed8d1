"""Host-side mirror of the reference Model API over the CUDA C-ABI.

    Model.build(schemas, cfg, params)        ~ Model<Real>::build + ParamStore
    model.forward_sample(sample)             ~ Model::forward_sample   (model.hpp:251)
    model.forward_with(sample, only_scenario)~ Model::forward_scoped   (model.hpp:265)
    model.forward_samples(samples)           concatenated forward_sample records
    model.forward_batch(packed) -> RecordArrays  the batched hot path
    infer_request(model, request)            ~ subgraph.hpp:47-62

Every compute step runs in libmtfm_cuda.so on the GPU; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import abi
from .schema import (BATCH_KEYS, InferenceRequest, ModelConfig, PredictionRecord, SchemaSet, normalize_batch,
                     pack_samples, sample_view_of_request)


@dataclass
class RecordArrays:
    user_id: np.ndarray
    scenario_id: np.ndarray
    exposure_index: np.ndarray
    task_index: np.ndarray
    logit: np.ndarray
    probability: np.ndarray

    def __len__(self):
        return len(self.user_id)


def _i32(v):
    return np.ascontiguousarray(np.asarray(v, dtype=np.int32))


class PreparedBatch:
    """A batch resident in HBM (mtfm_cuda_batch_prepare); run() enqueues the
    forward without host synchronisation, results() waits and copies."""

    def __init__(self, model: "Model", batch: dict, only_scenario: int = -1):
        self.model = model
        self.batch = normalize_batch(batch)
        self._pb = model._packed(self.batch)
        h = C.c_void_p()
        abi.check(abi.lib().mtfm_cuda_batch_prepare(model._h, C.byref(self._pb), only_scenario, C.byref(h)))
        self._h = h
        self.n_records = int(abi.lib().mtfm_cuda_count_records(model._h, C.byref(self._pb)))

    def update(self, batch: dict, only_scenario: int = -1):
        """Load another batch into this object's device buffers (mtfm_cuda_batch_update)."""
        self.batch = normalize_batch(batch)
        self._pb = self.model._packed(self.batch)
        abi.check(abi.lib().mtfm_cuda_batch_update(self.model._h, self._h, C.byref(self._pb), only_scenario))
        self.n_records = int(abi.lib().mtfm_cuda_count_records(self.model._h, C.byref(self._pb)))

    def run(self):
        abi.check(abi.lib().mtfm_cuda_batch_run(self.model._h, self._h))

    def results(self) -> RecordArrays:
        out, rec = self.model._record_buffers(self.n_records)
        abi.check(abi.lib().mtfm_cuda_batch_results(self.model._h, self._h, C.byref(rec)))
        n = int(rec.n_records)
        return RecordArrays(*(a[:n] for a in out))

    def fetch(self, which, dtype, count):
        dst = np.empty(count, dtype=dtype)
        got = abi.lib().mtfm_cuda_debug_fetch(self.model._h, self._h, which.encode(), abi.ptr(dst), dst.nbytes)
        if got < 0:
            raise abi.ContractError(f"debug_fetch({which}) failed")
        return dst

    def free(self):
        if self._h:
            abi.lib().mtfm_cuda_batch_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Model:
    def __init__(self, schemas: SchemaSet, cfg: ModelConfig, precision="bf16", device=0):
        self.schemas, self.cfg = schemas, cfg
        self.precision = precision
        L = abi.lib()
        h = cfg.hta
        md = abi.ModelDesc(h.d_model, h.blocks, h.target_layers, h.full_layers, h.heads, h.kv_heads,
                           abi.NORMS[h.norm] if isinstance(h.norm, str) else int(h.norm), h.eps, cfg.d_emb,
                           cfg.experts, cfg.d_expert)
        keep = []

        def arr(v):
            a = _i32(v if len(v) else [0])
            keep.append(a)
            return a.ctypes.data_as(abi._P32)

        hist, rt, sc = schemas.hist, schemas.rt, schemas.scenarios
        names = [t.encode() for s in sc for t in s.tasks]
        keep.append(names)
        tn = (C.c_char_p * max(1, len(names)))(*names)
        sd = abi.SchemaDesc(
            len(hist), arr([s.seq_id for s in hist]), arr([len(s.feature_vocabs) for s in hist]),
            arr([v for s in hist for v in s.feature_vocabs]),
            len(rt), arr([s.seq_id for s in rt]), arr([len(s.feature_vocabs) for s in rt]),
            arr([v for s in rt for v in s.feature_vocabs]),
            len(sc), arr([s.scenario_id for s in sc]), arr([len(s.user_feature_vocabs) for s in sc]),
            arr([len(s.cross_feature_vocabs) for s in sc]), arr([len(s.item_feature_vocabs) for s in sc]),
            arr([v for s in sc for v in (*s.user_feature_vocabs, *s.cross_feature_vocabs, *s.item_feature_vocabs)]),
            arr([len(s.tasks) for s in sc]), tn)
        out = C.c_void_p()
        prec = abi.PRECISION_BF16 if precision == "bf16" else abi.PRECISION_FP32_CHECK
        abi.check(L.mtfm_cuda_create(device, C.byref(md), C.byref(sd), prec, C.byref(out)))
        self._h = out
        self._tasks = {s.scenario_id: list(s.tasks) for s in sc}

    # ---- parameters (ParamStore, params.hpp:22-132)
    def param_specs(self):
        L = abi.lib()
        out = []
        r, c = C.c_int64(), C.c_int64()
        for i in range(L.mtfm_cuda_num_params(self._h)):
            n = L.mtfm_cuda_param_name(self._h, i, C.byref(r), C.byref(c))
            out.append((n.decode(), r.value, c.value))
        return out

    def set_param(self, name, value):
        v = np.ascontiguousarray(np.asarray(value, dtype=np.float32))
        if v.ndim == 1:
            v = v.reshape(1, -1)
        abi.check(abi.lib().mtfm_cuda_set_param(self._h, name.encode(), abi.ptr(v), v.shape[0], v.shape[1]))

    def set_params(self, params: dict):
        for name, _, _ in self.param_specs():
            if name not in params:
                raise abi.ConfigError(f"parameter not provided: {name}")
            self.set_param(name, params[name])

    @classmethod
    def build(cls, schemas, cfg, params, precision="bf16", device=0):
        m = cls(schemas, cfg, precision, device)
        m.set_params(params)
        return m

    # ---- scenario subgraph (subgraph.hpp:25-42)
    def restrict_to_scenario(self, scenario_id: int):
        """Turns this handle into a ScenarioSubgraph deployment: only the shared
        parameters and scenario_id's own are registered (param_specs() is the
        subgraph's ParamStore) and every forward is scoped to scenario_id."""
        abi.check(abi.lib().mtfm_cuda_restrict_to_scenario(self._h, int(scenario_id)))
        self.subgraph = int(scenario_id)
        return self

    @classmethod
    def build_subgraph(cls, schemas, cfg, sub_params, scenario_id, precision="bf16", device=0):
        """A model holding exactly extract_subgraph(model, scenario_id).params."""
        m = cls(schemas, cfg, precision, device).restrict_to_scenario(scenario_id)
        m.set_params(sub_params)
        return m

    # ---- forward
    def _packed(self, b):
        return abi.PackedBatch(len(b["user_id"]), len(b["seq_kind"]), len(b["ev_ts"]), len(b["exp_ts"]),
                               len(b["ev_feats"]), len(b["exp_feats"]),
                               *(abi.ptr(b[k]) for k in BATCH_KEYS))

    def _record_buffers(self, n):
        out = (np.empty(n, np.int64), np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n, np.int32),
               np.empty(n, np.float32), np.empty(n, np.float64))
        rec = abi.Records(n, 0, *(abi.ptr(a) for a in out))
        return out, rec

    def prepare(self, batch: dict, only_scenario=-1) -> PreparedBatch:
        return PreparedBatch(self, batch, only_scenario)

    def forward_batch(self, batch: dict, only_scenario=-1) -> RecordArrays:
        b = normalize_batch(batch)
        pb = self._packed(b)
        # capacity bound instead of a counting pass: every exposure yields at most
        # max-tasks records (the library reports the exact count)
        max_tasks = max((len(t) for t in self._tasks.values()), default=0)
        out, rec = self._record_buffers(int(len(b["exp_ts"])) * max_tasks)
        abi.check(abi.lib().mtfm_cuda_forward(self._h, C.byref(pb), only_scenario, C.byref(rec)))
        k = int(rec.n_records)
        return RecordArrays(*(a[:k] for a in out))

    def forward_samples(self, samples, only_scenario=-1, attach_labels=True):
        ra = self.forward_batch(pack_samples(samples), only_scenario)
        by_uid = {}
        for s in samples:
            by_uid.setdefault(s.user_id, []).append(s)
        recs = []
        # records are user-major in batch order; labels come from the host samples
        pos = 0
        for s in samples:
            n = sum(len(self._tasks.get(e.scenario_id, [])) for e in s.exposures
                    if only_scenario < 0 or e.scenario_id == only_scenario)
            for i in range(pos, pos + n):
                task = self._tasks[int(ra.scenario_id[i])][int(ra.task_index[i])]
                label = -1
                if attach_labels:
                    label = s.exposures[int(ra.exposure_index[i])].labels.get(task, -1)
                recs.append(PredictionRecord(int(ra.user_id[i]), int(ra.scenario_id[i]), int(ra.exposure_index[i]),
                                             task, float(ra.probability[i]), label))
            pos += n
        return recs

    def forward_sample(self, sample):
        return self.forward_samples([sample])

    def forward_with(self, sample, only_scenario=-1):
        return self.forward_samples([sample], only_scenario)

    # ---- training (Trainer::train_step, train.hpp:111-147; fp32 handles)
    def train_step(self, batch, labels, lr=3e-4, beta1=0.9, beta2=0.999, eps=1e-8, clip_norm=1.0, global_batch=0,
                   prepared: "PreparedBatch" = None):
        """One optimizer step over every user of `batch`; labels [n_exposures][max_tasks]
        (scenario task order, -1 absent). Returns TrainResult (loss, grad_norm, step)."""
        lab = np.ascontiguousarray(np.asarray(labels, dtype=np.int32))
        if lab.ndim == 1:
            lab = lab.reshape(-1, 1)
        pb = prepared if prepared is not None else self.prepare(batch)
        cfg = abi.TrainConfig(lr, beta1, beta2, eps, clip_norm, int(global_batch))
        res = abi.TrainResult()
        abi.check(abi.lib().mtfm_cuda_train_step(self._h, pb._h, abi.ptr(lab), lab.shape[1], C.byref(cfg), C.byref(res)))
        return res

    def prune_projections(self):
        """prune_model_projections (prune.hpp:92-103): 2:4 pattern on every f1/fuq/fkv/f2."""
        rep = abi.PruneReport()
        abi.check(abi.lib().mtfm_cuda_prune_projections(self._h, C.byref(rep)))
        return dict(groups_covered=rep.groups_covered, zeros_written=rep.zeros_written,
                    exempt_tail_rows=rep.exempt_tail_rows, pruned_params=rep.pruned_params)

    def set_sparse_mma(self, mode=2):
        """2:4 sparse tensor cores for f1/fuq/fkv/f2 (include/mtfm_cuda.h): mode 2 when the
        weights are 2:4 (default), 1 required, 0 dense. Returns whether the bf16 forward uses it."""
        active = C.c_int32(0)
        abi.check(abi.lib().mtfm_cuda_set_sparse_mma(self._h, int(mode), C.byref(active)))
        return bool(active.value)

    def get_param(self, name, rows, cols):
        out = np.empty((rows, cols), np.float32)
        abi.check(abi.lib().mtfm_cuda_get_param(self._h, name.encode(), abi.ptr(out), rows, cols))
        return out

    def get_grad(self, name, rows, cols):
        out = np.empty((rows, cols), np.float32)
        abi.check(abi.lib().mtfm_cuda_get_grad(self._h, name.encode(), abi.ptr(out), rows, cols))
        return out

    def dp_init(self, nranks, rank, unique_id: bytes):
        buf = (C.c_char * 128).from_buffer_copy(unique_id)
        abi.check(abi.lib().mtfm_cuda_dp_init(self._h, int(nranks), int(rank), C.cast(buf, C.c_void_p)))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_char * 128)()
        abi.check(abi.lib().mtfm_nccl_unique_id(C.cast(buf, C.c_void_p)))
        return bytes(buf)

    def last_stats(self):
        st = abi.RunStats()
        abi.check(abi.lib().mtfm_cuda_last_stats(self._h, C.byref(st)))
        return st

    def set_profiling(self, on=True):
        abi.check(abi.lib().mtfm_cuda_set_profiling(self._h, 1 if on else 0))

    def profile(self):
        """[(stage, ms, flops, bytes)] of the last run when profiling is on."""
        L = abi.lib()
        out = []
        ms, fl, by = C.c_double(), C.c_double(), C.c_double()
        for i in range(L.mtfm_cuda_profile_count(self._h)):
            n = L.mtfm_cuda_profile_entry(self._h, i, C.byref(ms), C.byref(fl), C.byref(by))
            out.append((n.decode(), ms.value, fl.value, by.value))
        return out

    def stream_handle(self):
        return abi.lib().mtfm_cuda_stream(self._h)

    def close(self):
        if getattr(self, "_h", None):
            abi.lib().mtfm_cuda_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def infer_requests(model: Model, requests):
    """Request-level serving at scale: many InferenceRequests scored in ONE
    forward, each request one user sample of the packed batch (its candidates
    as T tokens, tokenizer.hpp:138-153). Per request the records equal
    infer_request(model, sub, request) (subgraph.hpp:47-62): T tokens never see
    other users or each other. Returns one record list per request."""
    requests = list(requests)
    sub = getattr(model, "subgraph", -1)
    for r in requests:
        if sub >= 0 and r.scenario_id != sub:
            raise abi.IntegrityError(f"request scenario {r.scenario_id} does not match subgraph scenario {sub}")
    views = [sample_view_of_request(r) for r in requests]
    # a full model binds all scenarios: each sample only holds its request's scenario,
    # so the unscoped forward equals the per-request scoped ones
    ra = model.forward_batch(pack_samples(views), sub)
    out, pos = [], 0
    for r in requests:
        n = len(r.candidates) * len(model._tasks.get(r.scenario_id, []))
        recs = []
        for i in range(pos, pos + n):
            task = model._tasks[int(ra.scenario_id[i])][int(ra.task_index[i])]
            recs.append(PredictionRecord(int(ra.user_id[i]), int(ra.scenario_id[i]), int(ra.exposure_index[i]),
                                         task, float(ra.probability[i]), -1))
        out.append(recs)
        pos += n
    return out


def infer_request(model: Model, request: InferenceRequest):
    """subgraph.hpp:47-62: all candidates of one request packed as T tokens of
    one sequence, bound to the request's scenario only, no labels."""
    return model.forward_samples([sample_view_of_request(request)], only_scenario=request.scenario_id,
                                 attach_labels=False)
