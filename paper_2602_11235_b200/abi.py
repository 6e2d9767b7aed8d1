"""ctypes binding of include/mtfm_cuda.h (libmtfm_cuda.so, built in-tree).

There is no fallback: if the library is missing or the GPU is absent, the
calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmtfm_cuda.so")

OK, CONFIG_ERROR, INTEGRITY_ERROR, DIMENSION_ERROR, PARSE_ERROR, LOOKUP_ERROR, CONTRACT_ERROR, CUDA_ERROR = range(8)
PRECISION_BF16, PRECISION_FP32_CHECK = 0, 1
NORMS = {"valid": 0, "seqlen": 1, "none": 2}


class MtfmError(RuntimeError):
    """Base of the reference's exception taxonomy (errors.hpp:9-40)."""
    status = -1


class ConfigError(MtfmError):
    status = CONFIG_ERROR


class IntegrityError(MtfmError):
    status = INTEGRITY_ERROR


class DimensionError(MtfmError):
    status = DIMENSION_ERROR


class ParseError(MtfmError):
    status = PARSE_ERROR


class LookupError_(MtfmError):
    status = LOOKUP_ERROR


class ContractError(MtfmError):
    status = CONTRACT_ERROR


class CudaError(MtfmError):
    status = CUDA_ERROR


_BY_STATUS = {c.status: c for c in (ConfigError, IntegrityError, DimensionError, ParseError, LookupError_,
                                    ContractError, CudaError)}


class ModelDesc(C.Structure):
    _fields_ = [("d_model", C.c_int32), ("blocks", C.c_int32), ("target_layers", C.c_int32),
                ("full_layers", C.c_int32), ("heads", C.c_int32), ("kv_heads", C.c_int32), ("norm", C.c_int32),
                ("eps", C.c_double), ("d_emb", C.c_int32), ("experts", C.c_int32), ("d_expert", C.c_int32)]


_P32 = C.POINTER(C.c_int32)


class SchemaDesc(C.Structure):
    _fields_ = [("n_hist", C.c_int32), ("hist_ids", _P32), ("hist_nslots", _P32), ("hist_vocabs", _P32),
                ("n_rt", C.c_int32), ("rt_ids", _P32), ("rt_nslots", _P32), ("rt_vocabs", _P32),
                ("n_scen", C.c_int32), ("scen_ids", _P32), ("scen_nu", _P32), ("scen_nc", _P32), ("scen_ni", _P32),
                ("scen_vocabs", _P32), ("scen_ntasks", _P32), ("task_names", C.POINTER(C.c_char_p))]


class PackedBatch(C.Structure):
    _fields_ = [("n_users", C.c_int32), ("n_seqs", C.c_int32), ("n_events", C.c_int32), ("n_exposures", C.c_int32),
                ("n_ev_feats", C.c_int64), ("n_exp_feats", C.c_int64),
                ("user_id", C.c_void_p), ("seq_off", C.c_void_p), ("seq_kind", C.c_void_p),
                ("seq_schema", C.c_void_p), ("ev_off", C.c_void_p), ("ev_ts", C.c_void_p),
                ("ev_feat_off", C.c_void_p), ("ev_feats", C.c_void_p), ("exp_off", C.c_void_p),
                ("exp_scenario", C.c_void_p), ("exp_ts", C.c_void_p), ("exp_feat_off", C.c_void_p),
                ("exp_blk", C.c_void_p), ("exp_feats", C.c_void_p)]


class Records(C.Structure):
    _fields_ = [("capacity", C.c_int64), ("n_records", C.c_int64), ("user_id", C.c_void_p),
                ("scenario_id", C.c_void_p), ("exposure_index", C.c_void_p), ("task_index", C.c_void_p),
                ("logit", C.c_void_p), ("probability", C.c_void_p)]


class RunStats(C.Structure):
    _fields_ = [("kernel_launches", C.c_int64), ("algorithmic_flops", C.c_double), ("attention_flops", C.c_double),
                ("tokens", C.c_int64), ("targets", C.c_int64), ("records", C.c_int64)]


class ExposureStream(C.Structure):
    _fields_ = [("n_exposures", C.c_int32), ("n_feats", C.c_int64), ("user_id", C.c_void_p), ("scenario", C.c_void_p),
                ("ts", C.c_void_p), ("feat_off", C.c_void_p), ("blk", C.c_void_p), ("feats", C.c_void_p)]


class AggregationReport(C.Structure):
    _fields_ = [("n_exposure_records", C.c_int64), ("n_user_samples", C.c_int64), ("compression_ratio", C.c_double)]


class PackedSizes(C.Structure):
    _fields_ = [("n_users", C.c_int64), ("n_seqs", C.c_int64), ("n_events", C.c_int64), ("n_exposures", C.c_int64),
                ("n_ev_feats", C.c_int64), ("n_exp_feats", C.c_int64)]


class PackedBuffers(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("user_id", "seq_off", "seq_kind", "seq_schema", "ev_off", "ev_ts",
                                           "ev_feat_off", "ev_feats", "exp_off", "exp_scenario", "exp_ts",
                                           "exp_feat_off", "exp_blk", "exp_feats", "exp_src")]


class TrainConfig(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("clip_norm", C.c_double), ("global_batch", C.c_int64)]


class TrainResult(C.Structure):
    _fields_ = [("loss", C.c_double), ("grad_norm", C.c_double), ("step", C.c_int64), ("records", C.c_int64)]


class PruneReport(C.Structure):
    _fields_ = [("groups_covered", C.c_int64), ("zeros_written", C.c_int64), ("exempt_tail_rows", C.c_int64),
                ("pruned_params", C.c_int64)]


class DatasetInfo(C.Structure):
    _fields_ = [("format_version", C.c_int32), ("n_users", C.c_int64), ("n_chunks", C.c_int64),
                ("max_tasks", C.c_int32)]


# (name, restype, argtypes) — every symbol include/mtfm_cuda.h declares.
SIGNATURES = [
    ("mtfm_cuda_last_error", C.c_char_p, []),
    ("mtfm_cuda_version", C.c_char_p, []),
    ("mtfm_cuda_create", C.c_int, [C.c_int, C.POINTER(ModelDesc), C.POINTER(SchemaDesc), C.c_int32,
                                   C.POINTER(C.c_void_p)]),
    ("mtfm_cuda_destroy", C.c_int, [C.c_void_p]),
    ("mtfm_cuda_set_param", C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int64, C.c_int64]),
    ("mtfm_cuda_num_params", C.c_int64, [C.c_void_p]),
    ("mtfm_cuda_param_name", C.c_char_p, [C.c_void_p, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("mtfm_cuda_restrict_to_scenario", C.c_int, [C.c_void_p, C.c_int32]),
    ("mtfm_cuda_count_records", C.c_int64, [C.c_void_p, C.POINTER(PackedBatch)]),
    ("mtfm_cuda_forward", C.c_int, [C.c_void_p, C.POINTER(PackedBatch), C.c_int32, C.POINTER(Records)]),
    ("mtfm_cuda_batch_prepare", C.c_int, [C.c_void_p, C.POINTER(PackedBatch), C.c_int32, C.POINTER(C.c_void_p)]),
    ("mtfm_cuda_batch_update", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(PackedBatch), C.c_int32]),
    ("mtfm_cuda_batch_run", C.c_int, [C.c_void_p, C.c_void_p]),
    ("mtfm_cuda_batch_results", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(Records)]),
    ("mtfm_cuda_batch_free", C.c_int, [C.c_void_p]),
    ("mtfm_cuda_stream", C.c_void_p, [C.c_void_p]),
    ("mtfm_cuda_last_stats", C.c_int, [C.c_void_p, C.POINTER(RunStats)]),
    ("mtfm_cuda_set_profiling", C.c_int, [C.c_void_p, C.c_int32]),
    ("mtfm_cuda_profile_count", C.c_int64, [C.c_void_p]),
    ("mtfm_cuda_profile_entry", C.c_char_p, [C.c_void_p, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                             C.POINTER(C.c_double)]),
    ("mtfm_cuda_debug_gemm", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                       C.c_int64, C.c_int32, C.c_void_p]),
    ("mtfm_cuda_debug_fetch", C.c_int64, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_void_p, C.c_int64]),
    ("mtfm_cuda_aggregate_users", C.c_int, [C.c_int, C.c_void_p, C.c_int32, C.POINTER(ExposureStream),
                                            C.POINTER(PackedBatch), C.POINTER(C.c_void_p),
                                            C.POINTER(AggregationReport)]),
    ("mtfm_cuda_aggregate_sizes", C.c_int, [C.c_void_p, C.POINTER(PackedSizes)]),
    ("mtfm_cuda_aggregate_fetch", C.c_int, [C.c_void_p, C.POINTER(PackedBuffers)]),
    ("mtfm_cuda_aggregate_free", C.c_int, [C.c_void_p]),
    ("mtfm_cuda_prune_projections", C.c_int, [C.c_void_p, C.POINTER(PruneReport)]),
    ("mtfm_cuda_set_sparse_mma", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int32)]),
    ("mtfm_cuda_train_step", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(TrainConfig),
                                       C.POINTER(TrainResult)]),
    ("mtfm_cuda_get_param", C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int64, C.c_int64]),
    ("mtfm_cuda_get_grad", C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int64, C.c_int64]),
    ("mtfm_nccl_unique_id", C.c_int, [C.c_void_p]),
    ("mtfm_cuda_dp_init", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    ("mtfm_dataset_load", C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    ("mtfm_dataset_info", C.c_int, [C.c_void_p, C.POINTER(DatasetInfo)]),
    ("mtfm_dataset_schema_desc", C.c_int, [C.c_void_p, C.POINTER(SchemaDesc)]),
    ("mtfm_dataset_chunk", C.c_int, [C.c_void_p, C.c_int64, C.POINTER(PackedBatch), C.POINTER(C.POINTER(C.c_int32))]),
    ("mtfm_dataset_free", None, [C.c_void_p]),
]

_lib = None


def lib():
    """Loads libmtfm_cuda.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run python -m paper_2602_11235_b200.build")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status):
    if status != OK:
        msg = lib().mtfm_cuda_last_error().decode(errors="replace")
        raise _BY_STATUS.get(status, MtfmError)(msg)


def ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None and a.size else None
