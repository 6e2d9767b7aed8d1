"""B200-native (sm_100a) MTFM hot path: jagged user batches -> heterogeneous
tokenizer -> GQA Hybrid Target Attention stack -> MMoE heads, behind the C ABI
of include/mtfm_cuda.h (libmtfm_cuda.so). The shared library is loaded on
first use (abi.lib()) and there is no CPU fallback."""
from . import abi  # noqa: F401
from .aggregate import aggregate_users, pack_store, pack_stream  # noqa: F401
from .model import Model, PreparedBatch, RecordArrays, infer_request, infer_requests  # noqa: F401
from .schema import (BehaviorEvent, Candidate, Exposure, HTAConfig, InferenceRequest, ModelConfig,  # noqa: F401
                     PredictionRecord, ScenarioSchema, SchemaSet, SequenceRecord, SequenceSchema, UserSample,
                     pack_samples, sample_view_of_request)
