"""Dataset ingestion: the reference's line-delimited dataset
format parsed natively into packed jagged batches, bit-exact with what the
reference's own load_dataset (dataset_io.cpp:110-221) reads, with its error
taxonomy and line numbers (tests/golden/io/, tests/golden/io_expect.npz made
by oracle/ref_io.cpp). CPU: host-only parsing. GPU: scoring the chunks."""
import os

import numpy as np
import pytest

from golden_util import GOLDEN
from paper_2602_11235_b200 import abi
from paper_2602_11235_b200.ingest import load_dataset
from paper_2602_11235_b200.schema import BATCH_KEYS

IO = os.path.join(GOLDEN, "io")
EXPECT = {k.replace("__", "/"): v for k, v in np.load(os.path.join(GOLDEN, "io_expect.npz")).items()}
FILES = sorted(os.listdir(IO))
ERRORS = {"parse_error": abi.ParseError, "config_error": abi.ConfigError, "integrity_error": abi.IntegrityError,
          "lookup_error": abi.LookupError_}


def _concat(ds):
    parts = [ds.chunk(i) for i in range(ds.n_chunks)]
    out = {}
    for k in BATCH_KEYS:
        arrs = [p[0][k] for p in parts]
        if k in ("seq_off", "ev_off", "ev_feat_off", "exp_off", "exp_feat_off"):
            # chunk-local offsets -> global
            glob, base = [np.zeros(1, np.int64)], 0
            for a in arrs:
                glob.append(a[1:].astype(np.int64) + base)
                base += int(a[-1])
            out[k] = np.concatenate(glob)
        else:
            out[k] = np.concatenate(arrs) if arrs else np.zeros(0)
    labels = np.concatenate([p[1] for p in parts]) if parts else np.zeros((0, ds.max_tasks))
    return out, labels


@pytest.mark.parametrize("fn", FILES)
@pytest.mark.parametrize("chunk_users", [1, 3, 1024])
def test_ingest_matches_reference_load_dataset(fn, chunk_users):
    kind = bytes(EXPECT[fn + "/kind"]).decode()
    what = bytes(EXPECT[fn + "/what"]).decode()
    path = os.path.join(IO, fn)
    if kind != "ok":
        with pytest.raises(ERRORS[kind]) as ei:
            load_dataset(path, threads=4, chunk_users=chunk_users)
        got = str(ei.value)
        if "malformed" in what:  # nlohmann's own exception text after the prefix is not restated
            assert got.split(":")[:2] == what.split(":")[:2], (got, what)
        else:
            assert got == what
        return
    ds = load_dataset(path, threads=4, chunk_users=chunk_users)
    got, labels = _concat(ds)
    for k in BATCH_KEYS:
        assert np.array_equal(got[k].astype(np.int64), EXPECT[fn + "/" + k].astype(np.int64)), k
    mt = int(EXPECT[fn + "/max_tasks"][0])
    assert np.array_equal(labels.reshape(-1), EXPECT[fn + "/labels"]) and ds.max_tasks == mt
    assert ds.n_users == len(EXPECT[fn + "/user_id"])


@pytest.mark.gpu
def test_score_ingested_dataset_pipelined():
    """Chunks of the ingested file scored through the two-batch pipeline equal one
    forward over the whole dataset, and carry the file's labels."""
    from paper_2602_11235_b200 import Model, datagen
    from paper_2602_11235_b200.ingest import score_dataset
    from paper_2602_11235_b200.schema import ModelConfig, HTAConfig
    ds = load_dataset(os.path.join(IO, "dataset.jsonl"), chunk_users=7)
    cfg = ModelConfig(HTAConfig(d_model=64, blocks=1, target_layers=1, full_layers=1, heads=4, kv_heads=2))
    m = Model(ds.schemas, cfg)
    m.set_params(datagen.random_params(m.param_specs(), seed=1))
    parts = score_dataset(m, ds)
    whole, labels = _concat(ds)
    ref = m.forward_batch(whole)
    z = np.concatenate([p[0].logit for p in parts])
    assert np.array_equal(z, ref.logit)
    lab = np.concatenate([p[1] for p in parts])
    assert set(np.unique(lab)) <= {0, 1} and len(lab) == len(ref)
