"""Drop-in check on the GPU: oracle/_ref/ref_integration links the unmodified
reference (model, generator, forward_sample, infer_request) and
include/mtfm_cuda.hpp over libmtfm_cuda.so in one process and compares them
record by record."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "ref_integration")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("flag", ["", "--fp32"])
def test_reference_api_drop_in(flag):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/ref_integration not built (needs /root/reference at build time)")
    out = subprocess.run([BIN] + ([flag] if flag else []), capture_output=True, text=True, timeout=600)
    line = [l for l in out.stdout.splitlines() if l.startswith("{")][-1]
    r = json.loads(line)
    print(line)
    assert out.returncode == 0 and r["ok"], r
    assert r["records"] > 0
