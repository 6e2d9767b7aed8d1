"""One bf16 forward (and one fp32 check-mode forward) of a golden fixture, for
compute-sanitizer (racecheck / synccheck / memcheck) runs: python
scripts/sanitize_run.py <fixture> [bf16|fp32]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402
from golden_util import batch, model, ref_records  # noqa: E402
from helpers import from_oracle  # noqa: E402
from paper_2602_11235_b200 import Model  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tiny_j"
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
osch, ocfg, P = model(name)
sch, cfg = from_oracle(osch, ocfg)
m = Model.build(sch, cfg, P, precision=prec, device=0)
ra = m.forward_batch(batch(name))
_, z64, *_ = ref_records(name)
print(f"{name} {prec}: {len(ra)} records, max |dz| {np.max(np.abs(ra.logit - z64)):.3e}")
