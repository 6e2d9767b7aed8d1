"""The measurement the bench reports: per-stage algorithmic FLOPs add up to the
run's SURVEY 8(d) FLOP model (projections per complexity.hpp:54-64,
mask-aware attention, tokenizer MLPs, heads), so step_tflops is not inflated."""
import numpy as np
import pytest

from paper_2602_11235_b200 import Model, datagen

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("wl_name,users", [("small", 64), ("base", 64), ("paper", 4)])
def test_stage_flops_sum_to_algorithmic(wl_name, users):
    wl = datagen.WORKLOADS[wl_name]()
    b = datagen.generate(wl, n_users=users)
    m = Model(wl.schemas, wl.cfg, precision="bf16")
    m.set_params(datagen.random_params(m.param_specs(), seed=7))
    pb = m.prepare(b)
    m.set_profiling(True)
    for _ in range(2):  # the stage annotations use the visible-key sums of the previous results()
        pb.run()
        pb.results()
    prof = m.profile()
    m.set_profiling(False)
    total = sum(fl for _, _, fl, _ in prof)
    alg = m.last_stats().algorithmic_flops
    print(f"{wl_name}: stage sum {total:.6e} vs algorithmic {alg:.6e}")
    assert abs(total - alg) <= 1e-9 * alg
