"""Times gemm_tc_kernel (through mtfm_cuda_debug_gemm) against torch/cuBLAS on
the MTFM-small GEMM shapes under the MTFM_GEMM_* overrides set by the caller."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_11235_b200 import abi

L = abi.lib()
shapes = [("proj_full", 557056, 256, 640, 0), ("tok_mlp2", 557056, 512, 256, 1), ("fkv", 557056, 256, 128, 0),
          ("f2_resid", 557056, 256, 256, 2), ("tok_mlp1", 557056, 64, 512, 0),
          # MTFM-large shapes (M reduced to 2^20 rows)
          ("f2_L", 1048576, 1024, 1024, 2), ("tok2_L", 1048576, 2048, 1024, 1), ("projU_L", 1048576, 1024, 1024, 0),
          ("kv_L", 1048576, 1024, 512, 0)]
only = os.environ.get("SHAPE")
if only:
    shapes = [x for x in shapes if x[0] == only]
st = torch.cuda.current_stream()
tag = os.environ.get("TAG", "")
for name, M, K, N, epi in shapes:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    bt = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) / 16
    bias = torch.randn(N, device="cuda", dtype=torch.float32)
    out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if epi in (0, 3) else torch.float32)
    def run():
        abi.check(L.mtfm_cuda_debug_gemm(a.data_ptr(), bt.data_ptr(), bias.data_ptr(), out.data_ptr(), M, N, K, epi,
                                         C.c_void_p(st.cuda_stream)))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    # replay a captured graph of 10 launches: no host gaps inside the timed region
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        st = cs
        with torch.cuda.graph(g, stream=cs):
            for _ in range(10):
                run()
    st = torch.cuda.current_stream()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    ob = out.element_size()
    byts = M * K * 2 + N * K * 2 + M * N * ob * (2 if epi == 2 else 1)
    # correctness spot check
    ref = (a[:256].float() @ bt.float().t()) + bias
    if epi == 0:
        ref = torch.nn.functional.silu(ref)
    got = out[:256].float()
    err = "" if epi == 2 else " maxerr %.3g" % (got - ref).abs().max().item()
    tf = 2.0 * M * N * K / (ms / 1e3) / 1e12
    print(f"{tag:24s} {name:10s} {ms*1000:8.1f} us {byts/ms/1e6:7.0f} GB/s {tf:6.0f} TFLOP/s{err}", flush=True)
