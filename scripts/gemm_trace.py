"""One traced gemm_tc launch per shape (MTFM_GEMM_TRACE=1 prints CTA-0 clock stamps)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_11235_b200 import abi

L = abi.lib()
shapes = {"proj_full": (557056, 256, 640, 0), "tok_mlp2": (557056, 512, 256, 1), "fkv": (557056, 256, 128, 0),
          "f2_resid": (557056, 256, 256, 2), "tok_mlp1": (557056, 64, 512, 0)}
for name in os.environ.get("SHAPES", "fkv").split():
    M, K, N, epi = shapes[name]
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    bt = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) / 16
    bias = torch.randn(N, device="cuda", dtype=torch.float32)
    out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if epi in (0, 3) else torch.float32)
    st = torch.cuda.current_stream()
    for i in range(3):
        print(name, "run", i, file=sys.stderr, flush=True)
        abi.check(L.mtfm_cuda_debug_gemm(a.data_ptr(), bt.data_ptr(), bias.data_ptr(), out.data_ptr(), M, N, K, epi,
                                         C.c_void_p(st.cuda_stream)))
    torch.cuda.synchronize()
