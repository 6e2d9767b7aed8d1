"""cuBLAS (torch.matmul) timings of the MTFM-small GEMM shapes, for comparison
with gemm_tc_kernel (bf16 in/out, fp32 accumulate)."""
import torch
torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
shapes = {"proj_full (557056x256 @ 256x640)": (557056, 256, 640),
          "tok_mlp2 (557056x512 @ 512x256)": (557056, 512, 256),
          "fkv (557056x256 @ 256x128)": (557056, 256, 128),
          "f2 (557056x256 @ 256x256)": (557056, 256, 256),
          "tok_mlp1 (557056x64 @ 64x512)": (557056, 64, 512)}
for name, (M, K, N) in shapes.items():
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        c = a @ b
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    byts = (M * K + K * N + M * N) * 2
    print(f"{name:36s} {ms*1000:8.1f} us  {byts/ms/1e6:7.0f} GB/s  {2*M*K*N/ms/1e9:7.1f} TFLOP/s")
