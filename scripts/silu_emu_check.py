"""Float32 restatement of ptx::silu2_bf16_fma (csrc/ptx.cuh): the SFU-free SiLU
used for part of the attention scores. Prints its max relative error against
the exact s*sigmoid(s) over s in [-200, 200]; expected <= 8e-5."""
import numpy as np
f32 = np.float32
C = [f32(0.9999280571937561), f32(0.6932609677314758), f32(0.2426111400127411), f32(0.0551716648042202)]
M = f32(12582912.0)
def emu(s):
    s = s.astype(f32)
    t = (s * f32(-1.4426950408889634)).astype(f32)
    t = np.minimum(np.maximum(t, f32(-126)), f32(126))
    j = (t + M).astype(f32)
    n = (j - M).astype(f32)
    fr = (t - n).astype(f32)
    p = (fr * C[3] + C[2]).astype(f32)
    p = (p * fr + C[1]).astype(f32)
    p = (p * fr + C[0]).astype(f32)
    eb = (p.view(np.uint32) + (j.view(np.uint32) << np.uint32(23))).astype(np.uint32)
    e = eb.view(f32)
    nden = (e * f32(-1) + f32(-1)).astype(f32)
    r = (np.uint32(0xFEF311C3) - nden.view(np.uint32)).astype(np.uint32).view(f32)
    for _ in range(2):
        err = (nden * r + f32(1)).astype(f32)
        r = (r * err + r).astype(f32)
    return (s * r).astype(f32)
s = np.concatenate([np.linspace(-200, 200, 2000001), np.array([0.0, -0.0, 1e-30, -1e-30])]).astype(f32)
y = emu(s).astype(np.float64)
yt = s.astype(np.float64) / (1 + np.exp(-s.astype(np.float64)))
ae = np.abs(y - yt)
re = ae / np.maximum(np.abs(yt), 1e-30)
print("max abs err", ae.max(), "at", s[ae.argmax()])
m = np.abs(yt) > 1e-6
print("max rel err (|y|>1e-6)", re[m].max(), "at", s[m][re[m].argmax()])
# compare with tanh-based hardware-like formula in f32
h = (s * f32(0.5)).astype(f32)
y2 = (h + h * np.tanh(h.astype(np.float64)).astype(f32)).astype(np.float64)
print("tanh form (exact tanh) max rel err", (np.abs(y2 - yt) / np.maximum(np.abs(yt), 1e-30))[m].max())
