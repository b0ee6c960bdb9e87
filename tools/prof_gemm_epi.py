"""The FT-Transformer layer's four protected GEMMs (16K tokens, GPT-2-large shapes) with and
without their fused epilogues (head split, residual, GELU) vs the plain store + torch pass, and
cuBLAS. Median of per-iteration CUDA-event times, TFLOP/s of the GEMM.

python tools/prof_gemm_epi.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_02211_b200.ffn import AbftLinear  # noqa: E402


def med_ms(fn, iters=15):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


g = torch.Generator(device="cuda")
g.manual_seed(1)
t, d, dff = 16384, 1280, 5120
for name, n, k in (("qkv", 3 * d, d), ("o", d, d), ("ff1", dff, d), ("ff2", d, dff)):
    x = torch.empty((t, k), device="cuda").uniform_(-1, 1, generator=g).half()
    w = (torch.empty((n, k), device="cuda").uniform_(-1, 1, generator=g) / k ** 0.5).half()
    r = torch.empty((t, n), device="cuda").uniform_(-1, 1, generator=g).half()
    lin = AbftLinear(w, eps=5e-2)
    y = lin(x)
    fl = 2.0 * t * n * k
    res = {"plain": med_ms(lambda: lin(x, y)), "cublas": med_ms(lambda: x @ w.t())}
    if name == "qkv":
        res["head_split"] = med_ms(lambda: lin(x, head_split=(512, 20, 64)))
        res["plain+permute"] = med_ms(lambda: lin(x, y).view(32, 512, 3, 20, 64).permute(2, 0, 3, 1, 4).contiguous())
    else:
        res["resid_epi"] = med_ms(lambda: lin(x, residual=r))
        res["plain+add"] = med_ms(lambda: r + lin(x, y))
        if name == "ff1":
            res["gelu_epi"] = med_ms(lambda: lin(x, activation="gelu"))
            res["plain+gelu"] = med_ms(lambda: torch.nn.functional.gelu(lin(x, y)))
    print(f"{name} {t}x{n}x{k}: " + " | ".join(f"{kk} {v * 1e3:.1f} us {fl / v / 1e9:.0f}" for kk, v in res.items()),
          flush=True)
