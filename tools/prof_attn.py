"""Profiling driver: run the fused forward a few times on synthetic inputs.

python tools/prof_attn.py --mode efta-opt --b 2 --h 16 --s 8192 --d 128 --iters 3
(wrap in `ncu ... -k regex:efta_attn_fwd`)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_02211_b200 import EftaAttention, Thresholds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="efta-opt")
ap.add_argument("--b", type=int, default=2)
ap.add_argument("--h", type=int, default=16)
ap.add_argument("--s", type=int, default=8192)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--time", action="store_true")
ap.add_argument("--tok", action="store_true", help="fp16 token-major O output")
ap.add_argument("--causal", action="store_true")
a = ap.parse_args()
shape = (a.b, a.h, a.s, a.d)
q = torch.empty(shape, device="cuda").uniform_(-1, 1).half()
k = torch.empty(shape, device="cuda").uniform_(-1, 1).half()
v = torch.empty(shape, device="cuda").uniform_(-1, 1).half()
op = EftaAttention(*shape, mode=a.mode, thr=Thresholds(1e-4, 1e-3, 1e-3), token_major_out=a.tok, causal=a.causal)
for _ in range(a.iters):
    op(q, k, v)
torch.cuda.synchronize()
if a.time:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    op.desc.checksums_ready = 1
    e0.record()
    for _ in range(10):
        op(q, k, v)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    fl = (2 if a.causal else 4) * a.b * a.h * a.s * a.s * a.d
    print(f"{a.mode}{' tok' if a.tok else ''}{' causal' if a.causal else ''} {shape}: {ms:.3f} ms  {fl/ms/1e9:.1f} TFLOP/s  det={op.report().detections}")
