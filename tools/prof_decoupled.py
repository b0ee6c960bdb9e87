"""Time the decoupled baseline (mode "decoupled", csrc/decoupled.cu) beside EFTA-optimized on one
shape (kernel-side, CUDA events on the launching stream).
python tools/prof_decoupled.py --b 16 --h 16 --s 2048 --d 64"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_02211_b200 import EftaAttention, Thresholds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, default=16)
ap.add_argument("--h", type=int, default=16)
ap.add_argument("--s", type=int, default=2048)
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--only", default="")
a = ap.parse_args()
shape = (a.b, a.h, a.s, a.d)
q = torch.empty(shape, device="cuda").uniform_(-1, 1).half()
k = torch.empty(shape, device="cuda").uniform_(-1, 1).half()
v = torch.empty(shape, device="cuda").uniform_(-1, 1).half()
fl = 4 * a.b * a.h * a.s * a.s * a.d
res = {}
for mode, thr in (("efta-opt", Thresholds(1e-4, 1e-3, 1e-3)), ("decoupled", Thresholds(7e-6, 1e-3, 5e-3))):
    if a.only and mode != a.only:
        res[mode] = float("nan")
        continue
    op = EftaAttention(*shape, mode=mode, thr=thr)
    import time
    t0 = time.time()
    while time.time() - t0 < 1.0:  # warm-up: clocks ramp, lazy module loading
        op(q, k, v)
        torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.iters + 1)]
    ev[0].record()
    for it in range(a.iters):
        out = op(q, k, v)
        ev[it + 1].record()
    torch.cuda.synchronize()
    per = [ev[it].elapsed_time(ev[it + 1]) for it in range(a.iters)]
    ms = sorted(per)[len(per) // 2]  # median: a host hiccup between launches shows as GPU idle time
    print(f"  per-iteration ms: {[round(x, 3) for x in per]}")
    res[mode] = ms
    r = op.report()
    print(f"{mode:10s} {shape}: {ms:9.3f} ms  {fl / ms / 1e9:8.1f} TFLOP/s  det={r.detections} failed={r.failed}"
          f"  ws={op.workspace.numel() / 2**30:.2f} GiB")
    del op, out
    torch.cuda.empty_cache()
print(f"EFTA-optimized speed-up over decoupled: {res['decoupled'] / res['efta-opt']:.2f}x")
