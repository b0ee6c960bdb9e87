"""Decode step timing (csrc/decode.cu): B x H query rows against K/V caches of S keys, cache
checksums encoded once (steady-state decode). HBM bytes per step: K + V (+ KC, VC protected)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_02211_b200 import EftaDecode, Thresholds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, default=32)
ap.add_argument("--h", type=int, default=32)
ap.add_argument("--hkv", type=int, default=0)
ap.add_argument("--s", type=int, default=8192)
ap.add_argument("--d", type=int, default=128)
a = ap.parse_args()
hkv = a.hkv or a.h
q = torch.empty(a.b, a.h, a.d, device="cuda").uniform_(-1, 1).half()
k = torch.empty(a.b, hkv, a.s, a.d, device="cuda").uniform_(-1, 1).half()
v = torch.empty(a.b, hkv, a.s, a.d, device="cuda").uniform_(-1, 1).half()
for mode in ("efta-opt", "none"):
    op = EftaDecode(a.b, a.h, a.s, a.d, mode=mode, thr=Thresholds(1e-4, 1e-3, 1e-3), kv_heads=hkv)
    op.encode(k, v)
    for _ in range(3):
        op(q, k, v, cache_encoded=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        op(q, k, v, cache_encoded=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    kv_bytes = 2 * a.b * hkv * a.s * a.d * 2
    cs_bytes = (a.b * hkv * (a.s // 128) * 32 * a.d * 2 + a.b * hkv * a.s * 64 * 2) if mode == "efta-opt" else 0
    print(f"decode {mode:8s} B={a.b} H={a.h} Hkv={hkv} S={a.s} d={a.d}: {ms:.3f} ms  "
          f"{(kv_bytes + cs_bytes) / ms / 1e6:.0f} GB/s (K+V{'+KC+VC' if cs_bytes else ''})  "
          f"{kv_bytes / ms / 1e6:.0f} GB/s of K+V  det={op.report().detections}")
