"""Which check fires on the bench suite's causal inputs (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2504_02211_b200 import EftaAttention, Thresholds
dev = torch.device("cuda")
b, h, s_, d = 4, 32, 8192, 128
q = bench.synth_inputs(41, (b, h, s_, d), dev)
k = bench.synth_inputs(42, (b, h, s_, d), dev)
v = bench.synth_inputs(43, (b, h, s_, d), dev)
for thr in (Thresholds(1e-4, 1e-3, 1e-3), Thresholds(1e-4, 1e-2, 1e-3)):
    op = EftaAttention(b, h, s_, d, mode="efta-opt", thr=thr, device=dev, causal=True)
    o, m, l = op(q, k, v)
    rep = op.report()
    print(thr, rep.detections, rep.failed, rep.family_max)
    for e in rep.events[:10]:
        print("  ", e)
op = EftaAttention(b, h, s_, d, mode="efta-opt", thr=Thresholds(1e-4, 1e-3, 1e-3), device=dev, causal=False)
op(q, k, v)
rep = op.report()
print("non-causal", rep.detections, rep.family_max)
for e in rep.events[:5]:
    print("  ", e)
