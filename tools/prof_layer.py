"""FT-Transformer layer A/B: fused layouts (head-split QKV GEMM epilogue + token-major fp16
attention output) vs the torch head split / merge copies, protected and unprotected, at the
bench's C5 sweep (16K tokens, GPT-2-large shapes). Median of per-iteration CUDA-event times.

python tools/prof_layer.py [--iters 5]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_02211_b200 import FTTransformerLayer, Thresholds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
thr = Thresholds(1e-4, 1e-3, 1e-3)
layers = {(p, f): FTTransformerLayer(1280, 20, 5120, protect=p, thr=thr, seed=1, fused_layout=f != "copies",
                                     fused_gelu=f == "fused")
          for p in (True, False) for f in ("fused", "fused-nogelu", "copies")}


def med_ms(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


g = torch.Generator(device="cuda")
g.manual_seed(3)
for seq in (512, 2048, 8192, 16384):
    b = 16384 // seq
    x = torch.empty((b, seq, 1280), device="cuda").uniform_(-1, 1, generator=g).half()
    fl = layers[(True, "fused")].flops(b, seq)
    row = []
    for (p, f), lay in layers.items():
        ms = med_ms(lambda: lay(x))
        row.append(f"{'prot' if p else 'unprot'}/{f} {ms:.3f} ms {fl / ms / 1e9:.1f} TF/s")
    print(f"S={seq} B={b}: " + " | ".join(row), flush=True)
