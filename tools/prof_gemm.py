"""Time the strided-ABFT GEMM (and torch.matmul as a cuBLAS reference point).
python tools/prof_gemm.py --m 32768 --n 4096 --k 1024"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_02211_b200.ffn import AbftLinear  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=32768)
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--k", type=int, default=1024)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
x = torch.empty(a.m, a.k, device="cuda").uniform_(-1, 1).half()
w = (torch.empty(a.n, a.k, device="cuda").uniform_(-1, 1) / a.k ** 0.5).half()
lin = AbftLinear(w, eps=5e-2)
y = lin(x)
torch.cuda.synchronize()


def bench(fn):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.iters


ms = bench(lambda: lin(x, y))
ms_ref = bench(lambda: torch.matmul(x, w.t()))
fl = 2.0 * a.m * a.n * a.k
rep = lin.report()
err = (y.float() - torch.matmul(x, w.t()).float()).abs().max().item()
print(f"abft_gemm {a.m}x{a.n}x{a.k}: {ms:.3f} ms {fl/ms/1e9:.1f} TFLOP/s | cuBLAS fp16 {ms_ref:.3f} ms "
      f"{fl/ms_ref/1e9:.1f} TFLOP/s | det={rep.detections} max|y-ref|={err:.3e} clean_res={rep.family_max[1]:.2e}")
