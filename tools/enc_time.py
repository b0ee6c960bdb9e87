import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2504_02211_b200 import EftaAttention, Thresholds
for d in (128, 64):
    shape = (32, 32, 8192, 128) if d == 128 else (16, 16, 2048, 64)
    q, k, v = (torch.empty(shape, device="cuda").uniform_(-1, 1).half() for _ in range(3))
    for mode in ("efta-opt", "none"):
        op = EftaAttention(*shape, mode=mode, thr=Thresholds(1e-4, 1e-3, 1e-3))
        op(q, k, v); torch.cuda.synchronize()
        def t(ready, it=5):
            op.desc.checksums_ready = ready
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(it): op(q, k, v)
            e1.record(); torch.cuda.synchronize()
            return e0.elapsed_time(e1) / it
        full, kern = t(0), t(1)
        print(d, mode, "step %.3f ms  kernel %.3f ms  prepass %.3f ms" % (full, kern, full - kern))
