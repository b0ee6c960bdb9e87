"""End-to-end (host buffers) path at C4: PCIe bandwidth of the copies alone vs the chunked
efta_attn_fwd_host_f16 call for several chunk counts (EFTA_HOST_CHUNKS).

python tools/prof_e2e.py"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_02211_b200 import Thresholds, _lib  # noqa: E402

B, H, S, D = 32, 32, 8192, 128
shape = (B, H, S, D)
thr = Thresholds(1e-4, 1e-3, 1e-3)
hq, hk, hv = (torch.empty(shape, dtype=torch.float16).uniform_(-1, 1).pin_memory() for _ in range(3))
ho = torch.empty(shape, dtype=torch.float32).pin_memory()
hm = torch.empty(shape[:3], dtype=torch.float32).pin_memory()
hl = torch.empty(shape[:3], dtype=torch.float32).pin_memory()
dq = torch.empty(shape, dtype=torch.float16, device="cuda")
do = torch.empty(shape, dtype=torch.float32, device="cuda")


def wall(fn, n=2):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n


t = wall(lambda: dq.copy_(hq, non_blocking=True))
print(f"H2D {hq.numel() * 2 / t / 1e9:.1f} GB/s", flush=True)
t = wall(lambda: ho.copy_(do, non_blocking=True))
print(f"D2H {ho.numel() * 4 / t / 1e9:.1f} GB/s", flush=True)
s2 = torch.cuda.Stream()


def both():
    dq.copy_(hq, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)
    s2.synchronize()


t = wall(both)
print(f"H2D+D2H concurrent: {hq.numel() * 2 / 1e9:.2f} GB + {ho.numel() * 4 / 1e9:.2f} GB in {t * 1e3:.1f} ms", flush=True)
del dq, do
torch.cuda.empty_cache()
desc = _lib.AttnDesc(B, H, S, D, 128, 8, 0.0, 2, thr.eps1, thr.eps2, thr.eps_lin, 0, 0.0, 0, 0)
cnt = _lib.Counters()
fl = 4.0 * B * H * S * S * D
for ch in (16, 32, 48, 64):
    os.environ["EFTA_HOST_CHUNKS"] = str(ch)

    def step():
        _lib.check(_lib.lib.efta_attn_fwd_host_f16(
            C.byref(desc), hq.data_ptr(), hk.data_ptr(), hv.data_ptr(), ho.data_ptr(),
            hm.data_ptr(), hl.data_ptr(), None, 0, None, 0, None, 0, C.byref(cnt)))
    t = wall(step, 3)
    print(f"e2e chunks={ch}: {t * 1e3:.1f} ms  {fl / t / 1e12:.1f} TFLOP/s  det={cnt.detections}", flush=True)
