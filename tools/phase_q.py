"""Per-warp-quarter phase stamps of CTA (2,5) (EFTA_PROF build, alternating schedule):
EFTA_LIB=paper_2504_02211_b200/libefta_b200_prof.so python tools/phase_q.py --mode efta-opt"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_02211_b200 import EftaAttention, Thresholds, _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="efta-opt")
ap.add_argument("--d", type=int, default=128)
a = ap.parse_args()
shape = (8, 16, 8192, a.d)
q, k, v = (torch.empty(shape, device="cuda").uniform_(-1, 1).half() for _ in range(3))
op = EftaAttention(*shape, mode=a.mode, thr=Thresholds(1e-4, 1e-3, 1e-3))
op(q, k, v); op(q, k, v); torch.cuda.synchronize()
_lib.lib.efta_prof_buffer.restype = C.c_void_p
ptr = _lib.lib.efta_prof_buffer()
buf = np.zeros(64 * 32, np.uint64)
cudart = C.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else C.CDLL("libcudart.so")
cudart.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
cudart.cudaMemcpy(buf.ctypes.data, ptr, buf.nbytes, 2)
t = buf.reshape(64, 32).astype(np.int64)
base = t[8, 16 + 8]
print("block  S_ready[q0..3]              pre_exp[q0..3]              pre_bar[q0..3]              p_ready[q0..3]")
for j in range(8, 20):
    row = []
    for b in (8, 4, 0, 12):
        row.append(" ".join(f"{t[j, 16 + b + q] - base:6d}" for q in range(4)))
    print(f"{j:4d}   " + "   ".join(row))
for nm, b0, b1 in [("S_ready->pre_exp", 8, 4), ("pre_exp->pre_bar", 4, 0), ("pre_bar->p_ready", 0, 12)]:
    d = np.array([[t[j, 16 + b1 + q] - t[j, 16 + b0 + q] for q in range(4)] for j in range(8, 60)])
    print(f"{nm:18s} median per quarter", np.median(d, axis=0))
sk = np.array([t[j, 16:20].max() - t[j, 16:20].min() for j in range(8, 60)])
print("pre_bar skew (max-min over quarters) median", np.median(sk), "max", sk.max())
