"""Per-phase timing of one CTA (EFTA_PROF build): EFTA_PROF=1 python -m paper_2504_02211_b200.build
then EFTA_LIB=paper_2504_02211_b200/libefta_b200_prof.so python tools/phase_prof.py --mode none"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_02211_b200 import EftaAttention, Thresholds, _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="none")
ap.add_argument("--d", type=int, default=128)
a = ap.parse_args()
shape = (8, 16, 8192, a.d)
q = torch.empty(shape, device="cuda").uniform_(-1, 1).half()
k = torch.empty(shape, device="cuda").uniform_(-1, 1).half()
v = torch.empty(shape, device="cuda").uniform_(-1, 1).half()
op = EftaAttention(*shape, mode=a.mode, thr=Thresholds(1e-4, 1e-3, 1e-3))
op(q, k, v); torch.cuda.synchronize()
op(q, k, v); torch.cuda.synchronize()
_lib.lib.efta_prof_buffer.restype = C.c_void_p
ptr = _lib.lib.efta_prof_buffer()
buf = np.zeros(64 * 32, np.uint64)
cudart = C.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else C.CDLL("libcudart.so")
cudart.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
cudart.cudaMemcpy(buf.ctypes.data, ptr, buf.nbytes, 2)
t = buf.reshape(64, 32).astype(np.int64)
names = {7: "mma:s_free", 8: "row:pre_late", 15: "row:pre_exp", 0: "row:wait_S", 1: "row:S_ready", 2: "row:exp_done", 3: "row:sum_done", 4: "row:P_stored",
         5: "row:O_ready", 6: "row:p_ready", 10: "mma:iter", 11: "mma:S_issued", 12: "mma:P_ready",
         14: "mma:V_ready", 13: "mma:PV_issued", 16: "peer:wait_S", 17: "peer:S_ready", 18: "peer:exp_done",
         22: "peer:p_ready"}
base = t[8, 0]
print("iter  " + "  ".join(f"{names[s]:>13s}" for s in sorted(names)))
for j in range(8, 16):
    print(f"{j:4d}  " + "  ".join(f"{t[j, s] - base:13d}" for s in sorted(names)))
print("(the clock64 counters of the two CTAs of a pair are per-SM; compare within one CTA)")
per = np.diff(t[8:60, 0])
print("row period median", np.median(per))
for s_a, s_b, nm in [(9, 11, "S-issuer: issue S(j)"), (10, 12, "PV-issuer: wait P(j)"),
                     (12, 14, "PV-issuer: wait V(j)"), (14, 13, "PV-issuer: issue PV(j)"), (13, 10, "PV-issuer: to next iter"), (1, 8, "split: ld+max+xchg+exp"), (8, 3, "split: checks+or+P st"), (8, 5, "split: prod xchg"), (5, 7, "split: check+red.or"), (7, 3, "split: P st"), (3, 6, "split: to p_ready")] + [(0, 1, "wait S"), (1, 7, "tmem load S"), (7, 8, "max+exp"), (8, 9, "product check"),
                     (9, 15, "barrier.red.or"), (15, 2, "after or"), (2, 3, "checks+sum"), (3, 4, "P pack+store"),
                     (4, 5, "wait O(PV j-1)"), (5, 6, "correction+arrive"), (6, 0, "to next iter")]:
    dt = [(t[j, s_b] if (s_b not in (0, 10) or s_a == 9) else t[j + 1, s_b]) - t[j, s_a] for j in range(8, 60)]
    print(f"  {nm:20s} median {np.median(dt):8.0f} clk")
