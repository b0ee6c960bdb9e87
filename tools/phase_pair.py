"""Per-block phase timeline of the persistent CTA-pair kernel (EFTA_PROF build): CTA 2 (leader of
cluster 1), global key blocks g = 0..63 of that CTA (row warpgroup g & 1).
  EFTA_PROF=1 python -m paper_2504_02211_b200.build
  EFTA_LIB=paper_2504_02211_b200/libefta_b200_prof.so python tools/phase_pair.py --mode efta-opt --d 128
Slots (csrc/efta_attn_alt.cuh, efta_attn_pair.cuh): row warp 4/8: 0 wait S, 1 S ready, 15 early max
published, 8 before late-chain wait, 9 after it (+ tile decision), 2 S freed, 3 sums, 4 before
P-buffer wait, 5 after, 6 P ready; score issuer: 7 S-free seen for g, 11 S(g) issued; P.V issuer:
10 iteration start, 12 P(g) ready seen, 14 V(g) landed, 13 P.V(g) issued."""
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
ap.add_argument("--s", type=int, default=8192)
ap.add_argument("--b", type=int, default=8)
ap.add_argument("--h", type=int, default=16)
a = ap.parse_args()
shape = (a.b, a.h, a.s, a.d)
q, k, v = (torch.empty(shape, device="cuda").uniform_(-1, 1).half() for _ in range(3))
op = EftaAttention(*shape, mode=a.mode, thr=Thresholds(1e-4, 1e-3, 1e-3))
for _ in range(3):
    op(q, k, v)
torch.cuda.synchronize()
_lib.lib.efta_prof_buffer.restype = C.c_void_p
ptr = _lib.lib.efta_prof_buffer()
buf = np.zeros(64 * 64, np.uint64)
cudart = C.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else C.CDLL("libcudart.so")
cudart.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
cudart.cudaMemcpy(buf.ctypes.data, ptr, buf.nbytes, 2)
t = buf.reshape(64, 64).astype(np.int64)
print(f"{a.mode} d={a.d} S={a.s}; times in clk relative to S ready (slot 1) of the same block")
cols = [(0, "waitS"), (15, "early"), (8, "preLate"), (9, "postLt"), (2, "Sfree"), (3, "sums"), (4, "preOd"),
        (5, "postOd"), (6, "Prdy"), (11, "S_iss(g)"), (12, "PVseesP"), (13, "PV_iss")]
print("  g  period  " + " ".join(f"{n:>8s}" for _, n in cols))
per = []
for g in range(4, 62):
    base = t[g, 1]
    if base == 0:
        continue
    prev = t[g - 2, 1]
    per.append(base - prev)
    print(f"{g:3d} {base - prev:7d}  " + " ".join(f"{t[g, s] - base:8d}" for s, _ in cols))
per = np.array(per)
print(f"median row period per warpgroup (2 blocks): {np.median(per):.0f} clk -> {np.median(per) / 2:.0f} clk/block")
med = lambda s_a, s_b: np.median([t[g, s_b] - t[g, s_a] for g in range(6, 60)])  # noqa: E731
for a_, b_, nm in [(0, 1, "wait for S"), (1, 15, "TMEM load + max + early publish"), (15, 8, "exp stage"),
                   (8, 9, "late-chain wait + check + decision"), (9, 2, "late publish + S free"),
                   (2, 3, "factors + sums"), (3, 4, "P pack"), (4, 5, "wait P buffer (P.V j-1/j-2)"),
                   (5, 6, "P store + O rescale + arrive"), (6, 12, "P ready -> P.V issuer sees it"),
                   (12, 13, "P.V issue (incl. V wait)")]:
    print(f"  {nm:40s} median {med(a_, b_):8.0f} clk")
print("issuer: S(g) issued relative to S ready(g):", np.median([t[g, 1] - t[g, 11] for g in range(6, 60)]), "clk later")

# epilogue of warpgroup 1 (slots 32..39 at the tile's last block g): relative to its P ready
print("epilogue (last block g of a tile; clk after that block's P ready):")
for g in range(64):
    if t[g, 32] == 0:
        continue
    r = t[g, 6]
    print(f"  g={g}: fin wait {t[g, 32] - r}..{t[g, 33] - r}  o_final {t[g, 34] - r}  O read+o_free {t[g, 35] - r}"
          f"  range {t[g, 36] - r}  norm {t[g, 40] - r}  verify {t[g, 37] - r}  store {t[g, 38] - r}  flush {t[g, 39] - r}"
          f"  | next own block S ready {t[g + 2, 1] - r if g + 2 < 64 else -1}")
    if t[g, 44]:
        print(f"        per-warp O read {[int(t[g, 52 + w] - r) for w in range(4)]}  range {[int(t[g, 56 + w] - r) for w in range(4)]}")
        print(f"        sums {t[g, 41] - r}  per-warp norm done {[int(t[g, 48 + w] - r) for w in range(4)]}"
              f"  per-warp at the check barrier {[int(t[g, 44 + w] - r) for w in range(4)]}")
