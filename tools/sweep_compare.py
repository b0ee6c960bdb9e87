"""Detector curves (paper Fig. 8/10, reference src/campaign.cpp:261-357) on the GPU (C++ drop-in,
tools/sweep_gpu) and in the reference (oracle/_ref, run here on the host): same configuration,
calibration and trial seeds; each side calibrates its own base thresholds, as the reference
prescribes per backend. Writes one JSON object.
python tools/sweep_compare.py --n 512 --d 64 --trials 60 --out profiles/r02/threshold_sweep_512x64.json"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--cal-trials", type=int, default=60)
ap.add_argument("--safety", type=float, default=1.0)
ap.add_argument("--cal-seed", type=int, default=0xCA11B010)
ap.add_argument("--trials", type=int, default=60)
ap.add_argument("--seed", type=int, default=0x5EEB)
ap.add_argument("--points", type=int, default=10)
ap.add_argument("--out", default="")
a = ap.parse_args()
args = [str(x) for x in (a.n, a.d, a.cal_trials, a.safety, a.cal_seed, a.trials, a.seed, a.points)]
res = {"config": {"n": a.n, "d": a.d, "block": 128, "stride": 8, "mode": "efta-opt", "cal_trials": a.cal_trials,
                  "safety": a.safety, "trials": a.trials, "points": a.points,
                  "point_format": "[threshold multiplier, detection rate, false-alarm rate]"}}
r = subprocess.run([os.path.join(ROOT, "tools", "sweep_gpu"), *args], capture_output=True, text=True)
if r.returncode == 0:
    gpu = json.loads(r.stdout)
    res["gpu"] = {"base": gpu["base"], "points": gpu["points"]}
else:
    res["gpu"] = {"error": (r.stderr or r.stdout)[-300:]}
ref_so = os.path.join(ROOT, "oracle", "_ref", "libefta_ref.so")
if os.path.exists(ref_so):
    lib = C.CDLL(ref_so)
    P = C.POINTER(C.c_double)
    lib.eref_threshold_sweep.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                         C.c_uint64, C.c_int, C.c_uint64, C.c_int, P, P, P, P]
    base = (C.c_double * 3)()
    mult, det, fa = ((C.c_double * a.points)() for _ in range(3))
    rc = lib.eref_threshold_sweep(a.n, a.d, 128, 8, 2, a.cal_trials, a.safety, a.cal_seed, a.trials, a.seed,
                                  a.points, base, mult, det, fa)
    if rc == 0:
        res["reference"] = {"base": list(base), "points": [[mult[i], det[i], fa[i]] for i in range(a.points)]}
s = json.dumps(res, indent=1)
print(s)
if a.out:
    with open(a.out, "w") as fh:
        fh.write(s + "\n")
