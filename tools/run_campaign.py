"""GPU fault-injection campaign (C2: B=1, H=12, S=512, d=64, seeded single-bit flips in the score
accumulators, the softmax exponentials and the P.V accumulators) written in the reference's wire
formats: <out>/trials.csv and <out>/summary.json (src/campaign.cpp:359-372, tools/efta_main.cpp:87-162).

python tools/run_campaign.py --out gpurun_out/campaign --trials 20"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2504_02211_b200 import campaign  # noqa: E402
from paper_2504_02211_b200._lib import SITES  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/campaign")
ap.add_argument("--trials", type=int, default=20)
ap.add_argument("--heads", type=int, default=12)
ap.add_argument("--seq", type=int, default=512)
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--seed", type=int, default=7)
ap.add_argument("--calibrate", type=int, default=128)
ap.add_argument("--sites", default="GEMM1_OUT,EXP_OUT,GEMM2_ACC")
a = ap.parse_args()
sites = [SITES.index(s) for s in a.sites.split(",")]
thr, fam = campaign.calibrate_thresholds(a.seq, a.d, "efta-opt", a.calibrate, 2.0, a.seed ^ 0xCA11B7A7)
res = campaign.run_gpu_campaign(a.trials, a.heads, a.seq, a.d, sites=sites, seed=a.seed, thr=thr)
os.makedirs(a.out, exist_ok=True)
campaign.write_trials_csv(os.path.join(a.out, "trials.csv"), res["detail"])
j = campaign.write_summary_json(os.path.join(a.out, "summary.json"), res["detail"], "efta-opt", a.seq, a.d,
                                a.heads, thr, calibration={"calibration_trials": a.calibrate, "safety": 2.0,
                                                           "max_clean_exp": fam[0], "max_clean_out": fam[1],
                                                           "max_clean_lin": fam[2]})
print(j["stats"])
