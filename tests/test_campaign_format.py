"""Wire formats of the GPU campaign: trials.csv and summary.json written
with the reference's columns / keys (src/campaign.cpp:359-372, tools/efta_main.cpp:87-162).
CPU-only: synthetic records, no kernel launch."""
import csv
import json

import numpy as np

# the reference's header, restated from src/campaign.cpp:362-363
REF_HEADER = ("trial,head,seed,injected,fired,site,bit,fault,detections,corrections,recomputes,"
              "range_replacements,failed,argmax_ok,residual_out,rel_residual_out,outcome")


def _records():
    return [
        dict(trial=0, head=0, seed=123456789012345, injected=True, fired=True, fault="EXP_OUT:1:1:2:3:31",
             site="EXP_OUT", bit=31, detections=1, corrections=1, recomputes=1, range_replacements=0,
             failed=False, argmax_ok=True, residual_out=1.25e-7, rel_residual_out=3.0e-7, outcome="corrected"),
        dict(trial=0, head=1, seed=42, injected=True, fired=True, fault="REDUCE_SUM:0:3:4:0:30",
             site="REDUCE_SUM", bit=30, detections=1, corrections=3, recomputes=0, range_replacements=3,
             failed=False, argmax_ok=True, residual_out=0.5, rel_residual_out=0.75, outcome="range_restricted"),
        dict(trial=1, head=0, seed=7, injected=True, fired=True, fault="GEMM1_OUT:3:2:68:17:11",
             site="GEMM1_OUT", bit=11, detections=1, corrections=0, recomputes=0, range_replacements=0,
             failed=True, argmax_ok=False, residual_out=2.0, rel_residual_out=4.0, outcome="uncorrectable"),
    ]


def test_trials_csv_matches_reference_columns(tmp_path):
    from paper_2504_02211_b200.campaign import TRIALS_CSV_HEADER, write_trials_csv
    assert TRIALS_CSV_HEADER == REF_HEADER
    path = tmp_path / "trials.csv"
    write_trials_csv(str(path), _records())
    rows = list(csv.DictReader(open(path)))
    assert list(rows[0].keys()) == REF_HEADER.split(",")
    assert rows[0]["seed"] == "123456789012345" and rows[0]["injected"] == "1"
    assert rows[0]["residual_out"] == "1.25e-07"  # C++ ostream default (6 significant digits)
    assert rows[1]["range_replacements"] == "3" and rows[1]["outcome"] == "range_restricted"
    assert rows[2]["failed"] == "1" and rows[2]["argmax_ok"] == "0"


def test_summary_json_keys_and_stats(tmp_path):
    from paper_2504_02211_b200.attention import Thresholds
    from paper_2504_02211_b200.campaign import write_summary_json
    path = tmp_path / "summary.json"
    write_summary_json(str(path), _records(), "efta-opt", 512, 64, 12, Thresholds(1e-5, 1e-4, 1e-4),
                       calibration={"calibration_trials": 128, "safety": 2.0})
    j = json.load(open(path))
    assert set(j) == {"mode", "config", "thresholds", "stats"}
    assert j["mode"] == "efta-opt"
    assert j["config"] == {"seq_len": 512, "head_dim": 64, "block": 128, "stride": 8, "heads": 12,
                           "scale": 0.125}
    assert j["thresholds"]["calibrated"] is True and j["thresholds"]["eps1"] == 1e-5
    st = j["stats"]
    # CampaignStats (src/campaign.cpp:236-256): every key the reference writes
    assert set(st) == {"trials", "injected", "fired", "detected", "false_alarms", "corrected",
                       "range_restricted", "masked_benign", "range_contract", "uncorrectable",
                       "argmax_preserved", "max_corrected_residual", "coverage"}
    assert (st["trials"], st["fired"], st["detected"], st["corrected"], st["uncorrectable"]) == (3, 3, 3, 1, 1)
    assert st["argmax_preserved"] == 2 and st["max_corrected_residual"] == 1.25e-7
    assert abs(st["coverage"] - 2.0 / 3.0) < 1e-12


def test_rows_argmax_match():
    from paper_2504_02211_b200.campaign import rows_argmax_match
    a = np.array([[0.1, 0.5, 0.5], [1.0, 0.0, 0.0]], np.float32)  # ties: first index wins
    assert rows_argmax_match(a, a.copy())
    b = a.copy()
    b[0, 2] = 0.6
    assert not rows_argmax_match(a, b)
    c = a.copy()
    c[1, 1] = np.nan
    assert not rows_argmax_match(c, a)  # the reference's finite guard (src/campaign.cpp:130)
