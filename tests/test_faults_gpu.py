"""GPU fault-handling parity with the CPU reference under identical seeded fault plans, on the
fault-tap build of the production CTA-pair kernel (tests/fault_parity.py states the contract).

* acceptance sweep (reference acceptance check 4, tests/acceptance.cpp:125-211): every
  FaultSite x bits {31, 30, 29, 22, 21} x 20 reference-drawn coordinates, at d = 64 and d = 128
  (S = 512, block 128, stride 8): per record {fired, outcome, non-CLEAN events incl. row and
  col} identical to the reference, every mismatch explained by the margin rule, everything
  the reference absorbs absorbed;
* C2 campaign replay (BASELINE configs[1]: C1 shape, 20 trials x 12 heads, random plans over
  GEMM1_OUT / EXP_OUT / GEMM2_ACC, run_campaign's seeds): the same per-record contract.
"""
import pytest

from fault_parity import (acceptance_specs, campaign_specs, common_thresholds, run_parity,
                          summarize)

pytestmark = pytest.mark.gpu

SEQ = 512
ABSORBED = {"corrected", "masked_benign", "range_restricted", "range_contract", "clean"}


@pytest.fixture(scope="module", params=[64, 128])
def sweep(request):
    d = request.param
    thr, thr_g, thr_o = common_thresholds(SEQ, d)
    rows = run_parity(acceptance_specs(SEQ, d), SEQ, d, thr)
    s = summarize(rows, f"acceptance_sweep_d{d}",
                  dict(thresholds=(thr.eps1, thr.eps2, thr.eps_lin), thr_gpu=thr_g, thr_ref=thr_o))
    return dict(d=d, rows=rows, summary=s)


def test_sweep_no_false_alarms(sweep):
    assert all(r["false_alarm_g"] == 0 and r["false_alarm_o"] == 0 for r in sweep["rows"])


def test_sweep_gpu_absorbs_what_reference_absorbs(sweep):
    bad = [(r["spec"], r["oracle"], r["gpu"]) for r in sweep["rows"]
           if r["oracle"] in ABSORBED and r["gpu"] not in ABSORBED]
    assert not bad, bad[:8]


def test_sweep_records_identical_or_marginal(sweep):
    s = sweep["summary"]
    assert s["records"] == 800
    assert s["unexplained"] == 0, s["mismatches"][:10]
    # the margin rule may only explain a small fraction
    assert s["mismatched"] <= 0.03 * s["records"], s


@pytest.fixture(scope="module")
def c2():
    from paper_2504_02211_b200.campaign import SITES as S
    sites = [S.index("GEMM1_OUT"), S.index("EXP_OUT"), S.index("GEMM2_ACC")]
    thr, thr_g, thr_o = common_thresholds(SEQ, 64)
    rows = run_parity(campaign_specs(20, 12, SEQ, 64, sites, seed=7), SEQ, 64, thr)
    return dict(rows=rows, summary=summarize(rows, "c2_campaign",
                                             dict(thresholds=(thr.eps1, thr.eps2, thr.eps_lin),
                                                  thr_gpu=thr_g, thr_ref=thr_o)))


def test_c2_campaign_records_identical_or_marginal(c2):
    s = c2["summary"]
    assert s["records"] == 240
    assert s["unexplained"] == 0, s["mismatches"][:10]
    assert s["mismatched"] <= 0.03 * s["records"], s


def test_c2_campaign_fired_sets_identical(c2):
    assert all(r["fired_o"] == r["fired_g"] for r in c2["rows"])
