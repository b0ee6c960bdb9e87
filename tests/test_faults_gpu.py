"""GPU fault-handling parity with the CPU oracle under identical seeded fault plans.

Mirrors the reference's acceptance check 4 (tests/acceptance.cpp:125-211): every
site x bits {31,30,29,22,21} x seeded coordinates, at the GPU tile geometry
(block 128, stride 8) on a C1 head (S=512, d=64). Each side is classified
against its own fault-free twin with thresholds calibrated on its own clean runs
(reference calibrate_thresholds, src/campaign.cpp:261-297). Contract:
  * every fault the oracle absorbs is absorbed on the GPU (never uncorrectable);
  * the non-CLEAN check events (kind, block_i, block_j, status) agree exactly for
    the faults whose detection is not threshold-marginal;
  * the outcome classes agree for >= 95% of the sweep.
"""
import numpy as np
import pytest

from helpers import oracle

pytestmark = pytest.mark.gpu

SEQ, D, BLK, STR = 512, 64, 128, 8
BITS = (31, 30, 29, 22, 21)
COORDS = 4
ABSORBED = {"corrected", "masked_benign", "range_restricted", "range_contract", "clean"}


def _oracle_thresholds(trials=40, safety=2.0, seed=0xCA11B004):
    """calibrate_thresholds on the oracle: observe mode + per-iteration linear check."""
    orc = oracle()
    mx = {"exp_checksum": 0.0, "output_checksum": 0.0, "score_checksum": 0.0}
    for t in range(trials):
        q, k, v, _ = orc.gen_trial(orc.trial_seed(seed, t), SEQ, D, BLK, STR)
        r = orc.efta_forward(q, k, v, BLK, STR, mode="efta-opt",
                             thr=(np.inf, np.inf, np.inf), observe_linear=True)
        for kind in mx:
            v_ = r.max_residual(kind)
            if np.isfinite(v_):
                mx[kind] = max(mx[kind], v_)
    return (mx["exp_checksum"] * safety, mx["output_checksum"] * safety,
            mx["score_checksum"] * safety)


def _sweep_specs():
    """acceptance.cpp:137-158 coordinate scheme at block 128."""
    orc = oracle()
    from oracle import SITES
    out = []
    n = SEQ // BLK
    for s in range(8):
        for bit in BITS:
            # the reference draws coordinates from Rng(trial_seed(0xace4, s*64+bit)); we draw
            # them with the same generator through the oracle's random stream
            rnd = orc.random_matrix(orc.trial_seed(0xACE4, s * 64 + bit), 1, 4 * COORDS, 0.0, 1.0,
                                    half=False)[0]
            for c in range(COORDS):
                u = rnd[4 * c: 4 * c + 4]
                bi = int(u[0] * n)
                bj = 0 if s == 7 else int(u[1] * n)
                row = int(u[2] * BLK)
                bound = 1 if s in (3, 4) else (BLK if s <= 2 else D)
                col = int(u[3] * bound)
                seed = orc.trial_seed(0xBEEF00 + s, bit * 100 + c)
                out.append((SITES[s], (s, bi, bj, row, col, bit, 1), seed))
    return out


def _classify(out, ref, detections, rr, failed, final_l, site, eps2):
    from paper_2504_02211_b200.attention import FaultSpec
    from paper_2504_02211_b200.campaign import classify
    spec = FaultSpec(site, 0, 0, 0, 0, 0)
    return classify(out, ref, detections, rr, failed, final_l, spec, eps2)


@pytest.fixture(scope="module")
def sweep():
    import torch
    from paper_2504_02211_b200 import EftaAttention
    from paper_2504_02211_b200.attention import FaultSpec
    from paper_2504_02211_b200.campaign import calibrate_thresholds, per_head_report

    orc = oracle()
    specs = _sweep_specs()
    thr_o = _oracle_thresholds()
    thr_g, _ = calibrate_thresholds(SEQ, D, "efta-opt", trials=128, safety=2.0, seed=0xCA11B004)
    qs, ks, vs = [], [], []
    for _, _, seed in specs:
        q, k, v, _ = orc.gen_trial(seed, SEQ, D, BLK, STR)
        qs.append(q); ks.append(k); vs.append(v)
    n = len(specs)
    dev = lambda x: torch.from_numpy(np.stack(x)).half().cuda().view(1, n, SEQ, D)  # noqa: E731
    q, k, v = dev(qs), dev(ks), dev(vs)
    clean = EftaAttention(1, n, SEQ, D, mode="efta-opt", thr=thr_g, debug=True, ev_cap=1 << 14)
    o_ref, _, _ = clean(q, k, v)
    rep_clean = clean.report()
    faulted = EftaAttention(1, n, SEQ, D, mode="efta-opt", thr=thr_g, debug=True, ev_cap=1 << 14,
                            fired_cap=2 * n)
    faulted.set_faults([FaultSpec(*t, head=i) for i, (_, t, _) in enumerate(specs)])
    o_g, _, l_g = faulted(q, k, v)
    rep = faulted.report()
    det, rr, failed = per_head_report(rep.events, n)
    o_g = o_g.view(n, SEQ, D).cpu().numpy()
    o_ref = o_ref.view(n, SEQ, D).cpu().numpy()
    l_g = l_g.view(n, SEQ).cpu().numpy()
    gpu_events = {i: [] for i in range(n)}
    for e in rep.events:
        gpu_events[e["head"]].append((e["kind"], e["block_i"], e["block_j"], e["status"]))
    rows = []
    for i, (site, t, seed) in enumerate(specs):
        ro = orc.efta_forward(qs[i], ks[i], vs[i], BLK, STR, mode="efta-opt", thr=thr_o)
        rf = orc.efta_forward(qs[i], ks[i], vs[i], BLK, STR, mode="efta-opt", thr=thr_o, specs=[t])
        c_o = _classify(rf.o, ro.o, rf.detections, rf.range_replacements, rf.failed, rf.l, t[0],
                        thr_o[1])
        c_g = _classify(o_g[i], o_ref[i], det[i], rr[i], failed[i], l_g[i], t[0], thr_g.eps2)
        ev_o = sorted((e["kind"], e["block_i"], e["block_j"], e["status"])
                      for e in rf.detected_events())
        rows.append(dict(site=site, spec=t, oracle=c_o, gpu=c_g, ev_o=ev_o,
                         ev_g=sorted(gpu_events[i]), fired_o=bool(rf.fired)))
    return dict(rows=rows, false_alarms=rep_clean.detections, thr_o=thr_o, thr_g=thr_g)


def test_no_false_alarms_on_clean_twins(sweep):
    assert sweep["false_alarms"] == 0


def test_gpu_absorbs_everything_the_oracle_absorbs(sweep):
    bad = [r for r in sweep["rows"] if r["oracle"] in ABSORBED and r["gpu"] not in ABSORBED]
    assert not bad, bad[:5]


def test_outcome_classes_agree(sweep):
    rows = sweep["rows"]
    agree = sum(r["oracle"] == r["gpu"] for r in rows)
    mism = [(r["site"], r["spec"], r["oracle"], r["gpu"]) for r in rows if r["oracle"] != r["gpu"]]
    assert agree >= 0.95 * len(rows), (agree, len(rows), mism[:10])


def test_events_agree_for_non_marginal_faults(sweep):
    """Exponent / sign flips (bits 31, 30, 29) on the data sites are far above any
    threshold on both sides: their non-CLEAN events must match exactly."""
    data_sites = {"GEMM1_OUT", "EXP_OUT", "GEMM2_ACC", "NORMALIZE_OUT"}
    checked, bad = 0, []
    for r in sweep["rows"]:
        if r["site"] in data_sites and r["spec"][5] in (31, 30, 29) and r["fired_o"]:
            checked += 1
            if r["ev_o"] != r["ev_g"]:
                bad.append((r["site"], r["spec"], r["ev_o"], r["ev_g"]))
    assert checked > 20
    assert len(bad) <= 0.05 * checked, bad[:6]
