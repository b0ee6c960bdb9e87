"""Fault-handling parity harness: GPU (fault-tap build of the production CTA-pair kernel) vs the
CPU reference (oracle/_ref when built, else the bit-exact port) under identical seeded fault
plans and identical thresholds. Test infrastructure only.

Contract:
  * thresholds: each side is calibrated with the reference procedure (calibrate_thresholds,
    src/campaign.cpp:261-297: observation mode, worst clean residual per family x safety 2) on
    the same inputs; both sides then run with the per-family maximum of the two calibrations
    (neither side false-alarms, and one threshold decides for both);
  * per record: {fired, outcome class, non-CLEAN events (kind, block_i, block_j, status, row,
    col)} must be identical, unless the mismatch is explained by the margin rule (the two
    backends round differently: fp16 P, ex2.approx, tensor-core accumulation order):
      - near_threshold: an exp_checksum / output_checksum check of the faulted row block whose
        reference residual lies within a factor 4 of its threshold (eps1 resp. eps2) and that
        the upset moved (> 1.5x the fault-free twin's residual of the same check);
      - lin_margin: a GEMM1_OUT upset with eps_lin/4 < |after - before| < 4 eps_lin (the
        linear repair of the score tile decides between locating the cell and recomputing);
      - denominator_row: a corrupted or range-restricted denominator (REDUCE_SUM upset, or any
        range replacement) where both sides agree on the outcome and on every event but the
        located cell of the final output check: the row is divided by a wrong l, which scales its
        noise-level group residuals past eps2, so which cell gets the "largest correction" is
        picked by rounding.
    The marginal band (near_threshold or lin_margin, mismatched or not) is reported.
"""
from __future__ import annotations

import concurrent.futures as cf
import json
import os

import numpy as np

from helpers import oracle

SITES = ["GEMM1_OUT", "SUB_MAX", "EXP_OUT", "REDUCE_MAX", "REDUCE_SUM", "RESCALE_FACTOR",
         "GEMM2_ACC", "NORMALIZE_OUT"]
BLOCK, STRIDE = 128, 8
ACCEPT_BITS = (31, 30, 29, 22, 21)


def reference_oracle():
    """The unmodified reference when oracle/_ref was built (it travels with the repo snapshot),
    else the C restatement (bit-exact to it, tests/test_oracle.py)."""
    from oracle import Oracle
    try:
        return Oracle("ref")
    except FileNotFoundError:
        return oracle()


def acceptance_specs(seq, d, coords=20, bits=ACCEPT_BITS):
    """Reference acceptance check 4's fault list (tests/acceptance.cpp:131-161) at the GPU tile
    geometry: per (site, bit) an Rng(trial_seed(0xace4, s*64 + bit)) draws block_i, block_j
    (pinned 0 for NORMALIZE_OUT), row, col; the trial's inputs come from
    run_campaign(seed = trial_seed(0xbeef00 + s, bit*100 + c), 1 trial, 1 head)."""
    orc = oracle()
    nb = seq // BLOCK
    out = []
    for s in range(8):
        col_bound = 1 if s in (3, 4) else (BLOCK if s <= 2 else d)
        for bit in bits:
            bounds = []
            for _ in range(coords):
                bounds += [nb] + ([] if s == 7 else [nb]) + [BLOCK, col_bound]
            it = iter(orc.rng_below(orc.trial_seed(0xACE4, s * 64 + bit), bounds))
            for c in range(coords):
                bi = next(it)
                bj = 0 if s == 7 else next(it)
                row, col = next(it), next(it)
                seed = orc.trial_seed(0xBEEF00 + s, bit * 100 + c)
                out.append(((s, bi, bj, row, col, bit, 1), orc.trial_seed(seed, 0)))
    return out


def campaign_specs(n_trials, heads, seq, d, sites, seed):
    """run_campaign's random plans (src/campaign.cpp:172-185): per (trial, head) the head seed,
    q, k, v, then sample_random_plan from the same stream."""
    orc = oracle()
    out = []
    for t in range(n_trials):
        tseed = orc.trial_seed(seed, t)
        for h in range(heads):
            hseed = tseed if heads == 1 else orc.trial_seed(tseed, h)
            _, _, _, spec = orc.gen_trial(hseed, seq, d, BLOCK, STRIDE, sites=sites)
            out.append((spec, hseed))
    return out


def oracle_thresholds(seq, d, trials, seed, safety=2.0):
    """calibrate_thresholds (src/campaign.cpp:261-297) on the reference."""
    orc = reference_oracle()
    mx = {"exp_checksum": 0.0, "output_checksum": 0.0, "score_checksum": 0.0}

    def one(t):
        q, k, v, _ = orc.gen_trial(orc.trial_seed(seed, t), seq, d, BLOCK, STRIDE)
        r = orc.efta_forward(q, k, v, BLOCK, STRIDE, mode="efta-opt", thr=(np.inf, np.inf, np.inf),
                             observe_linear=True)
        return {kind: r.max_residual(kind) for kind in mx}

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for res in ex.map(one, range(trials)):
            for kind, v in res.items():
                if np.isfinite(v):
                    mx[kind] = max(mx[kind], v)
    return (mx["exp_checksum"] * safety, mx["output_checksum"] * safety, mx["score_checksum"] * safety)


def common_thresholds(seq, d, trials=64, seed=0xCA11B004):
    from paper_2504_02211_b200 import Thresholds
    from paper_2504_02211_b200.campaign import calibrate_thresholds
    thr_g, _ = calibrate_thresholds(seq, d, "efta-opt", trials=trials, safety=2.0, seed=seed)
    thr_o = oracle_thresholds(seq, d, trials, seed)
    thr = Thresholds(max(thr_g.eps1, thr_o[0]), max(thr_g.eps2, thr_o[1]), max(thr_g.eps_lin, thr_o[2]))
    return thr, (thr_g.eps1, thr_g.eps2, thr_g.eps_lin), thr_o


def _classify(out, ref, detections, rr, failed, final_l, site, eps2):
    from paper_2504_02211_b200.attention import FaultSpec
    from paper_2504_02211_b200.campaign import classify
    return classify(out, ref, detections, rr, failed, final_l, FaultSpec(site, 0, 0, 0, 0, 0), eps2)


def run_parity(plans, seq, d, thr):
    """plans: [(spec tuple (site, bi, bj, row, col, bit, trigger), head seed)]. Returns per-record
    dicts with both sides' outcome / fired / events and the margin explanation inputs."""
    from paper_2504_02211_b200.attention import FaultSpec
    from paper_2504_02211_b200.campaign import run_fault_records
    orc_in = oracle()
    ref = reference_oracle()
    ins = [orc_in.gen_trial(seed, seq, d, BLOCK, STRIDE)[:3] for _, seed in plans]
    qs = [q.astype(np.float16) for q, _, _ in ins]
    ks = [k.astype(np.float16) for _, k, _ in ins]
    vs = [v.astype(np.float16) for _, _, v in ins]
    specs = [FaultSpec(*t) for t, _ in plans]
    gpu = run_fault_records(qs, ks, vs, specs, thr)
    thr_t = (thr.eps1, thr.eps2, thr.eps_lin)

    def one(i):
        t, _ = plans[i]
        q, k, v = ins[i]
        r0 = ref.efta_forward(q, k, v, BLOCK, STRIDE, mode="efta-opt", thr=thr_t)
        r1 = ref.efta_forward(q, k, v, BLOCK, STRIDE, mode="efta-opt", thr=thr_t, specs=[t])
        oc = _classify(r1.o, r0.o, r1.detections, r1.range_replacements, r1.failed, r1.l, t[0], thr.eps2)
        ev = sorted((e["kind"], e["block_i"], e["block_j"], e["status"], e["row"], e["col"])
                    for e in r1.detected_events())
        def ratios(r):
            out = {}
            for e in r.events:
                if e["block_i"] != t[1] or not np.isfinite(e["residual"]):
                    continue
                den = thr.eps1 if e["kind"] == "exp_checksum" else (
                    thr.eps2 if e["kind"] == "output_checksum" else None)
                if den:
                    key = (e["kind"], e["block_j"])
                    out[key] = max(out.get(key, 0.0), e["residual"] / den)
            return out
        r_f, r_c = ratios(r1), ratios(r0)
        near = any(0.25 < v < 4.0 and v > 1.5 * r_c.get(key, 0.0) for key, v in r_f.items())
        fired = bool(r1.fired)
        dv = abs(float(r1.fired[0]["after"]) - float(r1.fired[0]["before"])) if fired else 0.0
        return dict(outcome=oc, fired=fired, events=ev, near=near, delta=dv,
                    range_replacements=r1.range_replacements, false_alarm=r0.detections)

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        orc_res = list(ex.map(one, range(len(plans))))
    rows = []
    for i, (t, seed) in enumerate(plans):
        o, g = orc_res[i], gpu[i]
        g_ev = [tuple(x) for x in g["events"]]
        same = o["fired"] == g["fired"] and o["outcome"] == g["outcome"] and o["events"] == g_ev
        lin = t[0] == 0 and 0.25 * thr.eps_lin < o["delta"] < 4.0 * thr.eps_lin
        strip = lambda ev: [e[:4] if e[0] == "output_checksum" else e for e in ev]  # noqa: E731
        range_row = ((t[0] == 4 or o["range_replacements"] > 0 or g["range_replacements"] > 0) and
                     o["fired"] == g["fired"] and o["outcome"] == g["outcome"] and
                     strip(o["events"]) == strip(g_ev))
        why = [] if same else [w for w, ok in (("near_threshold", o["near"]), ("lin_margin", lin),
                                                ("denominator_row", range_row)) if ok]
        rows.append(dict(spec=":".join([SITES[t[0]]] + [str(x) for x in t[1:6]]), site=SITES[t[0]], bit=t[5],
                         seed=seed, oracle=o["outcome"], gpu=g["outcome"], fired_o=o["fired"],
                         fired_g=g["fired"], ev_o=o["events"], ev_g=g_ev, same=same, explained=why,
                         band=o["near"] or lin, false_alarm_o=o["false_alarm"],
                         false_alarm_g=g["clean_false_alarms"]))
    return rows


def summarize(rows, name=None, extra=None):
    n = len(rows)
    mism = [r for r in rows if not r["same"]]
    unexplained = [r for r in mism if not r["explained"]]
    outc = {}
    for r in rows:
        outc.setdefault(r["oracle"], [0, 0])[0] += 1
        outc.setdefault(r["gpu"], [0, 0])[1] += 1
    s = dict(records=n, identical=n - len(mism), mismatched=len(mism), explained_by_margin=len(mism) - len(unexplained),
             unexplained=len(unexplained), marginal_band=sum(r["band"] for r in rows),
             marginal_band_identical=sum(r["band"] and r["same"] for r in rows),
             fired_oracle=sum(r["fired_o"] for r in rows), fired_gpu=sum(r["fired_g"] for r in rows),
             outcomes_oracle_gpu={k: v for k, v in sorted(outc.items())},
             mismatches=[(r["spec"], r["oracle"], r["gpu"], r["ev_o"], r["ev_g"], r["explained"])
                         for r in mism][:40])
    if extra:
        s.update(extra)
    out = os.environ.get("EFTA_PARITY_OUT")
    if out and name:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, f"{name}.json"), "w") as f:
            json.dump(s, f, indent=1, default=str)
    return s
