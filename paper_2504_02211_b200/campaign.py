"""GPU-backed fault-injection campaign — mirror of the reference's run_campaign /
classify_trial / calibrate_thresholds (reference src/campaign.cpp:123-297).

Trials are batched: every (trial, head) record of the reference becomes one
head of a single batched launch (heads are independent units), inputs and
fault plans are drawn with the reference's Rng stream (efta_gen_trial_f16, the
C++ host layer), and outcomes are classified on the host by the reference's
outcome ladder (efta_classify_trial).
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _lib
from ._lib import SITES, lib
from .attention import EftaAttention, FaultSpec, Thresholds

OUTCOMES = ["clean", "false_alarm", "corrected", "range_restricted", "masked_benign",
            "range_contract", "uncorrectable"]

lib.efta_trial_seed.restype = C.c_uint64
lib.efta_trial_seed.argtypes = [C.c_uint64, C.c_uint64]
lib.efta_gen_trial_f16.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_int), C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.POINTER(_lib.FaultSpec)]
lib.efta_classify_trial.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                    C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double]


def trial_seed(base: int, trial: int) -> int:
    return int(lib.efta_trial_seed(base, trial))


def gen_head(seed: int, n: int, d: int, block=128, stride=8, sites=None):
    """Reference Rng(seed): q, k, v = Matrix::random(n, d) in that order, then an
    optional sample_random_plan (src/campaign.cpp:177-185)."""
    q = np.empty((n, d), np.uint16)
    k = np.empty_like(q)
    v = np.empty_like(q)
    sites = list(sites or [])
    arr = (C.c_int * max(1, len(sites)))(*sites)
    spec = _lib.FaultSpec()
    rc = lib.efta_gen_trial_f16(seed, n, d, block, stride, arr, len(sites), q.ctypes.data,
                                k.ctypes.data, v.ctypes.data, C.byref(spec))
    if rc:
        raise _lib.ConfigError("gen_trial failed")
    f = None
    if sites:
        f = FaultSpec(spec.site, spec.block_i, spec.block_j, spec.row, spec.col, spec.bit,
                      spec.trigger)
    return q.view(np.float16), k.view(np.float16), v.view(np.float16), f


def classify(out: np.ndarray, ref: np.ndarray, detections: int, range_replacements: int,
             failed: bool, final_l: np.ndarray, spec, eps2: float) -> str:
    out = np.ascontiguousarray(out, np.float32)
    ref = np.ascontiguousarray(ref, np.float32)
    fl = np.ascontiguousarray(final_l, np.float32)
    red = spec is not None and spec.site in (SITES.index("REDUCE_MAX"), SITES.index("REDUCE_SUM"))
    o = lib.efta_classify_trial(out.shape[0], out.shape[1], out.ctypes.data, ref.ctypes.data,
                                detections, range_replacements, 1 if failed else 0, fl.ctypes.data,
                                fl.size, 1 if spec is not None else 0, 1 if red else 0, eps2)
    return OUTCOMES[o]


def per_head_report(events, n_heads):
    """Split device events by head (the device logs non-CLEAN events only)."""
    det = [0] * n_heads
    rr = [0] * n_heads
    failed = [False] * n_heads
    for e in events:
        h = e["head"]
        if e["status"] != "clean":
            det[h] += 1
        if e["kind"] == "rowsum_range":
            rr[h] += e["corrections"]
        if e["status"] in ("detected_uncorrectable", "nonfinite"):
            failed[h] = True
    return det, rr, failed


def calibrate_thresholds(seq_len, head_dim, mode="efta-opt", trials=64, safety=2.0, seed=1,
                         device="cuda"):
    """calibrate_thresholds (src/campaign.cpp:261-297) on the GPU: clean runs in
    observation mode (+ per-iteration linear residuals); each threshold is the worst
    clean residual of its family times `safety`. Trials run as heads of one launch."""
    qs, ks, vs = [], [], []
    for t in range(trials):
        q, k, v, _ = gen_head(trial_seed(seed, t), seq_len, head_dim)
        qs.append(q); ks.append(k); vs.append(v)
    dev = torch.device(device)
    q = torch.from_numpy(np.stack(qs)).to(dev).view(1, trials, seq_len, head_dim)
    k = torch.from_numpy(np.stack(ks)).to(dev).view(1, trials, seq_len, head_dim)
    v = torch.from_numpy(np.stack(vs)).to(dev).view(1, trials, seq_len, head_dim)
    op = EftaAttention(1, trials, seq_len, head_dim, mode=mode, thr=Thresholds.observe(),
                       observe_linear=True, debug=True, device=dev)
    op(q, k, v)
    rep = op.report()
    fe, fo, fl = rep.family_max
    thr = Thresholds(fe * safety if fe > 0 else math.inf, fo * safety if fo > 0 else math.inf,
                     fl * safety if fl > 0 else math.inf)
    return thr, rep.family_max


def run_fault_records(qs, ks, vs, specs, thr: Thresholds, mode="efta-opt", device="cuda"):
    """One batched pair of launches (fault-free twin, then faulted) over independent heads:
    head i gets inputs (qs[i], ks[i], vs[i]) [S, d] fp16 and fault spec specs[i] (or None).
    Returns per-head records with the reference classify_trial outcome, whether the fault
    fired, and the non-CLEAN events (kind, block_i, block_j, status, row, col)."""
    n_rec = len(qs)
    seq_len, head_dim = qs[0].shape
    dev = torch.device(device)
    shape = (1, n_rec, seq_len, head_dim)
    q = torch.from_numpy(np.stack(qs)).to(dev).view(shape)
    k = torch.from_numpy(np.stack(ks)).to(dev).view(shape)
    v = torch.from_numpy(np.stack(vs)).to(dev).view(shape)
    ev_cap = max(4096, 64 * n_rec)
    clean = EftaAttention(1, n_rec, seq_len, head_dim, mode=mode, thr=thr, debug=True,
                          ev_cap=ev_cap, device=dev)
    o_ref, _, _ = clean(q, k, v)
    rep_clean = clean.report()
    faulted = EftaAttention(1, n_rec, seq_len, head_dim, mode=mode, thr=thr, debug=True,
                            ev_cap=ev_cap, fired_cap=2 * n_rec, device=dev)
    hspecs = []
    for i, f in enumerate(specs):
        if f is not None:
            hspecs.append(FaultSpec(f.site, f.block_i, f.block_j, f.row, f.col, f.bit, f.trigger, head=i))
    faulted.set_faults(hspecs)
    o, m, l = faulted(q, k, v)
    rep = faulted.report(m, l)
    det, rr, failed = per_head_report(rep.events, n_rec)
    fired_heads = {f["spec"].head for f in rep.fired}
    o_np = o.view(n_rec, seq_len, head_dim).cpu().numpy()
    r_np = o_ref.view(n_rec, seq_len, head_dim).cpu().numpy()
    l_np = l.view(n_rec, seq_len).cpu().numpy()
    events = {i: [] for i in range(n_rec)}
    corr = [0] * n_rec
    reco = [0] * n_rec
    for e in rep.events:
        h = e["head"]
        corr[h] += e["corrections"]
        if e["kind"] in ("exp_checksum", "factor_range") and e["status"] == "corrected":
            reco[h] += 1
        if e["status"] != "clean":
            events[h].append((e["kind"], e["block_i"], e["block_j"], e["status"], e["row"], e["col"]))
    clean_det = [0] * n_rec
    for e in rep_clean.events:
        if e["status"] != "clean":
            clean_det[e["head"]] += 1
    out = []
    for i in range(n_rec):
        oc = classify(o_np[i], r_np[i], det[i], rr[i], failed[i], l_np[i], specs[i], thr.eps2)
        res = float(np.abs(o_np[i].astype(np.float64) - r_np[i]).max())
        ref_inf = float(np.abs(r_np[i]).max())
        out.append(dict(outcome=oc, fired=i in fired_heads, detections=det[i], corrections=corr[i],
                        recomputes=reco[i], range_replacements=rr[i], failed=failed[i],
                        events=sorted(events[i]), clean_false_alarms=clean_det[i],
                        argmax_ok=rows_argmax_match(o_np[i], r_np[i]), residual_out=res,
                        rel_residual_out=res / ref_inf if ref_inf > 0 else 0.0))
    return out


def run_gpu_campaign(n_trials=20, heads=12, seq_len=512, head_dim=64, sites=None, seed=7,
                     mode="efta-opt", thr: Thresholds | None = None, calibrate_trials=128,
                     device="cuda", fixed_plan=None):
    """run_campaign (src/campaign.cpp:154-259) with injection: one single-bit
    fault per (trial, head) record, classified against the fault-free twin. Runs the
    fault-tap build of the production CTA-pair kernel (debug=1) whenever the query-tile
    count is even."""
    if sites is None:
        sites = list(range(8))
    if thr is None:
        thr, _ = calibrate_thresholds(seq_len, head_dim, mode, calibrate_trials, 2.0,
                                      seed ^ 0xCA11B7A7, device)
    n_rec = n_trials * heads
    qs, ks, vs, specs, seeds = [], [], [], [], []
    for t in range(n_trials):
        tseed = trial_seed(seed, t)
        for h in range(heads):
            hseed = tseed if heads == 1 else trial_seed(tseed, h)
            seeds.append(hseed)
            q, k, v, f = gen_head(hseed, seq_len, head_dim, sites=None if fixed_plan else sites)
            if fixed_plan is not None:
                f = FaultSpec.parse(fixed_plan) if isinstance(fixed_plan, str) else fixed_plan
                f = FaultSpec(f.site, f.block_i, f.block_j, f.row, f.col, f.bit, f.trigger)
            qs.append(q); ks.append(k); vs.append(v); specs.append(f)
    recs = run_fault_records(qs, ks, vs, specs, thr, mode, device)
    records = []
    stats = {k2: 0 for k2 in OUTCOMES}
    for i, r in enumerate(recs):
        stats[r["outcome"]] += 1
        records.append(dict(trial=i // heads, head=i % heads, seed=seeds[i], injected=True,
                            fired=r["fired"], fault=specs[i].to_string(), spec=specs[i],
                            site=SITES[specs[i].site], bit=specs[i].bit, detections=r["detections"],
                            corrections=r["corrections"], recomputes=r["recomputes"],
                            range_replacements=r["range_replacements"], failed=r["failed"],
                            argmax_ok=r["argmax_ok"], residual_out=r["residual_out"],
                            rel_residual_out=r["rel_residual_out"], outcome=r["outcome"],
                            events=r["events"]))
    n_fired = sum(r["fired"] for r in records)
    bad = sum(1 for r in records if r["fired"] and r["outcome"] == "uncorrectable")
    return {"records": n_rec, "fired": n_fired, "coverage": 1.0 - bad / n_fired if n_fired else 1.0,
            "corrected": stats["corrected"], "masked_benign": stats["masked_benign"],
            "range_restricted": stats["range_restricted"],
            "range_contract": stats["range_contract"], "uncorrectable": stats["uncorrectable"],
            "false_alarms": sum(r["clean_false_alarms"] for r in recs),
            "thresholds": (thr.eps1, thr.eps2, thr.eps_lin), "detail": records}


# ---------------------------------------------------------------- wire formats
# trials.csv (src/campaign.cpp:359-372) and summary.json (tools/efta_main.cpp:117-162) written
# from GPU campaign records. Doubles follow C++ ostream defaults (6 significant digits).
TRIALS_CSV_HEADER = ("trial,head,seed,injected,fired,site,bit,fault,detections,corrections,recomputes,"
                     "range_replacements,failed,argmax_ok,residual_out,rel_residual_out,outcome")


def rows_argmax_match(a: np.ndarray, b: np.ndarray) -> bool:
    """rows_argmax_match (src/campaign.cpp:25-36) behind the finite guard of :130."""
    if a.shape != b.shape or not np.isfinite(a).all():
        return False
    return bool(np.array_equal(np.argmax(a, axis=1), np.argmax(b, axis=1)))


def _g(x: float) -> str:
    return f"{x:.6g}"


def write_trials_csv(path: str, records) -> None:
    with open(path, "w") as f:
        f.write(TRIALS_CSV_HEADER + "\n")
        for r in records:
            f.write(",".join([str(r["trial"]), str(r["head"]), str(r["seed"]), str(int(r["injected"])),
                              str(int(r["fired"])), r["site"], str(r["bit"]), r["fault"],
                              str(r["detections"]), str(r["corrections"]), str(r["recomputes"]),
                              str(r["range_replacements"]), str(int(r["failed"])), str(int(r["argmax_ok"])),
                              _g(r["residual_out"]), _g(r["rel_residual_out"]), r["outcome"]]) + "\n")


def campaign_stats(records) -> dict:
    """CampaignStats aggregation (src/campaign.cpp:236-256) + coverage (:103-111)."""
    st = dict(trials=0, injected=0, fired=0, detected=0, false_alarms=0, corrected=0, range_restricted=0,
              masked_benign=0, range_contract=0, uncorrectable=0, argmax_preserved=0,
              max_corrected_residual=0.0)
    for r in records:
        st["trials"] += 1
        st["injected"] += int(r["injected"])
        st["fired"] += int(r["fired"])
        st["detected"] += int(r["detections"] > 0)
        st["argmax_preserved"] += int(r["injected"] and r["argmax_ok"])
        o = r["outcome"]
        if o == "false_alarm":
            st["false_alarms"] += 1
        elif o != "clean":
            st[o] += 1
        if o == "corrected":
            st["max_corrected_residual"] = max(st["max_corrected_residual"], r["residual_out"])
    st["coverage"] = 1.0 - st["uncorrectable"] / st["fired"] if st["fired"] else 1.0
    return st


def write_summary_json(path: str, records, mode: str, seq_len: int, head_dim: int, heads: int,
                       thr: Thresholds, block: int = 128, stride: int = 8, scale: float | None = None,
                       calibration: dict | None = None) -> dict:
    """summary.json with the reference's mode / config / thresholds / stats keys. The reference's
    analytic `counters` and `overhead` blocks are CPU operation counts; the GPU reports measured
    time instead (bench.py), so they are omitted."""
    import json
    j = {"mode": {"efta-opt": "efta-opt", "efta": "efta", "none": "none"}[mode],
         "config": {"seq_len": seq_len, "head_dim": head_dim, "block": block, "stride": stride, "heads": heads,
                    "scale": scale if scale is not None else 1.0 / math.sqrt(head_dim)},
         "thresholds": {**({"calibrated": True, **calibration} if calibration else {"calibrated": False}),
                        "eps1": thr.eps1, "eps2": thr.eps2, "eps_lin": thr.eps_lin},
         "stats": campaign_stats(records)}
    with open(path, "w") as f:
        f.write(json.dumps(j, indent=2) + "\n")
    return j
