#!/usr/bin/env python3
"""bench.py — EFTA attention throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[3], "C4"): Llama-style attention B=32 H=32 S=8192
d_head=128 (1024 independent heads), fp16 Q/K/V (U(-1,1) on the fp16 grid like the
reference's Matrix::random), EFTA-optimized protection, block 128, stride 8.
Multi-GPU: one process per GPU; the 1024 global (batch x head) units
are split contiguously over the ranks (strong scaling, no collective on the data path;
the only collectives are the timing barrier / max-reduce).

One step = one protected forward over the rank's heads: checksum-encode prepass + the
fused attention kernel. value = 4*B*H*S^2*d FLOPs (the whole job) / max-over-ranks
device time.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B, H, S, D = 32, 32, 8192, 128
BLOCK, STRIDE = 128, 8
METRIC = "EFTA attention TFLOPS/GPU (EFTA-optimized fused forward)"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "r02", "attn_c4_traffic.json")


def flops(b, h, s, d):
    return 4.0 * b * h * s * s * d


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-campaign", action="store_true")
    ap.add_argument("--no-suite", action="store_true")
    return ap.parse_args()


# --------------------------------------------------------------------- dist
def dist_init(n):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    pg = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    else:
        torch.cuda.set_device(0)
    return rank, world, local, pg


def barrier(pg):
    import torch
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize()


def max_over_ranks(pg, x):
    import torch
    if pg is None:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock + throttle reasons via NVML during the timed region."""

    def __init__(self, index):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self.stop_ev.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        if self.nv is not None:
            self.t.join()

    def result(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- our arm
def synth_inputs(seed, shape, device):
    """U(-1,1) rounded to fp16 — the reference's Matrix::random distribution."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.empty(shape, dtype=torch.float32, device=device).uniform_(-1.0, 1.0, generator=g)
    return x.to(torch.float16)


def time_steps(fn, steps, warmup, pg):
    import torch
    for _ in range(warmup):
        fn()
    barrier(pg)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        fn()
    e1.record(st)
    barrier(pg)
    return e0.elapsed_time(e1) / steps  # ms per step on this rank


def cpu_baseline_ref(threads=None):
    """The unmodified reference (oracle/_ref) on C4 heads, one full head per host
    thread (efta_forward EFTA_OPTIMIZED, block 128, stride 8), timed by wall clock."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle  # test infrastructure: the CPU checker / baseline only
    which = "ref" if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libefta_ref.so")) else "port"
    orc = Oracle(which)
    ncpu = os.cpu_count() or 1
    threads = threads or ncpu
    heads = []
    for t in range(threads):
        q, k, v, _ = orc.gen_trial(orc.trial_seed(2024, t), S, D, BLOCK, STRIDE)
        heads.append((q, k, v))
    thr = (1e-5, 1e-4, 1e-4)

    def work(i):
        q, k, v = heads[i]
        orc.efta_forward(q, k, v, BLOCK, STRIDE, mode="efta-opt", thr=thr, ev_cap=1 << 14)

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    wall = time.perf_counter() - t0
    tf = threads * flops(1, 1, S, D) / wall / 1e12
    return {"value": tf, "unit": "TFLOP/s", "cores": threads,
            "kind": "reference" if which == "ref" else "port",
            "sample": f"{threads} C4 heads (S={S}, d={D}), one per host thread, EFTA_OPTIMIZED, "
                      f"block {BLOCK} stride {STRIDE}; wall {wall:.1f}s"}


def fault_campaign(n_trials=20):
    """C2-style campaign on the GPU: C1 shape (H=12, S=512, d=64), one random
    single-bit fault per (trial, head) over sites GEMM1_OUT / EXP_OUT / GEMM2_ACC,
    classified against the fault-free twin like the reference run_campaign."""
    from paper_2504_02211_b200.campaign import run_gpu_campaign
    st = run_gpu_campaign(n_trials=n_trials, heads=12, seq_len=512, head_dim=64,
                          sites=[0, 2, 6], seed=7)
    return st


def _time_cuda(fn, iters=5, warmup=2):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(iters):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def suite(dev):
    """The other BASELINE.json configs as secondary measurements (rank 0, N=1):
    C3 = BERT-large/GPT-2-medium attention B=16 H=16 S=2048 d=64 + the two strided-ABFT
    FFN GEMMs (d_model 1024, d_ff 4096, 32K tokens) against cuBLAS; C5 = the full
    FT-Transformer layer at GPT-2-large shapes over a 512..16K sequence sweep at 16K
    tokens, protected vs the unprotected twin of the same layer."""
    import torch
    from paper_2504_02211_b200 import AbftLinear, EftaAttention, FTTransformerLayer, Thresholds
    out = {}
    thr = Thresholds(1e-4, 1e-3, 1e-3)
    b, h, s_, d = 16, 16, 2048, 64
    q = synth_inputs(11, (b, h, s_, d), dev)
    k = synth_inputs(12, (b, h, s_, d), dev)
    v = synth_inputs(13, (b, h, s_, d), dev)
    c3 = {}
    for mode in ("efta-opt", "none"):
        op = EftaAttention(b, h, s_, d, mode=mode, thr=thr, device=dev)
        ms = _time_cuda(lambda: op(q, k, v))
        c3[f"attention_{mode}_tflops"] = round(flops(b, h, s_, d) / (ms * 1e-3) / 1e12, 2)
    del q, k, v
    t, dm, dff = 32768, 1024, 4096
    g = torch.Generator(device=dev)
    g.manual_seed(21)
    x = (torch.empty((t, dm), device=dev).uniform_(-1, 1, generator=g)).half()
    w1 = (torch.empty((dff, dm), device=dev).uniform_(-1, 1, generator=g) / math.sqrt(dm)).half()
    w2 = (torch.empty((dm, dff), device=dev).uniform_(-1, 1, generator=g) / math.sqrt(dff)).half()
    l1, l2 = AbftLinear(w1), AbftLinear(w2)
    y1 = l1(x)
    gf = 2.0 * t * dm * dff
    ms_p = _time_cuda(lambda: l2(l1(x, y1)))
    ms_u = _time_cuda(lambda: (x @ w1.t()) @ w2.t())
    c3["ffn_abft_tflops"] = round(2 * gf / (ms_p * 1e-3) / 1e12, 2)
    c3["ffn_cublas_tflops"] = round(2 * gf / (ms_u * 1e-3) / 1e12, 2)
    c3["ffn_ft_overhead_pct"] = round((ms_p / ms_u - 1) * 100, 2)
    c3["ffn_detections"] = l1.report().detections + l2.report().detections
    out["c3"] = c3
    del x, y1
    c5 = []
    lp = FTTransformerLayer(1280, 20, 5120, protect=True, thr=thr, seed=1, device=dev)
    lu = FTTransformerLayer(1280, 20, 5120, protect=False, thr=thr, seed=1, device=dev)
    for seq in (512, 2048, 8192, 16384):
        bb = 16384 // seq
        xx = (torch.empty((bb, seq, 1280), device=dev).uniform_(-1, 1, generator=g)).half()
        ms_p = _time_cuda(lambda: lp(xx), iters=3)
        ms_u = _time_cuda(lambda: lu(xx), iters=3)
        fl = lp.flops(bb, seq)
        c5.append({"seq_len": seq, "batch": bb, "protected_tflops": round(fl / (ms_p * 1e-3) / 1e12, 2),
                   "unprotected_tflops": round(fl / (ms_u * 1e-3) / 1e12, 2),
                   "ft_overhead_pct": round((ms_p / ms_u - 1) * 100, 2), "ms": round(ms_p, 3)})
    out["c5_layer_sweep"] = c5
    out["c5_detections"] = lp.report().detections
    del lp, lu, xx
    torch.cuda.empty_cache()
    # EFTA-optimized vs the decoupled baseline (csrc/decoupled.cu: traditional two-sided block
    # ABFT around cuBLAS GEMMs, DMR softmax, N^2 intermediates in HBM) on the paper's Table 1 / 2
    # head configurations at 16K tokens
    dec = []
    for (b, h, s_, d) in ((8, 16, 2048, 64), (1, 16, 16384, 64), (2, 32, 8192, 128)):
        q = synth_inputs(31, (b, h, s_, d), dev)
        k = synth_inputs(32, (b, h, s_, d), dev)
        v = synth_inputs(33, (b, h, s_, d), dev)
        row = {"batch": b, "heads": h, "seq_len": s_, "head_dim": d}
        for mode, th in (("efta-opt", thr), ("decoupled", Thresholds(7e-6, 1e-3, 5e-3))):
            op = EftaAttention(b, h, s_, d, mode=mode, thr=th, device=dev)
            ms = _time_cuda(lambda: op(q, k, v), iters=3)
            row[f"{mode}_ms"] = round(ms, 3)
            row[f"{mode}_detections"] = op.report().detections
            del op
            torch.cuda.empty_cache()
        row["efta_opt_speedup"] = round(row["decoupled_ms"] / row["efta-opt_ms"], 2)
        dec.append(row)
        del q, k, v
    out["decoupled_vs_efta_opt"] = dec
    # causal (decoder) attention on the pair kernel, a non-goal of the reference (F4):
    # useful work = half of the square, 2*B*H*S^2*d FLOPs
    cz = {}
    b, h, s_, d = 4, 32, 8192, 128
    q = synth_inputs(41, (b, h, s_, d), dev)
    k = synth_inputs(42, (b, h, s_, d), dev)
    v = synth_inputs(43, (b, h, s_, d), dev)
    for mode in ("efta-opt", "none"):
        op = EftaAttention(b, h, s_, d, mode=mode, thr=thr, device=dev, causal=True)
        ms = _time_cuda(lambda: op(q, k, v), iters=3)
        cz[f"causal_{mode}_tflops"] = round(flops(b, h, s_, d) / 2 / (ms * 1e-3) / 1e12, 2)
        cz[f"causal_{mode}_detections"] = op.report().detections
        del op
    cz["shape"] = {"batch": b, "heads": h, "seq_len": s_, "head_dim": d}
    out["causal"] = cz
    del q, k, v
    # KV-cache decode (F4): one query row per head against C4-sized caches, the caches'
    # checksum operands encoded once (steady-state decode); HBM-bound, bytes = K + V (+ KC, VC)
    from paper_2504_02211_b200 import EftaDecode
    b, h, s_, d = 32, 32, 8192, 128
    qd = synth_inputs(51, (b, h, d), dev)
    kd = synth_inputs(52, (b, h, s_, d), dev)
    vd = synth_inputs(53, (b, h, s_, d), dev)
    dz = {"shape": {"batch": b, "heads": h, "cache_len": s_, "head_dim": d}}
    for mode in ("efta-opt", "none"):
        op = EftaDecode(b, h, s_, d, mode=mode, thr=thr, device=dev)
        op.encode(kd, vd)
        ms = _time_cuda(lambda: op(qd, kd, vd, cache_encoded=True), iters=10)
        kv = 2 * b * h * s_ * d * 2
        cs = (b * h * (s_ // 128) * 32 * d * 2 + b * h * s_ * 64 * 2) if mode == "efta-opt" else 0
        dz[f"decode_{mode}_ms"] = round(ms, 4)
        dz[f"decode_{mode}_gbps"] = round((kv + cs) / (ms * 1e-3) / 1e9, 1)
        dz[f"decode_{mode}_detections"] = op.report().detections
        del op
    out["decode"] = dz
    del qd, kd, vd
    return out


def synth_heads(seed, start, count, device):
    """Heads [start, start+count) of the global C4 problem: head i is U(-1,1) on the fp16 grid
    from its own generator (seed, i), so every sharding of the global (b, h) index reproduces
    the same per-head inputs (the union over ranks is the single-GPU problem)."""
    import torch
    x = torch.empty((count, S, D), dtype=torch.float16, device=device)
    g = torch.Generator(device=device)
    tmp = torch.empty((S, D), dtype=torch.float32, device=device)
    for i in range(count):
        g.manual_seed(seed * 1_000_003 + start + i)
        tmp.uniform_(-1.0, 1.0, generator=g)
        x[i].copy_(tmp)
    return x


def fault_parity_c2():
    """Checker leg (not timed): the C2 campaign's 240 seeded plans replayed through the fault-tap
    build of the pair kernel and the CPU reference with common thresholds (tests/fault_parity.py):
    records identical in {fired, outcome, events incl. row/col}, mismatches explained by margin."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from fault_parity import campaign_specs, common_thresholds, run_parity, summarize  # test infrastructure
    thr, _, _ = common_thresholds(512, 64)
    rows = run_parity(campaign_specs(20, 12, 512, 64, [0, 2, 6], seed=7), 512, 64, thr)
    sm = summarize(rows)
    return {k2: sm[k2] for k2 in ("records", "identical", "mismatched", "explained_by_margin", "unexplained",
                                  "marginal_band", "fired_oracle", "fired_gpu")}


def ours(args):
    import torch
    rank, world, local, pg = dist_init(args.gpus)
    from paper_2504_02211_b200 import EftaAttention, Thresholds
    from paper_2504_02211_b200 import _lib
    from paper_2504_02211_b200.shard import shard_units
    dev = torch.device("cuda", torch.cuda.current_device())
    # global C4 problem: B*H = 1024 independent heads, split contiguously over the ranks
    # (no collective on the data path): strong scaling
    sh = shard_units(B * H, world, rank)
    nh = sh.count
    shape = (1, nh, S, D)
    q = synth_heads(1, sh.start, nh, dev).view(shape)
    k = synth_heads(2, sh.start, nh, dev).view(shape)
    v = synth_heads(3, sh.start, nh, dev).view(shape)
    thr = Thresholds(1e-4, 1e-3, 1e-3)
    op = EftaAttention(1, nh, S, D, mode="efta-opt", thr=thr, device=dev)
    op_none = EftaAttention(1, nh, S, D, mode="none", thr=thr, device=dev)
    o = torch.empty(shape, dtype=torch.float32, device=dev)
    m = torch.empty(shape[:3], dtype=torch.float32, device=dev)
    l = torch.empty(shape[:3], dtype=torch.float32, device=dev)

    step = lambda: op(q, k, v, o, m, l)  # noqa: E731
    with ClockSampler(local) as clk:
        ms = time_steps(step, args.steps, args.warmup, pg)
    ms_max = max_over_ranks(pg, ms)
    rep = op.report()
    total_flops = flops(B, H, S, D)  # the whole job: every rank's heads together
    value = total_flops / (ms_max * 1e-3) / 1e12

    # unprotected kernel (same kernel, MODE=NONE) for the FT overhead
    ms_none = max_over_ranks(pg, time_steps(lambda: op_none(q, k, v, o, m, l), args.steps,
                                            args.warmup, pg))
    # attention kernel alone (checksum operands already encoded): the roofline leg
    op.desc.checksums_ready = 1
    ms_kern = max_over_ranks(pg, time_steps(step, args.steps, 1, pg))
    op.desc.checksums_ready = 0

    peaks = json.load(open(PEAKS_PATH)) if os.path.exists(PEAKS_PATH) else {}
    peak = peaks.get("bf16_tflops_sustained") or 1400.0
    peak_burst = peaks.get("bf16_tflops") or 1590.0
    achieved = flops(1, nh, S, D) / (ms_kern * 1e-3) / 1e12  # per GPU (its own heads)
    traffic = None
    if os.path.exists(TRAFFIC_PATH):
        try:
            traffic = json.load(open(TRAFFIC_PATH)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f16",
        "data": "synthetic: U(-1,1) rounded to fp16 (the reference Matrix::random distribution), "
                "generated on device per head (seeded by the global head index)",
        "config": {"workload": "C4 Llama-style attention B=32 H=32 S=8192 d_head=128 (global), "
                               "batch x head sharded over the GPUs (strong scaling)",
                   "batch": B, "heads": H, "seq_len": S, "head_dim": D, "global_batch": B,
                   "heads_per_gpu": nh, "mode": "efta-opt", "block": BLOCK, "stride": STRIDE,
                   "parallelism": f"bh-shard{world}",
                   "l2": "inputs (3 x 2.1 GB fp16 at N=1) larger than L2 (126 MB)"},
        "unprotected_tflops": round(total_flops / (ms_none * 1e-3) / 1e12, 2),
        "ft_overhead_pct": round((ms_max / ms_none - 1.0) * 100.0, 2),
        "roofline": {"bound": "tensor", "achieved": round(achieved, 2), "peak": peak,
                     "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                     "frac_of_burst": round(achieved / peak_burst, 4),
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (kernel timed in a "
                                    "multi-second back-to-back loop)" if peaks else "fallback",
                     "kernel": "efta_attn_pair_kernel<128, EFTA_OPT> (CTA pairs, two alternating row warpgroups)",
                     "kernel_ms": round(ms_kern, 4), "traffic": traffic},
        "clocks": clk.result(),
        "gpu_launches": 2 * args.steps,  # checksum-encode prepass + fused attention per step
        "false_detections_in_timed_run": rep.detections,
    }
    # ---- e2e through the host C-ABI (pinned host buffers, copies in the timed region)
    if not args.no_e2e:
        desc = _lib.AttnDesc(1, nh, S, D, BLOCK, STRIDE, 0.0, 2, thr.eps1, thr.eps2, thr.eps_lin,
                             0, 0.0, 0, 0)
        hq = q.cpu().pin_memory()
        hk = k.cpu().pin_memory()
        hv = v.cpu().pin_memory()
        ho = torch.empty(shape, dtype=torch.float32).pin_memory()
        hm = torch.empty(shape[:3], dtype=torch.float32).pin_memory()
        hl = torch.empty(shape[:3], dtype=torch.float32).pin_memory()
        cnt = _lib.Counters()

        def e2e_step():
            _lib.check(_lib.lib.efta_attn_fwd_host_f16(
                C.byref(desc), hq.data_ptr(), hk.data_ptr(), hv.data_ptr(), ho.data_ptr(),
                hm.data_ptr(), hl.data_ptr(), None, 0, None, 0, None, 0, C.byref(cnt)))
        e2e_steps = max(1, min(3, args.steps))
        e2e_step()
        barrier(pg)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        barrier(pg)
        dt = max_over_ranks(pg, (time.perf_counter() - t0) / e2e_steps)
        line["e2e"] = {"value": round(total_flops / dt / 1e12, 2), "unit": "TFLOP/s",
                       "h2d_bytes_per_step": world * 3 * q.numel() * 2,
                       "d2h_bytes_per_step": world * (o.numel() * 4 + 2 * m.numel() * 4),
                       "steps": e2e_steps,
                       "path": "efta_attn_fwd_host_f16 (C-ABI, host buffers, synchronous), per rank on its heads"}
    if rank == 0 and world == 1:
        if not args.no_campaign:
            try:
                st = fault_campaign()
                line["fault_coverage_pct"] = round(100.0 * st["coverage"], 2)
                line["fault_campaign"] = {k2: st[k2] for k2 in ("records", "fired", "corrected",
                                                              "masked_benign", "range_restricted",
                                                              "range_contract", "uncorrectable",
                                                              "false_alarms")}
                line["fault_campaign"]["kernel"] = ("efta_attn_pair_kernel<64, EFTA_OPT, INJ> (fault-tap build "
                                                    "of the production pair kernel), GPU-calibrated thresholds")
                line["fault_campaign"]["uncorrectable_note"] = (
                    "single-bit score upsets at |delta| ~ eps1 that linear repair cannot locate; the reference "
                    "marks the same records uncorrectable (fault_parity)")
            except Exception as ex:  # reported, never fatal for the perf line
                line["fault_coverage_pct"] = None
                line["fault_campaign"] = {"error": str(ex)[:200]}
            try:
                line["fault_parity"] = fault_parity_c2()
            except Exception as ex:
                line["fault_parity"] = {"error": str(ex)[:200]}
        if not args.no_suite:
            try:
                line["suite"] = suite(dev)
            except Exception as ex:  # reported, never fatal for the perf line
                line["suite"] = {"error": str(ex)[:200]}
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_ref()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


# ------------------------------------------------------------ reference arm
def reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ncpu = os.cpu_count() or 1
    # warm-up: untimed, small sample (loads the library, faults in pages)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    which = "ref" if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libefta_ref.so")) else "port"
    orc = Oracle(which)
    for _ in range(args.warmup):
        q, k, v, _ = orc.gen_trial(1, 256, D, BLOCK, STRIDE)
        orc.efta_forward(q, k, v, BLOCK, STRIDE, mode="efta-opt", thr=(1e-5, 1e-4, 1e-4))
    vals = []
    t0 = time.perf_counter()
    res = None
    for _ in range(args.steps):
        res = cpu_baseline_ref(threads=ncpu)
        vals.append(res["value"])
    wall = time.perf_counter() - t0
    v = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(wall / args.steps * 1e3, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: reference Rng + Matrix::random Q/K/V (fp16 grid)",
        "config": {"workload": "C4 Llama-style attention B=32 H=32 S=8192 d_head=128 (global; bounded "
                               "sample: one head per host thread per step)",
                   "batch": B, "heads": H, "seq_len": S, "head_dim": D, "global_batch": B,
                   "mode": "efta-opt", "block": BLOCK, "stride": STRIDE},
        "cpu_baseline": {"value": round(v, 6), "unit": "TFLOP/s", "cores": ncpu,
                         "kind": res["kind"], "sample": res["sample"]},
        "e2e": {"value": round(v, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        reference(a)
    else:
        ours(a)
