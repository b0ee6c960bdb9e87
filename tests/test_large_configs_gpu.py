"""GPU parity at BASELINE.json's full sizes, on sampled units the CPU reference finishes in
seconds (heads and 128-row slabs are independent, src/campaign.cpp:175):

* C4 (B=32 H=32 S=8192 d=128, the bench workload): whole problem on the GPU, protected ==
  unprotected bit for bit, no false alarms; two heads (first and last) against the oracle;
* C3 attention (B=16 H=16 S=2048 d=64): eight heads sampled across the batch;
* the strided-ABFT FFN GEMMs at C3 (32768 x 1024 <-> 4096) and C5 (16384 x 1280 <-> 5120):
  sampled 128-row slabs x 256-wide output tiles against the reference's per-tile
  checksummed_gemm (product and checksum pair), then one upset per sampled tile located,
  reported and repaired like the reference's verify_locate_correct.
"""
import concurrent.futures as cf
import os

import numpy as np
import pytest

from helpers import oracle, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-2


def _uniform_half(shape, seed):
    import torch
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return torch.empty(shape, dtype=torch.float32, device="cuda").uniform_(-1.0, 1.0, generator=g).half()


def _oracle_heads(q, k, v, heads, mode="none"):
    orc = oracle()

    def one(h):
        return orc.efta_forward(q[h], k[h], v[h], 128, 8, mode=mode)

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(heads), os.cpu_count() or 1))) as ex:
        return dict(zip(heads, ex.map(one, heads)))


def test_c4_full_problem_parity():
    import torch
    from paper_2504_02211_b200 import EftaAttention, Thresholds
    b, h, s, d = 32, 32, 8192, 128
    q, k, v = (_uniform_half((b, h, s, d), 100 + i) for i in range(3))
    thr = Thresholds(1e-4, 1e-3, 1e-3)
    op = EftaAttention(b, h, s, d, mode="efta-opt", thr=thr)
    o, m, l = op(q, k, v)
    rep = op.report()
    assert rep.detections == 0 and not rep.failed, rep.events[:3]
    o_none, _, _ = EftaAttention(b, h, s, d, mode="none", thr=thr)(q, k, v)
    assert torch.equal(o.view(torch.int32), o_none.view(torch.int32))
    del o_none
    flat = (0, b * h - 1)
    qs = q.view(b * h, s, d)
    ks = k.view(b * h, s, d)
    vs = v.view(b * h, s, d)
    hq = {i: qs[i].float().cpu().numpy() for i in flat}
    hk = {i: ks[i].float().cpu().numpy() for i in flat}
    hv = {i: vs[i].float().cpu().numpy() for i in flat}
    refs = _oracle_heads(hq, hk, hv, list(flat))
    of, mf, lf = o.view(b * h, s, d), m.view(b * h, s), l.view(b * h, s)
    for i in flat:
        assert rel_err(of[i].cpu().numpy(), refs[i].o) <= TOL
        assert np.allclose(mf[i].cpu().numpy(), refs[i].m, rtol=1e-5, atol=1e-5)
        assert np.allclose(lf[i].cpu().numpy(), refs[i].l, rtol=1e-3)


def test_c3_attention_sampled_heads():
    from paper_2504_02211_b200 import EftaAttention, Thresholds
    b, h, s, d = 16, 16, 2048, 64
    q, k, v = (_uniform_half((b, h, s, d), 200 + i) for i in range(3))
    op = EftaAttention(b, h, s, d, mode="efta-opt", thr=Thresholds(1e-4, 1e-3, 1e-3))
    o, m, l = op(q, k, v)
    rep = op.report()
    assert rep.detections == 0 and not rep.failed
    heads = [0, 37, 66, 101, 130, 171, 200, 255]
    flat = lambda t: t.view(b * h, s, -1) if t.dim() == 4 else t.view(b * h, s)  # noqa: E731
    hq = {i: flat(q)[i].float().cpu().numpy() for i in heads}
    hk = {i: flat(k)[i].float().cpu().numpy() for i in heads}
    hv = {i: flat(v)[i].float().cpu().numpy() for i in heads}
    refs = _oracle_heads(hq, hk, hv, heads, mode="efta-opt")
    for i in heads:
        assert rel_err(flat(o)[i].cpu().numpy(), refs[i].o) <= TOL, i
        assert np.allclose(flat(m)[i].cpu().numpy(), refs[i].m, rtol=1e-5, atol=1e-5)
        assert np.allclose(flat(l)[i].cpu().numpy(), refs[i].l, rtol=1e-3)


FFN_SHAPES = [("c3_up", 32768, 1024, 4096), ("c3_down", 32768, 4096, 1024),
              ("c5_up", 16384, 1280, 5120), ("c5_down", 16384, 5120, 1280)]


@pytest.mark.parametrize("name,m,k,n", FFN_SHAPES)
def test_ffn_gemm_sampled_slabs(name, m, k, n):
    import torch
    from paper_2504_02211_b200.ffn import AbftLinear
    orc = oracle()
    x = _uniform_half((m, k), 300 + n)
    w = (_uniform_half((n, k), 400 + k).float() / np.sqrt(k)).half()
    lin = AbftLinear(w, eps=1e-2)
    cs = torch.empty((m, n // 256, 16), dtype=torch.float32, device="cuda")
    y = lin(x, fp32_out=True, checksums=cs)
    rep = lin.report()
    assert rep.detections == 0 and not rep.failed
    rng = np.random.default_rng(m + n + k)
    slabs = sorted(int(s) for s in rng.choice(m // 128, 2, replace=False))
    tiles = sorted(int(t) for t in rng.choice(n // 256, 2, replace=False))
    wn = w.float().cpu().numpy()
    xs = {s: x[s * 128:(s + 1) * 128].float().cpu().numpy() for s in slabs}
    jobs = [(s, t) for s in slabs for t in tiles]

    def one(st):
        s, t = st
        return orc.checksummed_gemm(xs[s], wn[t * 256:(t + 1) * 256].T.copy(), 8)

    with cf.ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        refs = dict(zip(jobs, ex.map(one, jobs)))
    y_np, cs_np = {}, {}
    worst = 0.0
    for (s, t), (c, c1, c2) in refs.items():
        yt = y[s * 128:(s + 1) * 128, t * 256:(t + 1) * 256].cpu().numpy()
        ct = cs[s * 128:(s + 1) * 128, t].cpu().numpy()
        # fp32 accumulation over K in a different order than the reference's k loop
        tol = 1e-5 * max(1.0, k / 1024)
        assert rel_err(yt, c) <= tol, (name, s, t, rel_err(yt, c))
        assert rel_err(ct[:, :8], c1) <= tol and rel_err(ct[:, 8:], c2) <= tol
        # the GPU's checksums verify the GPU product cleanly; residual sets the threshold below
        r = orc.verify_locate_correct(yt.copy(), ct[:, :8].copy(), ct[:, 8:].copy(), np.inf)
        worst = max(worst, r["residual"])
        y_np[(s, t)], cs_np[(s, t)] = yt, ct
    eps = max(8.0 * worst, 1e-6)
    # one upset per sampled tile: GPU (in-epilogue verify) vs the reference's verify on the same data
    faults = []
    for (s, t) in jobs:
        faults.append((s * 128 + int(rng.integers(0, 128)), t * 256 + int(rng.integers(0, 256)),
                       int(rng.choice([31, 30, 29, 22, 21, 18]))))
    dbg = AbftLinear(w, eps=eps, debug=True)
    dbg.set_faults(faults)
    y2 = dbg(x, fp32_out=True)
    rep2 = dbg.report()
    for (r, c, bit), (s, t) in zip(faults, jobs):
        ref_t = y_np[(s, t)].copy()
        ref_t[r - s * 128, c - t * 256] = orc.flip_bit(float(ref_t[r - s * 128, c - t * 256]), 32, bit)
        ro = orc.verify_locate_correct(ref_t, cs_np[(s, t)][:, :8].copy(), cs_np[(s, t)][:, 8:].copy(), eps)
        ev = [e for e in rep2.events if e["m_tile"] == s and e["n_tile"] == t]
        if ro["status"] == "clean":
            assert not ev, (name, r, c, bit, ev)
            continue
        assert len(ev) == 1, (name, r, c, bit, ev)
        e = ev[0]
        assert (e["status"], e["row"] - s * 128 if e["row"] >= 0 else -1, e["col"] - t * 256 if e["col"] >= 0 else -1,
                e["corrections"]) == (ro["status"], ro["row"], ro["col"], ro["corrections"]), (e, ro)
        got = y2[s * 128:(s + 1) * 128, t * 256:(t + 1) * 256].cpu().numpy()
        assert np.array_equal(got.view(np.uint32), ref_t.view(np.uint32)), (name, r, c, bit)
