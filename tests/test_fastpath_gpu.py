"""GPU tests of the fast (production) attention path beyond clean parity:

* the chunked, three-stream host entry point (efta_attn_fwd_host_f16, the reference-facing
  e2e call) reproduces the device entry point bit for bit;
* the rare recovery ladder of the CTA-pair kernel (alternating row warpgroups, c1-only score MMA,
  c2 on the CUDA cores) takes the same decisions as the single-CTA kernel when a checksum
  operand is corrupted in the workspace (a "natural" upset the tap variant cannot model).
"""
import ctypes as C
import os

import numpy as np
import pytest

from helpers import head_inputs

pytestmark = pytest.mark.gpu


def _dev(x):
    import torch
    return torch.from_numpy(x).to(torch.float16).cuda().contiguous()


@pytest.mark.parametrize("d,seq,heads", [(64, 512, 16), (128, 512, 6), (64, 256, 33)])
def test_host_path_chunked_matches_device(d, seq, heads):
    """(33 heads: chunks of 2 heads, 17 chunks used of the 32 allowed — every chunk's counters
    are merged, none read back uninitialised)"""
    import torch
    from paper_2504_02211_b200 import EftaAttention, Thresholds, _lib
    q, k, v, _ = head_inputs(4242 + d, heads, seq, d)
    thr = Thresholds(1e-4, 1e-3, 1e-3)
    op = EftaAttention(1, heads, seq, d, mode="efta-opt", thr=thr)
    o, m, l = op(_dev(q)[None], _dev(k)[None], _dev(v)[None])
    torch.cuda.synchronize()
    hq, hk, hv = (np.ascontiguousarray(x.astype(np.float16)) for x in (q, k, v))
    ho = np.empty((heads, seq, d), np.float32)
    hm = np.empty((heads, seq), np.float32)
    hl = np.empty((heads, seq), np.float32)
    desc = _lib.AttnDesc(1, heads, seq, d, 128, 8, 0.0, 2, thr.eps1, thr.eps2, thr.eps_lin, 0, 0.0, 0, 0)
    cnt = _lib.Counters()
    ev = (_lib.Event * 64)()
    _lib.check(_lib.lib.efta_attn_fwd_host_f16(
        C.byref(desc), hq.ctypes.data, hk.ctypes.data, hv.ctypes.data, ho.ctypes.data, hm.ctypes.data,
        hl.ctypes.data, None, 0, C.addressof(ev), 64, None, 0, C.byref(cnt)))
    assert np.array_equal(ho.view(np.uint32), o.cpu().numpy()[0].view(np.uint32))
    assert np.array_equal(hm, m.cpu().numpy()[0]) and np.array_equal(hl, l.cpu().numpy()[0])
    assert cnt.detections == 0 and cnt.failed == 0


def _corrupted_run(q, k, v, d, seq, heads, pair, target="kc"):
    import torch
    from paper_2504_02211_b200 import EftaAttention, Thresholds
    old = os.environ.pop("EFTA_NO_PAIR", None)
    if not pair:
        os.environ["EFTA_NO_PAIR"] = "1"
    try:
        op = EftaAttention(1, heads, seq, d, mode="efta-opt", thr=Thresholds(1e-4, 1e-3, 1e-3))
        qd, kd, vd = _dev(q)[None], _dev(k)[None], _dev(v)[None]
        op(qd, kd, vd)  # encodes the checksum operands into the workspace
        torch.cuda.synchronize()
        n = seq // 128
        if target == "kc":
            kc = op.workspace[: heads * n * 32 * d * 2].view(torch.float16).view(heads * n * 32, d)
            # c1_hi of group x=3, block j=1 of head 1: an upset in the checksum operand itself
            row = (1 * n + 1) * 32 + 3
            kc[row, 5] = kc[row, 5] * 4 + 8
        else:
            # an upset in K itself after encoding (key 1*128+37 of head 1): the score column
            # of that key is wrong in every query row and is the new row max of many rows, so
            # the recovery ladder repairs the running max (exercises the max-chain revision
            # of the alternating row-warpgroup schedule)
            kd[0, 1, 128 + 37, :] = kd[0, 1, 128 + 37, :] * 3 + 2
        op.desc.checksums_ready = 1
        o, m, l = op(qd, kd, vd)
        rep = op.report()
        return o.cpu().numpy()[0], rep
    finally:
        os.environ.pop("EFTA_NO_PAIR", None)
        if old is not None:
            os.environ["EFTA_NO_PAIR"] = old


@pytest.mark.parametrize("d,target", [(64, "kc"), (128, "kc"), (64, "k"), (128, "k")])
def test_pair_rare_ladder_matches_single_cta(d, target):
    seq, heads = 512, 2
    q, k, v, _ = head_inputs(99 + d, heads, seq, d)
    o_p, r_p = _corrupted_run(q, k, v, d, seq, heads, pair=True, target=target)
    o_s, r_s = _corrupted_run(q, k, v, d, seq, heads, pair=False, target=target)
    key = lambda e: (e["kind"], e["head"], e["block_i"], e["block_j"], e["status"], e["row"], e["col"])  # noqa: E731
    ev_p = sorted(key(e) for e in r_p.events)
    ev_s = sorted(key(e) for e in r_s.events)
    assert ev_p, "the corrupted checksum operand must be detected"
    assert all(e[1] == 1 and e[3] == 1 for e in ev_p), ev_p
    assert ev_p == ev_s, (ev_p, ev_s)
    assert r_p.detections == r_s.detections and r_p.failed == r_s.failed
    # both schedules repair the same cells: the outputs agree to accumulation-order noise
    assert np.abs(o_p - o_s).max() <= 2e-3 * np.abs(o_s).max()
