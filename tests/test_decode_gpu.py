"""KV-cache decode (csrc/decode.cu, a non-goal of the reference): one query
row per head against the K / V caches. efta_forward's query rows are independent, so a decode step
equals row 0 of the oracle's efta_forward(Q, K, V) with the decode query as Q's row 0 (the oracle
is pinned bit-exact to the reference): same O row within the north_star tolerance, the same m and
l, no events on clean inputs; upsets of the cached K after its checksums were encoded are detected
and repaired by the reference ladder on the row."""
import numpy as np
import pytest

from helpers import head_inputs, oracle, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-2


def _dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.float16).cuda().contiguous()


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("seq", [512, 1024])
@pytest.mark.parametrize("mode", ["none", "efta-opt"])
def test_decode_matches_oracle_row(d, seq, mode):
    from paper_2504_02211_b200 import Thresholds, efta_decode
    heads = 4
    q, k, v, _ = head_inputs(4100 + d + seq, heads, seq, d)
    qd = q[:, 5, :]  # the decode query: row 5 of each head's Q
    o, rep = efta_decode(_dev(qd), _dev(k), _dev(v), mode=mode, thr=Thresholds(1e-4, 1e-3, 1e-3))
    o = o.cpu().numpy()[0]
    m = rep.final_m.cpu().numpy()[0]
    l = rep.final_l.cpu().numpy()[0]
    orc = oracle()
    for h in range(heads):
        qq = q[h].copy()
        qq[0] = qd[h]
        ref = orc.efta_forward(qq, k[h], v[h], 128, 8, mode="none")
        assert rel_err(o[h], ref.o[0]) <= TOL, (h, rel_err(o[h], ref.o[0]))
        assert abs(m[h] - ref.m[0]) <= 1e-5 * max(1.0, abs(ref.m[0]))
        assert abs(l[h] - ref.l[0]) <= 1e-3 * ref.l[0]
    assert rep.detections == 0 and not rep.failed, rep.events[:4]


def test_decode_gqa_and_protected_equals_unprotected():
    """Grouped-query decode (8 query heads over 2 cache heads); EFTA-optimized and NONE give the
    same output bit for bit (the checks only read side-band values)."""
    from paper_2504_02211_b200 import Thresholds, efta_decode
    seq, d, h, hkv = 1024, 128, 8, 2
    q, _, _, _ = head_inputs(4200, h, seq, d)
    _, k, v, _ = head_inputs(4201, hkv, seq, d)
    qd = q[:, 0, :]
    o0, _ = efta_decode(_dev(qd), _dev(k), _dev(v), mode="none")
    o1, r1 = efta_decode(_dev(qd), _dev(k), _dev(v), mode="efta-opt", thr=Thresholds(1e-4, 1e-3, 1e-3))
    a0, a1 = o0.cpu().numpy()[0], o1.cpu().numpy()[0]
    assert np.array_equal(a0.view(np.uint32), a1.view(np.uint32))
    assert r1.detections == 0
    orc = oracle()
    for i in range(h):
        qq = q[i].copy()
        ref = orc.efta_forward(qq, k[i // (h // hkv)], v[i // (h // hkv)], 128, 8, mode="none")
        assert rel_err(a1[i], ref.o[0]) <= TOL


@pytest.mark.parametrize("d", [64, 128])
def test_decode_repairs_corrupted_cache_row(d):
    """A cached key (block 2, key 37 of head 1) is corrupted after its checksum operands were
    encoded (a memory upset in the cache): the block's exp-stage check fires, the linear repair
    restores the score and the row is recomputed; the output equals the clean decode."""
    import torch
    from paper_2504_02211_b200 import EftaDecode, Thresholds
    seq, heads = 1024, 2
    q, k, v, _ = head_inputs(4300 + d, heads, seq, d)
    qd, kd, vd = _dev(q[:, 3, :])[None], _dev(k)[None], _dev(v)[None]
    op = EftaDecode(1, heads, seq, d, mode="efta-opt", thr=Thresholds(1e-4, 1e-3, 1e-3))
    clean, _, _ = op(qd, kd, vd)
    clean = clean.cpu().numpy()[0]
    assert op.report().detections == 0
    op.encode(kd, vd)
    kd[0, 1, 2 * 128 + 37, :] = kd[0, 1, 2 * 128 + 37, :] * 3 + 1
    o, _, _ = op(qd, kd, vd, cache_encoded=True)
    rep = op.report()
    torch.cuda.synchronize()
    assert rep.detections > 0 and not rep.failed, rep.events
    assert {(e["kind"], e["head"], e["block_j"]) for e in rep.events} == {("exp_checksum", 1, 2)}
    assert rel_err(o.cpu().numpy()[0], clean) <= TOL


def test_decode_long_cache_no_false_alarms():
    """B=2, H=32, cache 8192 x 128 (a C4-sized decode step): no check fires; spot heads vs float64."""
    import torch
    from paper_2504_02211_b200 import Thresholds, efta_decode
    b, h, s, d = 2, 32, 8192, 128
    g = torch.Generator(device="cuda")
    g.manual_seed(23)
    q = torch.empty(b, h, d, device="cuda").uniform_(-1, 1, generator=g).half()
    k = torch.empty(b, h, s, d, device="cuda").uniform_(-1, 1, generator=g).half()
    v = torch.empty(b, h, s, d, device="cuda").uniform_(-1, 1, generator=g).half()
    o, rep = efta_decode(q, k, v, mode="efta-opt", thr=Thresholds(1e-4, 1e-3, 1e-3))
    assert rep.detections == 0 and not rep.failed, rep.events[:4]
    o = o.cpu().numpy()
    for bi, hi in ((0, 0), (1, 31)):
        qq = q[bi, hi].float().cpu().numpy().astype(np.float64)
        kk = k[bi, hi].float().cpu().numpy().astype(np.float64)
        vv = v[bi, hi].float().cpu().numpy().astype(np.float64)
        sc = kk @ qq / np.sqrt(d)
        p = np.exp(sc - sc.max())
        ref = p @ vv / p.sum()
        assert np.abs(o[bi, hi] - ref).max() <= TOL * np.abs(ref).max()
