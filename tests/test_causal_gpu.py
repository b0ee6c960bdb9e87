"""Causal (decoder) attention on the CTA-pair kernel (a non-goal of the
reference, so there is no reference run to be in parity with): key k is visible to
query q iff k <= q. Checked against a float64 causal softmax attention of the same fp16 inputs
(max-rel-err <= 1e-2, the north_star tolerance), protected == unprotected bit for bit, and the
recovery ladder of the masked diagonal blocks (exp-stage check on each group's visible cells)
repairing upsets of the score operand."""
import os

import numpy as np
import pytest

from helpers import head_inputs, rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _dev(x):
    import torch
    return torch.from_numpy(x).to(torch.float16).cuda().contiguous()


def causal_reference(q, k, v):
    """float64 causal attention of one head (inputs already on the fp16 grid)."""
    n, d = q.shape
    s = (q.astype(np.float64) @ k.astype(np.float64).T) / np.sqrt(d)
    s[np.triu_indices(n, 1)] = -np.inf
    m = s.max(axis=1, keepdims=True)
    p = np.exp(s - m)
    l = p.sum(axis=1, keepdims=True)
    return (p @ v.astype(np.float64)) / l, m[:, 0], l[:, 0]


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("seq", [256, 512, 2048])
@pytest.mark.parametrize("mode", ["none", "efta-opt"])
def test_causal_matches_float64_reference(d, seq, mode):
    from paper_2504_02211_b200 import Thresholds, efta_forward
    heads = 3
    q, k, v, _ = head_inputs(3100 + d + seq, heads, seq, d)
    o, rep = efta_forward(_dev(q), _dev(k), _dev(v), mode=mode, thr=Thresholds(1e-4, 1e-3, 1e-3), causal=True)
    o = o.cpu().numpy()
    m = rep.final_m.cpu().numpy()
    l = rep.final_l.cpu().numpy()
    for h in range(heads):
        ro, rm, rl = causal_reference(q[h], k[h], v[h])
        assert rel_err(o[h], ro) <= TOL, (h, rel_err(o[h], ro))
        assert np.allclose(m[h], rm, rtol=1e-5, atol=1e-5)
        assert np.allclose(l[h], rl, rtol=2e-3)
    assert rep.detections == 0 and not rep.failed, rep.events[:4]


@pytest.mark.parametrize("d", [64, 128])
def test_causal_protected_bit_identical_and_many_tiles(d):
    """EFTA-optimized == NONE bit for bit on the causal schedule (variable-length tiles handed out
    longest first), over enough heads that every cluster runs several tiles of unequal length."""
    from paper_2504_02211_b200 import Thresholds, efta_forward
    heads, seq = 160, 1024
    q, k, v, _ = head_inputs(3300 + d, heads, seq, d)
    o0, _ = efta_forward(_dev(q), _dev(k), _dev(v), mode="none", causal=True)
    o1, r1 = efta_forward(_dev(q), _dev(k), _dev(v), mode="efta-opt", thr=Thresholds(1e-4, 1e-3, 1e-3),
                          causal=True)
    a0, a1 = o0.cpu().numpy(), o1.cpu().numpy()
    assert np.array_equal(a0.view(np.uint32), a1.view(np.uint32))
    assert r1.detections == 0
    for h in (0, 77, 159):
        ro, _, _ = causal_reference(q[h], k[h], v[h])
        assert rel_err(a1[h], ro) <= TOL


def _corrupted(d, target, causal, q, k, v):
    import torch
    from paper_2504_02211_b200 import EftaAttention, Thresholds
    heads, seq = q.shape[0], q.shape[1]
    op = EftaAttention(1, heads, seq, d, mode="efta-opt", thr=Thresholds(1e-4, 1e-3, 1e-3), causal=causal)
    qd, kd, vd = _dev(q)[None], _dev(k)[None], _dev(v)[None]
    op(qd, kd, vd)  # encodes the checksum operands into the workspace
    torch.cuda.synchronize()
    n = seq // 128
    if target == "kc":
        kc = op.workspace[: heads * n * 32 * d * 2].view(torch.float16).view(heads * n * 32, d)
        row = (1 * n + 1) * 32 + 3  # c1_hi of group x = 3, key block 1, head 1
        kc[row, 5] = kc[row, 5] * 4 + 8
    else:
        kd[0, 1, 128 + 37, :] = kd[0, 1, 128 + 37, :] * 3 + 2
    op.desc.checksums_ready = 1
    o, m, l = op(qd, kd, vd)
    return o.cpu().numpy()[0], op.report()


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("target", ["kc", "k"])
def test_causal_recovery_ladder_matches_full_attention_ladder(d, target):
    """An upset in the score operand after the checksum prepass: a checksum row of key block 1
    (kc) or key 165 itself (k; its scores become the row max of many rows, so the ladder also
    repairs the running max). Block 1 is fully masked for query tile 0, the diagonal block of
    tile 1 and fully visible for tiles 2 and 3. Every affected tile is detected; tiles 2 and 3
    take exactly the decisions of the non-causal kernel on the same upset (same events incl.
    row / col); tiles 0 and 1 are repaired through the masked-block check (c1 minus the masked
    scores); every tile not declared uncorrectable equals the causal attention of the clean
    inputs."""
    heads, seq = 2, 512
    q, k, v, _ = head_inputs(3500 + d, heads, seq, d)
    oc, rc = _corrupted(d, target, True, q, k, v)
    on, rn = _corrupted(d, target, False, q, k, v)
    key = lambda e: (e["kind"], e["head"], e["block_i"], e["block_j"], e["status"], e["row"], e["col"])  # noqa: E731
    assert rc.detections > 0 and {e["head"] for e in rc.events} == {1}, rc.events[:6]
    assert sorted(key(e) for e in rc.events if e["block_i"] >= 2) == \
           sorted(key(e) for e in rn.events if e["block_i"] >= 2)
    low = [e for e in rc.events if e["block_i"] < 2]
    assert low and all(e["status"] == "corrected" for e in low) or target == "kc", low
    bad_tiles = {e["block_i"] for e in rc.events if e["status"] != "corrected"}
    for h in range(heads):
        ro, _, _ = causal_reference(q[h], k[h], v[h])
        for t in range(seq // 128):
            if h == 1 and t in bad_tiles:
                continue
            rows = slice(128 * t, 128 * t + 128)
            assert rel_err(oc[h][rows], ro[rows]) <= TOL, (h, t)


def test_causal_validation():
    from paper_2504_02211_b200 import EftaAttention, Thresholds, _lib
    with pytest.raises(_lib.ConfigError):
        EftaAttention(1, 2, 384, 64, mode="efta-opt", causal=True)  # odd block count
    with pytest.raises(_lib.ConfigError):
        EftaAttention(1, 2, 512, 64, mode="efta", causal=True)      # per-iteration check mode
    with pytest.raises(_lib.ConfigError):
        EftaAttention(1, 2, 512, 64, mode="efta-opt", debug=True, thr=Thresholds(), causal=True)


def test_causal_long_sequence_no_false_alarms():
    """S = 8192, d = 128, 32 heads (the bench's causal shape per batch entry): no check fires on
    clean inputs — in particular the rowsum range check on the rows with a single visible key —
    and sampled rows match float64 causal attention."""
    import torch
    from paper_2504_02211_b200 import Thresholds, efta_forward
    heads, seq, d = 32, 8192, 128
    g = torch.Generator(device="cuda")
    g.manual_seed(17)
    q, k, v = (torch.empty(heads, seq, d, device="cuda").uniform_(-1, 1, generator=g).half() for _ in range(3))
    o, rep = efta_forward(q, k, v, mode="efta-opt", thr=Thresholds(1e-4, 1e-3, 1e-3), causal=True)
    assert rep.detections == 0 and not rep.failed, rep.events[:4]
    o = o.cpu().numpy()
    qn, kn, vn = (x.float().cpu().numpy().astype(np.float64) for x in (q, k, v))
    for h in (0, 31):
        for r in (0, 1, 127, 128, 4095, 8191):
            s = qn[h, r] @ kn[h, : r + 1].T / np.sqrt(d)
            p = np.exp(s - s.max())
            ref = p @ vn[h, : r + 1] / p.sum()
            assert np.abs(o[h, r] - ref).max() <= TOL * max(np.abs(ref).max(), 1e-3), (h, r)
