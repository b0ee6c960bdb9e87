"""Fused layouts of the FT-Transformer layer (not reference features): the
strided-ABFT GEMM's head-split epilogue (a QKV projection writes [3, batch, heads, seq, head_dim])
and the attention's fp16 token-major O ([batch, seq, heads, head_dim], the output projection's
input). Both are stores of the same values the plain layouts hold, so every check is bit for bit
against the plain layout permuted in torch — clean, with injected upsets (the correction lands at
the split position) and for every attention configuration the pair kernel serves."""
import numpy as np
import pytest

from helpers import head_inputs

pytestmark = pytest.mark.gpu


def _bits(t):
    import torch
    return t.contiguous().view(torch.int16 if t.dtype == torch.float16 else torch.int32)


def _split_ref(y, seq, heads, hd):
    m, n = y.shape
    return y.view(m // seq, seq, n // (heads * hd), heads, hd).permute(2, 0, 3, 1, 4)


@pytest.mark.parametrize("m,seq,heads,hd,n", [
    (1024, 512, 10, 128, 3840),   # QKV of a 1280-wide model, 128-dim heads (pair GEMM)
    (1024, 256, 20, 64, 3840),    # 64-dim heads, 4 heads per 256-wide tile
    (384, 128, 3, 128, 768),      # two parts, part boundary inside tile 1; single-CTA GEMM (m % 256)
    (512, 512, 4, 64, 768),
])
@pytest.mark.parametrize("fp32", [False, True])
def test_gemm_head_split_equals_plain_permuted(m, seq, heads, hd, n, fp32):
    import torch
    from paper_2504_02211_b200 import AbftLinear
    g = torch.Generator(device="cuda")
    g.manual_seed(m + n + hd)
    x = torch.empty((m, 1024), device="cuda").uniform_(-1, 1, generator=g).half()
    w = (torch.empty((n, 1024), device="cuda").uniform_(-1, 1, generator=g) / 32).half()
    lin = AbftLinear(w, eps=1e-2)
    y = lin(x, fp32_out=fp32)
    ys = lin(x, fp32_out=fp32, head_split=(seq, heads, hd))
    assert ys.shape == (n // (heads * hd), m // seq, heads, seq, hd)
    assert torch.equal(_bits(ys), _bits(_split_ref(y, seq, heads, hd)))
    assert lin.report().detections == 0


@pytest.mark.parametrize("m", [1024, 384])
def test_gemm_head_split_correction_lands_at_split_position(m):
    """Upsets in the accumulator (debug build): the located / corrected value is rewritten at its
    head-split address, so the split output equals the plain corrected output permuted."""
    import torch
    from paper_2504_02211_b200 import AbftLinear
    seq, heads, hd, n = 128, 3, 128, 768
    g = torch.Generator(device="cuda")
    g.manual_seed(77)
    x = torch.empty((m, 512), device="cuda").uniform_(-1, 1, generator=g).half()
    w = (torch.empty((n, 512), device="cuda").uniform_(-1, 1, generator=g) / 16).half()
    lin = AbftLinear(w, eps=1e-2, debug=True)
    clean = lin(x)
    faults = [(5, 3, 31), (130, 400, 30), (m - 1, 767, 29), (200, 384, 24)]
    lin.set_faults(faults)
    y = lin(x)
    r_plain = lin.report()
    ys = lin(x, head_split=(seq, heads, hd))
    r_split = lin.report()
    assert r_plain.detections > 0 and r_split.detections == r_plain.detections
    assert [(e["row"], e["col"], e["status"]) for e in sorted(r_split.events, key=lambda e: e["row"])] == \
           [(e["row"], e["col"], e["status"]) for e in sorted(r_plain.events, key=lambda e: e["row"])]
    corrected = {(e["row"], e["col"]) for e in r_plain.events if e["status"] == "corrected"}
    for r, c, _ in faults:  # a corrected upset leaves the clean value
        if (r, c) in corrected:
            assert torch.equal(_bits(y[r, c]), _bits(clean[r, c]))
    assert torch.equal(_bits(ys), _bits(_split_ref(y, seq, heads, hd)))


def test_gemm_head_split_validation():
    import torch
    from paper_2504_02211_b200 import AbftLinear, _lib
    w = torch.zeros((768, 256), device="cuda", dtype=torch.float16)
    lin = AbftLinear(w)
    x = torch.zeros((256, 256), device="cuda", dtype=torch.float16)
    for bad in ((100, 3, 128), (128, 5, 128), (128, 3, 0)):
        with pytest.raises(_lib.ConfigError):
            lin(x, head_split=bad)


def _dev(x):
    import torch
    return torch.from_numpy(x).to(torch.float16).cuda().contiguous()


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("mode", ["none", "efta-opt"])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("kv", [0, 2])
def test_attention_token_major_fp16_equals_fp32_permuted(d, mode, causal, kv):
    import torch
    from paper_2504_02211_b200 import EftaAttention, Thresholds
    b, h, s = 2, 4, 512
    hk = kv or h
    q, _, _, _ = head_inputs(4100 + d, b * h, s, d)
    _, k, v, _ = head_inputs(4200 + d, b * hk, s, d)
    qd, kd, vd = _dev(q).view(b, h, s, d), _dev(k).view(b, hk, s, d), _dev(v).view(b, hk, s, d)
    thr = Thresholds(1e-4, 1e-3, 1e-3)
    a = EftaAttention(b, h, s, d, mode=mode, thr=thr, kv_heads=hk, causal=causal)
    t = EftaAttention(b, h, s, d, mode=mode, thr=thr, kv_heads=hk, causal=causal, token_major_out=True)
    o, m, l = a(qd, kd, vd)
    o16, m16, l16 = t(qd, kd, vd)
    assert o16.dtype == torch.float16 and o16.shape == (b, s, h, d)
    assert torch.equal(_bits(o16), _bits(o.half().permute(0, 2, 1, 3)))
    assert torch.equal(m, m16) and torch.equal(l, l16)
    assert t.report().detections == 0


def test_attention_token_major_with_fault_taps():
    """The tap build (debug, EFTA-optimized) writes the same token-major output; an upset of a
    score is repaired identically in both layouts."""
    import torch
    from paper_2504_02211_b200 import EftaAttention, FaultSpec, Thresholds
    b, h, s, d = 1, 3, 512, 64
    q, k, v, _ = head_inputs(4300, b * h, s, d)
    qd, kd, vd = (_dev(x).view(b, h, s, d) for x in (q, k, v))
    thr = Thresholds(1e-4, 1e-3, 1e-3)
    f = [FaultSpec.parse("GEMM1_OUT:1:2:3:4:30", head=2)]
    outs = []
    for tok in (False, True):
        op = EftaAttention(b, h, s, d, mode="efta-opt", thr=thr, debug=True, token_major_out=tok)
        op.set_faults(f)
        o, _, _ = op(qd, kd, vd)
        r = op.report()
        assert r.fired and r.detections > 0 and not r.failed
        outs.append((o, [(e["kind"], e["status"], e["row"], e["col"]) for e in r.events]))
    assert outs[0][1] == outs[1][1]
    assert torch.equal(_bits(outs[1][0]), _bits(outs[0][0].half().permute(0, 2, 1, 3)))


def test_attention_token_major_validation():
    from paper_2504_02211_b200 import EftaAttention, Thresholds, _lib
    with pytest.raises(_lib.ConfigError):
        EftaAttention(1, 2, 384, 64, mode="efta-opt", token_major_out=True)   # odd block count
    with pytest.raises(_lib.ConfigError):
        EftaAttention(1, 2, 512, 64, mode="efta", token_major_out=True)       # per-iteration check mode
    with pytest.raises(_lib.ConfigError):
        EftaAttention(1, 2, 512, 64, mode="decoupled", token_major_out=True)
    with pytest.raises(_lib.ConfigError):
        EftaAttention(1, 2, 512, 64, mode="none", debug=True, thr=Thresholds(), token_major_out=True)


@pytest.mark.parametrize("m,n,k", [(1024, 1280, 1280), (384, 5120, 1280)])
@pytest.mark.parametrize("act", [None, "gelu"])
@pytest.mark.parametrize("resid", [False, True])
def test_gemm_fused_epilogues_equal_torch_elementwise(m, n, k, act, resid):
    """y = gelu(half(x W^T)) (+ r) from the epilogue equals the fp16 GEMM followed by torch's
    F.gelu / `+` on fp16 tensors, bit for bit."""
    import torch
    from paper_2504_02211_b200 import AbftLinear
    g = torch.Generator(device="cuda")
    g.manual_seed(m + n)
    x = torch.empty((m, k), device="cuda").uniform_(-1, 1, generator=g).half()
    w = (torch.empty((n, k), device="cuda").uniform_(-2, 2, generator=g) / 32).half()
    r = torch.empty((m, n), device="cuda").uniform_(-3, 3, generator=g).half() if resid else None
    lin = AbftLinear(w, eps=1e-2)
    y = lin(x)
    ref = torch.nn.functional.gelu(y) if act else y
    if resid:
        ref = r + ref
    yf = lin(x, residual=r, activation=act)
    assert torch.equal(_bits(yf), _bits(ref))
    assert lin.report().detections == 0


def test_gemm_fused_epilogue_on_corrected_values():
    """A corrected upset is rewritten through the same epilogue (debug build)."""
    import torch
    from paper_2504_02211_b200 import AbftLinear
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x = torch.empty((512, 512), device="cuda").uniform_(-1, 1, generator=g).half()
    w = (torch.empty((768, 512), device="cuda").uniform_(-1, 1, generator=g) / 16).half()
    r = torch.empty((512, 768), device="cuda").uniform_(-1, 1, generator=g).half()
    lin = AbftLinear(w, eps=1e-2, debug=True)
    ref = torch.nn.functional.gelu(lin(x)) + r
    lin.set_faults([(7, 300, 31), (300, 7, 30)])
    y = lin(x, residual=r, activation="gelu")
    rep = lin.report()
    assert rep.detections == 2 and all(e["status"] == "corrected" for e in rep.events), rep.events
    assert torch.equal(_bits(y), _bits(ref))


@pytest.mark.parametrize("protect", [True, False])
@pytest.mark.parametrize("s", [512, 384])
def test_layer_fused_layouts_bit_identical(protect, s):
    """The layer with the fused layouts (head-split QKV GEMM, token-major fp16 O, residual /
    GELU epilogues) returns exactly what the copy-based layer returns (S = 384: odd block count,
    the attention keeps its fp32 output and the layer its merge copy). The unprotected twin's
    fused form (cuBLAS beta = 1 residuals) rounds differently: within fp16 tolerance."""
    import torch
    from paper_2504_02211_b200 import FTTransformerLayer
    a = FTTransformerLayer(d_model=1280, n_heads=20, d_ff=5120, protect=protect, seed=4, fused_layout=True)
    c = FTTransformerLayer(d_model=1280, n_heads=20, d_ff=5120, protect=protect, seed=4, fused_layout=False)
    g = torch.Generator(device="cuda")
    g.manual_seed(s)
    x = torch.empty((2, s, 1280), device="cuda").uniform_(-1, 1, generator=g).half()
    ya, yc = a(x), c(x)
    if protect:
        assert torch.equal(_bits(ya), _bits(yc))
    else:
        assert (ya.float() - yc.float()).abs().max().item() <= 1e-2 * yc.float().abs().max().item()
    assert a.report().detections == 0
    assert a._attn[(2, s)].token_major_out == (s == 512)
    np.testing.assert_equal(ya.shape, (2, s, 1280))


@pytest.mark.parametrize("n", [16384 * 5120, 1000003, 7])
def test_gelu_pass_bit_identical_to_torch(n):
    """csrc/elementwise.cu's GELU (the layer's FFN activation) equals F.gelu on fp16 bit for bit,
    including the ragged tail, infinities, huge / tiny magnitudes and subnormals (NaN as NaN)."""
    import torch
    from paper_2504_02211_b200.ffn import gelu_
    g = torch.Generator(device="cuda")
    g.manual_seed(n)
    x = (torch.randn(n, device="cuda", generator=g) * 4).half()
    special = torch.tensor([float("inf"), float("-inf"), float("nan"), 65504.0, -65504.0, 6e-8, -6e-8,
                            1e-5, -1e-5, 0.0, -0.0, -9.5, 9.5], device="cuda").half()
    x[: min(n, special.numel())] = special[: min(n, special.numel())]
    ref = torch.nn.functional.gelu(x)
    y = gelu_(x.clone())
    nan = torch.isnan(ref)
    assert torch.equal(torch.isnan(y), nan)
    assert torch.equal(_bits(y)[~nan], _bits(ref)[~nan])
