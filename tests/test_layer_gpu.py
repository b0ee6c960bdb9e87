"""GPU tests of the FT-Transformer layer: every linear module through the
strided-ABFT tcgen05 GEMM + EFTA attention, against an fp32 torch restatement of the same
layer, and clean (no detections) at GPT-2-large shapes."""
import math

import pytest

pytestmark = pytest.mark.gpu


def _ref_layer(layer, x):
    import torch
    b, s, d = x.shape
    w = {k: v.float() for k, v in layer.w.items()}
    x2 = x.float().reshape(b * s, d)
    qkv = (x2 @ w["qkv"].t()).half().float()
    qkv = qkv.view(b, s, 3, layer.n_heads, layer.head_dim).permute(2, 0, 3, 1, 4)
    q, k, v = qkv[0], qkv[1], qkv[2]
    att = torch.softmax((q @ k.transpose(-1, -2)) / math.sqrt(layer.head_dim), dim=-1) @ v
    o = att.permute(0, 2, 1, 3).reshape(b * s, d).half().float()
    h = x2 + (o @ w["o"].t()).half().float()
    f1 = torch.nn.functional.gelu((h.half().float() @ w["ff1"].t()).half().float())
    f = (f1.half().float() @ w["ff2"].t()).half().float()
    return (h + f).view(b, s, d)


@pytest.mark.parametrize("protect", [True, False])
def test_layer_matches_fp32_reference(protect):
    import torch
    from paper_2504_02211_b200 import FTTransformerLayer
    layer = FTTransformerLayer(d_model=1280, n_heads=20, d_ff=5120, protect=protect, seed=3)
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x = torch.empty((2, 512, 1280), device="cuda").uniform_(-1, 1, generator=g).half()
    y = layer(x).float()
    ref = _ref_layer(layer, x)
    err = (y - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-2, err
    rep = layer.report()
    assert rep.detections == 0 and not rep.failed, rep.events[:3]


def test_layer_protected_equals_unprotected_within_rounding():
    import torch
    from paper_2504_02211_b200 import FTTransformerLayer
    lp = FTTransformerLayer(d_model=1280, n_heads=20, d_ff=5120, protect=True, seed=9)
    lu = FTTransformerLayer(d_model=1280, n_heads=20, d_ff=5120, protect=False, seed=9)
    x = torch.empty((1, 1024, 1280), device="cuda").uniform_(-1, 1).half()
    a, b = lp(x).float(), lu(x).float()
    assert (a - b).abs().max().item() <= 1e-2 * b.abs().max().item()
