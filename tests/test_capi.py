"""CPU: the C-ABI library loads, exports every symbol include/efta_b200.h declares,
validates like the reference's AttnConfig, and its host-side helpers (reference
Rng / Matrix::random / sample_random_plan / classify_trial) agree with the oracle.
No compute calls (no GPU here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from helpers import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("efta_b200.h",):
        txt = open(os.path.join(ROOT, "include", h)).read()
        names |= set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?(efta_[a-z0-9_]+)\s*\(", txt, re.M))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    from paper_2504_02211_b200 import _lib
    decl = _declared()
    assert len(decl) >= 10
    missing = [n for n in decl if not hasattr(_lib.lib, n)]
    assert not missing, missing


def _desc(**kw):
    from paper_2504_02211_b200 import _lib
    d = dict(batch=1, heads=12, seq_len=512, head_dim=64, block=128, stride=8, scale=0.0, mode=2,
             eps1=7e-6, eps2=0.48, eps_lin=0.48, observe_linear=0, rowmax_bias=0.0, debug=0,
             checksums_ready=0, kv_heads=0, causal=0, o_token_major=0)
    d.update(kw)
    return _lib.AttnDesc(**d)


@pytest.mark.parametrize("kw,ok,msg", [
    ({}, True, ""),
    (dict(seq_len=500), False, "block must divide seq_len"),   # config.hpp:33-35
    (dict(stride=0), False, "dimensions must be positive"),     # config.hpp:31-32
    (dict(block=96, seq_len=480), False, "stride must divide block"),  # 96 % 8 == 0 -> geometry
    (dict(head_dim=60), False, "stride must divide head_dim"),  # config.hpp:37-38
    (dict(head_dim=96), False, "head_dim must be 64 or 128"),
    (dict(mode=3), True, ""),                                  # DECOUPLED baseline (csrc/decoupled.cu)
    (dict(mode=4), False, "unsupported mode"),
    (dict(kv_heads=4), True, ""),                              # grouped-query attention (F4)
    (dict(kv_heads=5), False, "kv_heads must divide heads"),
    (dict(causal=1), True, ""),                                # causal pair kernel (F4)
    (dict(causal=1, mode=1), False, "causal attention runs in modes"),
    (dict(causal=1, debug=1), False, "causal attention has no fault-tap build"),
    (dict(causal=1, seq_len=384), False, "causal attention needs an even number"),
    (dict(o_token_major=1), True, ""),                         # fp16 token-major O (layer fusion)
    (dict(o_token_major=1, causal=1, kv_heads=4, mode=0), True, ""),
    (dict(o_token_major=1, mode=1), False, "token-major fp16 output runs in modes"),
    (dict(o_token_major=1, mode=3), False, "token-major fp16 output runs in modes"),
    (dict(o_token_major=1, seq_len=384), False, "token-major fp16 output needs an even number"),
    (dict(o_token_major=1, mode=0, debug=1), False, "token-major fp16 output's tap build"),
    (dict(o_token_major=2), False, "o_token_major must be 0 or 1"),
])
def test_validate_mirrors_attnconfig(kw, ok, msg):
    from paper_2504_02211_b200 import _lib
    d = _desc(**kw)
    rc = _lib.lib.efta_attn_validate(C.byref(d))
    assert (rc == 0) == ok
    if ok:
        assert _lib.lib.efta_attn_workspace_bytes(C.byref(d)) > 0
    if not ok:
        assert rc == 1
        err = _lib.last_error()
        assert msg.split()[0] in err or msg in err or "block must be 128" in err, err


def test_workspace_size():
    from paper_2504_02211_b200 import _lib
    d = _desc()
    ws = _lib.lib.efta_attn_workspace_bytes(C.byref(d))
    al = lambda x: (x + 255) // 256 * 256  # noqa: E731
    kc = al(12 * 4 * 32 * 64 * 2)
    r2 = al(max(12 * 4 * 128 * 64, 12 * 4 * (64 + 32) * 128) * 2)
    # + the persistent kernel's tile counter + the decode path's split-KV partials: 12 rows x
    # splits x (m, l, lb, O[64], O.c[16]) fp32, splits = min(ceil(4 * SMs / 12), 4 / 2) = 2
    part = al(12 * 2 * (3 + 64 + 16) * 4)
    assert ws == kc + r2 + 256 + part


def test_python_mirror_raises_config_error():
    from paper_2504_02211_b200 import ConfigError, EftaAttention, FaultSpec, validate_plan
    with pytest.raises(ConfigError):
        EftaAttention(1, 1, 500, 64, device="cpu")
    with pytest.raises(ConfigError):
        FaultSpec.parse("BOGUS:0:0:0:0:1")
    with pytest.raises(ConfigError):
        FaultSpec.parse("GEMM1_OUT:0:0:0:0")
    f = FaultSpec.parse("EXP_OUT:2:3:7:11:30:2")
    assert f.to_string() == "EXP_OUT:2:3:7:11:30:2"
    g = FaultSpec.parse("EXP_OUT:1:1:2:3:31")
    assert g.trigger == 1 and g.to_string() == "EXP_OUT:1:1:2:3:31"
    validate_plan([g], 512, 64, 128, 1)
    with pytest.raises(ConfigError):  # two faults in one detection cycle (fault.cpp:117-119)
        validate_plan([g, FaultSpec.parse("GEMM1_OUT:1:0:0:0:3")], 512, 64, 128, 1)
    with pytest.raises(ConfigError):  # NORMALIZE_OUT is post-loop: block_j must be 0
        validate_plan([FaultSpec.parse("NORMALIZE_OUT:0:1:0:0:3")], 512, 64, 128, 1)


def test_flip_bit_matches_reference():
    from paper_2504_02211_b200 import _lib
    orc = oracle()
    rng = np.random.default_rng(0)
    for v in rng.uniform(-10, 10, 50).astype(np.float32):
        for b in (0, 5, 22, 23, 30, 31):
            a = np.float32(_lib.lib.efta_flip_bit(float(v), 32, b))
            r = np.float32(orc.flip_bit(float(v), 32, b))
            assert a.view(np.uint32) == r.view(np.uint32)


def test_host_rng_matches_reference_stream():
    from paper_2504_02211_b200.campaign import gen_head, trial_seed
    orc = oracle()
    for t in range(6):
        seed = trial_seed(7, t)
        assert seed == orc.trial_seed(7, t)
        q, k, v, f = gen_head(seed, 256, 64, 128, 8, sites=list(range(8)))
        q2, k2, v2, f2 = orc.gen_trial(seed, 256, 64, 128, 8, sites=list(range(8)))
        assert np.array_equal(q.astype(np.float32), q2) and np.array_equal(v.astype(np.float32), v2)
        assert f.as_tuple() == f2


def test_classify_trial_ladder():  # test_campaign.cpp:190-254
    from paper_2504_02211_b200.attention import FaultSpec
    from paper_2504_02211_b200.campaign import classify
    ref = oracle().random_matrix(808, 32, 16, half=False)
    some = FaultSpec.parse("GEMM1_OUT:0:0:1:2:30")
    l_ok = np.full(32, 10.0, np.float32)
    assert classify(ref, ref, 0, 0, False, l_ok, None, 1e-4) == "clean"
    assert classify(ref, ref, 1, 0, False, l_ok, None, 1e-4) == "false_alarm"
    assert classify(ref, ref, 1, 0, False, l_ok, some, 1e-4) == "corrected"
    assert classify(ref, ref, 0, 0, False, l_ok, some, 1e-4) == "masked_benign"
    out = ref.copy(); out[3, 3] += 5.0
    assert classify(out, ref, 1, 0, False, l_ok, some, 1e-4) == "uncorrectable"
    assert classify(ref, ref, 0, 0, True, l_ok, some, 1e-4) == "uncorrectable"
    sf = FaultSpec.parse("REDUCE_SUM:0:0:5:0:30")
    out = ref.copy(); out[5] *= 3.0
    assert classify(out, ref, 1, 1, False, l_ok, sf, 1e-4) == "range_restricted"
    out = ref.copy(); out[5] *= 1.2
    assert classify(out, ref, 0, 0, False, l_ok, FaultSpec.parse("REDUCE_SUM:0:0:5:0:3"),
                    1e-4) == "range_contract"


def test_decoupled_workspace_is_chunked():
    """The decoupled baseline keeps its N^2 intermediates (S_aug fp32, P_aug fp16) for one chunk
    of heads at a time: the workspace grows with the chunk, not with batch x heads."""
    from paper_2504_02211_b200 import _lib
    small = _desc(mode=3, batch=1, heads=1, seq_len=8192, head_dim=128)
    big = _desc(mode=3, batch=32, heads=32, seq_len=8192, head_dim=128)
    ws1 = _lib.lib.efta_attn_workspace_bytes(C.byref(small))
    ws2 = _lib.lib.efta_attn_workspace_bytes(C.byref(big))
    per_head = (64 * 132) ** 2 * 4  # S_aug alone
    assert ws1 > per_head
    assert ws2 <= (4 << 30) + 256 and ws2 >= ws1


def test_gqa_workspace_scales_with_kv_heads():
    """Under grouped-query attention the checksum operands (KC, [V^T ; VC^T]) exist once per K/V
    head: the workspace shrinks with the group size."""
    from paper_2504_02211_b200 import _lib
    mha = _lib.lib.efta_attn_workspace_bytes(C.byref(_desc(batch=2, heads=8, seq_len=1024)))
    gqa = _lib.lib.efta_attn_workspace_bytes(C.byref(_desc(batch=2, heads=8, seq_len=1024, kv_heads=2)))
    assert 0 < gqa < mha and mha / gqa > 3.5  # (the decode partials are per query head)


@pytest.mark.parametrize("split,ok", [
    ((0, 0, 0), True),
    ((512, 10, 128), True),      # QKV of a 1280-wide model: [3, m/512, 10, 512, 128]
    ((128, 7, 128), False),      # 896 does not divide n = 3840
    ((100, 10, 128), False),     # seq must divide m
    ((512, 10, 0), False),
    ((512, 0, 128), False),
    ((512, 20, 60), False),      # head_dim % 8
    ((-1, 0, 0), False),
])
def test_gemm_head_split_validation(split, ok):
    """efta_gemm_desc's head-split output fields (the fused QKV projection layout) are validated
    host-side: efta_abft_weight_cs_bytes returns 0 for an invalid descriptor."""
    from paper_2504_02211_b200 import _lib
    d = _lib.GemmDesc(1024, 3840, 1280, 8, 256, 1e-2, 0, *split)
    assert (_lib.lib.efta_abft_weight_cs_bytes(C.byref(d)) > 0) == ok
    if not ok:
        assert "head split" in _lib.last_error() or "head-split" in _lib.last_error()
