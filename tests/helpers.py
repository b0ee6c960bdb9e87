"""Shared test helpers: seeded reference inputs (oracle Rng) -> device tensors."""
import numpy as np

from oracle import Oracle  # noqa: E402  (tests/conftest.py puts oracle/ on sys.path)

_ORC = None


def oracle():
    global _ORC
    if _ORC is None:
        _ORC = Oracle("port")
    return _ORC


def head_inputs(base_seed: int, n_heads: int, seq: int, d: int, block=128, stride=8, sites=None):
    """Per-head inputs exactly as the reference campaign derives them
    (src/campaign.cpp:174-185): hseed = trial_seed(trial_seed(base, 0), h),
    q,k,v = Matrix::random in that order, then an optional random plan."""
    orc = oracle()
    tseed = orc.trial_seed(base_seed, 0)
    qs, ks, vs, specs = [], [], [], []
    for h in range(n_heads):
        hseed = tseed if n_heads == 1 else orc.trial_seed(tseed, h)
        q, k, v, spec = orc.gen_trial(hseed, seq, d, block, stride, sites=sites)
        qs.append(q); ks.append(k); vs.append(v); specs.append(spec)
    return np.stack(qs), np.stack(ks), np.stack(vs), specs


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = np.abs(b).max()
    return float(np.abs(a - b).max() / (scale if scale > 0 else 1.0))
