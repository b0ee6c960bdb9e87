"""B200-native (sm_100a) end-to-end fault-tolerant attention (EFTA, arXiv 2504.02211).

The compute lives in libefta_b200.so (CUDA kernels + C-ABI, include/efta_b200.h);
this package is the host-side mirror of the reference operator API. Attributes
are resolved lazily so `python -m paper_2504_02211_b200.build` works before the
library exists; any compute entry point raises if the library is missing.
"""
_ATTN = ("EftaAttention", "FaultSpec", "FTReport", "Thresholds", "efta_forward", "validate_plan",
         "EftaDecode", "efta_decode")
_LIB = ("ConfigError", "EftaError", "SITES", "KINDS", "STATUS")
_FFN = ("AbftLinear", "abft_gemm")
_LAYER = ("FTTransformerLayer",)


def __getattr__(name):
    if name in _ATTN:
        from . import attention
        return getattr(attention, name)
    if name in _LIB:
        from . import _lib
        return getattr(_lib, name)
    if name in _FFN:
        from . import ffn
        return getattr(ffn, name)
    if name in _LAYER:
        from . import layer
        return getattr(layer, name)
    raise AttributeError(name)


__all__ = list(_ATTN + _LIB + _FFN + _LAYER)
