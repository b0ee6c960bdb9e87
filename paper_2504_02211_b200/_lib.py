"""ctypes binding of libefta_b200.so (the C-ABI in include/efta_b200.h).

The shared library is the product: there is no Python or CPU fallback. If the
library is missing, importing this module raises (build it with
`python -m paper_2504_02211_b200.build`).
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EFTA_LIB") or os.path.join(PKG, "libefta_b200.so")

SITES = ["GEMM1_OUT", "SUB_MAX", "EXP_OUT", "REDUCE_MAX", "REDUCE_SUM",
         "RESCALE_FACTOR", "GEMM2_ACC", "NORMALIZE_OUT"]
MODES = {"none": 0, "efta": 1, "efta-opt": 2, "efta_optimized": 2, "decoupled": 3}
KINDS = ["score_checksum", "exp_checksum", "factor_range", "rowsum_range", "output_checksum",
         "dmr_softmax", "block_checksum"]
STATUS = ["clean", "corrected", "detected_uncorrectable", "nonfinite"]


class AttnDesc(C.Structure):
    _fields_ = [("batch", C.c_int), ("heads", C.c_int), ("seq_len", C.c_int),
                ("head_dim", C.c_int), ("block", C.c_int), ("stride", C.c_int),
                ("scale", C.c_float), ("mode", C.c_int), ("eps1", C.c_double),
                ("eps2", C.c_double), ("eps_lin", C.c_double), ("observe_linear", C.c_int),
                ("rowmax_bias", C.c_float), ("debug", C.c_int), ("checksums_ready", C.c_int),
                ("kv_heads", C.c_int), ("causal", C.c_int), ("o_token_major", C.c_int)]


class FaultSpec(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("head", "site", "block_i", "block_j", "row", "col", "bit",
                                        "trigger")]


class Event(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("kind", "head", "block_i", "block_j", "status", "row",
                                        "col", "violations", "corrections", "checksum_repair")] + \
               [("residual", C.c_double), ("delta", C.c_double)]


class Fired(C.Structure):
    _fields_ = [("spec", FaultSpec), ("before", C.c_float), ("after", C.c_float)]


class Counters(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("n_events", "n_fired", "detections", "corrections",
                                        "recomputes", "range_replacements", "failed", "pad_")] + \
               [("family_max", C.c_float * 3), ("pad2_", C.c_float)]


class GemmDesc(C.Structure):
    _fields_ = [("m", C.c_int), ("n", C.c_int), ("k", C.c_int), ("stride", C.c_int),
                ("n_tile", C.c_int), ("eps", C.c_double), ("debug", C.c_int),
                ("out_seq", C.c_int), ("out_heads", C.c_int), ("out_head_dim", C.c_int)]


class GemmFault(C.Structure):
    _fields_ = [("row", C.c_int), ("col", C.c_int), ("bit", C.c_int), ("pad_", C.c_int)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2504_02211_b200.build` "
            "(no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    lib.efta_last_error.restype = C.c_char_p
    lib.efta_attn_validate.argtypes = [C.POINTER(AttnDesc)]
    lib.efta_attn_workspace_bytes.restype = C.c_size_t
    lib.efta_attn_workspace_bytes.argtypes = [C.POINTER(AttnDesc)]
    lib.efta_attn_fwd_f16.argtypes = [C.POINTER(AttnDesc), vp, vp, vp, vp, vp, vp, vp, C.c_size_t,
                                      vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp]
    lib.efta_attn_fwd_host_f16.argtypes = [C.POINTER(AttnDesc), vp, vp, vp, vp, vp, vp, vp,
                                           C.c_int, vp, C.c_int, vp, C.c_int, vp]
    lib.efta_attn_encode_kv_f16.argtypes = [C.POINTER(AttnDesc), vp, vp, vp, vp, vp]
    lib.efta_decode_fwd_f16.argtypes = [C.POINTER(AttnDesc), vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp,
                                        C.c_int, vp, vp]
    lib.efta_flip_bit.restype = C.c_float
    lib.efta_flip_bit.argtypes = [C.c_float, C.c_int, C.c_int]
    if hasattr(lib, "efta_abft_gemm_f16"):
        lib.efta_abft_gemm_f16.argtypes = [C.POINTER(GemmDesc), vp, vp, vp, vp, vp, C.c_int, vp,
                                           C.c_int, vp, vp]
        lib.efta_abft_encode_weight_f16.argtypes = [C.POINTER(GemmDesc), vp, vp, vp]
        lib.efta_abft_weight_cs_bytes.restype = C.c_size_t
        lib.efta_abft_weight_cs_bytes.argtypes = [C.POINTER(GemmDesc)]
        lib.efta_abft_gemm_ex.argtypes = [C.POINTER(GemmDesc), vp, vp, vp, vp, C.c_int, vp, vp, C.c_int,
                                          vp, C.c_int, vp, vp]
        lib.efta_gelu_f16.argtypes = [vp, vp, C.c_size_t, vp]
        lib.efta_abft_gemm_fused_f16.argtypes = [C.POINTER(GemmDesc), vp, vp, vp, vp, vp, C.c_int, vp,
                                                 C.c_int, vp, C.c_int, vp, vp]
    return lib


lib = _load()

# exported symbols the header declares (checked by the CPU test-suite)
EXPORTS = ["efta_last_error", "efta_attn_validate", "efta_attn_workspace_bytes",
           "efta_attn_fwd_f16", "efta_attn_fwd_host_f16", "efta_attn_encode_kv_f16",
           "efta_flip_bit", "efta_abft_gemm_f16", "efta_abft_encode_weight_f16",
           "efta_abft_weight_cs_bytes", "efta_trial_seed", "efta_gen_trial_f16",
           "efta_classify_trial", "efta_abft_gemm_ex", "efta_abft_gemm_fused_f16", "efta_gelu_f16", "efta_encode_strided_f32",
           "efta_verify_workspace_bytes", "efta_verify_locate_correct_f32"]


def last_error() -> str:
    return lib.efta_last_error().decode()


class EftaError(RuntimeError):
    pass


class ConfigError(EftaError):
    """Mirror of the reference's efta::ConfigError (include/efta/config.hpp:9-11)."""


def check(rc: int):
    if rc == 0:
        return
    msg = last_error()
    if rc == 1:
        raise ConfigError(msg)
    raise EftaError(msg)
