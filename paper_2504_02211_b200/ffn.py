"""Strided-ABFT linear layers for the feed-forward block (FT-Transformer, arXiv 2504.02211).

    lin = AbftLinear(weight)        # weight: CUDA fp16 [out_features, in_features]
    y, rep = lin(x)                 # x: CUDA fp16 [tokens, in_features] -> y fp16

Mirrors the reference's checksummed_gemm + verify_locate_correct (reference
include/efta/abft.hpp:58-77) applied to every 256-wide output column tile; the
weight's strided checksum rows are encoded once at construction (weights are
static). The compute is libefta_b200.so's tcgen05 kernel (csrc/abft_gemm.cu).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import check, lib
from .attention import FTReport, KINDS, STATUS

_EXPORTS = ("efta_abft_gemm_f16", "efta_abft_gemm_ex", "efta_abft_gemm_fused_f16", "efta_abft_encode_weight_f16", "efta_abft_weight_cs_bytes")
for _n in _EXPORTS:
    if not hasattr(lib, _n):
        raise ImportError(f"libefta_b200.so lacks {_n}: rebuild the library")


class AbftLinear:
    def __init__(self, weight: torch.Tensor, eps: float = 1e-2, debug: bool = False,
                 ev_cap: int = 4096):
        if weight.dtype != torch.float16 or not weight.is_cuda or weight.dim() != 2:
            raise _lib.ConfigError("AbftLinear: weight must be a 2-D CUDA fp16 tensor [N, K]")
        self.weight = weight.contiguous()
        self.n, self.k = self.weight.shape
        self.eps = eps
        self.debug = debug
        desc = _lib.GemmDesc(128, self.n, self.k, 8, 256, eps, 1 if debug else 0)
        check(_validate(desc))
        nbytes = lib.efta_abft_weight_cs_bytes(C.byref(desc))
        self.wcs = torch.empty(nbytes // 2, dtype=torch.float16, device=weight.device)
        check(lib.efta_abft_encode_weight_f16(C.byref(desc), self.weight.data_ptr(),
                                              self.wcs.data_ptr(),
                                              torch.cuda.current_stream(weight.device).cuda_stream))
        dev = weight.device
        self.counters = torch.zeros(C.sizeof(_lib.Counters), dtype=torch.uint8, device=dev)
        self.ev_cap = ev_cap
        self.events = torch.zeros(ev_cap * C.sizeof(_lib.Event), dtype=torch.uint8, device=dev)
        self.faults = None
        self.n_faults = 0

    def set_faults(self, faults):
        """faults: iterable of (row, col, bit) in global output coordinates."""
        faults = list(faults or [])
        self.n_faults = len(faults)
        if not faults:
            self.faults = None
            return
        arr = (_lib.FaultSpec * len(faults))(
            *[_lib.FaultSpec(0, 0, r, 0, 0, c, b, 1) for (r, c, b) in faults])
        self.faults = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).to(self.weight.device)

    def __call__(self, x: torch.Tensor, y: torch.Tensor | None = None, fp32_out: bool = False,
                 checksums: torch.Tensor | None = None, head_split: tuple | None = None,
                 residual: torch.Tensor | None = None, activation: str | None = None):
        """y = x @ weight.T (fp16, or fp32 with fp32_out). checksums, if given: a CUDA fp32
        tensor [tokens, out_features/256, 16] receiving each output tile's tensor-core
        c1[8] | c2[8] per row (the reference's ChecksumPair per 256-wide tile).
        head_split = (seq, heads, head_dim): y comes back [parts, tokens/seq, heads, seq,
        head_dim] (parts = out_features / (heads*head_dim)), written by the GEMM epilogue —
        a fused QKV projection hands Q, K, V to the attention without a permute copy.
        residual (fp16 [tokens, out_features]) / activation ("gelu"): element-wise epilogues on
        the verified fp16 value, y = gelu(half(x @ W.T)) (+ residual) — the residual adds and
        the FFN activation of a transformer layer without extra passes over HBM."""
        if x.dtype != torch.float16 or not x.is_cuda or x.dim() != 2 or x.shape[1] != self.k:
            raise _lib.ConfigError("AbftLinear: x must be CUDA fp16 [tokens, in_features]")
        x = x.contiguous()
        m = x.shape[0]
        split = (0, 0, 0)
        shape = (m, self.n)
        if head_split is not None:
            seq, heads, hd = (int(v) for v in head_split)
            split = (seq, heads, hd)
            if seq <= 0 or heads <= 0 or hd <= 0 or m % seq or self.n % (heads * hd):
                raise _lib.ConfigError("AbftLinear: head_split must tile [tokens, out_features]")
            shape = (self.n // (heads * hd), m // seq, heads, seq, hd)
        if y is None:
            y = torch.empty(shape, dtype=torch.float32 if fp32_out else torch.float16, device=x.device)
        if checksums is not None and (checksums.dtype != torch.float32 or checksums.numel() != m * (self.n // 256) * 16):
            raise _lib.ConfigError("AbftLinear: checksums must be fp32 [tokens, out/256, 16]")
        desc = _lib.GemmDesc(m, self.n, self.k, 8, 256, self.eps, 1 if self.debug else 0, *split)
        faults = self.faults.data_ptr() if self.faults is not None else None
        st = torch.cuda.current_stream(x.device).cuda_stream
        if residual is not None or activation is not None:
            if activation not in (None, "gelu"):
                raise _lib.ConfigError("AbftLinear: activation must be None or 'gelu'")
            if residual is not None and (residual.dtype != torch.float16 or not residual.is_cuda
                                         or residual.shape != (m, self.n)):
                raise _lib.ConfigError("AbftLinear: residual must be CUDA fp16 [tokens, out_features]")
            if checksums is not None:
                raise _lib.ConfigError("AbftLinear: the fused epilogues return no tile checksums")
            res = residual.contiguous() if residual is not None else None
            check(lib.efta_abft_gemm_fused_f16(
                C.byref(desc), x.data_ptr(), self.weight.data_ptr(), self.wcs.data_ptr(), y.data_ptr(),
                res.data_ptr() if res is not None else None, 1 if activation == "gelu" else 0,
                faults, self.n_faults, self.events.data_ptr(), self.ev_cap, self.counters.data_ptr(), st))
            return y
        check(lib.efta_abft_gemm_ex(
            C.byref(desc), x.data_ptr(), self.weight.data_ptr(), self.wcs.data_ptr(), y.data_ptr(),
            1 if y.dtype == torch.float32 else 0, checksums.data_ptr() if checksums is not None else None,
            self.faults.data_ptr() if self.faults is not None else None, self.n_faults,
            self.events.data_ptr(), self.ev_cap, self.counters.data_ptr(),
            torch.cuda.current_stream(x.device).cuda_stream))
        return y

    def report(self) -> FTReport:
        cnt = _lib.Counters.from_buffer_copy(bytes(self.counters.cpu().numpy()))
        rep = FTReport(mode="abft", detections=cnt.detections, corrections=cnt.corrections,
                       failed=bool(cnt.failed), family_max=tuple(cnt.family_max))
        ne = min(cnt.n_events, self.ev_cap)
        if ne:
            raw = bytes(self.events[: ne * C.sizeof(_lib.Event)].cpu().numpy())
            for i in range(ne):
                e = _lib.Event.from_buffer_copy(raw, i * C.sizeof(_lib.Event))
                rep.events.append(dict(kind=KINDS[e.kind], n_tile=e.head, m_tile=e.block_i,
                                       status=STATUS[e.status], row=e.row, col=e.col,
                                       violations=e.violations, corrections=e.corrections,
                                       checksum_repair=e.checksum_repair, residual=e.residual,
                                       delta=e.delta))
        return rep


def gelu_(x: torch.Tensor) -> torch.Tensor:
    """In-place erf GELU of a CUDA fp16 tensor (csrc/elementwise.cu; bit-identical to F.gelu)."""
    if x.dtype != torch.float16 or not x.is_cuda or not x.is_contiguous():
        raise _lib.ConfigError("gelu_: x must be a contiguous CUDA fp16 tensor")
    check(lib.efta_gelu_f16(x.data_ptr(), x.data_ptr(), x.numel(), torch.cuda.current_stream(x.device).cuda_stream))
    return x


def _validate(desc) -> int:
    # efta_abft_weight_cs_bytes returns 0 on an invalid descriptor and sets the error
    return 0 if lib.efta_abft_weight_cs_bytes(C.byref(desc)) else 1


def abft_gemm(x: torch.Tensor, weight: torch.Tensor, eps: float = 1e-2):
    """One-shot protected linear: returns (y, FTReport)."""
    lin = AbftLinear(weight, eps=eps)
    y = lin(x)
    return y, lin.report()
