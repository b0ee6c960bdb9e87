"""Host-side mirror of the reference operator API for the EFTA hot path.

    efta_forward(q, k, v, mode, thr, faults, ...)  ->  (O, FTReport)

mirrors efta::efta_forward (reference include/efta/efta.hpp:86-89): same
modes (NONE / EFTA / EFTA_OPTIMIZED), same Thresholds (snvr.hpp:17-30), same
fault-site vocabulary and FaultSpec text format (fault.hpp:16-47), and an
FTReport carrying the same fields (events, detections, corrections,
recomputes, range_replacements, failed, final_m, final_l). Tensors live on the
GPU (torch is used for device memory and streams only); all compute runs in
libefta_b200.so through its C-ABI.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import torch

from . import _lib
from ._lib import SITES, KINDS, STATUS, MODES, check, lib

INF = math.inf


@dataclass
class Thresholds:
    """Reference Thresholds (include/efta/snvr.hpp:17-30)."""
    eps1: float = 7e-6
    eps2: float = 0.48
    eps_lin: float = 0.48

    @staticmethod
    def observe() -> "Thresholds":
        return Thresholds(INF, INF, INF)


@dataclass
class FaultSpec:
    """Reference FaultSpec (include/efta/fault.hpp:36-47) + the flat head index."""
    site: int
    block_i: int
    block_j: int
    row: int
    col: int
    bit: int
    trigger: int = 1
    head: int = 0

    @staticmethod
    def parse(text: str, head: int = 0) -> "FaultSpec":
        """SITE:i:j:row:col:bit[:trigger] (reference src/fault.cpp:48-76)."""
        parts = text.split(":")
        if len(parts) not in (6, 7):
            raise _lib.ConfigError(
                f"fault spec: expected SITE:i:j:row:col:bit[:trigger], got '{text}'")
        if parts[0] not in SITES:
            raise _lib.ConfigError(f"fault spec: unknown site '{parts[0]}'")
        try:
            vals = [int(x) for x in parts[1:]]
        except ValueError:
            raise _lib.ConfigError(f"fault spec: bad integer field in '{text}'") from None
        return FaultSpec(SITES.index(parts[0]), *vals[:5], vals[5] if len(vals) == 6 else 1,
                         head=head)

    def to_string(self) -> str:
        s = f"{SITES[self.site]}:{self.block_i}:{self.block_j}:{self.row}:{self.col}:{self.bit}"
        return s + (f":{self.trigger}" if self.trigger != 1 else "")

    def as_tuple(self) -> tuple:
        return (self.site, self.block_i, self.block_j, self.row, self.col, self.bit, self.trigger)


def validate_plan(specs, seq_len: int, head_dim: int, block: int = 128, heads: int = 1):
    """FaultPlan::validate (reference src/fault.cpp:100-121): coordinates in range
    and at most one spec per (head, row-block)."""
    n = seq_len // block
    seen = set()
    for f in specs:
        if not 0 <= f.head < heads:
            raise _lib.ConfigError("fault plan: head out of range")
        if not 0 <= f.block_i < n:
            raise _lib.ConfigError("fault plan: block_i out of range")
        post = f.site == SITES.index("NORMALIZE_OUT")
        if not 0 <= f.block_j < (1 if post else n):
            raise _lib.ConfigError("fault plan: block_j out of range")
        if not 0 <= f.row < block:
            raise _lib.ConfigError("fault plan: row out of range")
        bound = block if f.site <= 2 else (1 if f.site in (3, 4) else head_dim)
        if not 0 <= f.col < bound:
            raise _lib.ConfigError("fault plan: col out of range for site")
        if not 0 <= f.bit <= 31:
            raise _lib.ConfigError("fault plan: bit out of range")
        if f.trigger < 1:
            raise _lib.ConfigError("fault plan: trigger must be >= 1")
        key = (f.head, f.block_i)
        if key in seen:
            raise _lib.ConfigError(
                f"fault plan: multiple faults in one detection cycle (row-block {f.block_i})")
        seen.add(key)


@dataclass
class FTReport:
    """Reference FTReport (include/efta/efta.hpp:50-72), device-side edition:
    `events` holds the non-CLEAN check outcomes only."""
    mode: str
    events: list = field(default_factory=list)
    detections: int = 0
    corrections: int = 0
    recomputes: int = 0
    range_replacements: int = 0
    failed: bool = False
    final_m: torch.Tensor | None = None
    final_l: torch.Tensor | None = None
    fired: list = field(default_factory=list)
    family_max: tuple = (0.0, 0.0, 0.0)  # worst clean residual: exp, out, lin

    def max_residual(self, kind: str) -> float:
        v = [e["residual"] for e in self.events if e["kind"] == kind]
        return max(v) if v else -INF


def _desc(b, h, s, d, mode, thr, scale, observe_linear, rowmax_bias, debug, block, stride, kv_heads=0,
          causal=False):
    return _lib.AttnDesc(b, h, s, d, block, stride, float(scale), MODES[mode], float(thr.eps1),
                         float(thr.eps2), float(thr.eps_lin), 1 if observe_linear else 0,
                         float(rowmax_bias), 1 if debug else 0, 0, int(kv_heads), 1 if causal else 0)


def _as_bhsd(x: torch.Tensor):
    if x.dim() == 2:
        return x.unsqueeze(0).unsqueeze(0)
    if x.dim() == 3:
        return x.unsqueeze(0)
    return x


class EftaAttention:
    """Pre-planned fused forward for a fixed shape: owns the workspace, the
    counters and the event/fired buffers, so repeated calls allocate nothing
    (the form bench.py times)."""

    def __init__(self, batch, heads, seq_len, head_dim, mode="efta-opt", thr=None, scale=0.0,
                 observe_linear=False, rowmax_bias=0.0, debug=False, block=128, stride=8,
                 ev_cap=4096, fired_cap=256, device="cuda", kv_heads=None, causal=False,
                 token_major_out=False):
        self.shape = (batch, heads, seq_len, head_dim)
        # token_major_out: O comes back fp16 [batch, seq_len, heads, head_dim] (the output
        # projection's input, written by the kernel's epilogue) instead of fp32 [b, h, s, d]
        self.token_major_out = bool(token_major_out)
        # grouped-query attention: K / V carry kv_heads heads (query head h reads h // group)
        self.kv_heads = heads if not kv_heads else int(kv_heads)
        self.mode = mode
        self.thr = thr or Thresholds()
        self.desc = _desc(batch, heads, seq_len, head_dim, mode, self.thr, scale, observe_linear,
                          rowmax_bias, debug, block, stride, self.kv_heads, causal)
        self.desc.o_token_major = 1 if token_major_out else 0
        check(lib.efta_attn_validate(C.byref(self.desc)))
        ws = lib.efta_attn_workspace_bytes(C.byref(self.desc))
        dev = torch.device(device)
        self.workspace = torch.empty(ws, dtype=torch.uint8, device=dev)
        self.counters = torch.zeros(C.sizeof(_lib.Counters), dtype=torch.uint8, device=dev)
        self.ev_cap, self.fired_cap = ev_cap, fired_cap
        self.events = torch.zeros(max(1, ev_cap) * C.sizeof(_lib.Event), dtype=torch.uint8, device=dev)
        self.fired = torch.zeros(max(1, fired_cap) * C.sizeof(_lib.Fired), dtype=torch.uint8, device=dev)
        self.faults = None
        self.n_faults = 0

    def set_faults(self, specs):
        specs = list(specs or [])
        self.n_faults = len(specs)
        if not specs:
            self.faults = None
            return
        arr = (_lib.FaultSpec * len(specs))(
            *[_lib.FaultSpec(f.head, f.site, f.block_i, f.block_j, f.row, f.col, f.bit, f.trigger)
              for f in specs])
        host = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8)
        self.faults = host.to(self.workspace.device)

    def __call__(self, q, k, v, o=None, m=None, l=None, stream=None):
        b, h, s, d = self.shape
        for t, hh in ((q, h), (k, self.kv_heads), (v, self.kv_heads)):
            if t.dtype != torch.float16 or not t.is_cuda or not t.is_contiguous():
                raise _lib.ConfigError("efta_forward: q/k/v must be contiguous CUDA fp16 tensors")
            if t.numel() != b * hh * s * d:
                raise _lib.ConfigError("attention: Q/K/V must all be seq_len x head_dim")
        if o is None:
            o = (torch.empty((b, s, h, d), dtype=torch.float16, device=q.device) if self.token_major_out
                 else torch.empty((b, h, s, d), dtype=torch.float32, device=q.device))
        if m is None:
            m = torch.empty((b, h, s), dtype=torch.float32, device=q.device)
        if l is None:
            l = torch.empty((b, h, s), dtype=torch.float32, device=q.device)
        st = stream if stream is not None else torch.cuda.current_stream(q.device)
        check(lib.efta_attn_fwd_f16(
            C.byref(self.desc), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
            m.data_ptr(), l.data_ptr(), self.workspace.data_ptr(), self.workspace.numel(),
            self.faults.data_ptr() if self.faults is not None else None, self.n_faults,
            self.events.data_ptr(), self.ev_cap, self.fired.data_ptr(), self.fired_cap,
            self.counters.data_ptr(), st.cuda_stream))
        return o, m, l

    def report(self, m=None, l=None) -> FTReport:
        """Copies the device-side counters / events back (synchronises)."""
        cnt = _lib.Counters.from_buffer_copy(bytes(self.counters.cpu().numpy()))
        rep = FTReport(mode=self.mode, detections=cnt.detections, corrections=cnt.corrections,
                       recomputes=cnt.recomputes, range_replacements=cnt.range_replacements,
                       failed=bool(cnt.failed), final_m=m, final_l=l,
                       family_max=tuple(cnt.family_max))
        ne = min(cnt.n_events, self.ev_cap)
        if ne:
            raw = bytes(self.events[: ne * C.sizeof(_lib.Event)].cpu().numpy())
            for i in range(ne):
                e = _lib.Event.from_buffer_copy(raw, i * C.sizeof(_lib.Event))
                rep.events.append(dict(kind=KINDS[e.kind], head=e.head, block_i=e.block_i,
                                       block_j=e.block_j, status=STATUS[e.status], row=e.row,
                                       col=e.col, violations=e.violations,
                                       corrections=e.corrections,
                                       checksum_repair=e.checksum_repair, residual=e.residual,
                                       delta=e.delta))
        nf = min(cnt.n_fired, self.fired_cap)
        if nf:
            raw = bytes(self.fired[: nf * C.sizeof(_lib.Fired)].cpu().numpy())
            for i in range(nf):
                f = _lib.Fired.from_buffer_copy(raw, i * C.sizeof(_lib.Fired))
                sp = f.spec
                rep.fired.append(dict(spec=FaultSpec(sp.site, sp.block_i, sp.block_j, sp.row,
                                                     sp.col, sp.bit, sp.trigger, head=sp.head),
                                      before=f.before, after=f.after))
        return rep


def efta_forward(q, k, v, mode="efta-opt", thr: Thresholds | None = None, faults=None,
                 scale=0.0, observe_linear=False, rowmax_bias=0.0, debug=None, block=128,
                 stride=8, ev_cap=4096, causal=False):
    """One protected (or plain) attention forward. q/k/v: CUDA fp16 [S,d], [BH,S,d]
    or [B,H,S,d]. Returns (O fp32 with q's shape, FTReport)."""
    shape = q.shape
    q4, k4, v4 = (_as_bhsd(x).contiguous() for x in (q, k, v))
    b, h, s, d = q4.shape
    kv_heads = k4.shape[1]  # fewer K/V heads than query heads: grouped-query attention
    specs = []
    for f in faults or []:
        specs.append(FaultSpec.parse(f) if isinstance(f, str) else f)
    if specs:
        validate_plan(specs, s, d, block, b * h)
    if debug is None:
        debug = bool(specs) or observe_linear
    op = EftaAttention(b, h, s, d, mode=mode, thr=thr, scale=scale, observe_linear=observe_linear,
                       rowmax_bias=rowmax_bias, debug=debug, block=block, stride=stride,
                       ev_cap=ev_cap, device=q.device, kv_heads=kv_heads, causal=causal)
    op.set_faults(specs)
    o, m, l = op(q4, k4, v4)
    rep = op.report(m.reshape(shape[:-1]), l.reshape(shape[:-1]))
    return o.reshape(shape), rep


class EftaDecode:
    """KV-cache decode (not a reference feature): one query row per head
    against K / V caches [batch, kv_heads, seq_len, head_dim] — the reference algorithm for that
    row (row 0 of efta_forward(q, K, V)) with EFTA-optimized checks, HBM-bound (csrc/decode.cu).
    Owns the workspace holding the cache's checksum operands: `encode(k, v)` once, then decode
    steps with `cache_encoded=True` skip re-encoding."""

    def __init__(self, batch, heads, seq_len, head_dim, mode="efta-opt", thr=None, scale=0.0,
                 kv_heads=None, ev_cap=1024, device="cuda"):
        self.shape = (batch, heads, seq_len, head_dim)
        self.kv_heads = heads if not kv_heads else int(kv_heads)
        self.mode = mode
        self.thr = thr or Thresholds()
        self.desc = _desc(batch, heads, seq_len, head_dim, mode, self.thr, scale, False, 0.0, False, 128, 8,
                          self.kv_heads)
        check(lib.efta_attn_validate(C.byref(self.desc)))
        dev = torch.device(device)
        self.workspace = torch.empty(lib.efta_attn_workspace_bytes(C.byref(self.desc)), dtype=torch.uint8, device=dev)
        self.counters = torch.zeros(C.sizeof(_lib.Counters), dtype=torch.uint8, device=dev)
        self.ev_cap = ev_cap
        self.events = torch.zeros(max(1, ev_cap) * C.sizeof(_lib.Event), dtype=torch.uint8, device=dev)

    def encode(self, k, v, stream=None):
        """Checksum operands of the caches into the workspace (efta_attn_encode_kv_f16)."""
        st = stream if stream is not None else torch.cuda.current_stream(k.device)
        ws = self.workspace.data_ptr()
        b, h, s, d = self.shape
        kc_bytes = ((b * self.kv_heads * (s // 128) * 32 * d * 2) + 255) // 256 * 256
        check(lib.efta_attn_encode_kv_f16(C.byref(self.desc), k.data_ptr(), v.data_ptr(), ws, ws + kc_bytes,
                                          st.cuda_stream))

    def __call__(self, q, k, v, o=None, cache_encoded=False, stream=None):
        b, h, s, d = self.shape
        for t_, n_ in ((q, b * h * d), (k, b * self.kv_heads * s * d), (v, b * self.kv_heads * s * d)):
            if t_.dtype != torch.float16 or not t_.is_cuda or not t_.is_contiguous() or t_.numel() != n_:
                raise _lib.ConfigError("efta_decode: q [B,H,d] and k/v [B,H_kv,S,d] contiguous CUDA fp16")
        if o is None:
            o = torch.empty((b, h, d), dtype=torch.float32, device=q.device)
        m = torch.empty((b, h), dtype=torch.float32, device=q.device)
        l = torch.empty((b, h), dtype=torch.float32, device=q.device)
        self.desc.checksums_ready = 1 if cache_encoded else 0
        st = stream if stream is not None else torch.cuda.current_stream(q.device)
        check(lib.efta_decode_fwd_f16(C.byref(self.desc), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                      m.data_ptr(), l.data_ptr(), self.workspace.data_ptr(), self.workspace.numel(),
                                      self.events.data_ptr(), self.ev_cap, self.counters.data_ptr(),
                                      st.cuda_stream))
        return o, m, l

    def report(self) -> FTReport:
        cnt = _lib.Counters.from_buffer_copy(bytes(self.counters.cpu().numpy()))
        rep = FTReport(mode=self.mode, detections=cnt.detections, corrections=cnt.corrections,
                       recomputes=cnt.recomputes, range_replacements=cnt.range_replacements,
                       failed=bool(cnt.failed), family_max=tuple(cnt.family_max))
        ne = min(cnt.n_events, self.ev_cap)
        if ne:
            raw = bytes(self.events[: ne * C.sizeof(_lib.Event)].cpu().numpy())
            for i in range(ne):
                e = _lib.Event.from_buffer_copy(raw, i * C.sizeof(_lib.Event))
                rep.events.append(dict(kind=KINDS[e.kind], head=e.head, block_i=e.block_i, block_j=e.block_j,
                                       status=STATUS[e.status], row=e.row, col=e.col, violations=e.violations,
                                       corrections=e.corrections, checksum_repair=e.checksum_repair,
                                       residual=e.residual, delta=e.delta))
        return rep


def efta_decode(q, k, v, mode="efta-opt", thr: Thresholds | None = None, scale=0.0):
    """One decode step: q [B, H, d] (or [H, d]), k / v [B, H_kv, S, d] (or [H_kv, S, d]).
    Returns (O fp32 [B, H, d], FTReport)."""
    if q.dim() == 2:
        q, k, v = q[None], k[None], v[None]
    b, h, d = q.shape
    _, hkv, s, _ = k.shape
    op = EftaDecode(b, h, s, d, mode=mode, thr=thr, scale=scale, kv_heads=hkv, device=q.device)
    o, m, l = op(q.contiguous(), k.contiguous(), v.contiguous())
    rep = op.report()
    rep.final_m, rep.final_l = m, l
    return o, rep
