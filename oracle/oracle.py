"""ctypes binding for the CPU checkers under oracle/ — TEST INFRASTRUCTURE ONLY.

`Oracle("port")` loads liboracle.so (our C restatement, efta_oracle.c);
`Oracle("ref")` loads _ref/libefta_ref.so (the unmodified reference compiled
from /root/reference by oracle/Makefile). Both expose the same C ABI
(oracle_abi.h). Only tests/, __graft_entry__.smoke() and bench.py's CPU legs
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

SITES = ["GEMM1_OUT", "SUB_MAX", "EXP_OUT", "REDUCE_MAX", "REDUCE_SUM",
         "RESCALE_FACTOR", "GEMM2_ACC", "NORMALIZE_OUT"]
MODES = {"none": 0, "efta": 1, "efta-opt": 2, "decoupled": 3}  # decoupled: the reference (_ref) only
KINDS = ["score_checksum", "exp_checksum", "factor_range", "rowsum_range", "output_checksum",
         "dmr_softmax", "block_checksum"]
STATUS = ["clean", "corrected", "detected_uncorrectable", "nonfinite"]


class FaultSpecC(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("site", "block_i", "block_j", "row", "col", "bit", "trigger")]


class EventC(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("kind", "block_i", "block_j", "status", "row", "col",
                                        "violations", "corrections", "checksum_repair", "pad_")] + \
               [("residual", C.c_double), ("delta", C.c_double)]


class FiredC(C.Structure):
    _fields_ = [("spec", FaultSpecC), ("before", C.c_float), ("after", C.c_float)]


class SummaryC(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("detections", "corrections", "recomputes",
                                        "range_replacements", "failed", "n_events", "n_fired",
                                        "pad_")] + \
               [(n, C.c_uint64) for n in ("flops_main", "flops_checksum", "flops_verify",
                                           "intermediate_elems", "flops_main_gemm_scores",
                                           "flops_cs_gemm_scores", "flops_main_gemm_output",
                                           "flops_cs_gemm_output", "exp_checks", "output_checks")]


class VerifyReportC(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("status", "row", "col", "violations", "corrections",
                                        "checksum_repair")] + \
               [("residual", C.c_double), ("delta", C.c_double)]


def spec_tuple(s) -> tuple:
    return (s.site, s.block_i, s.block_j, s.row, s.col, s.bit, s.trigger)


def parse_spec(text: str) -> tuple:
    """FaultSpec::parse text format SITE:i:j:row:col:bit[:trigger] (src/fault.cpp:48-76)."""
    parts = text.split(":")
    if len(parts) not in (6, 7):
        raise ValueError(f"fault spec: expected SITE:i:j:row:col:bit[:trigger], got '{text}'")
    site = SITES.index(parts[0])
    vals = [int(x) for x in parts[1:]]
    trig = vals[5] if len(vals) == 6 else 1
    return (site, vals[0], vals[1], vals[2], vals[3], vals[4], trig)


@dataclass
class ForwardResult:
    o: np.ndarray
    m: np.ndarray
    l: np.ndarray
    events: list = field(default_factory=list)
    fired: list = field(default_factory=list)
    detections: int = 0
    corrections: int = 0
    recomputes: int = 0
    range_replacements: int = 0
    failed: bool = False
    summary: SummaryC | None = None

    def max_residual(self, kind: str) -> float:
        vals = [e["residual"] for e in self.events if e["kind"] == kind]
        return max(vals) if vals else float("-inf")

    def detected_events(self) -> list:
        return [e for e in self.events if e["status"] != "clean"]


_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")


class Oracle:
    def __init__(self, which: str = "port"):
        path = os.path.join(HERE, "liboracle.so") if which == "port" else \
            os.path.join(HERE, "_ref", "libefta_ref.so")
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.which = which
        self.lib = C.CDLL(path)
        p = "eorc_" if which == "port" else "eref_"
        self._p = p
        L = self.lib
        fn = lambda n: getattr(L, p + n)  # noqa: E731
        self._last_error = fn("last_error")
        self._last_error.restype = C.c_char_p
        self._trial_seed = fn("trial_seed")
        self._trial_seed.restype = C.c_uint64
        self._trial_seed.argtypes = [C.c_uint64, C.c_uint64]
        self._gen_trial = fn("gen_trial")
        self._gen_trial.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.POINTER(C.c_int), C.c_int, _f32p, _f32p, _f32p,
                                    C.POINTER(FaultSpecC)]
        self._random_matrix = fn("random_matrix")
        self._random_matrix.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_double, C.c_double,
                                        C.c_int, _f32p]
        self._below = fn("rng_below_seq")
        self._below.argtypes = [C.c_uint64, C.c_int, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        self._flip = fn("flip_bit")
        self._flip.restype = C.c_float
        self._flip.argtypes = [C.c_float, C.c_int, C.c_int]
        self._f2h = fn("float_to_half_bits")
        self._f2h.restype = C.c_uint16
        self._f2h.argtypes = [C.c_float]
        self._h2f = fn("half_bits_to_float")
        self._h2f.restype = C.c_float
        self._h2f.argtypes = [C.c_uint16]
        self._fwd = fn("efta_forward")
        self._fwd.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_int,
                              C.c_double, C.c_double, C.c_double, C.c_int, C.c_float,
                              _f32p, _f32p, _f32p, _f32p, _f32p, _f32p,
                              C.POINTER(FaultSpecC), C.c_int, C.POINTER(EventC), C.c_int,
                              C.POINTER(FiredC), C.c_int, C.POINTER(SummaryC)]
        self._std = fn("standard_attention")
        self._std.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_float,
                              _f32p, _f32p, _f32p, _f32p]
        self._enc = fn("encode_strided")
        self._enc.argtypes = [C.c_int, C.c_int, C.c_int, _f32p, _f32p, _f32p]
        self._csg = fn("checksummed_gemm")
        self._csg.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _f32p, _f32p, _f32p, _f32p,
                              _f32p]
        self._vlc = fn("verify_locate_correct")
        self._vlc.argtypes = [C.c_int, C.c_int, C.c_int, _f32p, _f32p, _f32p, C.c_double,
                              C.POINTER(C.c_double), C.POINTER(VerifyReportC)]

    # ---- primitives -------------------------------------------------------
    def last_error(self) -> str:
        return self._last_error().decode()

    def trial_seed(self, base: int, trial: int) -> int:
        return int(self._trial_seed(base, trial))

    def gen_trial(self, seed: int, n: int, d: int, block: int = 128, stride: int = 8,
                  sites=None):
        q = np.empty((n, d), np.float32)
        k = np.empty_like(q)
        v = np.empty_like(q)
        spec = FaultSpecC()
        sites = list(sites or [])
        arr = (C.c_int * max(1, len(sites)))(*sites)
        rc = self._gen_trial(seed, n, d, block, stride, arr, len(sites), q, k, v, C.byref(spec))
        if rc:
            raise ValueError(self.last_error())
        return q, k, v, (spec_tuple(spec) if sites else None)

    def random_matrix(self, seed: int, rows: int, cols: int, lo=-1.0, hi=1.0, half=True):
        out = np.empty((rows, cols), np.float32)
        self._random_matrix(seed, rows, cols, lo, hi, 1 if half else 0, out)
        return out

    def rng_below(self, seed: int, bounds) -> list:
        """Rng(seed).below(b) for each b in order (include/efta/rng.hpp:31-38)."""
        n = len(bounds)
        bb = (C.c_uint32 * max(1, n))(*bounds)
        out = (C.c_uint32 * max(1, n))()
        self._below(seed, n, bb, out)
        return [int(out[i]) for i in range(n)]

    def flip_bit(self, v: float, width: int, bit: int) -> float:
        return float(self._flip(v, width, bit))

    def f2h(self, f: float) -> int:
        return int(self._f2h(f))

    def h2f(self, h: int) -> float:
        return float(self._h2f(h))

    # ---- hot path -----------------------------------------------------------
    def efta_forward(self, q, k, v, block=128, stride=8, scale=0.0, mode="efta-opt",
                     thr=(7e-6, 0.48, 0.48), specs=(), observe_linear=False, rowmax_bias=0.0,
                     ev_cap=None) -> ForwardResult:
        n, d = q.shape
        nb = n // block if block > 0 else 0
        if ev_cap is None:
            ev_cap = max(64, 4 * nb * (nb + 2) + 16) + (4 * n if mode == "decoupled" else 0)
        o = np.zeros((n, d), np.float32)
        m = np.zeros(n, np.float32)
        l = np.zeros(n, np.float32)
        specs = [parse_spec(s) if isinstance(s, str) else tuple(s) for s in specs]
        sp = (FaultSpecC * max(1, len(specs)))(*[FaultSpecC(*s) for s in specs])
        ev = (EventC * ev_cap)()
        fired = (FiredC * 16)()
        summ = SummaryC()
        rc = self._fwd(n, d, block, stride, scale, MODES[mode], thr[0], thr[1], thr[2],
                       1 if observe_linear else 0, rowmax_bias,
                       np.ascontiguousarray(q, np.float32), np.ascontiguousarray(k, np.float32),
                       np.ascontiguousarray(v, np.float32), o, m, l, sp, len(specs), ev, ev_cap,
                       fired, 16, C.byref(summ))
        if rc:
            raise ValueError(self.last_error())
        events = []
        for i in range(min(summ.n_events, ev_cap)):
            e = ev[i]
            events.append(dict(kind=KINDS[e.kind], block_i=e.block_i, block_j=e.block_j,
                               status=STATUS[e.status], row=e.row, col=e.col,
                               violations=e.violations, corrections=e.corrections,
                               checksum_repair=e.checksum_repair, residual=e.residual,
                               delta=e.delta))
        fl = [dict(spec=spec_tuple(fired[i].spec), before=fired[i].before, after=fired[i].after)
              for i in range(min(summ.n_fired, 16))]
        return ForwardResult(o=o, m=m, l=l, events=events, fired=fl,
                             detections=summ.detections, corrections=summ.corrections,
                             recomputes=summ.recomputes,
                             range_replacements=summ.range_replacements,
                             failed=bool(summ.failed), summary=summ)

    def standard_attention(self, q, k, v, block=128, stride=8, scale=0.0):
        n, d = q.shape
        o = np.zeros((n, d), np.float32)
        if self._std(n, d, block, stride, scale, q, k, v, o):
            raise ValueError(self.last_error())
        return o

    def encode_strided(self, t, stride):
        t = np.ascontiguousarray(t, np.float32)
        rows, cols = t.shape
        c1 = np.zeros((rows, stride), np.float32)
        c2 = np.zeros_like(c1)
        if self._enc(rows, cols, stride, t, c1, c2):
            raise ValueError(self.last_error())
        return c1, c2

    def checksummed_gemm(self, a, bt, stride):
        a = np.ascontiguousarray(a, np.float32)
        bt = np.ascontiguousarray(bt, np.float32)
        m, kd = a.shape
        w = bt.shape[1]
        c = np.zeros((m, w), np.float32)
        c1 = np.zeros((m, stride), np.float32)
        c2 = np.zeros_like(c1)
        if self._csg(m, kd, w, stride, a, bt, c, c1, c2):
            raise ValueError(self.last_error())
        return c, c1, c2

    def verify_locate_correct(self, t, c1, c2, eps, row_eps_mult=None):
        """Repairs t in place (like the reference's Matrix&); returns the report dict."""
        rows, cols = t.shape
        stride = c1.shape[1]
        rep = VerifyReportC()
        mult = None
        if row_eps_mult is not None:
            mult = (C.c_double * rows)(*row_eps_mult)
        if self._vlc(rows, cols, stride, t, np.ascontiguousarray(c1, np.float32),
                     np.ascontiguousarray(c2, np.float32), eps, mult, C.byref(rep)):
            raise ValueError(self.last_error())
        return dict(status=STATUS[rep.status], row=rep.row, col=rep.col,
                    violations=rep.violations, corrections=rep.corrections,
                    checksum_repair=rep.checksum_repair, residual=rep.residual, delta=rep.delta)
