"""FT-Transformer layer (arXiv 2504.02211 Fig. 1 / SURVEY.md §8(f) F1): every linear module
through the strided-ABFT tcgen05 GEMM, attention through the fused EFTA kernel.

    layer = FTTransformerLayer(d_model=1280, n_heads=20, d_ff=5120)   # GPT-2-large shapes
    y = layer(x)                  # x: CUDA fp16 [batch, seq, d_model] -> y fp16
    rep = layer.report()          # merged FT outcome of the 4 GEMMs + attention

Structure (the paper applies strided ABFT to "all linear modules"):
    qkv = X Wqkv^T      (AbftLinear, N = 3 d_model)
    O   = EFTA(Q, K, V) (EftaAttention, EFTA-optimized)
    h   = X + O Wo^T    (AbftLinear)
    y   = h + GELU(h W1^T) W2^T   (AbftLinear x 2)
The head split and merge are epilogue layouts of the protected kernels (the QKV GEMM writes
[3, batch, heads, seq, head_dim], the attention writes fp16 token-major O) and the residual adds
and GELU are epilogue ops of the protected GEMMs, applied to the verified values
(fused_layout=False: the same layer with torch copies and element-wise ops, bit-identical).
No normalisation layers: the reference protects only the GEMMs and the attention.
The GELU is csrc/elementwise.cu's HBM-bound pass (bit-identical to F.gelu; in the ff1 epilogue
it measured slower, fused_gelu=True). `protect=False` builds the unprotected twin of the same
layer (cuBLAS linears with the residual adds as beta = 1 epilogues, the same GELU pass, the same
attention kernel in mode NONE with the fp16 token-major output, a torch head-split copy) for the
FT-overhead comparison.
"""
from __future__ import annotations

import math

import torch

from .attention import EftaAttention, FTReport, Thresholds
from .ffn import AbftLinear, gelu_


def _weight(n, k, gen, device):
    w = torch.empty((n, k), dtype=torch.float32, device=device).uniform_(-1.0, 1.0, generator=gen)
    return (w / math.sqrt(k)).to(torch.float16)


class FTTransformerLayer:
    def __init__(self, d_model=1280, n_heads=20, d_ff=5120, protect=True, thr=None, gemm_eps=1e-2,
                 seed=0, device="cuda", fused_layout=True, fused_gelu=False):
        if d_model % n_heads:
            raise ValueError("d_model must be a multiple of n_heads")
        self.d_model, self.n_heads, self.d_ff = d_model, n_heads, d_ff
        self.head_dim = d_model // n_heads
        self.protect = protect
        self.fused_layout = fused_layout  # False: the head split / merge as torch copies (A/B)
        self.fused_gelu = fused_gelu      # True: GELU in the ff1 epilogue (measured slower: erff in the epilogue warps)
        self.thr = thr or Thresholds(1e-4, 1e-3, 1e-3)
        gen = torch.Generator(device=device)
        gen.manual_seed(seed)
        self.w = {name: _weight(n, k, gen, device)
                  for name, (n, k) in (("qkv", (3 * d_model, d_model)), ("o", (d_model, d_model)),
                                       ("ff1", (d_ff, d_model)), ("ff2", (d_model, d_ff)))}
        self.lin = {name: AbftLinear(w, eps=gemm_eps) for name, w in self.w.items()} if protect else None
        self._attn = {}

    def _linear(self, name, x):
        if self.protect:
            return self.lin[name](x)
        return x @ self.w[name].t()

    def _attention(self, b, s):
        key = (b, s)
        if key not in self._attn:
            # the fp16 token-major O output runs on the CTA-pair kernel (even seq / 128 blocks)
            tok = self.fused_layout and (s // 128) % 2 == 0
            self._attn[key] = EftaAttention(b, self.n_heads, s, self.head_dim,
                                            mode="efta-opt" if self.protect else "none", thr=self.thr,
                                            device=self.w["o"].device, token_major_out=tok)
        return self._attn[key]

    def flops(self, b, s):
        t = b * s
        lin = 2.0 * t * (4 * self.d_model * self.d_model + 2 * self.d_model * self.d_ff)
        return lin + 4.0 * b * self.n_heads * s * s * self.head_dim

    def __call__(self, x: torch.Tensor) -> torch.Tensor:
        b, s, d = x.shape
        t = b * s
        x2 = x.reshape(t, d)
        attn = self._attention(b, s)
        split = (s, self.n_heads, self.head_dim)
        if self.protect and attn.token_major_out:
            # the QKV GEMM's epilogue writes [3, b, h, s, dh] and the attention's epilogue fp16
            # token-major O [b, s, h, dh] = the O projection's input: no head split / merge copies
            qkv = self.lin["qkv"](x2, head_split=split)
        else:
            qkv = self._linear("qkv", x2)                               # [t, 3d] (cuBLAS twin)
            qkv = qkv.view(b, s, 3, self.n_heads, self.head_dim).permute(2, 0, 3, 1, 4).contiguous()
        o, _, _ = attn(qkv[0], qkv[1], qkv[2])
        if attn.token_major_out:
            o = o.view(t, d)                                            # fp16, already token-major
        else:
            o = o.to(torch.float16).permute(0, 2, 1, 3).reshape(t, d)  # [b, h, s, dh] fp32
        if self.fused_layout and self.protect:
            # residual adds and GELU in the protected GEMMs' epilogues (after verification)
            h = self.lin["o"](o, residual=x2)
            f1 = self.lin["ff1"](h, activation="gelu") if self.fused_gelu else gelu_(self.lin["ff1"](h))
            return self.lin["ff2"](f1, residual=h).view(b, s, d)
        if self.fused_layout:
            # unprotected twin: the residual adds as cuBLAS beta = 1 epilogues
            h = torch.addmm(x2, o, self.w["o"].t())
            f1 = gelu_(h @ self.w["ff1"].t())
            return torch.addmm(h, f1, self.w["ff2"].t()).view(b, s, d)
        h = x2 + self._linear("o", o)
        f = self._linear("ff2", torch.nn.functional.gelu(self._linear("ff1", h)))
        return (h + f).view(b, s, d)

    def report(self) -> FTReport:
        rep = FTReport(mode="layer")
        parts = [a.report() for a in self._attn.values()]
        if self.protect:
            parts += [lin.report() for lin in self.lin.values()]
        for r in parts:
            rep.events += r.events
            rep.detections += r.detections
            rep.corrections += r.corrections
            rep.recomputes += r.recomputes
            rep.range_replacements += r.range_replacements
            rep.failed = rep.failed or r.failed
        return rep
