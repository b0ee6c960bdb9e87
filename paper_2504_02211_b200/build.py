"""In-tree build of libefta_b200.so for sm_100a (nvcc, parallel per translation unit).

python -m paper_2504_02211_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build_prof" if os.environ.get("EFTA_PROF") == "1" else
                     (f"_build_{os.environ['EFTA_VARIANT']}" if os.environ.get("EFTA_VARIANT") else "_build"))
PROF = os.environ.get("EFTA_PROF") == "1"   # phase-timestamp build (tools/phase_prof.py)
VARIANT = os.environ.get("EFTA_VARIANT", "")  # experiment builds: extra -D flags, separate .so
LIB = os.path.join(PKG, "libefta_b200_prof.so" if PROF else
                   (f"libefta_b200_{VARIANT}.so" if VARIANT else "libefta_b200.so"))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr"] + (["-DEFTA_PROF"] if os.environ.get("EFTA_PROF") == "1" else []) + \
        os.environ.get("EFTA_DEFS", "").split()

# translation units: (source, extra defines) — the attention instantiations are
# split per head dim so they compile in parallel
UNITS = [
    ("efta_capi.cu", []),
    ("efta_attn_inst.cu", ["-DEFTA_INST_D=64"]),
    ("efta_attn_inst.cu", ["-DEFTA_INST_D=128"]),
    ("efta_attn_inst.cu", ["-DEFTA_INST_D=64", "-DEFTA_INST_INJ=1"]),
    ("efta_attn_inst.cu", ["-DEFTA_INST_D=128", "-DEFTA_INST_INJ=1"]),
    ("efta_attn_inst.cu", ["-DEFTA_INST_D=64", "-DEFTA_INST_CAUSAL=1"]),
    ("efta_attn_inst.cu", ["-DEFTA_INST_D=128", "-DEFTA_INST_CAUSAL=1"]),
    ("abft_gemm.cu", []),
    ("abft_verify.cu", []),
    ("efta_host.cu", []),
    ("decoupled.cu", []),
    ("decode.cu", []),
    ("elementwise.cu", []),
]


def _deps():
    files = []
    for d in (CSRC, os.path.join(PKG, "..", "include")):
        for f in os.listdir(d):
            if f.endswith((".cu", ".cuh", ".h", ".hpp")):
                files.append(os.path.join(d, f))
    return files


def _obj(src, defs):
    tag = "_".join(x[2:].replace("EFTA_INST_", "").replace("=", "") for x in defs) or "base"
    return os.path.join(BUILD, f"{os.path.splitext(src)[0]}_{tag}.o")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _deps())


def _compile(src, defs, log, force=False):
    obj = _obj(src, defs)
    if not force and os.path.exists(obj):
        t = os.path.getmtime(obj)
        if all(os.path.getmtime(f) <= t for f in _deps()):
            return obj
    cmd = [NVCC, *ARCH, *FLAGS, *defs, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src} {defs}:\n{r.stderr[-4000:]}")
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    units = [(s, d) for s, d in UNITS if os.path.exists(os.path.join(CSRC, s))]
    with cf.ThreadPoolExecutor(max_workers=len(units)) as ex:
        futs = [ex.submit(_compile, s, d, _obj(s, d) + ".log", force) for s, d in units]
        objs = [f.result() for f in futs]
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-lcuda", "-lcublas",
           "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
