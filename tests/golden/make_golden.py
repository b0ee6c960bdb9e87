"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED reference
(oracle/_ref/libefta_ref.so, built by oracle/Makefile from /root/reference).

Run in the build container (where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py
The fixtures are small .npz files; they pin the oracle restatement
(oracle/efta_oracle.c) on machines that cannot build the reference.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from oracle import Oracle  # noqa: E402

EVENT_KEYS = ("kind", "block_i", "block_j", "status", "row", "col", "violations", "corrections")

# (name, seq, d, block, stride, mode, thresholds, fault specs)
CASES = [
    ("c1_head_none", 256, 64, 128, 8, "none", (7e-6, 0.48, 0.48), []),
    ("c1_head_opt", 256, 64, 128, 8, "efta-opt", (1e-5, 1e-4, 1e-4), []),
    ("d128_head_opt", 256, 128, 128, 8, "efta-opt", (1e-5, 1e-4, 1e-4), []),
    # the reference unit test's fixed single faults (tests/test_efta.cpp:107-173), N=64 d=32 B=16
    *[(f"kat_{s.split(':')[0].lower()}_{i}", 64, 32, 16, 8, "efta-opt", (7e-6, 1e-4, 1e-4), [s])
      for i, s in enumerate(["GEMM1_OUT:1:2:3:4:30", "SUB_MAX:0:1:5:6:31", "EXP_OUT:2:1:7:8:31",
                             "REDUCE_MAX:1:1:2:0:30", "REDUCE_MAX:1:2:2:0:29",
                             "REDUCE_SUM:0:3:4:0:30", "RESCALE_FACTOR:3:1:2:9:31",
                             "GEMM2_ACC:2:2:8:10:30", "NORMALIZE_OUT:1:0:3:12:22"])],
    # the same sites at the GPU geometry (block 128), C1 head shape
    *[(f"b128_{s.split(':')[0].lower()}", 512, 64, 128, 8, "efta-opt", (1e-5, 1e-4, 1e-4), [s])
      for s in ["GEMM1_OUT:1:2:3:4:30", "EXP_OUT:2:1:7:8:31", "GEMM2_ACC:2:2:8:10:30",
                "REDUCE_SUM:0:3:4:0:30", "NORMALIZE_OUT:1:0:3:12:22"]],
]


def main():
    ref = Oracle("ref")
    index = {}
    for name, n, d, b, s, mode, thr, specs in CASES:
        seed = 99 if name.startswith("kat") else ref.trial_seed(4242, len(index))
        q, k, v, _ = ref.gen_trial(seed, n, d, b, s)
        res = ref.efta_forward(q, k, v, b, s, mode=mode, thr=thr, specs=specs)
        ev = np.array([[e[k_] if not isinstance(e[k_], str) else
                        (["score_checksum", "exp_checksum", "factor_range", "rowsum_range",
                          "output_checksum"].index(e[k_]) if k_ == "kind" else
                         ["clean", "corrected", "detected_uncorrectable", "nonfinite"].index(e[k_]))
                        for k_ in EVENT_KEYS] for e in res.events], dtype=np.int32).reshape(-1, len(EVENT_KEYS))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), seed=np.uint64(seed), o=res.o,
                            m=res.m, l=res.l, events=ev,
                            summary=np.array([res.detections, res.corrections, res.recomputes,
                                              res.range_replacements, int(res.failed)], np.int32))
        index[name] = dict(seq=n, d=d, block=b, stride=s, mode=mode, thr=list(thr), specs=specs,
                           seed=int(seed))
    with open(os.path.join(HERE, "index.json"), "w") as fh:
        json.dump(index, fh, indent=1)
    print(f"wrote {len(index)} fixtures")


if __name__ == "__main__":
    main()
