"""GPU decoupled FT baseline (csrc/decoupled.cu) against the reference's own
decoupled_ft_forward (src/decoupled.cpp:98-282, compiled into oracle/_ref): three kernels with
the N^2 intermediates in HBM, traditional two-sided block checksums, DMR softmax.

Parity contract: outputs within the north_star tolerance; per fault, the same outcome
(fired, detected, failed) and the same non-CLEAN events (kind, block_i, block_j, status,
row, col) as the reference for upsets far above the detection thresholds (bit 30 / 31 / 29
flips), the reference test's single-fault cases (tests/test_efta.cpp:277-313) re-run at the
B=128 tile geometry."""
import os

import numpy as np
import pytest

from helpers import head_inputs, rel_err

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "libefta_ref.so")
TOL = 1e-2
# the reference test's thresholds for the decoupled baseline (tests/test_efta.cpp:281)
THR = (7e-6, 1e-3, 5e-3)


def _ref():
    from oracle import Oracle
    if not os.path.exists(REF):
        pytest.fail("oracle/_ref/libefta_ref.so missing: build it with `make -C oracle` where "
                    "/root/reference exists (it travels with the repo snapshot)")
    return Oracle("ref")


def _dev(x):
    import torch
    return torch.from_numpy(x).to(torch.float16).cuda().contiguous()


def _events(evs):
    return sorted((e["kind"], e["block_i"], e["block_j"], e["status"], e["row"], e["col"])
                  for e in evs if e["status"] != "clean")


@pytest.mark.parametrize("d,seq,heads", [(64, 512, 12), (128, 512, 3), (64, 1024, 2), (128, 256, 4)])
def test_decoupled_clean_matches_reference(d, seq, heads):
    from paper_2504_02211_b200 import Thresholds, efta_forward
    q, k, v, _ = head_inputs(4321 + d + seq, heads, seq, d)
    o, rep = efta_forward(_dev(q), _dev(k), _dev(v), mode="decoupled", thr=Thresholds(*THR))
    o = o.cpu().numpy()
    m = rep.final_m.cpu().numpy()
    l = rep.final_l.cpu().numpy()
    ref = _ref()
    for h in range(heads):
        r = ref.efta_forward(q[h], k[h], v[h], 128, 8, mode="decoupled", thr=THR)
        assert rel_err(o[h], r.o) <= TOL, (h, rel_err(o[h], r.o))
        assert np.allclose(m[h], r.m, rtol=1e-5, atol=1e-5)
        assert np.allclose(l[h], r.l, rtol=1e-4)
    assert rep.detections == 0, rep.events[:4]
    assert not rep.failed


FAULTS = [
    # tests/test_efta.cpp:277-313 (re-targeted to B=128 coordinates)
    "GEMM1_OUT:0:1:2:3:30", "EXP_OUT:1:1:3:4:30", "REDUCE_SUM:2:0:5:0:30", "GEMM2_ACC:1:0:2:7:30",
    # every other site the decoupled pipeline taps, large upsets
    "NORMALIZE_OUT:1:0:3:12:30", "SUB_MAX:1:2:3:4:30", "REDUCE_MAX:1:0:3:0:30",
    "GEMM1_OUT:3:0:127:127:31", "GEMM1_OUT:2:3:64:5:29", "GEMM2_ACC:3:0:0:63:31",
    "EXP_OUT:0:3:100:90:29", "NORMALIZE_OUT:2:0:10:50:31",
    # a fault on the second evaluation of the duplicated softmax (trigger 2): the reference
    # compares evaluation 2 with evaluation 3 and declares the row uncorrectable
    "EXP_OUT:1:1:3:4:30:2",
]


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("spec", FAULTS)
def test_decoupled_fault_outcome_matches_reference(d, spec):
    from paper_2504_02211_b200 import FaultSpec, Thresholds, efta_forward
    seq = 512
    q, k, v, _ = head_inputs(99 + d, 1, seq, d)
    ref = _ref()
    clean = ref.efta_forward(q[0], k[0], v[0], 128, 8, mode="decoupled", thr=THR)
    r = ref.efta_forward(q[0], k[0], v[0], 128, 8, mode="decoupled", thr=THR, specs=[spec])
    f = FaultSpec.parse(spec, head=0)
    o, rep = efta_forward(_dev(q), _dev(k), _dev(v), mode="decoupled", thr=Thresholds(*THR), faults=[f])
    o = o.cpu().numpy()[0]
    assert len(rep.fired) == len(r.fired) == 1
    assert (rep.detections > 0) == (r.detections > 0)
    assert rep.failed == r.failed, (rep.events, r.events)
    assert _events(rep.events) == _events(r.events), (_events(rep.events), _events(r.events))
    if not r.failed:
        # repaired: the output equals the clean run within the tolerance
        assert rel_err(o, clean.o) <= TOL


def test_decoupled_many_heads_and_chunks(monkeypatch):
    """More heads than one workspace chunk holds (EFTA_DECOUPLED_CHUNK_MB shrinks the chunk to
    one head): the host loop over head chunks (csrc/decoupled.cu forward) covers every head;
    two faults on different heads are both repaired and reported against their flat index."""
    import torch
    monkeypatch.setenv("EFTA_DECOUPLED_CHUNK_MB", "40")
    from paper_2504_02211_b200 import FaultSpec, Thresholds, efta_forward
    heads, seq, d = 6, 2048, 64
    q, k, v, _ = head_inputs(2024, heads, seq, d)
    faults = [FaultSpec.parse("GEMM1_OUT:3:7:11:12:30", head=1), FaultSpec.parse("GEMM2_ACC:9:0:5:6:30", head=4)]
    o, rep = efta_forward(_dev(q), _dev(k), _dev(v), mode="decoupled", thr=Thresholds(*THR), faults=faults)
    o0, rep0 = efta_forward(_dev(q), _dev(k), _dev(v), mode="efta-opt", thr=Thresholds(1e-4, 1e-3, 1e-3))
    assert not rep.failed and rep.detections == 2, rep.events
    assert sorted(e["head"] for e in rep.events) == [1, 4]
    assert rel_err(o.cpu().numpy(), o0.cpu().numpy()) <= TOL
    torch.cuda.synchronize()
