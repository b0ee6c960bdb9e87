"""CPU, world_size 2 over gloo: the multi-GPU layout of SURVEY.md §8(e) — (batch x head) units
split contiguously over ranks with fault specs routed by head, FFN token rows split in 128-row
blocks with replicated weights — computed per rank (the CPU oracle stands in for the GPU kernel
here) and gathered: identical to the single-rank result, events included. Plus the
max-over-ranks timing reduction bench.py uses."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2504_02211_b200.shard import route_faults, shard_tokens, shard_units

SEQ, D, HEADS = 256, 64, 6
SPECS = ["EXP_OUT:1:0:5:7:30", "GEMM2_ACC:0:1:100:3:29", "GEMM1_OUT:1:1:64:90:22"]
SPEC_HEADS = [0, 3, 5]
TOKENS, K, N = 512, 128, 256


def test_shard_units_cover_and_balance():
    for n in (1, 7, 12, 256, 1024, 1025):
        for w in (1, 2, 4, 8):
            shards = [shard_units(n, w, r) for r in range(w)]
            assert shards[0].start == 0 and shards[-1].stop == n
            for a, b in zip(shards, shards[1:]):
                assert a.stop == b.start
            sizes = [s.count for s in shards]
            assert max(sizes) - min(sizes) <= 1


def test_shard_tokens_aligned():
    for w in (1, 2, 4, 8):
        sh = [shard_tokens(32768, w, r) for r in range(w)]
        assert sh[0].start == 0 and sh[-1].stop == 32768
        assert all(s.start % 128 == 0 and s.count % 128 == 0 for s in sh)


def test_route_faults():
    from paper_2504_02211_b200.attention import FaultSpec
    specs = [FaultSpec.parse("EXP_OUT:0:1:2:3:30", head=h) for h in (0, 5, 6, 11)]
    s = shard_units(12, 2, 1)  # heads 6..11
    local = route_faults(specs, s)
    assert [f.head for f in local] == [0, 5]


def _inputs(h):
    from helpers import oracle
    orc = oracle()
    q, k, v, _ = orc.gen_trial(orc.trial_seed(99, h), SEQ, D, 128, 8)
    return q, k, v


def _specs():
    from paper_2504_02211_b200.attention import FaultSpec
    return [FaultSpec.parse(t, head=h) for t, h in zip(SPECS, SPEC_HEADS)]


def _heads_result(start, count, specs):
    """Run heads [start, start+count) with their routed (local) specs; return global records."""
    from helpers import oracle
    orc = oracle()
    out = []
    thr = (1e-5, 1e-4, 1e-4)
    for i in range(count):
        q, k, v = _inputs(start + i)
        mine = [f.as_tuple() for f in specs if f.head == i]
        r = orc.efta_forward(q, k, v, 128, 8, mode="efta-opt", thr=thr, specs=mine)
        ev = sorted((start + i, e["kind"], e["block_i"], e["block_j"], e["status"], e["row"], e["col"])
                    for e in r.detected_events())
        out.append((start + i, r.o.tobytes(), ev, len(r.fired)))
    return out


def _ffn_rows(start, count):
    from helpers import oracle
    orc = oracle()
    x = orc.random_matrix(7, TOKENS, K)[start:start + count]
    w = orc.random_matrix(8, K, N)
    c, c1, c2 = orc.checksummed_gemm(x, w, 8)
    return [(start + r, c[r].tobytes(), c1[r].tobytes(), c2[r].tobytes()) for r in range(count)]


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_02211_b200.shard import gather_units, max_over_ranks, route_faults, shard_tokens, shard_units
    sh = shard_units(HEADS, world, rank)
    local = route_faults(_specs(), sh)
    att = gather_units(_heads_result(sh.start, sh.count, local), dist)
    ts = shard_tokens(TOKENS, world, rank)
    ffn = gather_units(_ffn_rows(ts.start, ts.count), dist)
    t = max_over_ranks(10.0 + rank, dist, device="cpu")
    dist.barrier()
    if rank == 0:
        q.put((att, ffn, t, (sh.start, sh.count)))
    dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_two_rank_gloo_shards_compute_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    att, ffn, t, sh0 = q.get(timeout=170)
    for p in ps:
        p.join(30)
    assert sh0 == (0, 3)
    # single-rank reference: all heads, global specs (local index == global index)
    single = _heads_result(0, HEADS, _specs())
    assert [a[0] for a in att] == list(range(HEADS))
    assert att == single  # outputs bit for bit, events (with global heads), fired counts
    assert sum(a[3] for a in att) == len(SPECS) and sum(len(a[2]) > 0 for a in att) >= 2
    assert ffn == _ffn_rows(0, TOKENS)
    assert t == 11.0
