"""CPU, world_size 2 over gloo: the multi-GPU host logic (batch x head sharding,
fault routing, max-over-ranks timing) that bench.py and the campaign use."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2504_02211_b200.shard import route_faults, shard_units


def test_shard_units_cover_and_balance():
    for n in (1, 7, 12, 256, 1024, 1025):
        for w in (1, 2, 4, 8):
            shards = [shard_units(n, w, r) for r in range(w)]
            assert shards[0].start == 0 and shards[-1].stop == n
            for a, b in zip(shards, shards[1:]):
                assert a.stop == b.start
            sizes = [s.count for s in shards]
            assert max(sizes) - min(sizes) <= 1


def test_route_faults():
    from paper_2504_02211_b200.attention import FaultSpec
    specs = [FaultSpec.parse("EXP_OUT:0:1:2:3:30", head=h) for h in (0, 5, 6, 11)]
    s = shard_units(12, 2, 1)  # heads 6..11
    local = route_faults(specs, s)
    assert [f.head for f in local] == [0, 5]


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_02211_b200.shard import max_over_ranks, shard_units
    sh = shard_units(1024, world, rank)
    t = max_over_ranks(10.0 + rank, dist, device="cpu")
    dist.barrier()
    q.put((rank, sh.start, sh.count, t))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_gloo_sharding_and_max_timing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=100) for _ in ps)
    for p in ps:
        p.join(30)
    assert res[0][1:3] == (0, 512) and res[1][1:3] == (512, 512)
    assert res[0][3] == res[1][3] == 11.0
