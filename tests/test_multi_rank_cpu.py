"""World-size-2 gloo tests of the replica (N > 1) host logic used by bench.py.

The path does not shard inside an image, so N GPUs run N replicas: these tests check the
rank bookkeeping, the barrier, the max-over-ranks time and the whole-job rate on CPU.
"""
import os
import socket

import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1707_02018_b200 import replicas
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        info = replicas.rank_info()
        assert (info.world, info.rank) == (world, rank)
        replicas.barrier(world)
        t = replicas.max_over_ranks(1.0 + rank, world)            # rank 1 is the slow one
        rate = replicas.whole_job_rate(4.0, 0.5 + 0.5 * rank, world)   # 4 images per rank
        sh = list(replicas.shard(7, world, rank))
        q.put((rank, t, rate, sh))
    finally:
        dist.destroy_process_group()


def test_replicas_world2_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    for rank, t, rate, _ in res:
        assert t == 2.0                       # max over ranks, seen identically on both
        assert rate == pytest.approx(8.0 / 1.0)   # 8 images over the slowest rank's 1.0 s
    shards = [s for *_, s in res]
    assert shards[0] + shards[1] == list(range(7))


@pytest.mark.parametrize("n,world", [(0, 1), (1, 2), (4, 4), (5, 2), (8, 3), (16, 8)])
def test_shard_partitions_units(n, world):
    from paper_1707_02018_b200 import replicas
    seen = []
    sizes = []
    for r in range(world):
        s = replicas.shard(n, world, r)
        seen.extend(s)
        sizes.append(len(s))
    assert seen == list(range(n))
    assert max(sizes) - min(sizes) <= 1


def test_shard_rejects_bad_args():
    from paper_1707_02018_b200 import replicas
    with pytest.raises(ValueError):
        replicas.shard(4, 2, 2)
    with pytest.raises(ValueError):
        replicas.shard(-1, 2, 0)


def test_single_rank_is_identity():
    from paper_1707_02018_b200 import replicas
    assert replicas.max_over_ranks(3.5, 1) == 3.5
    assert replicas.whole_job_rate(4, 2.0, 1) == 2.0
