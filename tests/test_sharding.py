"""CPU, world_size 2 over gloo: the N>1 bench path -- stream sharding with no
data-path collective, max-over-ranks timing, per-rank independence of the
codec (each rank's streams reproduce the single-process results)."""

import hashlib
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2602_03529_b200.shard import rank_streams, strong_streams


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import hashlib

    import torch
    import torch.distributed as dist
    from oracle import semstream_oracle as O
    from oracle.synth import make_clip
    from paper_2602_03529_b200.shard import max_over_ranks, rank_streams

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = rank_streams(rank, world, 2)
    digests = {}
    for sid in mine:
        clip = make_clip("moving-square", 48, 40, 9, seed=sid)
        res = O.pipeline_gop(clip.gop(0), 2 + sid % 2, gop_id=0, drop_rate=0.1)
        digests[sid] = hashlib.sha256(np.stack(res["frames"]).tobytes()).hexdigest()
    ms = max_over_ranks(10.0 + 5.0 * rank)
    dist.barrier()
    q.put((rank, mine, digests, ms))
    dist.destroy_process_group()


def test_two_rank_sharding_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort()
    assert got[0][1] == [0, 1] and got[1][1] == [2, 3]          # disjoint, weak scaling
    assert all(r[3] == 15.0 for r in got)                       # max over ranks
    # each rank's streams equal a single-process run of the same streams
    from oracle import semstream_oracle as O
    from oracle.synth import make_clip
    for _, mine, digests, _ in got:
        for sid in mine:
            clip = make_clip("moving-square", 48, 40, 9, seed=sid)
            res = O.pipeline_gop(clip.gop(0), 2 + sid % 2, gop_id=0, drop_rate=0.1)
            assert digests[sid] == hashlib.sha256(np.stack(res["frames"]).tobytes()).hexdigest()


def test_shard_helpers():
    assert rank_streams(1, 4, 3) == [3, 4, 5]
    assert sorted(sum((strong_streams(r, 4, 10) for r in range(4)), [])) == list(range(10))
    with pytest.raises(ValueError):
        rank_streams(4, 4, 1)
