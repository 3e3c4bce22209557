"""Multi-process host logic of the env-sharded path on CPU (gloo, world_size 2)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_15352_b200.dist import env_slice, fold_digests, gather_stats, max_over_ranks


def test_env_slice_partitions():
    for n in (0, 1, 7, 4096, 32768, 32771):
        for world in (1, 2, 3, 8):
            parts = [env_slice(n, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        env_slice(10, 2, 2)


def test_fold_is_order_dependent_and_deterministic():
    d = [3, 0xFFFFFFFFFFFFFFFF, 12345678901234567, 0]
    assert fold_digests(d) == fold_digests(list(d))
    assert fold_digests(d) != fold_digests(d[::-1])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_total = 10
        a, b = env_slice(n_total, world, rank)
        # per-env digests of a fake render: a pure function of the global env index
        digests = [(e * 0x9E3779B97F4A7C15 + 7) & 0xFFFFFFFFFFFFFFFF for e in range(a, b)]
        frames = (b - a) * 3
        elapsed = 1000 + 500 * rank
        total, tmax, digs = gather_stats(frames, fold_digests(digests), elapsed)
        m = max_over_ranks(float(rank) + 0.5)
        q.put((rank, total, tmax, digs, m))
    finally:
        dist.destroy_process_group()


def test_gather_stats_gloo_two_ranks():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    for rank, total, tmax, digs, m in out:
        assert total == 10 * 3
        assert tmax == 1500
        assert m == 1.5
        # rank-sliced digests equal per-slice folds of the single-process digest list
        ref = [(e * 0x9E3779B97F4A7C15 + 7) & 0xFFFFFFFFFFFFFFFF for e in range(10)]
        assert digs == [fold_digests(ref[:5]), fold_digests(ref[5:])]


def test_single_process_passthrough():
    assert not dist.is_initialized()
    assert gather_stats(5, 42, 100) == (5, 100, [42])
    assert max_over_ranks(2.5) == 2.5
