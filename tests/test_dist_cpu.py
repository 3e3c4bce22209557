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


def _digest(a) -> int:
    import hashlib
    return int.from_bytes(hashlib.blake2b(a.tobytes(), digest_size=7).digest(), "little")


def _stream_worker(rank, world, port, q):
    """bench.scene_stream over gloo: rank 0 generates and broadcasts the scenes
    (C3), rank 1 receives them and places its own envs' cameras."""
    import sys
    import numpy as np
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    import gg_inputs as gi
    from paper_2510_15352_b200.dist import gather_env_digests
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        E = 24
        wl = gi.Workload("c4", n_envs=E * world, n_sets=2, env_range=(rank * E, (rank + 1) * E), n_scenes=3,
                         n_gauss=1500, sh_degree=1)
        cpu = torch.device("cpu")
        sums = [float(sum(float(x.double().sum()) for x in arrs[:5])) for _, arrs in
                bench.scene_stream(wl, rank, world, cpu, cpu)]
        # per-env "digests" that are a function of the env's inputs only
        dig = torch.tensor([_digest(wl.viewmats[:, e]) for e in range(E)], dtype=torch.int64)
        q.put((rank, sums, wl.viewmats.copy(), wl.binding.copy(), gather_env_digests(dig)))
    finally:
        dist.destroy_process_group()


def test_scene_broadcast_and_global_env_slices_gloo():
    """Rank-sliced inputs of a 2-rank run equal the single-process workload's
    (every input is a function of the global env index), the broadcast scenes
    equal the generated ones, and the gathered per-env digests come back in
    global env order (SURVEY §8(e) determinism checks, C3 scene broadcast)."""
    import numpy as np
    import gg_inputs as gi
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_stream_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = gi.Workload("c4", n_envs=48, n_sets=2, n_scenes=3, n_gauss=1500, sh_degree=1)
    ref_sums = [float(sum(float(np.asarray(a, np.float64).sum()) for a in
                          (sc.means, sc.scales, sc.quats, sc.opacities, sc.sh))) for _, sc in full.scenes(n_proc=1)]
    for rank, sums, vm, binding, digs in out:
        assert sums == ref_sums
        assert np.array_equal(vm, full.viewmats[:, rank * 24:(rank + 1) * 24])
        assert np.array_equal(binding, full.binding[rank * 24:(rank + 1) * 24])
    assert out[0][4] == out[1][4]                  # both ranks see all digests, rank (= global env) order
    ref_dig = [_digest(full.viewmats[:, e]) for e in range(48)]
    assert out[0][4] == ref_dig
