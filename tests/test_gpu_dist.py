"""Multi-rank determinism of the env-sharded path on the GPU (-m gpu).

SURVEY §8(e) checks, made real: bench.py run as 2 ranks (torchrun, gloo for
the host collectives: both ranks share the one B200 of this pool, and no
kernel of either rank waits on the other) renders envs [0, E) and [E, 2E) of
one global env set; the per-env digests of both ranks, folded in global env
order, must equal a single-process render of all 2E envs.  That is both
checks at once: a rank-sliced run equals a 1-GPU run, and an env rendered on
another rank (env E.. on rank 1 here, on rank 0 in the 1-process run) gives
the same bits.  The multi-scene case also exercises the C3 scene broadcast
(rank 0 generates, rank 1 receives).
"""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench(args, nproc=1):
    base = [sys.executable, "bench.py"] + args + ["--steps", "1", "--warmup", "1", "--no-e2e", "--no-cpu"]
    if nproc > 1:
        base = ([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
                 "--master-addr", "127.0.0.1", f"--master-port={_port()}"] + base[1:] + ["--dist-backend", "gloo"])
    r = subprocess.run(base, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")][-1]
    return json.loads(line)


@pytest.mark.parametrize("cfg", [["--config", "c3", "--gaussians", "200000"],
                                 ["--config", "c4", "--scenes", "6", "--gaussians", "100000"]])
def test_rank_sliced_digest_equals_single_process(cfg):
    one = _bench(cfg + ["--envs", "64"])
    two = _bench(cfg + ["--envs", "32"], nproc=2)
    assert one["config"]["total_envs"] == two["config"]["total_envs"] == 64
    assert two["n_gpus"] == 2
    assert one["digest"] == two["digest"], (one["digest"], two["digest"])
