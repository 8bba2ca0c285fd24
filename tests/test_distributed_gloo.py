"""World-size-2 gloo run of the sharded batch (row blocks + gather + mirror),
with the pinned CPU oracle as the per-rank compute function (the CUDA compute
is covered by the gpu tests; here the host-side multi-process logic is)."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

REPO = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, tri, q, count=11):
    sys.path.insert(0, str(REPO))
    import torch.distributed as dist

    from oracle import oracle as orc
    from paper_2007_16135_b200.distributed import sharded_batch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(3)
    series = [(rng.standard_normal((int(n), 2)), np.arange(int(n), dtype=float))
              for n in rng.integers(1, 40, size=count)]

    def compute(b0, b1):
        block = np.zeros((b1 - b0, len(series)))
        for li, i in enumerate(range(b0, b1)):
            for j in range(i if tri else 0, len(series)):
                a, b = series[i], series[j]
                block[li, j] = orc.twed(a[0], a[1], b[0], b[1], 0.5, 0.25, 2)
        return block

    full = sharded_batch(len(series), len(series), tri, compute)
    if rank == 0:
        want = orc.twed_batch(series, None, 0.5, 0.25, 2, symmetric=tri, threads=1)
        q.put(bool(np.array_equal(full.numpy(), want)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,count", [(2, 11), (3, 11), (3, 2)])
@pytest.mark.parametrize("tri", [False, True])
def test_sharded_batch(world, count, tri):
    """Ragged series, unequal row blocks (and an empty block when there are
    fewer rows than ranks); every rank sends exactly its rows to rank 0."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, tri, q, count)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
