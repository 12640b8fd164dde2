"""Multi-GPU host logic on CPU: balanced factor partition + world_size-2 gloo gather of the
per-factor blocks to rank 0 (the N>1 path of bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2109_07073_b200.sharding import gather_blocks, partition_factors


def test_partition_tiles_and_balances():
    rng = np.random.default_rng(0)
    counts = rng.integers(15000, 20001, size=4445)
    for world in (1, 2, 3, 4, 8):
        parts = partition_factors(counts, world)
        assert parts[0][0] == 0 and parts[-1][1] == len(counts)
        for a, b in zip(parts, parts[1:]):
            assert a[1] == b[0]
        loads = [counts[b:e].sum() for b, e in parts]
        assert max(loads) - min(loads) <= 2 * counts.max()
    assert partition_factors([], 3) == [(0, 0)] * 3
    assert partition_factors([5], 2) in ([(0, 1), (1, 1)], [(0, 0), (0, 1)])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, F, D, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    counts = [len(range(*p)) for p in partition_factors(np.full(F, 20000), world)]
    b, e = partition_factors(np.full(F, 20000), world)[rank]
    # stand-in for this rank's linearized blocks: row f holds f (global factor id)
    local = torch.arange(b, e, dtype=torch.float64)[:, None].repeat(1, D)
    out = gather_blocks(local, counts, dst=0)
    if rank == 0:
        q.put(out.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("F", [7, 4445])
def test_gloo_gather_world2(F):
    world, D = 2, 121
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, F, D, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got.shape == (F, D)
    assert np.array_equal(got[:, 0], np.arange(F, dtype=np.float64))
