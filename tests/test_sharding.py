"""Multi-GPU host logic on CPU: balanced factor partition, world_size-2 gloo gather of the
per-factor blocks to rank 0 (the N>1 path of bench.py), and the sharded LM with
the CPU oracle standing in for each rank's GPU graph."""
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


class _OracleShard:
    """A rank's factor range served by the CPU oracle (stand-in for its FactorGraph)."""

    def __init__(self, frames, maps, ij):
        self.frames, self.maps, self.ij = frames, maps, np.asarray(ij).reshape(-1, 2)

    def linearize_raw(self, poses):
        import oracle_ctypes as O

        out = np.zeros((len(self.ij), 121))
        inl = np.zeros(len(self.ij), np.int32)
        for f, (i, j) in enumerate(self.ij):
            r = O.linearize(*self.frames[j], self.maps[i], poses[i], poses[j])
            out[f], inl[f] = r["raw"], r["inliers"]
        return out, inl

    def evaluate(self, poses):
        import oracle_ctypes as O

        err = np.zeros(len(self.ij))
        inl = np.zeros(len(self.ij), np.int32)
        for f, (i, j) in enumerate(self.ij):
            err[f], inl[f] = O.evaluate(*self.frames[j], self.maps[i], poses[i], poses[j])
        return err, inl


def _lm_problem():
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import oracle_ctypes as O

    rng = O.Rng(77)
    base_m, base_c = rng.gaussian_cloud(1500, 6.0)
    frames, truth = [], []
    for k in range(5):
        T = rng.random_pose(0.02, 0.2) if k else O.IDENTITY.copy()
        # every frame observes the same structure from its own pose
        m, c = O.transform_cloud(base_m, base_c, O.inverse(T))
        frames.append((m.astype(np.float32).astype(np.float64), O.cov9(c.reshape(-1, 9))))
        truth.append(T)
    maps = [O.OracleMap(m, c, 1.0) for m, c in frames]
    ij = [(i, j) for j in range(1, 5) for i in range(j)]
    init = np.stack([O.compose(T, rng.random_pose(0.01, 0.05)) if k else T for k, T in enumerate(truth)])
    return frames, maps, ij, init


def _lm_worker(rank, world, port, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2109_07073_b200 import optimizer as LM
    from paper_2109_07073_b200.sharding import ShardedFactorGraph

    frames, maps, ij, init = _lm_problem()
    parts = partition_factors([len(frames[j][0]) for _, j in ij], world)
    b, e = parts[rank]
    g = ShardedFactorGraph(_OracleShard(frames, maps, ij[b:e]), ij, [p[1] - p[0] for p in parts], len(init))
    poses, rep = LM.optimize(g, init, settings=LM.LmSettings(max_iterations=5), device_assembly=False, gpu_solve=False)
    q.put((rank, poses, rep.iterations, rep.final_error))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_sharded_lm_matches_single_process():
    from paper_2109_07073_b200 import optimizer as LM

    frames, maps, ij, init = _lm_problem()
    single = _OracleShard(frames, maps, ij)

    class _Full:
        _ij = np.asarray(ij)
        num_poses = len(init)

        def linearize_raw(self, poses):
            return single.linearize_raw(poses)

        def total_error(self, poses):
            err, _ = single.evaluate(poses)
            return float(np.cumsum(err)[-1])

    ref_poses, ref = LM.optimize(_Full(), init, settings=LM.LmSettings(max_iterations=5), device_assembly=False,
                                 gpu_solve=False)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, poses, its, err in results:
        assert its == ref.iterations and err == ref.final_error  # identical decisions on every rank
        assert np.array_equal(poses, ref_poses)


@pytest.mark.gpu
def test_sharded_graph_with_gpu_factor_graph_world1():
    """ShardedFactorGraph around a GPU FactorGraph (world size 1, gloo): same LM as the bare graph."""
    import paper_2109_07073_b200 as V
    from paper_2109_07073_b200 import optimizer as LM
    from paper_2109_07073_b200.sharding import ShardedFactorGraph

    frames, maps, ij, init = _lm_problem()
    ctx = V.default_context(0)
    clouds = [V.PointCloud(m.astype(np.float32), V.cov6_from(c), ctx) for m, c in frames]
    gmaps = V.GaussianVoxelMap.build_batch(clouds, 1.0)
    graph = V.FactorGraph([V.MatchingCostFactor(i, j, clouds[j], gmaps[i]) for i, j in ij], len(init))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        sharded = ShardedFactorGraph(graph, ij, [len(ij)], len(init))
        p1, r1 = LM.optimize(sharded, init, settings=LM.LmSettings(max_iterations=5), device_assembly=False,
                             gpu_solve=False)
        p2, r2 = LM.optimize(graph, init, settings=LM.LmSettings(max_iterations=5), device_assembly=False,
                             gpu_solve=False)
    finally:
        dist.destroy_process_group()
    assert r1.iterations == r2.iterations and r1.final_error == r2.final_error
    assert np.array_equal(p1, p2)


class _OracleRankShare:
    """A rank's share served by the CPU oracle: blocks(poses) -> [count, 122] rows (block + inliers),
    the RankShare interface (stand-in for FactorGraph.create_range on the rank's GPU)."""

    device = "cpu"

    def __init__(self, frames, maps, ij):
        self.inner = _OracleShard(frames, maps, ij)

    def blocks(self, poses):
        raw, inl = self.inner.linearize_raw(poses.numpy())
        return torch.from_numpy(np.concatenate([raw, inl[:, None].astype(np.float64)], axis=1))


def _gathered_worker(rank, world, port, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2109_07073_b200 import optimizer as LM
    from paper_2109_07073_b200.sharding import GatheredGraph

    frames, maps, ij, init = _lm_problem()
    parts = partition_factors([len(frames[j][0]) for _, j in ij], world)
    b, e = parts[rank]
    g = GatheredGraph(_OracleRankShare(frames, maps, ij[b:e]), [p[1] - p[0] for p in parts], len(init), ij)
    if rank == 0:
        poses, rep = LM.optimize(g, init, settings=LM.LmSettings(max_iterations=5), device_assembly=False,
                                 gpu_solve=False)
        raw, inl = g.linearize_raw(poses)  # one more gathered step: the blocks themselves
        g.stop()
        q.put((poses, rep.iterations, rep.final_error, [(t.error, t.lam, t.accepted) for t in rep.trace], raw, inl))
    else:
        q.put(("served", g.serve()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_gathered_lm_world2_matches_single_process():
    """One process per device (the torchrun path): rank 1 serves its share's linearizations, rank 0
    gathers every step's blocks in factor order and runs the LM on them — the gathered blocks, the
    trace and the poses equal the single-process run bit for bit (world size 2, gloo)."""
    from paper_2109_07073_b200 import optimizer as LM

    frames, maps, ij, init = _lm_problem()
    single = _OracleShard(frames, maps, ij)

    class _Full:
        _ij = np.asarray(ij)
        num_poses = len(init)

        def linearize_raw(self, poses):
            return single.linearize_raw(poses)

        def total_error(self, poses):
            raw, _ = single.linearize_raw(poses)
            return float(np.cumsum(raw[:, 120])[-1])

    ref_poses, ref = LM.optimize(_Full(), init, settings=LM.LmSettings(max_iterations=5), device_assembly=False,
                                 gpu_solve=False)
    ref_raw, ref_inl = single.linearize_raw(ref_poses)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gathered_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    root = [r for r in results if not isinstance(r[0], str)][0]
    served = [r for r in results if isinstance(r[0], str)][0]
    poses, its, err, trace, raw, inl = root
    assert its == ref.iterations and err == ref.final_error
    assert trace == [(t.error, t.lam, t.accepted) for t in ref.trace]
    assert np.array_equal(poses, ref_poses)
    assert np.array_equal(raw, ref_raw) and np.array_equal(inl, ref_inl)
    assert served[1] >= ref.iterations + 1  # rank 1 linearized its share at every step
