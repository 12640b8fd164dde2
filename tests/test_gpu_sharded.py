"""Multi-GPU split of ONE graph behind the C ABI, exercised on one GPU: several
contexts on device 0 stand in for the devices of a box (the code path is the same — per-shard
streams, cross-stream events, the root's assembly kernel reading the shards' blocks through their
device pointers). Bar: bit-identical to the single-context graph — blocks, errors, assembled
systems and the native LM's trace and poses."""
import numpy as np
import pytest
import torch

import oracle_ctypes as O

V = pytest.importorskip("paper_2109_07073_b200")

pytestmark = pytest.mark.gpu


def _problem(ctxs, nframes=9, n=2500, seed=501):
    """The same clouds / maps replicated on every context; factors (j-d -> j) plus loop closures."""
    rng = O.Rng(seed)
    data = []
    for _ in range(nframes):
        m, c = rng.gaussian_cloud(n, 10.0)
        data.append((m.astype(np.float32), V.cov6_from(c)))
    links = [(j - d, j) for j in range(1, nframes) for d in (1, 2) if j - d >= 0] + [(nframes - 1, 0)]
    if nframes > 5:
        links.append((5, 1))
    lists = []
    for ctx in ctxs:
        clouds = V.PointCloud.upload_batch([d[0] for d in data], [d[1] for d in data], ctx)
        maps = V.GaussianVoxelMap.build_batch(clouds, [1.0] * nframes)
        lists.append([V.MatchingCostFactor(i, j, clouds[j], maps[i]) for i, j in links])
    poses = np.stack([rng.random_pose(0.05, 0.5) for _ in range(nframes)])
    return lists, poses


@pytest.fixture(scope="module")
def ctxs():
    return [V.default_context(0), V.Context(0), V.Context(0)]


def test_range_graphs_tile_the_full_graph(ctxs):
    lists, poses = _problem(ctxs[:1])
    full = V.FactorGraph(lists[0], len(poses))
    F = full.num_factors()
    ref_raw, ref_inl = full.linearize_raw(poses)
    ref_err, _ = full.evaluate(poses)
    for cuts in ([0, F], [0, 5, F], [0, 1, 7, 12, F]):
        raws, inls, errs = [], [], []
        for a, b in zip(cuts, cuts[1:]):
            g = V.FactorGraph.create_range(lists[0], len(poses), a, b - a)
            assert g.num_factors() == b - a
            r, i = g.linearize_raw(poses)
            raws.append(r), inls.append(i), errs.append(g.evaluate(poses)[0])
        assert np.array_equal(np.concatenate(raws), ref_raw) and np.array_equal(np.concatenate(inls), ref_inl)
        assert np.array_equal(np.concatenate(errs), ref_err)


@pytest.mark.parametrize("shards,copy", [(2, False), (3, False), (2, True)])
def test_sharded_graph_bit_identical(ctxs, monkeypatch, shards, copy):
    if copy:  # gather by peer copies instead of reading the shards' blocks in place
        monkeypatch.setenv("VGICP_SHARD_COPY", "1")
    use = ctxs[:shards]
    lists, poses = _problem(use)
    full = V.FactorGraph(lists[0], len(poses))
    sh = V.FactorGraph.sharded(lists, len(poses))
    assert sh.num_shards() == shards
    ranges = [sh.shard_range(r) for r in range(shards)]
    assert ranges[0][0] == 0 and sum(c for _, c in ranges) == full.num_factors()
    assert sh.num_points() == full.num_points()
    a, ai = full.linearize_raw(poses)
    b, bi = sh.linearize_raw(poses)
    assert np.array_equal(a, b) and np.array_equal(ai, bi)
    assert np.array_equal(full.evaluate(poses)[0], sh.evaluate(poses)[0])
    # device variants return root-device memory
    F = full.num_factors()
    dp = torch.from_numpy(np.ascontiguousarray(poses)).cuda()
    d1 = torch.empty((F, 121), dtype=torch.float64, device="cuda")
    d2 = torch.empty_like(d1)
    i1 = torch.empty(F, dtype=torch.int32, device="cuda")
    i2 = torch.empty_like(i1)
    torch.cuda.synchronize()
    full.linearize_device(dp.data_ptr(), d1.data_ptr(), i1.data_ptr())
    sh.linearize_device(dp.data_ptr(), d2.data_ptr(), i2.data_ptr())
    full.ctx.synchronize()
    sh.ctx.synchronize()
    assert torch.equal(d1, d2) and torch.equal(i1, i2)
    # assembled systems (the root reads the shards' blocks) and the linearization's errors
    fixed = np.zeros(len(poses), np.uint8)
    fixed[0] = 1
    full.assembly_plan(fixed)
    sh.assembly_plan(fixed)
    for x, y in zip(full.linearize_assembled(poses), sh.linearize_assembled(poses)):
        assert np.array_equal(x, y)
    assert np.array_equal(full.linearized_errors()[0], sh.linearized_errors()[0])
    # the native LM (vgicp_graph_optimize) on the sharded graph: the same trace and poses
    from paper_2109_07073_b200 import optimizer as LM

    monkeypatch.setenv("VGICP_LM_NO_HOST_BAND", "1")  # the device band solver on the root
    p1, r1 = LM.optimize_native(full, poses)
    p2, r2 = LM.optimize_native(sh, poses)
    assert [(t.error, t.lam, t.accepted) for t in r1.trace] == [(t.error, t.lam, t.accepted) for t in r2.trace]
    assert r1.reason == r2.reason and r1.final_error == r2.final_error and np.array_equal(p1, p2)


def test_assemble_external_blocks_equals_device_assembly(ctxs):
    """vgicp_graph_assemble_device over blocks produced elsewhere (here: the concatenated range
    graphs' blocks, as gathered over NCCL from the ranks) == linearize_assembled_device."""
    lists, poses = _problem(ctxs[:1])
    full = V.FactorGraph(lists[0], len(poses))
    plan = full.assembly_plan(np.eye(1, len(poses), dtype=np.uint8)[0])
    S, P = plan.num_slots, len(plan.pairs)
    F = full.num_factors()
    dp = torch.from_numpy(np.ascontiguousarray(poses)).cuda()
    a1 = torch.empty((S + P) * 36 + S * 6, dtype=torch.float64, device="cuda")
    a2 = torch.empty_like(a1)
    torch.cuda.synchronize()
    full.linearize_assembled_device(dp.data_ptr(), a1.data_ptr())
    full.ctx.synchronize()
    blocks = torch.empty((F, 121), dtype=torch.float64, device="cuda")
    inl = torch.empty(F, dtype=torch.int32, device="cuda")
    half = F // 2
    for a, b in ((0, half), (half, F)):
        g = V.FactorGraph.create_range(lists[0], len(poses), a, b - a)
        g.linearize_device(dp.data_ptr(), blocks[a:b].data_ptr(), inl[a:b].data_ptr())
        g.ctx.synchronize()
    full.assemble_device(blocks.data_ptr(), a2.data_ptr())
    full.ctx.synchronize()
    assert torch.equal(a1, a2)


def test_gathered_graph_nccl_world1_matches_graph(ctxs):
    """The torchrun path (sharding.GatheredGraph over NCCL) at world size 1 on this GPU: RankShare
    (create_range) + the gather + the root's assembly of the gathered blocks give the same LM as the
    graph itself, bit for bit."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2109_07073_b200 import optimizer as LM
    from paper_2109_07073_b200.sharding import GatheredGraph, RankShare

    lists, poses = _problem(ctxs[:1])
    full = V.FactorGraph(lists[0], len(poses))
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(sock.getsockname()[1])
    sock.close()
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        F = full.num_factors()
        share = RankShare(V.FactorGraph.create_range(lists[0], len(poses), 0, F), 0, F, torch.device("cuda", 0))
        gg = GatheredGraph(share, [F], len(poses), full._ij, root_graph=full)
        p1, r1 = LM.optimize(gg, poses)
        raw, inl = gg.linearize_raw(poses)
        gg.stop()
    finally:
        dist.destroy_process_group()
    p2, r2 = LM.optimize(full, poses)
    assert [(t.error, t.lam, t.accepted) for t in r1.trace] == [(t.error, t.lam, t.accepted) for t in r2.trace]
    assert np.array_equal(p1, p2)
    ref_raw, ref_inl = full.linearize_raw(poses)
    assert np.array_equal(raw, ref_raw) and np.array_equal(inl, ref_inl)


def test_sharded_edge_cases(ctxs):
    """More shards than needed (an empty range), range graphs of zero factors, mismatched factor
    lists (validation), and a one-shard sharded graph — all behave like the plain graph."""
    lists, poses = _problem(ctxs[:3], nframes=3, n=800, seed=502)
    two = [fl[:2] for fl in lists]  # 2 factors over 3 shards: at least one shard is empty
    full = V.FactorGraph(two[0], len(poses))
    sh = V.FactorGraph.sharded(two, len(poses))
    counts = [sh.shard_range(r)[1] for r in range(3)]
    assert sum(counts) == 2 and 0 in counts
    a, ai = full.linearize_raw(poses)
    b, bi = sh.linearize_raw(poses)
    assert np.array_equal(a, b) and np.array_equal(ai, bi)
    one = V.FactorGraph.sharded(two[:1], len(poses))
    assert one.num_shards() == 1 and np.array_equal(one.linearize_raw(poses)[0], a)
    empty = V.FactorGraph.create_range(lists[0], len(poses), 1, 0)
    assert empty.num_factors() == 0 and empty.linearize_raw(poses)[0].shape == (0, 121)
    with pytest.raises(ValueError):
        V.FactorGraph.create_range(lists[0], len(poses), 2, len(lists[0]))  # beyond the list
    with pytest.raises(ValueError):  # the shards' lists must describe the same factors
        V.FactorGraph.sharded([lists[0], lists[1][::-1]], len(poses))


def test_mixed_float32_float64_batch_build(ctxs):
    """One build_batch call with float32 clouds (hand-written build) and float64 clouds (sort-based
    build) interleaved returns every map in its slot, identical to single builds."""
    rng = O.Rng(503)
    clouds = []
    for k in range(6):
        m, c = rng.gaussian_cloud(600 + 200 * k, 6.0)
        if k % 2:
            clouds.append(V.PointCloud(m + 1e-7, c, ctxs[0]))  # not float32-exact -> float64 cloud
        else:
            clouds.append(V.PointCloud(m.astype(np.float32), V.cov6_from(c), ctxs[0]))
    assert [c.is_f64() for c in clouds] == [False, True] * 3
    res = [1.0, 0.5, 2.0, 1.0, 0.7, 1.3]
    batch = V.GaussianVoxelMap.build_batch(clouds, res)
    for c, r, b in zip(clouds, res, batch):
        s = V.GaussianVoxelMap(c, r)
        assert b.resolution() == r
        for x, y in zip(b.export(), s.export()):
            assert np.array_equal(x, y)


def test_upload_batch_all_empty_and_single(ctxs):
    out = V.PointCloud.upload_batch([np.zeros((0, 3), np.float32)] * 3, None, ctxs[0])
    assert [len(c) for c in out] == [0, 0, 0]
    m = np.random.default_rng(6).uniform(-5, 5, (100, 3)).astype(np.float32)
    one = V.PointCloud.upload_batch([m], [np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (100, 1))], ctxs[0])
    assert len(one) == 1 and len(one[0]) == 100 and one[0].has_covariances()


def test_replicated_clouds_maps_and_sharded_graph(ctxs):
    """vgicp_cloud_replicate / vgicp_voxelmap_replicate copy the device state whole: the replicas
    export the same maps, give the same factor blocks, and a sharded graph over replicas (the usual
    way to build one: upload / build once, replicate) equals the single-context graph bit for bit —
    hand-built and sort-based (float64) maps, hash-table and rank lookups alike."""
    import os

    lists, poses = _problem(ctxs[:1], nframes=6, n=1500, seed=504)
    f0 = lists[0]
    full = V.FactorGraph(f0, len(poses))
    m0 = f0[0].target_voxels
    r1 = m0.replicate(ctxs[1])
    for x, y in zip(m0.export(), r1.export()):
        assert np.array_equal(x, y)
    pts = np.random.default_rng(8).uniform(-10, 10, (500, 3))
    assert np.array_equal(m0.lookup(pts), r1.lookup(pts))  # hash table built on demand on the replica
    sh = V.FactorGraph.sharded_replicas(f0, len(poses), ctxs[:3])
    assert sh.num_shards() == 3
    a, ai = full.linearize_raw(poses)
    b, bi = sh.linearize_raw(poses)
    assert np.array_equal(a, b) and np.array_equal(ai, bi)
    # a float64 (sort-based) map and its cloud replicate too
    rng = O.Rng(505)
    m, c = rng.gaussian_cloud(800, 5.0)
    c64 = V.PointCloud(m + 1e-7, c, ctxs[0])
    g64 = V.GaussianVoxelMap(c64, 0.5)
    g64r = g64.replicate(ctxs[2])
    for x, y in zip(g64.export(), g64r.export()):
        assert np.array_equal(x, y)
    src = f0[1].source_points
    fa = V.FactorGraph([V.MatchingCostFactor(0, 1, c64, m0)], 2).linearize_raw(poses[:2])
    fb = V.FactorGraph([V.MatchingCostFactor(0, 1, c64.replicate(ctxs[1]), r1)], 2).linearize_raw(poses[:2])
    assert np.array_equal(fa[0], fb[0]) and np.array_equal(fa[1], fb[1])
    assert src is not None


def test_sharded_replicas_float64_rare_path(ctxs):
    """float64 clouds with rank-deficient covariances (every hit's M near singular: the fp64 LDLT
    decides on the source's float64 covariance, read through the cloud's point index / covariance
    arrays) replicated onto the other contexts: the sharded graph's blocks, inliers and errors are
    bit-identical to the single graph's, whose inliers equal the oracle's."""
    rng = np.random.default_rng(77)
    frames, clouds = [], []
    for _ in range(4):
        m = rng.normal(size=(3000, 3)) * 6.0 + 1e-9  # not float32-exact
        v = rng.normal(size=(3000, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        c = 0.05 * v[:, :, None] * v[:, None, :]  # rank 1
        frames.append((m, c.reshape(-1, 9)))
        clouds.append(V.PointCloud(m, c, ctxs[0]))
    assert all(c.is_f64() for c in clouds)
    maps = V.GaussianVoxelMap.build_batch(clouds, [1.0] * 4)
    links = [(0, 1), (1, 2), (2, 3), (0, 2), (1, 3)]
    factors = [V.MatchingCostFactor(i, j, clouds[j], maps[i]) for i, j in links]
    poses = np.stack([np.concatenate([np.eye(3).reshape(9), rng.normal(size=3) * 0.05]) for _ in range(4)])
    full = V.FactorGraph(factors, 4)
    ref_raw, ref_inl = full.linearize_raw(poses)
    for k, (i, j) in enumerate(links):
        om = O.OracleMap(*frames[i], 1.0)
        assert int(ref_inl[k]) == O.linearize(*frames[j], om, poses[i], poses[j])["inliers"]
    sh = V.FactorGraph.sharded_replicas(factors, 4, ctxs[:3])
    raw, inl = sh.linearize_raw(poses)
    assert np.array_equal(raw, ref_raw) and np.array_equal(inl, ref_inl)
    assert np.array_equal(sh.evaluate(poses)[0], full.evaluate(poses)[0])
