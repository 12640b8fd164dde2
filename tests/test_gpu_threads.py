"""Several host threads, one context each, on the same GPU at once (include/vgicp_b200.h: "one host
thread drives a context"): map builds, overlap queries, graph linearization and the native LM run
concurrently (ctypes releases the GIL inside every C ABI call) and give bit-for-bit the results of a
serial run — the library holds no unsynchronised process-wide state on these paths (per-device
kernel attributes, thread-local error strings, per-context scratch and streams).
"""
import threading

import numpy as np
import pytest

import oracle_ctypes as O
from helpers import contract_inputs

V = pytest.importorskip("paper_2109_07073_b200")

pytestmark = pytest.mark.gpu

THREADS = 4


def scene(seed):
    rng = O.Rng(seed)
    frames = []
    for _ in range(5):
        m, _, c6 = contract_inputs(*rng.gaussian_cloud(6000, 12.0))
        frames.append((m, c6))
    poses = np.stack([rng.random_pose(0.03, 0.3) for _ in range(5)])
    return frames, poses


def work(ctx, frames, poses):
    clouds = [V.PointCloud(m, c6, ctx) for m, c6 in frames]
    maps = V.GaussianVoxelMap.build_batch(clouds, [1.0, 0.5, 1.0, 2.0, 1.0])
    exports = [mp.export() for mp in maps]
    rels = [O.compose(O.inverse(poses[i]), poses[i + 1]) for i in range(4)]
    hits = V.overlap_hits(clouds[1:], rels, maps[:4])
    factors = [V.MatchingCostFactor(i, j, clouds[j], maps[i]) for i in range(5) for j in range(i + 1, 5)]
    graph = V.FactorGraph(factors, 5, ctx=ctx)
    raws = [graph.linearize_raw(poses) for _ in range(5)]
    err, inl = graph.evaluate(poses)
    from paper_2109_07073_b200 import optimizer as LM

    fixed = np.zeros(5, np.uint8)
    fixed[0] = 1
    lm_poses, rep = LM.optimize_native(graph, poses, fixed=fixed, settings=LM.LmSettings(max_iterations=5))
    return exports, np.asarray(hits), raws, err, inl, np.asarray(lm_poses), rep.final_error, rep.iterations


def same(a, b):
    if isinstance(a, (list, tuple)):
        return len(a) == len(b) and all(same(x, y) for x, y in zip(a, b))
    return np.array_equal(np.asarray(a), np.asarray(b))


def test_threads_with_own_contexts_match_serial():
    inputs = [scene(900 + t) for t in range(THREADS)]
    serial_ctx = V.Context(0)
    serial = [work(serial_ctx, *inputs[t]) for t in range(THREADS)]
    results, errors = [None] * THREADS, []
    barrier = threading.Barrier(THREADS)

    def run(t):
        try:
            ctx = V.Context(0)
            barrier.wait()
            out = None
            for _ in range(3):  # repeat to overlap the phases of different threads
                out = work(ctx, *inputs[t])
            ctx.synchronize()
            results[t] = out
        except Exception as e:  # surfaced below
            errors.append((t, repr(e)))

    threads = [threading.Thread(target=run, args=(t,)) for t in range(THREADS)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for t in range(THREADS):
        assert same(results[t], serial[t]), t
