"""Generates tests/golden/c3_links.npy: the factor list of BASELINE config C3 (450-frame figure-eight,
seed 1, 20k points per scan, 1.0 m voxels), selected by the reference's rule (pipeline.cpp:135-141:
each frame's <= 10 highest-overlap predecessors with overlap > 0.025 at the ground-truth relative
pose) with the CPU ORACLE's overlap_rate (oracle/: voxelmap.cpp:119-135 restated) — exact hit
counts, so the list is what the reference would build. The --impl reference bench arm reads it
instead of re-running 101k overlap probes on the host; tests check it against the GPU selection.

  python tests/golden/make_c3_links.py [--frames 450] [--procs N]
"""
import argparse
import os
import sys
from multiprocessing import Pool

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

_STATE = {}


def _init(frames):
    import oracle_ctypes as O
    from bench_workloads import synthetic as S
    from bench_workloads import workloads as W

    seq = S.generate(W.c3_spec(frames=frames))
    pts = [m.astype(np.float64) for m in seq.scans]
    unit = [O.unit_covariances(len(p)) for p in pts]  # overlap reads keys only
    _STATE.update(O=O, pts=pts, gt=seq.ground_truth, maps={}, unit=unit)


def _row(j):
    from bench_workloads.workloads import pose_inv, pose_mul

    O, pts, gt = _STATE["O"], _STATE["pts"], _STATE["gt"]
    out = []
    for i in range(j):
        if i not in _STATE["maps"]:
            _STATE["maps"][i] = O.OracleMap(pts[i], _STATE["unit"][i], 1.0, threads=1)
        out.append(((i, j), O.overlap_rate(pts[j], pose_mul(pose_inv(gt[i]), gt[j]), _STATE["maps"][i], threads=1)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=450)
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.abspath(__file__)), "c3_links.npy"))
    a = ap.parse_args()
    from bench_workloads.workloads import select_links

    with Pool(a.procs, initializer=_init, initargs=(a.frames,)) as pool:
        rows = pool.map(_row, range(1, a.frames), chunksize=1)
    overlaps = dict(kv for r in rows for kv in r)
    links = np.array(select_links(overlaps, a.frames, 10, 0.025), np.int32).reshape(-1, 2)
    np.save(a.out, links)
    print(f"{len(links)} links -> {a.out}")


if __name__ == "__main__":
    main()
