import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2109_07073_b200 as V
from paper_2109_07073_b200 import optimizer as LM
from bench_workloads import workloads as W
ctx = V.default_context(0)
sc = W.make_scans(W.c1_spec(), ctx=ctx)
tgt = V.PointCloud(sc.means[0], sc.cov6[0], ctx); src = V.PointCloud(sc.means[1], sc.cov6[1], ctx)
vmap = V.GaussianVoxelMap(tgt, 1.0)
poses = np.stack([sc.gt[0], LM.compose(sc.gt[1], LM.se3_exp([0.0, 0.0, 0.01, 0.1, 0.0, 0.0]))])
for chunk in (0, 512, 1024, 2048):
    g = V.FactorGraph([V.MatchingCostFactor(0, 1, src, vmap)], 2, chunk=chunk)
    dP = torch.tensor(poses, dtype=torch.float64, device="cuda"); dO = torch.zeros((1, 121), dtype=torch.float64, device="cuda"); dI = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream(); 
    for _ in range(10): g.linearize_device(dP.data_ptr(), dO.data_ptr(), dI.data_ptr())
    ctx.synchronize()
    t = time.perf_counter()
    for _ in range(200): g.linearize_device(dP.data_ptr(), dO.data_ptr(), dI.data_ptr())
    ctx.synchronize(); dev = (time.perf_counter() - t) / 200 * 1e3
    t = time.perf_counter()
    for _ in range(200): g.linearize_raw(poses)
    host = (time.perf_counter() - t) / 200 * 1e3
    print(f"chunk {chunk}: back-to-back device launches {dev:.4f} ms/launch, host call {host:.4f} ms")
