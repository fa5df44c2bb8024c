"""rs_contingency throughput (experiments): 256 frames x ~117K points."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2003_00575_b200 import evaluation as ev

B, n = 256, 117000
g = np.random.default_rng(0)
gt = torch.from_numpy(g.integers(0, 80, size=B * n).astype(np.int32)).cuda()
pred = torch.from_numpy(g.integers(0, 120, size=B * n).astype(np.int32)).cuda()
off = torch.arange(B + 1, dtype=torch.int64, device="cuda") * n
for _ in range(3):
    ev.contingency_batch(gt, pred, off)
torch.cuda.synchronize()
import time
t0 = time.perf_counter()
for _ in range(10):
    f, *_ = ev.contingency_batch(gt, pred, off)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 10
print(f"contingency_batch (incl. table read-back): {dt*1e3:.2f} ms for {B} frames, {B*n/dt/1e9:.2f} G points/s")
t0 = time.perf_counter()
out = ev.match_instances_batch(gt, pred, off, ev.EvalConfig(min_gt_points=100))
print(f"match_instances_batch: {(time.perf_counter()-t0)*1e3:.1f} ms, {sum(len(o) for o in out)} instances")
