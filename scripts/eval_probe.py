"""rs_contingency throughput: the instance-scoring counting step for 256
config-1 frames (131072 points each): gt = labels of the default pipeline,
pred = labels of the core variant (two different segmentations of the same
frames, so the table has realistic overlaps), plus the random-label stress case."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import evaluation as ev, synthetic

frames = synthetic.make_batch(1, device="cuda")
m = synthetic.sensor_for(synthetic.CONFIGS[1])
gt = rs.Pipeline(m, rs.PipelineConfig()).segment_batch(frames).labels.flatten().contiguous()
pred = rs.Pipeline(m, rs.PipelineConfig(ground_removal=False, min_cluster_points=1)).segment_batch(
    frames).labels.flatten().contiguous()
B, n = frames.shape[0], frames[0].numel()
off = torch.arange(B + 1, dtype=torch.int64, device="cuda") * n
print(ev.contingency_device_ms(gt, pred, off), "ms device (segmentations)")
g = np.random.default_rng(0)
rg = torch.from_numpy(g.integers(0, 80, size=B * n).astype(np.int32)).cuda()
rp = torch.from_numpy(g.integers(0, 120, size=B * n).astype(np.int32)).cuda()
print(ev.contingency_device_ms(rg, rp, off), "ms device (random labels, spilling)")
t0 = time.perf_counter()
out = ev.match_instances_batch(gt, pred, off, ev.EvalConfig(min_gt_points=100))
print(f"match_instances_batch: {(time.perf_counter()-t0)*1e3:.1f} ms, {sum(len(o) for o in out)} instances")
