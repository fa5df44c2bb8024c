"""Run the fused kernel a few times on one config (for ncu / compute-sanitizer)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import synthetic

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=1)
p.add_argument("--batch", type=int, default=64)
p.add_argument("--iters", type=int, default=3)
p.add_argument("--skip", type=int, default=0)
p.add_argument("--core", action="store_true")
p.add_argument("--rows", type=int, default=0)
p.add_argument("--offsets", default="", help="Map Connection offsets 'dy,dx;dy,dx' (overrides --skip)")
p.add_argument("--preset", default="", help="Map Connection preset (mc1, mc6, mc14)")
p.add_argument("--cap", type=int, default=0, help="node capacity cap (forces the in-kernel overflow path)")
p.add_argument("--check", action="store_true", help="compare with the CPU oracle")
a = p.parse_args()
spec = synthetic.CONFIGS[a.config]
frames = synthetic.make_batch(a.config, a.batch, device="cuda")
pat = (rs.MCPattern(tuple(tuple(int(x) for x in o.split(",")) for o in a.offsets.split(";")))
       if a.offsets else rs.preset_pattern(a.preset) if a.preset else rs.skip_pattern(a.skip))
cfg = (rs.PipelineConfig(mc_pattern=pat, ground_removal=False, min_cluster_points=1)
       if a.core else rs.PipelineConfig(mc_pattern=pat))
pipe = rs.Pipeline(synthetic.sensor_for(spec), cfg, rows_per_cta=a.rows, node_capacity=a.cap)
torch.cuda.synchronize()
for _ in range(a.iters):
    pipe.segment_batch(frames)
torch.cuda.synchronize()
if a.check:
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from oracle import oracle
    res = pipe.segment_batch(frames)
    wl, wn, _ = oracle.segment_batch(frames.cpu().numpy(), pipe.packed)
    assert (res.labels.cpu().numpy() == wl).all() and (res.n_clusters.cpu().numpy() == wn).all(), "mismatch"
    print("oracle check ok")
print("ok", pipe.rows_per_cta, pipe.ctas_per_frame, pipe.smem_bytes)
