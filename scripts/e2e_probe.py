"""e2e through rs_segment_batch_host: with / without cluster sizes, timing per call."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import synthetic

spec = synthetic.CONFIGS[1]
frames = synthetic.make_batch(1, device="cuda")
pipe = rs.Pipeline(synthetic.sensor_for(spec), rs.PipelineConfig())
B = frames.shape[0]
h_in = torch.empty(frames.shape, dtype=torch.float32, pin_memory=True); h_in.copy_(frames); h_in = h_in.numpy()
h_lab = torch.empty(frames.shape, dtype=torch.int32, pin_memory=True).numpy()
h_ncl = torch.empty((B,), dtype=torch.int32, pin_memory=True).numpy()
h_sz = torch.empty((B, pipe.sizes_stride), dtype=torch.int64, pin_memory=True).numpy()
for name, kw in [("full", dict(cluster_sizes=h_sz)), ("no sizes", dict(cluster_sizes=False))]:
    for _ in range(3):
        pipe.segment_batch_host(h_in, h_lab, h_ncl, **kw)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); pipe.segment_batch_host(h_in, h_lab, h_ncl, **kw); ts.append(time.perf_counter() - t0)
    t = sorted(ts)[5]
    print(f"{name:9s}: {t*1e3:.2f} ms/call  {B/t:,.0f} frames/s")
