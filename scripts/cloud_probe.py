"""Point-cloud path on the config-1 batch (experiments): run a few steps for ncu."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import cloud, synthetic

spec = synthetic.CONFIGS[1]
frames = synthetic.make_batch(1, int(sys.argv[1]) if len(sys.argv) > 1 else 256, device="cuda")
pipe = rs.Pipeline(synthetic.sensor_for(spec), rs.PipelineConfig())
m = pipe.model
r = frames.double()
el = torch.as_tensor(np.asarray(m.channel_angles), dtype=torch.float64, device="cuda")[:, None]
az = (torch.arange(m.width, dtype=torch.float64, device="cuda") + 0.5) * m.azimuth_step
keep = r > 0
xyz = torch.stack([r * torch.cos(el) * torch.cos(az), r * torch.cos(el) * torch.sin(az), r * torch.sin(el).expand_as(r)], -1)
pts = xyz[keep].contiguous()
off = torch.zeros(frames.shape[0] + 1, dtype=torch.int64, device="cuda")
off[1:] = torch.cumsum(keep.flatten(1).sum(1), 0)
for _ in range(3):
    ranges, pidx, _ = cloud.project_batch(pts, off, m)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); cloud.project_batch(pts, off, m); e1.record(); torch.cuda.synchronize()
print("project ms", e0.elapsed_time(e1), "points", pts.shape[0])
