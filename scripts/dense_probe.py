"""Throughput when every frame takes the node-capacity overflow path (experiments)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import synthetic

for cid in (1, 3):
    spec = synthetic.CONFIGS[cid]
    frames = synthetic.make_batch(cid, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for cap in (0, 32):
        pipe = rs.Pipeline(synthetic.sensor_for(spec), rs.PipelineConfig(), node_capacity=cap)
        for _ in range(2):
            pipe.segment_batch(frames)
        ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(10)]
        for e0, e1 in ev:
            flush.zero_(); e0.record(); pipe.segment_batch(frames); e1.record()
        torch.cuda.synchronize()
        ts = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ev)
        print(f"config {cid} node_capacity={cap or 'auto'}: {ts[5]:8.1f} us  {frames.shape[0] / ts[5] * 1e6:,.0f} frames/s")
