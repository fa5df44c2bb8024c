"""Kernel time when the fast kernel stops after phase N (experiments only)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import _native, synthetic

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
spec = synthetic.CONFIGS[cid]
frames = synthetic.make_batch(cid, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
names = {1: "A+bits", 2: "R runs", 9: "U gather", 3: "U unite", 4: "flatten+sizes", 5: "X cross", 6: "Z resolve",
         7: "K+assign", 8: "run labels", 0: "full"}
prev = 0.0
for stop in (1, 2, 9, 3, 4, 5, 6, 7, 8, 0):
    pipe = rs.Pipeline(synthetic.sensor_for(spec), rs.PipelineConfig())
    pipe.rs_config = _native.make_config(pipe.packed, stop_after=stop)
    for _ in range(5):
        pipe.segment_batch(frames)
    ts = []
    for _ in range(30):
        flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); pipe.segment_batch(frames); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[len(ts) // 2] * 1e3
    print(f"stop after {stop} ({names[stop]:14s}): {t:7.1f} us  (+{t - prev:6.1f})")
    prev = t
