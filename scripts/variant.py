"""Time experimental kernel variants selected through rs_config.reserved[1] codes
(experiments only) and check their labels against the default path."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import _native, synthetic

cid = int(sys.argv[1])
codes = [int(c) for c in sys.argv[2:]] or [0]
spec = synthetic.CONFIGS[cid]
frames = synthetic.make_batch(cid, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ref = None
for code in [0] + codes:
    pipe = rs.Pipeline(synthetic.sensor_for(spec), rs.PipelineConfig())
    pipe.rs_config = _native.make_config(pipe.packed, stop_after=code)
    out = pipe.segment_batch(frames)
    torch.cuda.synchronize()
    if ref is None:
        ref = out.labels.clone()
    same = bool(torch.equal(ref, out.labels))
    ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(40)]
    for e0, e1 in ev:
        flush.zero_()
        e0.record(); pipe.segment_batch(frames); e1.record()
    torch.cuda.synchronize()
    ts = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ev)
    print(f"code {code:3d}: {ts[len(ts) // 2]:7.1f} us  labels==default {same}")
