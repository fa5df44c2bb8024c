"""Time single Map Connection offsets on config 1 (experiments)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import synthetic

frames = synthetic.make_batch(1, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
frames = synthetic.make_batch(cid, device="cuda")
for offs in [(), ((0, 2),), ((2, 0),), ((0, 2), (2, 0)), ((1, 1),), ((3, 0),), ((2, 2),),
             rs.preset_pattern("mc6").offsets, rs.preset_pattern("mc14").offsets]:
    pipe = rs.Pipeline(synthetic.sensor_for(synthetic.CONFIGS[cid]), rs.PipelineConfig(mc_pattern=rs.MCPattern(offs)))
    for _ in range(3):
        pipe.segment_batch(frames)
    ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(20)]
    for e0, e1 in ev:
        flush.zero_(); e0.record(); pipe.segment_batch(frames); e1.record()
    torch.cuda.synchronize()
    ts = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ev)
    print(f"{str(offs)[:40]:40s} {ts[10]:8.1f} us  R={pipe.rows_per_cta} C={pipe.ctas_per_frame}")
