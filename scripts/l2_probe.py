"""Kernel time under three L2 regimes between timed steps (experiments):
flush (512 MiB write), none with one input batch, none with two alternating batches."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import synthetic

spec = synthetic.CONFIGS[1]
f0 = synthetic.make_batch(1, device="cuda")
f1 = synthetic.make_batch(1, device="cuda", first_seed=256)
pipe = rs.Pipeline(synthetic.sensor_for(spec), rs.PipelineConfig())
lab = [torch.empty(f0.shape, dtype=torch.int32, device="cuda") for _ in range(2)]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for mode in ("flush", "none-1buf", "none-2buf", "flush", "none-2buf"):
    for _ in range(3):
        pipe.segment_batch(f0)
    ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(40)]
    for i, (e0, e1) in enumerate(ev):
        if mode == "flush":
            flush.zero_()
        x = f1 if (mode == "none-2buf" and i % 2) else f0
        e0.record(); pipe.segment_batch(x, labels=lab[i % 2]); e1.record()
    torch.cuda.synchronize()
    ts = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ev)
    print(f"{mode:10s} median {ts[20]:7.1f} us  mean {sum(ts)/len(ts):7.1f}")
