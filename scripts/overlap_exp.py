"""Experiment: concurrency of a bits-only launch (stop_after=1) with full launches."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import _native, synthetic

spec = synthetic.CONFIGS[1]
frames = synthetic.make_batch(1, device="cuda")
half_a, half_b = frames[:128].contiguous(), frames[128:].contiguous()
m = synthetic.sensor_for(spec)
full = rs.Pipeline(m, rs.PipelineConfig())
bits = rs.Pipeline(m, rs.PipelineConfig())
bits.rs_config = _native.make_config(bits.packed, stop_after=1)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        flush.zero_(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return sorted(ts)[n // 2]

def seq():
    bits.segment_batch(half_a); full.segment_batch(half_b)
def conc():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): bits.segment_batch(half_a, stream=s1)
    with torch.cuda.stream(s2): full.segment_batch(half_b, stream=s2)
    cur.wait_stream(s1); cur.wait_stream(s2)
print("bits 128:", t(lambda: bits.segment_batch(half_a)))
print("full 128:", t(lambda: full.segment_batch(half_b)))
print("sequential bits+full:", t(seq))
print("concurrent bits||full:", t(conc))
print("full 256:", t(lambda: full.segment_batch(frames)))
