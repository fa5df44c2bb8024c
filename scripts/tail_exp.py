"""Experiment: split the batch into a full first wave + a finer-grained tail launch."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import synthetic

frames = synthetic.make_batch(1, device="cuda")
m = synthetic.sensor_for(synthetic.CONFIGS[1])
p32 = rs.Pipeline(m, rs.PipelineConfig())
p16 = rs.Pipeline(m, rs.PipelineConfig(), rows_per_cta=16)
p8 = rs.Pipeline(m, rs.PipelineConfig(), rows_per_cta=8)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
lab = torch.empty(frames.shape, dtype=torch.int32, device="cuda")
ncl = torch.empty(256, dtype=torch.int32, device="cuda")
szs = torch.empty((256, p32.sizes_stride), dtype=torch.int64, device="cuda")

def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    # like bench.py: the flush runs on the GPU while the host enqueues the
    # step, so host launch latency stays outside the events
    ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(n)]
    for e0, e1 in ev:
        flush.zero_()
        e0.record(); fn(); e1.record()
    torch.cuda.synchronize()
    ts = [e0.elapsed_time(e1) * 1e3 for e0, e1 in ev]
    return sorted(ts)[n // 2]

def split(k, tail):
    def fn():
        p32.segment_batch(frames[:k], labels=lab[:k], n_clusters=ncl[:k], cluster_sizes=szs[:k])
        tail.segment_batch(frames[k:], labels=lab[k:], n_clusters=ncl[k:], cluster_sizes=szs[k:])
    return fn
print("all R32:", t(lambda: p32.segment_batch(frames, labels=lab, n_clusters=ncl, cluster_sizes=szs)))
for k in (148, 140, 160, 200):
    print(f"R32[:{k}] + R16 tail:", t(split(k, p16)), f"  + R8 tail:", t(split(k, p8)))
for b in (64, 128, 148, 192, 256, 296):
    print(f"R32 batch {b}:", t(lambda: p32.segment_batch(frames[:b] if b <= 256 else torch.cat([frames, frames[:b-256]]))))
