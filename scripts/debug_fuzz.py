"""Reproduce a failing fuzz seed: mismatching cells and their neighbourhood."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np, torch
import paper_2003_00575_b200 as rs
from oracle import oracle
from test_gpu_fuzz import _case
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 29
model, cfg, frames, rows, cap = _case(seed)
for c in ([cap] if len(sys.argv) < 3 else [int(x) for x in sys.argv[2:]]):
    pipe = rs.Pipeline(model, cfg, device="cuda:0", rows_per_cta=rows, node_capacity=c)
    print("cap", c, pipe.plan, cfg.mc_pattern)
    res = pipe.segment_batch(torch.as_tensor(frames).cuda())
    torch.cuda.synchronize()
    for b in range(frames.shape[0]):
        wl, ws = oracle.segment_frame(frames[b], pipe.packed)
        got = res.label_image(b)
        bad = np.argwhere(got.labels != wl)
        print(f" frame {b}: {len(bad)} mismatches, ncl got {got.cluster_count} want {len(ws) - 1}")
        for r, cc in bad[:10]:
            print(f"   ({r},{cc}) got {got.labels[r, cc]} want {wl[r, cc]}")
