"""Repeat fuzz seeds many times (race hunting): python scripts/stress_fuzz.py REPS SEED[:CAP] ..."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np, torch
import paper_2003_00575_b200 as rs
from oracle import oracle
from test_gpu_fuzz import _case
reps = int(sys.argv[1])
for spec in sys.argv[2:]:
    seed, _, capo = spec.partition(":")
    model, cfg, frames, rows, cap = _case(int(seed))
    cap = int(capo) if capo else cap
    pipe = rs.Pipeline(model, cfg, device="cuda:0", rows_per_cta=rows, node_capacity=cap)
    x = torch.as_tensor(frames).cuda()
    want = [oracle.segment_frame(frames[b], pipe.packed)[0] for b in range(frames.shape[0])]
    bad = 0
    for it in range(reps):
        res = pipe.segment_batch(x)
        got = res.labels.cpu().numpy()
        for b in range(frames.shape[0]):
            n = int((got[b] != want[b]).sum())
            if n:
                bad += 1
                if bad <= 3:
                    idx = np.argwhere(got[b] != want[b])[:4]
                    print(f"  seed {seed} cap {cap} rep {it} frame {b}: {n} mismatches at {idx.tolist()}")
    print(f"seed {seed} cap {cap} rows {rows} plan {pipe.plan['fast_ctas']}x{pipe.plan['fast_rows']}: {bad} bad frames of {reps * frames.shape[0]}")
