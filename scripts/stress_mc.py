"""Determinism stress of the Map Connection paths at full batch (race hunting):
every repetition's labels must equal the first run's, whose first frames are
checked against the oracle.  python scripts/stress_mc.py [REPS]"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import synthetic
from oracle import oracle

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for cid, name, pat in ((1, "S1", rs.skip_pattern(1)), (2, "S1", rs.skip_pattern(1)), (4, "S2", rs.skip_pattern(2)),
                       (1, "mc6", rs.preset_pattern("mc6")), (1, "mc14", rs.preset_pattern("mc14")),
                       (3, "mc6", rs.preset_pattern("mc6"))):
    frames = synthetic.make_batch(cid, device="cuda")
    pipe = rs.Pipeline(synthetic.sensor_for(synthetic.CONFIGS[cid]), rs.PipelineConfig(mc_pattern=pat))
    ref = pipe.segment_batch(frames)
    torch.cuda.synchronize()
    ref_l, ref_n = ref.labels.clone(), ref.n_clusters.clone()
    host = frames[:4].cpu().numpy()
    ok = all(np.array_equal(ref_l[b].cpu().numpy(), oracle.segment_frame(host[b], pipe.packed)[0]) for b in range(4))
    bad = 0
    for _ in range(reps):
        out = pipe.segment_batch(frames)
        bad += int(not (torch.equal(out.labels, ref_l) and torch.equal(out.n_clusters, ref_n)))
    torch.cuda.synchronize()
    print(f"config {cid} {name}: first 4 frames == oracle {ok}; {bad} of {reps} repetitions differ from the first run")
