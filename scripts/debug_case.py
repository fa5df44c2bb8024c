import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np, torch
import golden
import paper_2003_00575_b200 as rs
key = sys.argv[1] if len(sys.argv) > 1 else "r000"
m, cfg, ranges, labels, sizes, st = golden.case("random", key)
pipe = rs.Pipeline(m, cfg)
print(pipe.plan)
x = torch.from_numpy(ranges).cuda()[None]
lab = torch.full((1,) + ranges.shape, -7, dtype=torch.int32, device="cuda")
res = pipe.segment_batch(x, labels=lab)
torch.cuda.synchronize()
print("ncl", res.n_clusters.cpu().numpy(), "want", len(sizes) - 1)
print("got\n", res.labels[0].cpu().numpy()[:4])
print("want\n", labels[:4])
ws = pipe.workspace(1, torch.cuda.current_stream())
print("ws", ws[:16].view(torch.int32).cpu().numpy())
