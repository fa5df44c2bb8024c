"""Per-phase CTA timing from the RS_PHASE_PROF build (clock64 deltas)."""
import argparse
import ctypes
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
os.environ["RS_LIB"] = str(ROOT / "paper_2003_00575_b200" / "_lib" / "librangeseg_b200_prof.so")
sys.path.insert(0, str(ROOT))

import numpy as np
import torch

import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import _native, synthetic

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=1)
p.add_argument("--batch", type=int, default=256)
p.add_argument("--core", action="store_true")
p.add_argument("--skip", type=int, default=0)
p.add_argument("--rows", type=int, default=0)
p.add_argument("--offsets", default="", help="Map Connection offsets 'dy,dx;dy,dx' (overrides --skip)")
a = p.parse_args()
names = ["A bits", "B edges/MC", "R runs", "U unions", "U flatten", "U sizes", "cs1+ovf", "X cross",
         "cs2", "Z resolve", "cs3+K kept", "cs4+prefix", "run labels", "cs5", "cell labels"]
spec = synthetic.CONFIGS[a.config]
frames = synthetic.make_batch(a.config, a.batch, device="cuda")
pat = (rs.MCPattern(tuple(tuple(int(x) for x in o.split(",")) for o in a.offsets.split(";")))
       if a.offsets else rs.skip_pattern(a.skip))
cfg = (rs.PipelineConfig(mc_pattern=pat, ground_removal=False, min_cluster_points=1)
       if a.core else rs.PipelineConfig(mc_pattern=pat))
pipe = rs.Pipeline(synthetic.sensor_for(spec), cfg, rows_per_cta=a.rows)
for _ in range(3):
    pipe.segment_batch(frames)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record(); pipe.segment_batch(frames); ev[1].record(); torch.cuda.synchronize()
n = min(8192, a.batch * pipe.ctas_per_frame)
buf = np.zeros((n, 24), dtype=np.int64)
_native.check(_native.lib().rs_phase_profile(buf.ctypes.data_as(ctypes.c_void_p), n))
NM = len(names) + 1
d = np.diff(buf[:, :NM], axis=1).astype(np.float64)
tot = buf[:, NM - 1] - buf[:, 0]
print(f"kernel {ev[0].elapsed_time(ev[1])*1e3:.1f} us, plan R={pipe.rows_per_cta} C={pipe.ctas_per_frame} "
      f"smem={pipe.smem_bytes}, CTAs profiled {n}")
print(f"CTA lifetime cycles: mean {tot.mean():.0f} p50 {np.median(tot):.0f} p90 {np.percentile(tot,90):.0f}")
for i, nm in enumerate(names):
    print(f"  {nm:16s} mean {d[:, i].mean():9.0f}  p90 {np.percentile(d[:, i], 90):9.0f}  "
          f"share {100*d[:, i].mean()/tot.mean():5.1f}%")
gs, ge = buf[:, 16], buf[:, 17]
t0 = gs.min()
print(f"globaltimer: start spread {(gs.max()-t0)/1e3:.1f} us, last end {(ge.max()-t0)/1e3:.1f} us, "
      f"mean life {(ge-gs).mean()/1e3:.1f} us")
order = np.argsort(gs)
qs = [0, 0.1, 0.25, 0.5, 0.58, 0.75, 0.9, 1.0]
print("start-time quantiles (us):", " ".join(f"{q:.2f}:{(np.quantile(gs, q)-t0)/1e3:.1f}" for q in qs))
print("end-time quantiles (us):  ", " ".join(f"{q:.2f}:{(np.quantile(ge, q)-t0)/1e3:.1f}" for q in qs))
print("distinct SMs used:", len(np.unique(buf[:, 18])))
sub = [("gather", 3, 19), ("hook", 19, 20), ("unite", 20, 4)]
ok = (buf[:, 19] > 0) & (buf[:, 20] > 0)
for nm, i, j in sub:
    d2 = (buf[ok, j] - buf[ok, i]).astype(np.float64)
    print(f"  U.{nm:10s} mean {d2.mean():9.0f}  p90 {np.percentile(d2, 90):9.0f}")
inband = (buf[:, 21] > 0) & (buf[:, 21] < buf[:, 6])   # Map Connections inside the band (marks before the size pass)
okb = (buf[:, 21] > 0) & (buf[:, 22] > 0) & (buf[:, 23] > 0) & ~inband
if okb.any():   # step M (Map Connections) inside "Z resolve"
    for nm, i, j in [("M.compress", 9, 21), ("M.runs", 21, 22), ("M.list unite", 22, 23), ("M.cs2b+Z", 23, 10)]:
        d3 = (buf[okb, j] - buf[okb, i]).astype(np.float64)
        print(f"  {nm:14s} mean {d3.mean():9.0f}  p90 {np.percentile(d3, 90):9.0f}  max {d3.max():9.0f}")
oka = inband & (buf[:, 22] > 0) & (buf[:, 23] > 0)
if oka.any():   # Map Connections inside the band (last round; inside "U sizes"): heads listed, chains tested + united, re-flatten
    for nm, i, j in [("mc.heads (last round: 5 = first)", 5, 21), ("mc.chains", 21, 23), ("mc.reflatten", 23, 22), ("sizes", 22, 6)]:
        d3 = (buf[oka, j] - buf[oka, i]).astype(np.float64)
        print(f"  {nm:16s} mean {d3.mean():9.0f}  p90 {np.percentile(d3, 90):9.0f}  max {d3.max():9.0f}")
C = pipe.ctas_per_frame
if C > 1:
    rank = np.arange(n) % C
    print("per band (CTA rank in the cluster): mean cycles of each phase")
    print("  " + " ".join(f"{nm[:10]:>10s}" for nm in names))
    for k in range(C):
        m = rank == k
        print(f"k={k} " + " ".join(f"{d[m, i].mean():10.0f}" for i in range(len(names))))
