"""Counters of the run-level Map Connection pass (library built with
-DRS_MC_STATS, via RS_LIB): (run, offset) items, partner runs compared,
differing roots, cell pairs tested, unions -- per batch."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import _native, synthetic

for cid, pat in ((1, "S1"), (1, "mc6"), (1, "mc14"), (4, "S1")):
    spec = synthetic.CONFIGS[cid]
    frames = synthetic.make_batch(cid, device="cuda")
    p = rs.skip_pattern(1) if pat == "S1" else rs.preset_pattern(pat)
    pipe = rs.Pipeline(synthetic.sensor_for(spec), rs.PipelineConfig(mc_pattern=p))
    out = (ctypes.c_int64 * 8)()
    lib = _native.lib()
    lib.rs_mc_stats(out, 1)
    pipe.segment_batch(frames)
    torch.cuda.synchronize()
    lib.rs_mc_stats(out, 1)
    print(cid, pat, "words-with-cells %d heads %d live-chains %d chain-cells %d unions %d (per batch)" % tuple(out[:5]))
