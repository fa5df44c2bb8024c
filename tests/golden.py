"""Loader for tests/golden/*.npz (written by tests/golden/make_golden.py from the
Python reference).  Rebuilds the sensor model and PipelineConfig of each case
with this package's host code."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2003_00575_b200 import (DistanceThreshold, GroundParams, MCPattern,
                                   PipelineConfig, SensorModel)

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def load(name):
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def model(store, key):
    step, mount, width = store[f"{key}/geom"]
    return SensorModel(store[f"{key}/angles"], float(step), float(mount), width=int(width))


def config(store, key):
    c = json.loads(str(store[f"{key}/cfg"][0]))
    return PipelineConfig(ground=GroundParams(theta_deg=c["theta"], keep_above_z=c["keep_above"]),
                          threshold=DistanceThreshold(c["d_max"]),
                          mc_pattern=MCPattern(tuple(tuple(o) for o in c["offsets"])),
                          min_cluster_points=c["min_points"], ground_removal=c["ground"])


def unpack(store, key, shape):
    n = int(np.prod(shape))
    return np.unpackbits(store[key])[:n].reshape(shape).astype(bool)


def frame_cases():
    """(case key, frame key) for every pipeline run in frames.npz."""
    st = load("frames")
    out = []
    for k in st:
        if k.endswith("/labels"):
            case = k[: -len("/labels")]
            out.append((case, case.split("/")[0]))
    return sorted(out)


def random_cases():
    st = load("random")
    return sorted({k.split("/")[0] for k in st})


def case(group, case_key, frame_key=None):
    """-> (model, config, ranges, labels, sizes, stages or None)."""
    st = load(group)
    frame_key = frame_key or case_key
    m = model(st, frame_key)
    cfg = config(st, case_key)
    ranges = st[f"{frame_key}/ranges"]
    H, W = ranges.shape
    stages = None
    if f"{case_key}/ground" in st:
        stages = (unpack(st, f"{case_key}/ground", (H, W)),
                  unpack(st, f"{case_key}/horizontal", (H, W)),
                  unpack(st, f"{case_key}/vertical", (H - 1, W)))
    return m, cfg, ranges, st[f"{case_key}/labels"], st[f"{case_key}/sizes"], stages
