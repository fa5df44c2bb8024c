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


# ---------------------------------------------------------------- project ----
def project_cases():
    return sorted({k.rsplit("/", 1)[0] for k in load("project")})


def project_case(key):
    st = load("project")
    m = SensorModel(st[f"{key}/angles_deg"], float(st[f"{key}/step_deg"]), float(st[f"{key}/mount"]),
                    width=int(st[f"{key}/width"]))
    return m, {k.rsplit("/", 1)[1]: v for k, v in st.items() if k.rsplit("/", 1)[0] == key}


def unstable_cells(points, model, rel=1e-12):
    """Cells a point may land in when its elevation sits within ``rel`` of a
    channel midpoint / field-of-view edge, or its azimuth within ``rel`` of a
    column edge.  There the decision turns on the last ulp of asin / atan2,
    which differ between libraries (numpy's vectorised float64 arcsin is not the
    C library's; CUDA's is a third).  Returns a bool [H, W] mask and the number
    of such points.  Everywhere else projection results must be bit-identical.
    """
    H, W = model.height, model.width
    p = np.asarray(points, dtype=np.float64)[:, :3]
    r = np.sqrt((p[:, 0] * p[:, 0] + p[:, 1] * p[:, 1]) + p[:, 2] * p[:, 2])
    ok = r > 0
    el = np.arcsin(np.clip(np.divide(p[:, 2], r, where=ok, out=np.zeros_like(r)), -1, 1))
    ang = np.asarray(model.channel_angles, dtype=np.float64)
    desc = ang[0] > ang[-1]
    asc = ang[::-1] if desc else ang
    bounds = np.concatenate([(asc[1:] + asc[:-1]) / 2, [asc[0] - (asc[1] - asc[0]) / 2,
                                                       asc[-1] + (asc[-1] - asc[-2]) / 2]])
    near_el = (np.abs(el[:, None] - bounds[None, :]) <= rel * np.maximum(1.0, np.abs(bounds))).any(1)
    az = np.arctan2(p[:, 1], p[:, 0])
    az = np.where(az < 0, az + 2 * np.pi, az)
    q = az / model.azimuth_step
    near_az = (np.abs(q - np.round(q)) <= rel * np.maximum(1.0, np.abs(q))) | \
              (np.abs(az - 2 * np.pi) <= rel) | (np.abs(az) <= rel)
    amb = ok & (near_el | near_az)
    mask = np.zeros((H, W), bool)
    for i in np.flatnonzero(amb):
        row = int(np.argmin(np.abs(asc - el[i])))
        row = H - 1 - row if desc else row
        col = int(np.floor(q[i])) % W
        for dr in (-1, 0, 1):
            for dc in (-1, 0, 1):
                rr = row + dr
                if 0 <= rr < H:
                    mask[rr, (col + dc) % W] = True
    return mask, int(amb.sum())


# ------------------------------------------------------------------- eval ----
def eval_cases():
    return sorted({k.split("/")[0] for k in load("eval")})


def eval_case(key):
    st = load("eval")
    matches = [tuple(m) for m in json.loads(str(st[f"{key}/matches"][0]))]
    summary = json.loads(str(st[f"{key}/summary"][0]))
    return st[f"{key}/gt"], st[f"{key}/pred"], int(st[f"{key}/min_gt_points"]), matches, summary


def pack_bits(bits):
    """bool [..., W] -> uint32 [..., ceil(W/32)], bit c%32 of word c/32 (the
    rs_fast_planes layout)."""
    bits = np.asarray(bits, dtype=bool)
    W = bits.shape[-1]
    wpr = (W + 31) // 32
    pad = np.zeros(bits.shape[:-1] + (wpr * 32,), dtype=bool)
    pad[..., :W] = bits
    return np.packbits(pad, axis=-1, bitorder="little").view(np.uint32)


def planes_from_masks(ranges, ground, horizontal, vertical):
    """Presence / left-edge / up-edge planes from the reference's stage outputs
    (extract_ground mask, build_connectivity horizontal / vertical images)."""
    H, W = ranges.shape
    pres = (ranges > 0) & ~ground
    left = np.roll(horizontal, 1, axis=1) if W > 1 else np.zeros_like(horizontal)
    up = np.zeros((H, W), dtype=bool)
    up[1:] = vertical
    return np.stack([pack_bits(pres), pack_bits(left), pack_bits(up)])
