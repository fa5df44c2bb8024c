"""Generate the golden fixtures by running the Python reference itself.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports ``rangeseg`` from /root/reference/pkg/src, feeds it seeded inputs and
records its float32 constant tables, stage masks (``extract_ground``,
``build_connectivity``) and final ``Pipeline.segment_range_image`` labels and
cluster sizes.  The .npz files it writes are committed; tests read only them,
so nothing at test time touches /root/reference.

Case groups:
  tables.npz   f32 tables of SensorModel / ground_bounds / thresholds for 7 geometries
  frames.npz   full-size frames (config 0-4 generator, reference stock scenes) x configs
  random.npz   60 small random frames with random MC patterns, ground on/off
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import rangeseg as R  # noqa: E402  (the reference)
from rangeseg import synthetic as RS  # noqa: E402

from paper_2003_00575_b200 import synthetic as S  # noqa: E402  (input generator only)

OUT = Path(__file__).resolve().parent
F32 = np.float32

ALL_OFFSETS = sorted(set(R.preset_pattern("mc6").offsets) | set(R.preset_pattern("mc14").offsets)
                     | {(1, -4), (7, -3), (0, 5), (1, 1), (2, -1)})


def geometry(name):
    if name == "c0":
        return dict(angles=np.linspace(2.0, -24.8, 64), step=360 / 2048, mount=1.73, width=2048)
    if name == "c2":
        return dict(angles=np.linspace(22.5, -22.5, 128), step=360 / 2048, mount=1.8, width=2048)
    if name == "c3":
        return dict(angles=np.linspace(15.0, -25.0, 32), step=360 / 1024, mount=1.5, width=1024)
    if name == "hdl64":
        m = R.default_model()
    elif name == "fixture":
        m = RS.fixture_model()
    elif name == "small":
        m = R.uniform_model(8, top_deg=-2.0, step_deg=2.0, azimuth_step_deg=22.5, mount_height_m=1.5)
    elif name == "ascending":
        m = R.SensorModel([-20.0, -17.0, -14.0, -11.0, -8.0, -5.0], 45.0, 1.5, width=8)
    return dict(angles=m.channel_angles_deg.copy(), step=m.azimuth_step_deg,
                mount=m.mount_height, width=m.width)


def ref_model(g):
    return R.SensorModel(g["angles"], g["step"], g["mount"], width=g["width"])


def put_geometry(store, key, g):
    store[f"{key}/angles"] = np.asarray(g["angles"], dtype=np.float64)
    store[f"{key}/geom"] = np.array([g["step"], g["mount"], g["width"]], dtype=np.float64)


def make_tables():
    store = {}
    for name in ("c0", "c2", "c3", "hdl64", "fixture", "small", "ascending"):
        g = geometry(name)
        m = ref_model(g)
        put_geometry(store, name, g)
        H, W = m.height, m.width
        store[f"{name}/sin_ch"] = m.sin_channel.astype(F32)
        store[f"{name}/sin_a"] = m.sin_vertical.astype(F32)
        store[f"{name}/cos_a"] = m.cos_vertical.astype(F32)
        for theta in (5.0, 10.0):
            try:
                lo, hi = R.ground.ground_bounds(m, theta)
                store[f"{name}/lo_{theta:g}"] = lo.astype(F32)
                store[f"{name}/hi_{theta:g}"] = hi.astype(F32)
            except ValueError:
                pass
        offs = [o for o in ALL_OFFSETS if o[0] < H and abs(o[1]) < W] + [(0, 1), (1, 0)]
        for dy, dx in offs:
            store[f"{name}/tc_{dy}_{dx}"] = m.pair_constant(dy, dx).astype(F32).ravel()
        store[f"{name}/keep_above"] = np.asarray(
            R.GroundParams().resolve_keep_above(m), dtype=F32)
    for d in (0.8, 0.4, 0.9, 0.25):
        store[f"dmax/{d:g}"] = np.asarray(R.DistanceThreshold(d).d_max_sq, dtype=F32)
    np.savez_compressed(OUT / "tables.npz", **store)
    print("tables.npz", len(store), "arrays")


PIPE_CONFIGS = {
    "default": dict(preset="none", ground=True, min_points=100),
    "mc1": dict(preset="mc1", ground=True, min_points=100),
    "mc6": dict(preset="mc6", ground=True, min_points=100),
    "mc14": dict(preset="mc14", ground=True, min_points=100),
    "core": dict(preset="none", ground=False, min_points=1),
    "core_mc1": dict(preset="mc1", ground=False, min_points=1),
}


def ref_config(c, offsets=None, theta=10.0, keep_above=None, d_max=0.8):
    pattern = R.MCPattern(tuple(offsets)) if offsets is not None else R.preset_pattern(c["preset"])
    return R.PipelineConfig(ground=R.GroundParams(theta_deg=theta, keep_above_z=keep_above),
                            threshold=R.DistanceThreshold(d_max), mc_pattern=pattern,
                            min_cluster_points=c["min_points"], ground_removal=c["ground"])


def run_case(store, key, g, ranges, c, stages=False, offsets=None, **kw):
    m = ref_model(g)
    cfg = ref_config(c, offsets, **kw)
    ri = R.from_ranges(ranges)
    li, _ = R.Pipeline(m, cfg).segment_range_image(ri)
    store[f"{key}/labels"] = li.labels.astype(np.int32)
    store[f"{key}/sizes"] = li.cluster_sizes.astype(np.int64)
    store[f"{key}/cfg"] = np.array([json.dumps(dict(
        offsets=[list(o) for o in cfg.mc_pattern.offsets], ground=cfg.ground_removal,
        min_points=cfg.min_cluster_points, theta=cfg.ground.theta_deg,
        keep_above=cfg.ground.keep_above_z, d_max=cfg.threshold.d_max))])
    if stages:
        if cfg.ground_removal:
            gm = R.extract_ground(ri, R.height_image(ri, m), m, cfg.ground)
        else:
            gm = R.GroundMask(mask=~ri.valid_mask())
        conn = R.build_connectivity(ri, gm, m, cfg.threshold)
        store[f"{key}/ground"] = np.packbits(gm.mask)
        store[f"{key}/horizontal"] = np.packbits(conn.horizontal)
        store[f"{key}/vertical"] = np.packbits(conn.vertical)
    return li


def make_frames():
    store = {}
    frames = {
        "c0": (geometry("c0"), S.make_batch(0, 1).numpy()[0]),
        "c1s7": (geometry("c0"), S.make_batch(1, 1, first_seed=7).numpy()[0]),
        "c2": (geometry("c2"), S.make_batch(2, 1).numpy()[0]),
        "c3": (geometry("c3"), S.make_batch(3, 1).numpy()[0]),
        "c4": (geometry("c0"), S.make_batch(4, 1).numpy()[0]),
    }
    fx = RS.fixture_model()
    frames["twobox"] = (geometry("fixture"), RS.two_box_scene(fx)[0])
    frames["occluder"] = (geometry("fixture"), RS.two_box_scene(fx, occlusion_gap=True)[0])
    for fname, (g, ranges) in frames.items():
        put_geometry(store, fname, g)
        store[f"{fname}/ranges"] = ranges.astype(F32)
        names = PIPE_CONFIGS if fname in ("c0", "c4") else ("default", "mc1", "core")
        for cname in names:
            li = run_case(store, f"{fname}/{cname}", g, ranges, PIPE_CONFIGS[cname],
                          stages=cname in ("default", "core"))
            print(fname, cname, li.cluster_count)
    # non-default parameters on the config-0 frame
    g, ranges = frames["c0"]
    run_case(store, "c0/theta5_d04", g, ranges, PIPE_CONFIGS["default"], stages=True,
             theta=5.0, d_max=0.4)
    run_case(store, "c0/keep_m05_mc", g, ranges, PIPE_CONFIGS["default"], stages=True,
             offsets=[(1, -4), (0, 5), (7, -3)], keep_above=-0.5, d_max=0.9)
    np.savez_compressed(OUT / "frames.npz", **store)
    print("frames.npz", len(store), "arrays")


def make_random():
    store = {}
    rng = np.random.default_rng(20260809)
    n = 60
    for i in range(n):
        H = int(rng.integers(2, 21))
        W = int(rng.integers(1, 25))
        top = float(rng.choice([-2.0, 3.0, 20.0]))
        g = dict(angles=top - 1.0 * np.arange(H), step=360.0 / W, mount=1.7, width=W)
        ranges = rng.uniform(0.5, 12.0, size=(H, W)).astype(F32)
        ranges[rng.random((H, W)) < 0.3] = 0.0
        offsets = []
        for _ in range(int(rng.integers(0, 5))):
            dy = int(rng.integers(0, min(H - 1, 3) + 1))
            dx = int(rng.integers(-min(W - 1, 3), min(W - 1, 3) + 1))
            if dy == 0 and dx == 0:
                if W == 1:
                    continue
                dx = 1
            offsets.append((dy, dx))
        c = dict(preset="none", ground=bool(rng.random() < 0.5), min_points=int(rng.choice([1, 1, 3, 6])))
        key = f"r{i:03d}"
        put_geometry(store, key, g)
        store[f"{key}/ranges"] = ranges
        run_case(store, key, g, ranges, c, stages=True, offsets=offsets)
    np.savez_compressed(OUT / "random.npz", **store)
    print("random.npz", n, "cases")


if __name__ == "__main__":
    make_tables()
    make_frames()
    make_random()
