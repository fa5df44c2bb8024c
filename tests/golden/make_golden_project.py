"""Golden fixtures for the point-cloud path, recorded from
the Python reference itself in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_project.py

For each (sensor model, cloud) case it stores the reference's
``range_image.project`` outputs (ranges, point_index, n_dropped,
n_overwritten) and ``labels_to_points`` for a random label image.  Clouds are
seeded and include the edge cases the projection rules have: collisions with
equal ranges (highest point index wins), points on channel midpoints and on
the half-gap field-of-view edges, azimuth bin edges and the -pi/pi seam, the
origin, and float32-valued input.  Writes tests/golden/project.npz.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import rangeseg as R  # noqa: E402  (the reference)
from rangeseg.range_image import labels_to_points, project  # noqa: E402

OUT = Path(__file__).resolve().parent / "project.npz"


def models():
    return {
        "hdl64": R.default_model(),
        "c0": R.SensorModel(np.linspace(2.0, -24.8, 64), 360 / 2048, 1.73, width=2048),
        "c2": R.SensorModel(np.linspace(22.5, -22.5, 128), 360 / 2048, 1.8, width=2048),
        "ascending": R.SensorModel([-20.0, -17.0, -14.0, -11.0, -8.0, -5.0], 45.0, 1.5, width=8),
        "partial": R.SensorModel(np.linspace(10.0, -10.0, 16), 1.5, 1.7, width=200),
    }


def sph(r, elev_deg, az_deg):
    e, a = np.radians(elev_deg), np.radians(az_deg)
    return np.stack([r * np.cos(e) * np.cos(a), r * np.cos(e) * np.sin(a), r * np.sin(e)], axis=-1)


def clouds(m, g):
    ang = m.channel_angles_deg
    asc = np.sort(ang)
    step = m.azimuth_step_deg
    out = {}
    out["cube"] = g.uniform(-40, 40, size=(6000, 3))
    # realistic: every channel x column with noise and dropout, plus repeats
    el = np.repeat(ang, 64)
    az = np.tile(np.arange(64) * step * 3.7, ang.size)
    r = g.uniform(1, 60, size=el.size)
    pts = sph(r, el + g.normal(0, 0.02, el.size), az + g.normal(0, 0.01, az.size))
    out["scan"] = np.concatenate([pts, pts[::7]])          # exact duplicates: ties
    # channel midpoints, FOV edges, azimuth bin edges and the seam
    mids = (asc[1:] + asc[:-1]) / 2
    gap_lo, gap_hi = (asc[1] - asc[0]) / 2, (asc[-1] - asc[-2]) / 2
    edges_el = np.concatenate([mids, [asc[0] - gap_lo, asc[-1] + gap_hi,
                                      asc[0] - gap_lo - 1e-9, asc[-1] + gap_hi + 1e-9]])
    e2 = np.repeat(edges_el, 9)
    a2 = np.tile(np.array([0.0, step, 2 * step, 179.999999, 180.0, -180.0, -step, -1e-12, 359.9]),
                 edges_el.size)
    out["edges"] = np.concatenate([sph(g.uniform(2, 30, e2.size), e2, a2),
                                   np.zeros((3, 3)),                       # origin: dropped
                                   [[5.0, 0.0, 0.0], [5.0, 0.0, 0.0],      # equal ranges, one cell
                                    [3.0, -0.0, 0.0], [-4.0, 0.0, 0.0], [-4.0, -0.0, 0.0]]])
    out["f32"] = g.uniform(-25, 25, size=(3000, 3)).astype(np.float32)
    out["wide"] = np.concatenate([g.uniform(-80, 80, size=(2000, 4)),       # extra column ignored
                                  np.ones((5, 4))])
    return out


def main():
    g = np.random.default_rng(20031)
    store = {}
    for mname, m in models().items():
        for cname, pts in clouds(m, g).items():
            key = f"{mname}/{cname}"
            ri = project(pts, m)
            labels = g.integers(0, 9, size=ri.ranges.shape).astype(np.int32)
            store[f"{key}/points"] = np.asarray(pts)
            store[f"{key}/angles_deg"] = m.channel_angles_deg
            store[f"{key}/step_deg"] = np.float64(m.azimuth_step_deg)
            store[f"{key}/mount"] = np.float64(m.mount_height)
            store[f"{key}/width"] = np.int64(m.width)
            store[f"{key}/ranges"] = ri.ranges
            store[f"{key}/point_index"] = ri.point_index
            store[f"{key}/counts"] = np.array([ri.n_points, ri.n_dropped, ri.n_overwritten], np.int64)
            store[f"{key}/labels"] = labels
            store[f"{key}/point_labels"] = labels_to_points(labels, ri)
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT} ({len(store)} arrays)")


if __name__ == "__main__":
    main()
