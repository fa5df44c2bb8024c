"""Seeded synthetic range images for BASELINE.json's five configs.

No public dataset is named by BASELINE.json and the reference's real data
(SemanticKITTI, test_acceptance.py:236-255) is not available, so these frames
stand in for it.  The scanner is ray cast analytically, in the manner of the
reference's own fixture renderer (synthetic.py:58-95: beam at the column
centre ``(c + 0.5) * step``, ground plane at z = 0 of the ground frame, sensor
at the mount height), extended with what the configs ask for and the
reference renderer lacks: vertical cylinders, 0.1 m poles, a max-range cut,
Gaussian range noise, i.i.d. dropout and stripe dropout.

Generator choices the configs leave open (documented in DESIGN.md):

* object centres: radius ~ U(r_lo, r_hi) (radius-uniform), azimuth ~ U(0, 2 pi);
* box footprint U(0.5, 5) x U(0.5, 5) m, height U(1, 3) m, yaw 0, on the ground;
* order: ray cast -> max-range cut -> + N(0, sigma) in float64 -> float32 ->
  dropout (zeroed cells) -> clamp at 0;
* config 3 has no stated max range: 100 m; config 4 has no stated noise: 0.02 m;
* config 4 poles: 0.1 x 0.1 m, height U(1.5, 4) m, radius U(4, 50) m; stripes are
  finite segments (horizontal: 1..S+1 rows x U(16, 256) columns, vertical:
  1..S+1 columns x U(4, 32) rows) drawn until >= 30% of cells are dropped.

Scene parameters, noise and dropout come from ``numpy.random.default_rng((config,
seed))``; the ray cast runs in float64 torch on any device (IEEE ops only, so
CPU and GPU produce the same bits).  This module is input generation, not part
of the segmentation path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .sensor import SensorModel, fov_model


@dataclass(frozen=True)
class SceneSpec:
    name: str
    H: int
    W: int
    top_deg: float
    bottom_deg: float
    mount: float
    batch: int
    n_boxes: tuple            # (lo, hi) inclusive box count per frame
    box_radius: tuple
    n_cylinders: int = 0
    cyl_radius: tuple = (3.0, 60.0)
    n_poles: int = 0
    pole_radius: tuple = (4.0, 50.0)
    max_range: float = 80.0
    noise: float = 0.02
    dropout: float = 0.05
    stripe_dropout: float = 0.0
    skip: int = 0             # S: stripe widths are 1..S+1
    ground_only: bool = False


CONFIGS = {
    0: SceneSpec("c0_hdl64_single", 64, 2048, 2.0, -24.8, 1.73, 1, (40, 40), (4.0, 50.0)),
    1: SceneSpec("c1_hdl64_b256", 64, 2048, 2.0, -24.8, 1.73, 256, (10, 80), (4.0, 50.0)),
    2: SceneSpec("c2_os128_b128", 128, 2048, 22.5, -22.5, 1.8, 128, (120, 120), (3.0, 60.0),
                 n_cylinders=60, cyl_radius=(3.0, 60.0), max_range=100.0, dropout=0.08),
    3: SceneSpec("c3_vlp32_b1024", 32, 1024, 15.0, -25.0, 1.5, 1024, (20, 20), (2.0, 30.0),
                 max_range=100.0, noise=0.03, dropout=0.03),
    4: SceneSpec("c4_stress_b256", 64, 2048, 2.0, -24.8, 1.73, 256, (0, 0), (4.0, 50.0),
                 n_poles=200, dropout=0.0, stripe_dropout=0.30, ground_only=True),
}


def sensor_for(spec: SceneSpec) -> SensorModel:
    return fov_model(spec.H, spec.top_deg, spec.bottom_deg, spec.W, spec.mount)


def _place(rng, n, r_lo, r_hi):
    rad = rng.uniform(r_lo, r_hi, size=n)
    az = rng.uniform(0.0, 2.0 * math.pi, size=n)
    return rad * np.cos(az), rad * np.sin(az)


def _scene_objects(spec: SceneSpec, rng):
    """Boxes as (lo[3], hi[3]) and cylinders as (cx, cy, rho, h), float64."""
    boxes = []
    n_box = int(rng.integers(spec.n_boxes[0], spec.n_boxes[1] + 1))
    cx, cy = _place(rng, n_box, *spec.box_radius)
    for i in range(n_box):
        sx, sy = rng.uniform(0.5, 5.0, size=2)
        sz = rng.uniform(1.0, 3.0)
        lo = (cx[i] - sx / 2, cy[i] - sy / 2, 0.0)
        hi = (cx[i] + sx / 2, cy[i] + sy / 2, sz)
        if lo[0] - 0.5 < 0.0 < hi[0] + 0.5 and lo[1] - 0.5 < 0.0 < hi[1] + 0.5:
            shift = (max(sx, sy) / 2 + 1.0) / max(math.hypot(cx[i], cy[i]), 1e-6)
            lo = (lo[0] + cx[i] * shift, lo[1] + cy[i] * shift, 0.0)
            hi = (hi[0] + cx[i] * shift, hi[1] + cy[i] * shift, sz)
        boxes.append((lo, hi))
    px, py = _place(rng, spec.n_poles, *spec.pole_radius)
    for i in range(spec.n_poles):
        h = rng.uniform(1.5, 4.0)
        boxes.append(((px[i] - 0.05, py[i] - 0.05, 0.0), (px[i] + 0.05, py[i] + 0.05, h)))
    cyls = []
    qx, qy = _place(rng, spec.n_cylinders, *spec.cyl_radius)
    for i in range(spec.n_cylinders):
        cyls.append((qx[i], qy[i], rng.uniform(0.2, 0.6), rng.uniform(1.0, 2.0)))
    return boxes, cyls


def _stripes(spec: SceneSpec, rng):
    H, W = spec.H, spec.W
    drop = np.zeros((H, W), dtype=bool)
    target = spec.stripe_dropout * H * W
    while drop.sum() < target:
        w = int(rng.integers(1, spec.skip + 2))
        if rng.random() < 0.5:     # horizontal segment: w rows x L columns (wraps)
            r = int(rng.integers(0, H))
            c0, L = int(rng.integers(0, W)), int(rng.integers(16, 257))
            cols = (c0 + np.arange(L)) % W
            drop[r:r + w][:, cols] = True
        else:                      # vertical segment: L rows x w columns
            c = int(rng.integers(0, W))
            r0, L = int(rng.integers(0, H)), int(rng.integers(4, 33))
            cols = (c + np.arange(w)) % W
            drop[r0:r0 + L][:, cols] = True
    return drop


def _beams(model: SensorModel, device):
    phi = (np.arange(model.width) + 0.5) * model.azimuth_step
    cd, sd = model.cos_channel[:, None], model.sin_channel[:, None]
    dx = cd * np.cos(phi)[None, :]
    dy = cd * np.sin(phi)[None, :]
    dz = np.broadcast_to(sd, (model.height, model.width))
    return [torch.from_numpy(np.ascontiguousarray(a)).to(device) for a in (dx, dy, dz)]


def _cast(model: SensorModel, objects, device):
    """First-hit distance per beam for one frame (float64, inf = miss)."""
    d = _beams(model, device)
    oz = model.mount_height
    org = (0.0, 0.0, oz)
    tbest = torch.where(d[2] < 0, (0.0 - oz) / d[2], torch.full_like(d[2], math.inf))
    boxes, cyls = objects
    inv = [1.0 / torch.where(a == 0, torch.full_like(a, 1e-300), a) for a in d]
    for lo, hi in boxes:
        tn = torch.full_like(tbest, -math.inf)
        tf = torch.full_like(tbest, math.inf)
        for ax in range(3):
            t1 = (lo[ax] - org[ax]) * inv[ax]
            t2 = (hi[ax] - org[ax]) * inv[ax]
            tn = torch.maximum(tn, torch.minimum(t1, t2))
            tf = torch.minimum(tf, torch.maximum(t1, t2))
        t = torch.where((tn <= tf) & (tn > 1e-9), tn, torch.full_like(tn, math.inf))
        tbest = torch.minimum(tbest, t)
    for cx, cy, rho, h in cyls:
        ox, oy = -cx, -cy
        a = d[0] * d[0] + d[1] * d[1]
        b = 2.0 * (d[0] * ox + d[1] * oy)
        c = ox * ox + oy * oy - rho * rho
        disc = b * b - 4.0 * a * c
        ok = (disc >= 0) & (a > 0)
        t = (-b - torch.sqrt(torch.clamp(disc, min=0.0))) / (2.0 * a)
        z = oz + t * d[2]
        side = ok & (t > 1e-9) & (z >= 0.0) & (z <= h)
        tc = (h - oz) / torch.where(d[2] == 0, torch.full_like(d[2], 1e-300), d[2])
        xc, yc = tc * d[0] + ox, tc * d[1] + oy
        cap = (d[2] < 0) & (tc > 1e-9) & (xc * xc + yc * yc <= rho * rho)
        tt = torch.where(side, t, torch.full_like(t, math.inf))
        tt = torch.minimum(tt, torch.where(cap, tc, torch.full_like(tc, math.inf)))
        tbest = torch.minimum(tbest, tt)
    return tbest


def render_frame(spec: SceneSpec, seed: int, config_id: int, device="cpu",
                 model: SensorModel | None = None) -> torch.Tensor:
    """One seeded frame of ``spec`` as float32 [H, W] on ``device``."""
    model = model or sensor_for(spec)
    rng = np.random.default_rng((config_id, seed))
    objects = ([], []) if spec.ground_only and spec.n_poles == 0 else _scene_objects(spec, rng)
    t = _cast(model, objects, device)
    t = torch.where(torch.isfinite(t) & (t <= spec.max_range), t, torch.zeros_like(t))
    noise = torch.from_numpy(rng.normal(0.0, spec.noise, size=(spec.H, spec.W))).to(device)
    r = torch.where(t > 0, t + noise, t).to(torch.float32)
    keep = rng.random((spec.H, spec.W)) >= spec.dropout
    if spec.stripe_dropout > 0:
        keep &= ~_stripes(spec, rng)
    r = r * torch.from_numpy(keep).to(device)
    return torch.clamp(r, min=0.0).contiguous()


def make_batch(config_id: int, batch: int | None = None, device="cpu",
               first_seed: int = 0) -> torch.Tensor:
    """Frames ``first_seed .. first_seed+batch-1`` of config ``config_id`` as [B, H, W]."""
    spec = CONFIGS[config_id]
    n = spec.batch if batch is None else batch
    model = sensor_for(spec)
    out = torch.empty((n, spec.H, spec.W), dtype=torch.float32, device=device)
    for i in range(n):
        out[i] = render_frame(spec, first_seed + i, config_id, device, model)
    return out
