"""Seeded randomized parity: random geometries, parameters, Map Connection
patterns, band heights and node capacities, GPU against the CPU oracle
(bit-exact labels and sizes).  Complements the hand-picked cases in
test_gpu_parity.py with combinations nobody thought of."""

import os

import numpy as np
import pytest
import torch

import paper_2003_00575_b200 as rs
from oracle import oracle

pytestmark = pytest.mark.gpu


def _case(seed):
    g = np.random.default_rng(1000 + seed)
    H = int(g.integers(2, 80))
    W = int(g.choice([1, 2, 7, 31, 32, 33, 96, 127, 128, 129, 300, 512, 1000, 2048]))
    top = float(g.uniform(-5, 25))
    step = float(g.uniform(0.1, min(2.0, 50.0 / H)))   # elevations stay in (-30, 25) deg
    model = rs.SensorModel(top - step * np.arange(H), 360.0 / W, float(g.uniform(0.5, 2.5)), width=W)
    offs = []
    for _ in range(int(g.integers(0, 6))):
        dy = int(g.integers(0, min(H, 6)))
        dx = int(g.integers(-min(W - 1, 40), min(W, 41)))
        if dy == 0 and dx <= 0:
            dx = -dx
        if (dy, dx) != (0, 0) and (dy, dx) not in offs and abs(dx) < W:
            offs.append((dy, dx))
    cfg = rs.PipelineConfig(
        ground=rs.GroundParams(theta_deg=float(g.uniform(1, 30)),
                               keep_above_z=None if g.random() < 0.5 else float(g.uniform(-3, 1))),
        threshold=rs.DistanceThreshold(d_max=float(g.uniform(0.1, 3.0))),
        mc_pattern=rs.MCPattern(tuple(offs)),
        min_cluster_points=int(g.choice([1, 2, 5, 30])),
        ground_removal=bool(g.random() < 0.7))
    B = int(g.integers(1, 5))
    frames = np.exp(g.uniform(np.log(0.3), np.log(60.0), size=(B, H, W))).astype(np.float32)
    frames[g.random(frames.shape) < g.uniform(0, 0.5)] = 0
    if g.random() < 0.3:                       # smooth surfaces: long runs, big components
        frames = np.where(frames > 0, np.float32(g.uniform(2, 20)), frames).astype(np.float32)
    rows = int(g.choice([r for r in (0, 0, 1, 3, 8, 16, 31, 64) if r == 0 or -(-H // r) <= 16]))
    cap = int(g.choice([0, 0, 0, 40, 600]))
    return model, cfg, frames, rows, cap


@pytest.mark.parametrize("seed", range(int(os.environ.get("RS_FUZZ_N", "60"))))
def test_fuzz_vs_oracle(seed, cuda):
    model, cfg, frames, rows, cap = _case(seed)
    try:
        pipe = rs.Pipeline(model, cfg, device="cuda:0", rows_per_cta=rows, node_capacity=cap)
    except ValueError as e:   # e.g. a band height the plan cannot use for this geometry
        pytest.skip(str(e))
    res = pipe.segment_batch(torch.as_tensor(frames).cuda())
    torch.cuda.synchronize()
    for b in range(frames.shape[0]):
        wl, ws = oracle.segment_frame(frames[b], pipe.packed)
        got = res.label_image(b)
        assert np.array_equal(got.labels, wl), f"{int((got.labels != wl).sum())} label mismatches"
        assert np.array_equal(got.cluster_sizes, ws)
