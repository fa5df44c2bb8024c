"""The stages as separate GPU calls (paper_2003_00575_b200.stages: height_image,
extract_ground, build_connectivity) against the
reference's recorded stage outputs (tests/golden/frames.npz) and the
reference's float32 formulas restated in numpy (exact IEEE float32 ops)."""

import numpy as np
import pytest

import golden
import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import stages

pytestmark = pytest.mark.gpu

CASES = [(c, f) for c, f in golden.frame_cases()
         if golden.load("frames").get(f"{c}/ground") is not None][:12]


@pytest.mark.parametrize("case_key,frame_key", CASES)
def test_stages_match_reference(case_key, frame_key, cuda):
    m, cfg, ranges, _, _, (g_want, h_want, v_want) = golden.case("frames", case_key, frame_key)
    ri = rs.from_ranges(ranges)
    z = stages.height_image(ri, m)
    want_z = ranges * m.sin_channel[:, None].astype(np.float32)
    want_z += np.float32(m.mount_height)
    want_z = np.where(ranges > 0, want_z, np.float32(np.nan)).astype(np.float32)
    assert np.array_equal(z, want_z, equal_nan=True)
    if cfg.ground_removal:
        gm = stages.extract_ground(ri, z, m, cfg.ground)
        assert np.array_equal(gm.mask, g_want)
    gm = stages.GroundMask(mask=g_want)
    conn = stages.build_connectivity(ri, gm, m, cfg.threshold)
    assert np.array_equal(conn.horizontal, h_want)
    assert np.array_equal(conn.vertical, v_want)


def test_caller_inputs_are_used(rng, cuda):
    """A caller's own height image / ground mask decide, as in the reference."""
    m = rs.default_model()
    ranges = rng.uniform(1, 30, size=(m.height, m.width)).astype(np.float32)
    ri = rs.from_ranges(ranges)
    low = np.full(ranges.shape, -100.0, np.float32)      # everything low enough
    high = np.full(ranges.shape, 100.0, np.float32)      # nothing low enough
    g_low = stages.extract_ground(ri, low, m).mask
    g_high = stages.extract_ground(ri, high, m).mask
    assert not g_high.any() and g_low.sum() >= 0
    everything = stages.GroundMask(mask=np.ones(ranges.shape, bool))
    conn = stages.build_connectivity(ri, everything, m)
    assert not conn.horizontal.any() and not conn.vertical.any()
    with pytest.raises(ValueError):
        stages.extract_ground(ri, low[:-1], m)
    with pytest.raises(ValueError):
        stages.height_image(rs.from_ranges(ranges[:-1]), m)
