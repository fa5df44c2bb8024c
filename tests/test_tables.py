"""Host-side float32 constant tables are bit-identical to the reference's.

Golden values: SensorModel / ground_bounds / DistanceThreshold of the Python
reference cast to float32 (sensor.py:97-141, ground.py:76-92,
connectivity.py:21-31), recorded by tests/golden/make_golden.py.
"""

import numpy as np
import pytest

import golden
from paper_2003_00575_b200 import (DistanceThreshold, GroundParams, PipelineConfig,
                                   MCPattern, pack_tables)

GEOMS = ("c0", "c2", "c3", "hdl64", "fixture", "small", "ascending")


def _bits(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


@pytest.mark.parametrize("name", GEOMS)
def test_tables_bit_identical(name):
    st = golden.load("tables")
    m = golden.model(st, name)
    H, W = m.height, m.width
    offs = sorted({tuple(int(x) for x in k.split("/")[1][3:].split("_"))
                   for k in st if k.startswith(f"{name}/tc_")})
    mc = [o for o in offs if o not in ((0, 1), (1, 0))]
    for theta in (5.0, 10.0):
        if f"{name}/lo_{theta:g}" not in st:
            with pytest.raises(ValueError):
                pack_tables(m, PipelineConfig(ground=GroundParams(theta_deg=theta)))
            continue
        pt = pack_tables(m, PipelineConfig(ground=GroundParams(theta_deg=theta),
                                           mc_pattern=MCPattern(tuple(mc))))
        assert np.array_equal(_bits(pt.section("lo")), _bits(st[f"{name}/lo_{theta:g}"]))
        assert np.array_equal(_bits(pt.section("hi")), _bits(st[f"{name}/hi_{theta:g}"]))
    pt = pack_tables(m, PipelineConfig(ground_removal=False, mc_pattern=MCPattern(tuple(mc))))
    assert np.array_equal(_bits(pt.section("sin_ch")), _bits(st[f"{name}/sin_ch"]))
    assert np.array_equal(_bits(pt.section("sin_a")), _bits(st[f"{name}/sin_a"]))
    assert np.array_equal(_bits(pt.section("cos_a")), _bits(st[f"{name}/cos_a"]))
    assert np.array_equal(_bits(pt.section("two_cos_v")), _bits(st[f"{name}/tc_1_0"]))
    if W > 1:
        assert _bits(pt.two_cos_h) == _bits(st[f"{name}/tc_0_1"][0])
    for k, (dy, dx) in enumerate(pt.offsets):
        want = st[f"{name}/tc_{dy}_{dx}"]
        got = pt.section("two_cos_off", k)
        if dy == 0:
            assert np.all(_bits(got) == _bits(want[0]))
        else:
            assert np.array_equal(_bits(got[:H - dy]), _bits(want))
    assert _bits(pt.keep_above) == _bits(st[f"{name}/keep_above"])
    assert _bits(pt.mount) == _bits(np.float32(m.mount_height))


@pytest.mark.parametrize("d", [0.8, 0.4, 0.9, 0.25])
def test_threshold_square_bits(d):
    st = golden.load("tables")
    m = golden.model(st, "small")
    pt = pack_tables(m, PipelineConfig(threshold=DistanceThreshold(d)))
    assert _bits(pt.d_max_sq) == _bits(st[f"dmax/{d:g}"])


def test_default_threshold_is_064f():
    m = golden.model(golden.load("tables"), "c0")
    assert _bits(pack_tables(m, PipelineConfig()).d_max_sq) == 0x3F23D70A
