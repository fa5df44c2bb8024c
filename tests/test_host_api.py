"""Host logic that runs without a GPU: parameter objects, validation errors
(mirroring the reference's ValueError conditions), planning and the C ABI
library's exported symbols."""

import ctypes
import math
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import _native

ROOT = Path(__file__).resolve().parents[1]


# -- patterns (map_connections.py:23-70; reference tests test_map_connections.py:24-58)
def test_preset_sizes():
    assert len(rs.preset_pattern("mc1")) == 2
    assert len(rs.preset_pattern("mc6")) == 6
    assert len(rs.preset_pattern("mc14")) == 14
    assert len(rs.preset_pattern("none")) == 0


def test_mc14_is_diagonal():
    assert all(dy == dx for dy, dx in rs.preset_pattern("mc14").offsets)


def test_unknown_preset_rejected():
    with pytest.raises(ValueError):
        rs.preset_pattern("mc99")


def test_pattern_canonicalizes_and_dedupes():
    p = rs.MCPattern(((0, -2), (0, 2), (-1, 3), (1, -3)))
    assert p.offsets == ((0, 2), (1, -3))


def test_parse_offsets():
    assert rs.parse_offsets("0,2;2,0 ; 3,3").offsets == ((0, 2), (2, 0), (3, 3))


def test_zero_offset_rejected():
    with pytest.raises(ValueError):
        rs.MCPattern(((0, 0),))


def test_skip_count_mapping():
    assert rs.skip_pattern(0).offsets == ()
    assert set(rs.skip_pattern(1).offsets) == set(rs.preset_pattern("mc1").offsets)
    assert set(rs.skip_pattern(2).offsets) == {(0, 2), (2, 0), (0, 3), (3, 0)}
    with pytest.raises(ValueError):
        rs.skip_pattern(-1)


# -- parameter validation (ground.py:40-43, connectivity.py:29-30, sensor.py:68-95)
def test_params_validation():
    with pytest.raises(ValueError):
        rs.GroundParams(theta_deg=0.0)
    with pytest.raises(ValueError):
        rs.GroundParams(theta_deg=95.0)
    with pytest.raises(ValueError):
        rs.GroundParams(keep_above_z=math.nan)
    with pytest.raises(ValueError):
        rs.DistanceThreshold(0.0)
    assert rs.DistanceThreshold(0.8).d_max_sq == pytest.approx(0.64)


def test_sensor_validation():
    with pytest.raises(rs.SensorConfigError):
        rs.SensorModel([1.0], 0.1, 1.0)
    with pytest.raises(rs.SensorConfigError):
        rs.SensorModel([1.0, 2.0, 1.5], 0.1, 1.0)
    with pytest.raises(rs.SensorConfigError):
        rs.SensorModel([1.0, 2.0], 0.0, 1.0)
    with pytest.raises(rs.SensorConfigError):
        rs.SensorModel([1.0, 2.0], 1.0, 1.0, width=400)
    assert rs.default_model().shape == (64, 4000)


def test_load_sensor_model_yaml(tmp_path):
    p = tmp_path / "s.yaml"
    p.write_text("channels: 64\nvertical_fov: [2.0, -23.2]\nazimuth_step_deg: 0.09\n"
                 "mount_height_m: 1.73\n")
    m = rs.load_sensor_model(p)
    assert m.shape == (64, 4000)
    m2 = rs.load_sensor_model(m.to_dict())
    assert np.array_equal(m2.channel_angles, m.channel_angles)
    with pytest.raises(rs.SensorConfigError):
        rs.load_sensor_model({"channels": 2})


def test_offset_beyond_frame_rejected():
    m = rs.uniform_model(4, top_deg=-2.0, step_deg=1.0, azimuth_step_deg=90.0,
                         mount_height_m=1.7, width=4)
    with pytest.raises(ValueError):
        rs.pack_tables(m, rs.PipelineConfig(mc_pattern=rs.MCPattern(((5, 0),))))
    with pytest.raises(ValueError):
        rs.pack_tables(m, rs.PipelineConfig(mc_pattern=rs.MCPattern(((0, 4),))))


def test_extreme_geometry_rejected_with_ground_on():
    m = rs.uniform_model(4, top_deg=-80.0, step_deg=4.0, azimuth_step_deg=45.0,
                         mount_height_m=1.5)
    with pytest.raises(ValueError):
        rs.pack_tables(m, rs.PipelineConfig(ground=rs.GroundParams(theta_deg=15.0)))
    rs.pack_tables(m, rs.PipelineConfig(ground_removal=False))   # bypass never checks


def test_from_ranges_validation():
    with pytest.raises(ValueError):
        rs.from_ranges(np.zeros(5, np.float32))
    with pytest.raises(ValueError):
        rs.from_ranges(np.full((2, 2), np.nan, np.float32))
    with pytest.raises(ValueError):
        rs.from_ranges(np.full((2, 2), -1.0, np.float32))
    assert rs.from_ranges(np.ones((2, 3))).ranges.dtype == np.float32


# -- the C ABI library ---------------------------------------------------------
def _header_symbols():
    text = (ROOT / "include" / "rangeseg_b200.h").read_text()
    return set(re.findall(r"^\w[\w\s\*]*?\b(rs_\w+)\s*\(", text, flags=re.M))


def test_library_exports_every_header_symbol():
    lib = _native.lib()
    declared = _header_symbols()
    assert declared == set(_native.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.rs_version() == 300


def test_tables_count_matches_layout():
    lib = _native.lib()
    for H, n in ((64, 0), (64, 14), (2, 1)):
        assert lib.rs_tables_count(H, n) == rs.PackedTables.size(H, n)


@pytest.mark.parametrize("H,W,R,C", [(64, 2048, 32, 2), (32, 1024, 32, 1), (8, 16, 8, 1),
                                     (3, 5, 3, 1), (128, 2048, None, None),
                                     (64, 4000, None, None), (200, 1000, None, None)])
def test_plan(H, W, R, C):
    m = rs.fov_model(H, 2.0, -20.0, W, 1.7)
    cfg = _native.make_config(rs.pack_tables(m, rs.PipelineConfig()))
    r, c, smem = _native.plan(cfg)
    if R is not None:
        assert (r, c) == (R, C)
    assert c <= 16 and r * c >= H and r * (c - 1) < H
    assert smem <= 227 * 1024


def test_plan_rejects_bad_config():
    m = rs.fov_model(8, 2.0, -20.0, 16, 1.7)
    cfg = _native.make_config(rs.pack_tables(m, rs.PipelineConfig()))
    cfg.offsets[0][0], cfg.offsets[0][1] = 0, -1
    cfg.n_offsets = 1
    with pytest.raises(ValueError, match="canonical"):
        _native.plan(cfg)
    cfg.n_offsets = 0
    cfg.height = 1
    with pytest.raises(ValueError):
        _native.plan(cfg)


def test_plan_rejects_frames_beyond_a_cluster():
    m = rs.fov_model(512, 20.0, -20.0, 8192, 1.7)
    with pytest.raises(ValueError):
        rs.Pipeline(m, rs.PipelineConfig(ground_removal=False), device="cpu")


def test_pipeline_refuses_cpu_device():
    m = rs.fov_model(8, 2.0, -20.0, 16, 1.7)
    pipe = rs.Pipeline(m, device="cpu")
    import torch
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        pipe.segment_batch(torch.zeros((1, 8, 16)))


def test_reserved_fields_rejected():
    """reserved[1]/[2] are experiment hooks: a production build rejects them."""
    m = rs.fov_model(8, 2.0, -20.0, 16, 1.7)
    cfg = _native.make_config(rs.pack_tables(m, rs.PipelineConfig()))
    cfg.reserved[1] = 3
    with pytest.raises(ValueError, match="reserved"):
        _native.plan(cfg)
    cfg.reserved[1] = 0
    cfg.reserved[2] = 1
    with pytest.raises(ValueError, match="reserved"):
        _native.plan(cfg)


def test_plan_prefers_fast_kernel_when_dense_cannot_hold():
    """H=512, W=1024: no dense plan (17 bands of 31 rows) but 8 fast bands fit."""
    m = rs.fov_model(512, 20.0, -20.0, 1024, 1.7)
    cfg = _native.make_config(rs.pack_tables(m, rs.PipelineConfig(ground_removal=False)))
    d = _native.plan_detail(cfg)
    assert d["fast"] == 1 and d["fast_ctas"] <= 16


def _host_call(cfg, batch, sizes_stride, with_sizes=True):
    import ctypes
    lib = _native.lib()
    H, W = cfg.height, cfg.width
    tab = np.zeros(lib.rs_tables_count(H, cfg.n_offsets), np.float32)
    rg = np.zeros((max(batch, 1), H, W), np.float32)
    lab = np.zeros((max(batch, 1), H, W), np.int32)
    ncl = np.zeros(max(batch, 1), np.int32)
    sz = np.zeros((max(batch, 1), max(sizes_stride, 1)), np.int64)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)   # noqa: E731
    return lib.rs_segment_batch_host(ctypes.byref(cfg), p(tab), p(rg), batch, p(lab), p(ncl),
                                     p(sz) if with_sizes else None, sizes_stride)


def test_host_entry_checks_sizes_stride_before_any_launch():
    m = rs.fov_model(8, 2.0, -20.0, 16, 1.7)
    cfg = _native.make_config(rs.pack_tables(m, rs.PipelineConfig(min_cluster_points=1)))
    need = 8 * 16 + 1
    assert _host_call(cfg, 2, need - 1) == _native.RS_EINVAL
    assert b"sizes_stride" in _native.lib().rs_last_error()
    assert _host_call(cfg, 2, -5) == _native.RS_EINVAL
    assert _host_call(cfg, -1, need) == _native.RS_EINVAL
    assert _host_call(cfg, 0, need) == _native.RS_OK


def test_device_entry_checks_alignment_and_stride():
    import ctypes
    lib = _native.lib()
    m = rs.fov_model(8, 2.0, -20.0, 128, 1.7)
    cfg = _native.make_config(rs.pack_tables(m, rs.PipelineConfig(min_cluster_points=1)))
    fake = ctypes.c_void_p(0x10000)
    # misaligned labels pointer
    st = lib.rs_segment_batch(ctypes.byref(cfg), fake, fake, 1, ctypes.c_void_p(0x10004), fake, None, 0, None)
    assert st == _native.RS_EINVAL and b"aligned" in lib.rs_last_error()
    st = lib.rs_segment_batch(ctypes.byref(cfg), fake, fake, 1, fake, fake, fake, 10, None)
    assert st == _native.RS_EINVAL and b"sizes_stride" in lib.rs_last_error()


def test_plan_cache_keeps_errors_per_config():
    m = rs.fov_model(8, 2.0, -20.0, 16, 1.7)
    good = _native.make_config(rs.pack_tables(m, rs.PipelineConfig()))
    bad = _native.make_config(rs.pack_tables(m, rs.PipelineConfig()))
    bad.rows_per_cta = 99
    for _ in range(3):
        assert _native.plan(good)[1] >= 1
        with pytest.raises(ValueError, match="rows_per_cta"):
            _native.plan(bad)


def test_small_batches_get_thinner_bands():
    m = rs.fov_model(64, 2.0, -24.8, 2048, 1.73)
    cfg = _native.make_config(rs.pack_tables(m, rs.PipelineConfig()))
    big = _native.plan_batch(cfg, 256)
    assert (big["fast_rows"], big["fast_ctas"]) == (32, 2) == (_native.plan_detail(cfg)["fast_rows"], 2)
    one = _native.plan_batch(cfg, 1)
    assert one["fast"] and one["fast_ctas"] == 16 and one["fast_rows"] == 4
    assert _native.plan_batch(cfg, 40)["fast_ctas"] == 4
    # an explicit band height is kept
    cfg.rows_per_cta = 32
    assert _native.plan_batch(cfg, 1)["fast_rows"] == 32


def test_torch_extension_loads_and_matches_abi():
    """The thin PyTorch extension (csrc/torch_ext.cpp) links the same C ABI."""
    ext = _native.torch_ext()
    assert ext.abi_version() == _native.lib().rs_version()
    assert hasattr(ext, "segment_batch")
