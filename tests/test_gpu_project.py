"""GPU point-cloud path: rs_project / rs_labels_to_points /
Pipeline.segment_cloud against the reference's recorded outputs
(tests/golden/project.npz) and the CPU oracle.  Projection results must be
bit-identical except on cells that a point within 1e-12 relative of a channel
midpoint, the field-of-view edge or a column edge can reach (there asin /
atan2 last-ulp differences between libraries decide; tests/golden.py
unstable_cells), and those points are counted."""

import numpy as np
import pytest
import torch

import golden
import paper_2003_00575_b200 as rs
from oracle import oracle
from paper_2003_00575_b200 import cloud, synthetic

pytestmark = pytest.mark.gpu


def _assert_projection(got_ranges, got_pidx, got_counts, want_ranges, want_pidx, want_counts, unstable, n_amb):
    st = ~unstable
    assert np.array_equal(got_ranges[st].view(np.uint32), want_ranges[st].view(np.uint32))
    assert np.array_equal(got_pidx[st], want_pidx[st])
    assert abs(int(got_counts[0]) - int(want_counts[0])) <= n_amb
    assert abs(int(got_counts[1]) - int(want_counts[1])) <= 2 * n_amb
    if n_amb == 0:
        assert np.array_equal(got_ranges.view(np.uint32), want_ranges.view(np.uint32))
        assert np.array_equal(got_pidx, want_pidx)
        assert (int(got_counts[0]), int(got_counts[1])) == (int(want_counts[0]), int(want_counts[1]))


@pytest.mark.parametrize("key", golden.project_cases())
def test_project_matches_reference(key, cuda):
    m, c = golden.project_case(key)
    ri = rs.project(c["points"], m)
    unstable, n_amb = golden.unstable_cells(c["points"], m)
    _assert_projection(ri.ranges, ri.point_index, (ri.n_dropped, ri.n_overwritten),
                       c["ranges"], c["point_index"], c["counts"][1:], unstable, n_amb)
    assert ri.n_points == c["counts"][0]


@pytest.mark.parametrize("key", golden.project_cases())
def test_labels_to_points_matches_reference(key, cuda):
    m, c = golden.project_case(key)
    ri = rs.RangeImage(ranges=c["ranges"], point_index=c["point_index"], n_points=int(c["counts"][0]))
    assert np.array_equal(rs.labels_to_points(c["labels"], ri), c["point_labels"])


def _random_clouds(g, model, n_clouds):
    clouds = []
    for _ in range(n_clouds):
        n = int(g.integers(1, 40000))
        kind = g.integers(0, 3)
        if kind == 0:
            pts = g.uniform(-60, 60, size=(n, 3))
        elif kind == 1:   # scan-like: every channel, random azimuths, some exact duplicates
            el = g.choice(model.channel_angles, size=n) + g.normal(0, 1e-3, n)
            az = g.uniform(-np.pi, np.pi, n)
            r = g.uniform(0.5, 90, n)
            pts = np.stack([r * np.cos(el) * np.cos(az), r * np.cos(el) * np.sin(az), r * np.sin(el)], 1)
            pts = np.concatenate([pts, pts[: n // 5]])
        else:             # float32-valued with a fourth column
            pts = np.concatenate([g.uniform(-30, 30, size=(n, 3)), g.uniform(0, 1, size=(n, 1))], 1)
            pts = pts.astype(np.float32).astype(np.float64)
        clouds.append(np.ascontiguousarray(pts))
    return clouds


@pytest.mark.parametrize("cid", [0, 2, 3])
def test_batched_projection_vs_oracle(cid, rng, cuda):
    model = synthetic.sensor_for(synthetic.CONFIGS[cid])
    clouds = _random_clouds(rng, model, 6)
    width = max(c.shape[1] for c in clouds)
    pts = np.concatenate([np.pad(c, ((0, 0), (0, width - c.shape[1]))) for c in clouds])
    off = np.cumsum([0] + [c.shape[0] for c in clouds]).astype(np.int64)
    ranges, pidx, counts = cloud.project_batch(torch.from_numpy(pts).cuda(), torch.from_numpy(off).cuda(), model)
    ranges, pidx, counts = ranges.cpu().numpy(), pidx.cpu().numpy(), counts.cpu().numpy()
    for b, c in enumerate(clouds):
        wr, wp, wd, wo = oracle.project(c, model)
        unstable, n_amb = golden.unstable_cells(c, model)
        _assert_projection(ranges[b], pidx[b], counts[b], wr, wp, (wd, wo), unstable, n_amb)


def test_segment_cloud_matches_oracle_composition(rng, cuda):
    """segment_cloud == oracle project -> oracle segment_frame -> oracle
    labels_to_points (pipeline.py:133-158), for clouds rendered from the
    config-1 scenes (so clusters are real objects) plus noise points."""
    spec = synthetic.CONFIGS[1]
    model = synthetic.sensor_for(spec)
    pipe = rs.Pipeline(model, rs.PipelineConfig(), device="cuda:0")
    frames = synthetic.make_batch(1, 3, "cpu").numpy()
    el = np.asarray(model.channel_angles)[:, None]
    az = (np.arange(model.width) + 0.5) * model.azimuth_step
    clouds = []
    for f in frames:
        r = f.astype(np.float64)
        keep = r > 0
        x = (r * np.cos(el) * np.cos(az))[keep]
        y = (r * np.cos(el) * np.sin(az))[keep]
        z = (r * np.sin(el) * np.ones_like(az))[keep]
        pts = np.stack([x, y, z], 1)
        pts = np.concatenate([pts, rng.uniform(-50, 50, size=(2000, 3))])
        clouds.append(pts[rng.permutation(len(pts))])
    outs = pipe.segment_clouds(clouds)
    for pts, (seg, _) in zip(clouds, outs):
        wr, wp, wd, wo = oracle.project(pts, model)
        unstable, n_amb = golden.unstable_cells(pts, model)
        assert n_amb == 0
        wl, ws = oracle.segment_frame(wr, pipe.packed)
        assert np.array_equal(seg.label_image.labels, wl)
        assert np.array_equal(seg.label_image.cluster_sizes, ws)
        assert np.array_equal(seg.point_labels, oracle.labels_to_points(wl, wp, len(pts)))
    one, _ = pipe.segment_cloud(clouds[0])
    assert np.array_equal(one.point_labels, outs[0][0].point_labels)


def test_reference_projection_rules(cuda):
    """The reference's own unit cases (test_range_image.py:20-133)."""
    m = rs.default_model()
    ri = rs.project(np.array([[10.0, 0.0, 0.0]]), m)          # on-axis -> the 0 deg channel
    assert ri.ranges[5, 0] == np.float32(10.0) and ri.n_dropped == 0 and ri.n_overwritten == 0
    ri = rs.project(np.array([[7.0, 0.0, 0.0], [5.0, 0.0, 0.0]]), m)
    assert ri.ranges[5, 0] == np.float32(5.0) and ri.point_index[5, 0] == 1 and ri.n_overwritten == 1
    ri = rs.project(np.array([[10.0, 0.0, 0.0], [1.0, 0.0, 5.0]]), m)
    assert ri.n_dropped == 1 and ri.n_projected == 1
    labels = np.full(ri.shape, 3, dtype=np.int32)
    assert rs.labels_to_points(labels, ri)[1] == 0             # dropped point: background
    ri = rs.project(np.array([[5.0, 0.0, 0.0]] * 4), m)        # equal ranges: highest index wins
    assert ri.point_index[5, 0] == 3 and ri.n_overwritten == 3
    az = np.radians(0.09 * 1.5)
    ri = rs.project(np.array([[10 * np.cos(az), 10 * np.sin(az), 0.0]]), m)
    assert ri.ranges[5, 1] > 0                                  # azimuth column convention
    g = np.random.default_rng(5)
    pts = g.uniform(-40, 40, size=(5000, 3))
    ri = rs.project(pts, m)
    assert ri.n_dropped + ri.n_overwritten + ri.n_projected == len(pts)
    with pytest.raises(ValueError):
        rs.project(np.empty((0, 3)), m)
    with pytest.raises(ValueError):
        rs.labels_to_points(np.ones((4, 8), np.int32), rs.from_ranges(np.ones((4, 8), np.float32)))
    seg, _ = rs.Pipeline(m, rs.PipelineConfig(), device="cuda:0").segment_cloud(np.empty((0, 3)))
    assert seg.point_labels.size == 0 and seg.label_image.cluster_sizes[0] == m.height * m.width


def test_scan_files_batch_end_to_end(rng, tmp_path, cuda):
    """KITTI .bin scans -> one pinned upload (io_formats.load_scans_pinned) ->
    project / segment / labels_to_points on the device -> .label files, equal
    to per-scan segment_cloud and to the oracle composition."""
    from paper_2003_00575_b200 import io_formats as io
    model = rs.default_model()
    pipe = rs.Pipeline(model, rs.PipelineConfig(min_cluster_points=10), device="cuda:0")
    paths = []
    for k in range(4):
        pts = rng.uniform(-35, 35, size=(int(rng.integers(5000, 30000)), 3)).astype(np.float32)
        io.write_velodyne_bin(tmp_path / f"{k:06d}.bin", pts, rng.uniform(0, 1, len(pts)))
        paths.append(tmp_path / f"{k:06d}.bin")
    x, off = io.load_scans_pinned(paths)
    ranges, pidx, _ = cloud.project_batch(x, off, model)
    res = pipe.segment_batch(ranges)
    plab = cloud.labels_to_points_batch(res.labels, pidx, off).cpu().numpy()
    offs = off.cpu().numpy()
    for k, p in enumerate(paths):
        pts = io.read_velodyne_bin(p)
        mine = plab[offs[k]:offs[k + 1]]
        seg, _ = pipe.segment_cloud(pts)
        assert np.array_equal(mine, seg.point_labels)
        wr, wp, _, _ = oracle.project(pts, model)
        wl, _ = oracle.segment_frame(wr, pipe.packed)
        assert np.array_equal(mine, oracle.labels_to_points(wl, wp, len(pts)))
        io.write_instance_labels(tmp_path / f"{k:06d}.label", mine)
        assert np.array_equal(io.read_instance_labels(tmp_path / f"{k:06d}.label", len(pts)), mine)
