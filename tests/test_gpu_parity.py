"""GPU parity: the sm_100a path (through the C ABI) against the reference's
recorded outputs (tests/golden) and against the CPU oracle on the five
BASELINE configs.  Bar: bit-exact int32 labels and int64 cluster sizes
(integer work), bit-exact ground / edge masks (float32 decisions computed in
the reference's op order — the 1e-6 tolerance band of north_star is not used,
the count of mismatches must be 0)."""

import numpy as np
import pytest
import torch

import golden
import paper_2003_00575_b200 as rs
from oracle import oracle
from paper_2003_00575_b200 import synthetic

pytestmark = pytest.mark.gpu


def _run(model, cfg, frames, **kw):
    pipe = rs.Pipeline(model, cfg, device="cuda:0", **kw)
    x = torch.as_tensor(np.ascontiguousarray(frames, dtype=np.float32)).cuda()
    if x.dim() == 2:
        x = x[None]
    res = pipe.segment_batch(x)
    torch.cuda.synchronize()
    return pipe, res


def _assert_frame(res, b, labels, sizes):
    got = res.label_image(b)
    assert np.array_equal(got.labels, labels), \
        f"{int((got.labels != labels).sum())} label mismatches"
    assert np.array_equal(got.cluster_sizes, sizes)


# ---------------------------------------------------------------- golden -----
@pytest.mark.parametrize("case_key,frame_key", golden.frame_cases())
def test_golden_frames(case_key, frame_key, cuda):
    m, cfg, ranges, labels, sizes, stages = golden.case("frames", case_key, frame_key)
    pipe, res = _run(m, cfg, ranges)
    _assert_frame(res, 0, labels, sizes)
    if stages is not None:
        g, h, v = pipe.stage_masks(torch.from_numpy(ranges).cuda()[None])
        for got, want in zip((g, h, v), stages):
            assert int((got[0].cpu().numpy() != want).sum()) == 0


@pytest.mark.parametrize("key", golden.random_cases())
@pytest.mark.parametrize("rows", [0, 1, 2])
def test_golden_random_frames(key, rows, cuda):
    m, cfg, ranges, labels, sizes, stages = golden.case("random", key)
    if rows and -(-m.height // rows) > 16:
        pytest.skip("more bands than a cluster holds")
    pipe, res = _run(m, cfg, ranges, rows_per_cta=rows)
    _assert_frame(res, 0, labels, sizes)
    g, h, v = pipe.stage_masks(torch.from_numpy(ranges).cuda()[None])
    for got, want in zip((g, h, v), stages):
        assert np.array_equal(got[0].cpu().numpy(), want)


# --------------------------------------------------- BASELINE configs vs oracle
VARIANTS = {
    "default": rs.PipelineConfig(),
    "core": rs.PipelineConfig(ground_removal=False, min_cluster_points=1),
    "S1": rs.PipelineConfig(mc_pattern=rs.skip_pattern(1)),
    "mc14_core": rs.PipelineConfig(mc_pattern=rs.preset_pattern("mc14"),
                                   ground_removal=False, min_cluster_points=1),
}


@pytest.fixture(scope="module")
def config_frames():
    out = {}
    for cid, n in ((0, 1), (1, 12), (2, 6), (3, 24), (4, 12)):
        out[cid] = synthetic.make_batch(cid, n, device="cuda:0")
    return out


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("cid", [0, 1, 2, 3, 4])
def test_configs_vs_oracle(cid, variant, config_frames):
    model = synthetic.sensor_for(synthetic.CONFIGS[cid])
    cfg = VARIANTS[variant]
    frames = config_frames[cid]
    pipe = rs.Pipeline(model, cfg, device="cuda:0")
    res = pipe.segment_batch(frames)
    host = frames.cpu().numpy()
    want_l, want_n, want_s = oracle.segment_batch(host, pipe.packed, sizes_stride=pipe.sizes_stride)
    torch.cuda.synchronize()
    got_l = res.labels.cpu().numpy()
    got_n = res.n_clusters.cpu().numpy()
    got_s = res.cluster_sizes.cpu().numpy()
    assert np.array_equal(got_n, want_n)
    assert int((got_l != want_l).sum()) == 0
    for b in range(host.shape[0]):
        k = int(want_n[b])
        assert np.array_equal(got_s[b, :k + 1], want_s[b, :k + 1])


@pytest.mark.parametrize("rows", [1, 3, 5, 8, 16])
def test_band_height_does_not_change_labels(rows, config_frames):
    model = synthetic.sensor_for(synthetic.CONFIGS[1])
    frames = config_frames[1][:4]
    cfg = rs.PipelineConfig(mc_pattern=rs.preset_pattern("mc6"), ground_removal=False,
                            min_cluster_points=3)
    if -(-64 // rows) > 16:
        pytest.skip("more bands than a cluster holds")
    base = rs.Pipeline(model, cfg, device="cuda:0").segment_batch(frames)
    alt = rs.Pipeline(model, cfg, device="cuda:0", rows_per_cta=rows).segment_batch(frames)
    torch.cuda.synchronize()
    assert torch.equal(base.labels, alt.labels)
    assert torch.equal(base.n_clusters, alt.n_clusters)


def test_full_headline_batch_vs_oracle(cuda):
    """Config 1 at its full size (256 frames, 2^25 cells), reference defaults."""
    frames = synthetic.make_batch(1, device="cuda:0")
    model = synthetic.sensor_for(synthetic.CONFIGS[1])
    pipe = rs.Pipeline(model, rs.PipelineConfig(), device="cuda:0")
    res = pipe.segment_batch(frames)
    want_l, want_n, want_s = oracle.segment_batch(frames.cpu().numpy(), pipe.packed,
                                                  sizes_stride=pipe.sizes_stride)
    torch.cuda.synchronize()
    assert np.array_equal(res.n_clusters.cpu().numpy(), want_n)
    assert int((res.labels.cpu().numpy() != want_l).sum()) == 0
    got_s = res.cluster_sizes.cpu().numpy()
    for b in range(frames.shape[0]):
        k = int(want_n[b])
        assert np.array_equal(got_s[b, :k + 1], want_s[b, :k + 1])


# ------------------------------------------------------------------ edges ---
def _random_model(H, W):
    return rs.SensorModel(-2.0 - 1.0 * np.arange(H), 360.0 / W, 1.7, width=W)


@pytest.mark.parametrize("H,W", [(2, 1), (2, 2), (3, 1), (2, 33), (17, 3), (64, 5), (5, 2048),
                                 (31, 31), (40, 700)])
def test_odd_shapes_vs_oracle(H, W, rng, cuda):
    model = _random_model(H, W)
    frames = rng.uniform(0.5, 12.0, size=(3, H, W)).astype(np.float32)
    frames[rng.random(frames.shape) < 0.3] = 0
    for cfg in (rs.PipelineConfig(ground_removal=False, min_cluster_points=1),
                rs.PipelineConfig(ground_removal=False, min_cluster_points=2,
                                  mc_pattern=rs.MCPattern(tuple(
                                      o for o in ((0, 2), (1, -1), (1, 1), (2, 0))
                                      if o[0] < H and abs(o[1]) < W)))):
        pipe, res = _run(model, cfg, frames)
        for b in range(3):
            wl, ws = oracle.segment_frame(frames[b], pipe.packed)
            _assert_frame(res, b, wl, ws)


@pytest.mark.parametrize("keep", [None, -1e30, -50.0, -1.7, -0.25, 0.0, 0.3, 2.5, 1e30])
def test_height_threshold_edges_vs_oracle(keep, rng, cuda):
    """The kernel replaces z = v*sin + mount <= keep_above by one product
    against a per-row threshold found by exact search (rs_common.cuh
    z_threshold); check it on rows with positive, zero and negative sines and
    on ranges from subnormal to huge, ground mask and labels against the
    oracle (ground.py:112-140 restated)."""
    H, W = 24, 256
    # elevations +6 .. -17 deg in 1 deg steps: row 6 is exactly 0 deg (sin 0)
    model = rs.SensorModel(6.0 - 1.0 * np.arange(H), 360.0 / W, 1.7, width=W)
    frames = np.exp(rng.uniform(np.log(0.05), np.log(200.0), size=(3, H, W))).astype(np.float32)
    frames[rng.random(frames.shape) < 0.15] = 0
    frames[0, :, :8] = np.float32(1e-40)           # subnormal ranges
    frames[0, :, 8:16] = np.float32(3e38)          # near FLT_MAX
    frames[1] = np.float32(5.0)                    # flat ring: many ties at the bound
    cfg = rs.PipelineConfig(ground=rs.GroundParams(theta_deg=12.0, keep_above_z=keep),
                            min_cluster_points=1)
    pipe, res = _run(model, cfg, frames)
    g, _, _ = pipe.stage_masks(torch.as_tensor(frames).cuda())
    for b in range(3):
        wl, ws, wg, _, _ = oracle.segment_frame(frames[b], pipe.packed, stages=True)
        assert np.array_equal(g[b].cpu().numpy(), wg)
        _assert_frame(res, b, wl, ws)


@pytest.mark.parametrize("H,W,rows", [(32, 256, 4), (48, 2048, 16), (64, 1024, 0), (20, 96, 2), (36, 64, 8)])
def test_in_band_map_connections_vs_oracle(H, W, rows, rng, cuda):
    """Map Connections united inside the band (rs_mc.cuh: mc_axis_heads /
    mc_chain_finish) and, for rows whose partner row lies in a band above,
    during the cross-band step (mc_axis_cross): partner rows one and several
    bands up (dy > rows_per_cta), horizontal offsets wider than a word,
    negative dx across the azimuth seam, skip offsets with their detour
    filter, many offsets (one round each), sparse speckle (long hook chains)
    and a fully linked frame with holes (every chain united at once)."""
    model = _random_model(H, W)
    frames = rng.uniform(0.5, 12.0, size=(4, H, W)).astype(np.float32)
    frames[rng.random(frames.shape) < 0.25] = 0
    frames[1] = 7.0                               # everything linked ...
    frames[1, :, ::3] = 0                         # ... but for every third column
    frames[2] = 7.0
    frames[2, 1::2, :] = 0                        # every second row missing: only (2k, 0) links rows
    frames[3, rng.random((H, W)) < 0.6] = 0       # speckle
    cand = ((0, 2), (2, 0), (0, 3), (3, 0), (9, 0), (5, 3), (0, 40), (7, -2), (1, -1), (2, 2), (17, 17),
            (4, -33), (0, W // 2), (H - 1, 1))
    offs = tuple(o for o in cand if o[0] < H and abs(o[1]) < W and (o[0] > 0 or o[1] > 0))
    for cfg in (rs.PipelineConfig(ground_removal=False, min_cluster_points=1, mc_pattern=rs.MCPattern(offs)),
                rs.PipelineConfig(ground_removal=False, min_cluster_points=2, mc_pattern=rs.skip_pattern(3)),
                rs.PipelineConfig(min_cluster_points=5, mc_pattern=rs.MCPattern(((2, 0), (4, 0), (1, 1))))):
        pipe, res = _run(model, cfg, frames, rows_per_cta=rows)
        for b in range(frames.shape[0]):
            wl, ws = oracle.segment_frame(frames[b], pipe.packed)
            _assert_frame(res, b, wl, ws)


@pytest.mark.parametrize("H,W,rows", [(64, 2048, 0), (33, 300, 8), (40, 96, 16), (24, 4096, 0)])
def test_step_a_map_connections_vs_oracle(H, W, rows, rng, cuda):
    """Offsets with dy <= 2 and 0 <= dx <= 31 (at most four) are tested in
    step A from registers (rs_fast.cuh, MCA): partners in the previous word,
    before the chunk, across the azimuth seam and above the band, mixed with
    offsets that take the per-lane path (dy >= 3, dx < 0, a fifth one)."""
    model = _random_model(H, W)
    frames = rng.uniform(0.5, 12.0, size=(3, H, W)).astype(np.float32)
    frames[rng.random(frames.shape) < 0.25] = 0
    frames[1] = 7.0                               # everything linked
    frames[1, :, ::3] = 0
    offs = ((0, 31), (1, 30), (2, 17), (0, 5), (2, 0), (3, 1), (1, -3))
    offs = tuple(o for o in offs if o[0] < H and abs(o[1]) < W)
    for cfg in (rs.PipelineConfig(ground_removal=False, min_cluster_points=1, mc_pattern=rs.MCPattern(offs)),
                rs.PipelineConfig(ground_removal=False, min_cluster_points=3,
                                  mc_pattern=rs.MCPattern(((0, 2), (2, 0))))):
        pipe, res = _run(model, cfg, frames, rows_per_cta=rows)
        for b in range(3):
            wl, ws = oracle.segment_frame(frames[b], pipe.packed)
            _assert_frame(res, b, wl, ws)


def test_empty_and_full_frames(cuda):
    model = synthetic.sensor_for(synthetic.CONFIGS[0])
    frames = np.zeros((3, 64, 2048), np.float32)
    frames[1] = 10.0                              # one wrap-around component
    frames[2, :, ::2] = 10.0                      # isolated vertical lines
    for cfg in (rs.PipelineConfig(ground_removal=False, min_cluster_points=1),
                rs.PipelineConfig(ground_removal=False, min_cluster_points=65)):
        pipe, res = _run(model, cfg, frames)
        for b in range(3):
            wl, ws = oracle.segment_frame(frames[b], pipe.packed)
            _assert_frame(res, b, wl, ws)
    assert int(res.n_clusters[0]) == 0
    assert int(res.n_clusters[1]) == 1


def test_serpentine_component(cuda):
    """A single snake through every row: the longest possible cross-band chain."""
    H, W = 64, 256
    model = _random_model(H, W)
    f = np.zeros((H, W), np.float32)
    for r in range(0, H, 2):
        f[r, :] = 5.0
        f[r + 1, (W - 1) if (r // 2) % 2 == 0 else 0] = 5.0 if r + 1 < H else 0
    f[:, 1::17] = 0.0
    cfg = rs.PipelineConfig(ground_removal=False, min_cluster_points=1)
    for rows in (4, 8, 16):
        pipe, res = _run(model, cfg, f, rows_per_cta=rows)
        wl, ws = oracle.segment_frame(f, pipe.packed)
        _assert_frame(res, 0, wl, ws)


def test_rotation_equivariance(config_frames):
    model = synthetic.sensor_for(synthetic.CONFIGS[1])
    f = config_frames[1][:2]
    cfg = rs.PipelineConfig(ground_removal=False, min_cluster_points=1)
    pipe = rs.Pipeline(model, cfg, device="cuda:0")
    a = pipe.segment_batch(f).labels.cpu().numpy()
    b = pipe.segment_batch(torch.roll(f, 731, dims=2)).labels.cpu().numpy()
    for i in range(2):
        ra = np.roll(a[i], 731, axis=1)
        # same partition up to naming
        pairs = set(zip(ra.ravel().tolist(), b[i].ravel().tolist()))
        assert len(pairs) == len(set(ra.ravel().tolist()))


def test_determinism(config_frames):
    model = synthetic.sensor_for(synthetic.CONFIGS[4])
    pipe = rs.Pipeline(model, rs.PipelineConfig(ground_removal=False, min_cluster_points=1,
                                                mc_pattern=rs.preset_pattern("mc1")),
                       device="cuda:0")
    outs = [pipe.segment_batch(config_frames[4]).labels.clone() for _ in range(3)]
    assert all(torch.equal(outs[0], o) for o in outs[1:])


# --------------------------------------------------------------- host API ---
def test_segment_range_image_api(cuda):
    m, cfg, ranges, labels, sizes, _ = golden.case("frames", "occluder/mc1", "occluder")
    li, rec = rs.Pipeline(m, cfg).segment_range_image(rs.from_ranges(ranges))
    assert np.array_equal(li.labels, labels)
    assert np.array_equal(li.cluster_sizes, sizes)
    assert li.cluster_count == 2
    assert rec.stage_sum() <= rec.total + 0.5
    with pytest.raises(ValueError):
        rs.Pipeline(m, cfg).segment_range_image(rs.from_ranges(ranges[:, :10]))


def test_segment_in_parallel_matches_serial(cuda):
    m, cfg, a, *_ = golden.case("frames", "twobox/default", "twobox")
    _, _, b, *_ = golden.case("frames", "occluder/default", "occluder")
    frames = [a, b, a]
    serial = [rs.Pipeline(m, cfg).segment_range_image(rs.from_ranges(f))[0] for f in frames]
    par = rs.segment_in_parallel(frames, m, cfg)
    for s, p in zip(serial, par):
        assert np.array_equal(s.labels, p.labels)
        assert np.array_equal(s.cluster_sizes, p.cluster_sizes)


def test_host_buffer_entry_matches_device(config_frames):
    model = synthetic.sensor_for(synthetic.CONFIGS[1])
    pipe = rs.Pipeline(model, rs.PipelineConfig(), device="cuda:0")
    f = config_frames[1]
    dev = pipe.segment_batch(f)
    host = torch.empty(f.shape, dtype=torch.float32, pin_memory=True)
    host.copy_(f)
    lab, ncl, sz = pipe.segment_batch_host(host.numpy())
    torch.cuda.synchronize()
    assert np.array_equal(lab, dev.labels.cpu().numpy())
    assert np.array_equal(ncl, dev.n_clusters.cpu().numpy())
    dsz = dev.cluster_sizes.cpu().numpy()
    for b in range(f.shape[0]):
        assert np.array_equal(sz[b, :ncl[b] + 1], dsz[b, :ncl[b] + 1])


def test_batch_zero_and_errors(cuda):
    model = synthetic.sensor_for(synthetic.CONFIGS[3])
    pipe = rs.Pipeline(model, device="cuda:0")
    res = pipe.segment_batch(torch.zeros((0, 32, 1024), device="cuda:0"))
    assert res.labels.shape == (0, 32, 1024)
    with pytest.raises(ValueError):
        pipe.segment_batch(torch.zeros((1, 32, 1000), device="cuda:0"))
    with pytest.raises(ValueError):
        pipe.segment_batch(torch.zeros((1, 32, 1024), device="cuda:0", dtype=torch.float64))


# ------------------------------------------- node-capacity overflow path -----
@pytest.mark.parametrize("cap", [32, 700, 2000])
@pytest.mark.parametrize("cid,variant", [(1, "default"), (4, "core"), (3, "S1")])
def test_node_capacity_overflow_path(cap, cid, variant, config_frames):
    """Frames whose bands hold more runs than the node capacity are finished by
    the fast kernel's global-memory union-find over cells (rs_overflow.cuh);
    results must not change."""
    model = synthetic.sensor_for(synthetic.CONFIGS[cid])
    cfg = VARIANTS[variant]
    frames = config_frames[cid]
    pipe = rs.Pipeline(model, cfg, device="cuda:0", node_capacity=cap)
    assert pipe.plan["fast"] and pipe.plan["may_overflow"]
    want_l, want_n, want_s = oracle.segment_batch(frames.cpu().numpy(), pipe.packed,
                                                  sizes_stride=pipe.sizes_stride)
    for _ in range(2):    # repeat calls: nothing carried over between them
        res = pipe.segment_batch(frames)
        torch.cuda.synchronize()
        assert np.array_equal(res.n_clusters.cpu().numpy(), want_n)
        assert int((res.labels.cpu().numpy() != want_l).sum()) == 0
        got_s = res.cluster_sizes.cpu().numpy()
        for b in range(frames.shape[0]):
            k = int(want_n[b])
            assert np.array_equal(got_s[b, :k + 1], want_s[b, :k + 1])


@pytest.mark.parametrize("variant", ["default", "core", "S1"])
def test_natural_overflow_noise_frames(variant):
    """Frames of independent random ranges: almost every cell is its own run,
    far above the node capacity, mixed with ordinary frames in one batch."""
    spec = synthetic.CONFIGS[1]
    model = synthetic.sensor_for(spec)
    g = np.random.default_rng(11)
    H, W = spec.H, spec.W
    noise = g.uniform(1.0, 60.0, size=(3, H, W)).astype(np.float32)
    noise[1, : H // 2] = 0.0                       # only the lower band overflows
    noise[2, H // 2:] = np.float32(7.5)             # upper band overflows, lower band one component
    frames = torch.cat([synthetic.make_batch(1, 2, device="cuda:0"),
                        torch.from_numpy(noise).cuda()])
    pipe = rs.Pipeline(model, VARIANTS[variant], device="cuda:0")
    assert pipe.plan["may_overflow"]
    want_l, want_n, want_s = oracle.segment_batch(frames.cpu().numpy(), pipe.packed,
                                                  sizes_stride=pipe.sizes_stride)
    res = pipe.segment_batch(frames)
    torch.cuda.synchronize()
    assert np.array_equal(res.n_clusters.cpu().numpy(), want_n)
    assert np.array_equal(res.labels.cpu().numpy(), want_l)
    got_s = res.cluster_sizes.cpu().numpy()
    for b in range(frames.shape[0]):
        k = int(want_n[b])
        assert np.array_equal(got_s[b, :k + 1], want_s[b, :k + 1])


@pytest.mark.parametrize("cid,variant", [(1, "default"), (2, "core"), (4, "S1"), (3, "mc14_core")])
def test_dense_kernel_when_fast_plan_impossible(cid, variant, config_frames):
    """Band heights the fast kernel cannot hold (64 rows of 2048 cells, or more
    rows than a 1024-wide frame needs) run rs_dense_kernel over the batch; the
    results are the same as the oracle's."""
    model = synthetic.sensor_for(synthetic.CONFIGS[cid])
    pipe = rs.Pipeline(model, VARIANTS[variant], device="cuda:0", rows_per_cta=64)
    if pipe.plan["fast"]:
        pytest.skip("the fast plan holds this geometry")
    frames = config_frames[cid][:4]
    want_l, want_n, want_s = oracle.segment_batch(frames.cpu().numpy(), pipe.packed,
                                                  sizes_stride=pipe.sizes_stride)
    res = pipe.segment_batch(frames)
    torch.cuda.synchronize()
    assert np.array_equal(res.n_clusters.cpu().numpy(), want_n)
    assert np.array_equal(res.labels.cpu().numpy(), want_l)
    got_s = res.cluster_sizes.cpu().numpy()
    for b in range(frames.shape[0]):
        k = int(want_n[b])
        assert np.array_equal(got_s[b, :k + 1], want_s[b, :k + 1])
