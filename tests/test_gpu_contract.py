"""GPU parity at full BASELINE batch sizes, the fused kernel's own edge
decisions, and the input / output contract of the drop-in boundary.

* Labels, counts and sizes of every BASELINE config at its FULL batch (1, 256,
  128, 1024 and 256 frames) for the four variants, against the CPU oracle
  (oracle/, pinned to the reference's outputs in test_oracle_golden.py).
* ``rs_fast_planes``: the presence / left / up / Map Connection bit planes the
  hot kernel itself built (sign-folded slope window, per-row height
  threshold — rewrites of ground.py:112-140 that rs_stage_kernel does not
  use), compared bit for bit with the reference's recorded stage masks and
  with the oracle's planes.  North_star allows mismatches within 1e-6 of the
  threshold; the bar here is zero.
* Input contract (range_image.py:47-54): NaN / inf / negative ranges are
  flagged by the kernel (n_clusters = -1) and raise ValueError at the
  host-buffer entry and in ``segment_range_image``; -0.0 passes.
"""

import numpy as np
import pytest
import torch

import golden
import paper_2003_00575_b200 as rs
from oracle import oracle
from paper_2003_00575_b200 import _native, synthetic

pytestmark = pytest.mark.gpu

VARIANTS = {
    "default": rs.PipelineConfig(),
    "core": rs.PipelineConfig(ground_removal=False, min_cluster_points=1),
    "S1": rs.PipelineConfig(mc_pattern=rs.skip_pattern(1)),
    "mc14_core": rs.PipelineConfig(mc_pattern=rs.preset_pattern("mc14"),
                                   ground_removal=False, min_cluster_points=1),
}

_FRAMES = {}


def full_frames(cid):
    if cid not in _FRAMES:
        _FRAMES.clear()   # one config resident at a time
        _FRAMES[cid] = synthetic.make_batch(cid, device="cuda:0")
    return _FRAMES[cid]


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("cid", [0, 1, 2, 3, 4])
def test_full_batch_vs_oracle(cid, variant, cuda):
    frames = full_frames(cid)
    assert frames.shape[0] == synthetic.CONFIGS[cid].batch
    pipe = rs.Pipeline(synthetic.sensor_for(synthetic.CONFIGS[cid]), VARIANTS[variant], device="cuda:0")
    res = pipe.segment_batch(frames)
    host = frames.cpu().numpy()
    want_l, want_n, want_s = oracle.segment_batch(host, pipe.packed, sizes_stride=pipe.sizes_stride)
    torch.cuda.synchronize()
    got_n = res.n_clusters.cpu().numpy()
    assert np.array_equal(got_n, want_n)
    bad = np.nonzero((res.labels.cpu().numpy() != want_l).reshape(len(host), -1).any(1))[0]
    assert bad.size == 0, f"{bad.size} of {len(host)} frames differ (first {bad[:5]})"
    got_s = res.cluster_sizes.cpu().numpy()
    for b in range(host.shape[0]):
        k = int(want_n[b])
        assert np.array_equal(got_s[b, :k + 1], want_s[b, :k + 1])


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("cid", [0, 1, 2, 3, 4])
def test_fast_kernel_edge_decisions_vs_oracle(cid, variant, cuda):
    """Every presence / edge / Map Connection decision of the hot kernel, at full batch."""
    frames = full_frames(cid)
    pipe = rs.Pipeline(synthetic.sensor_for(synthetic.CONFIGS[cid]), VARIANTS[variant], device="cuda:0")
    planes, res = pipe.fast_planes(frames)
    want = oracle.planes_batch(frames.cpu().numpy(), pipe.packed)
    got = planes.cpu().numpy().view(np.uint32)
    diff = np.unpackbits((got ^ want).view(np.uint8)).sum()
    assert diff == 0, f"{diff} edge/presence decisions differ"
    # the export does not change the labels
    ref = pipe.segment_batch(frames)
    torch.cuda.synchronize()
    assert torch.equal(ref.labels, res.labels)


@pytest.mark.parametrize("case_key,frame_key", golden.frame_cases())
def test_fast_kernel_planes_vs_reference_masks(case_key, frame_key, cuda):
    m, cfg, ranges, labels, sizes, stages = golden.case("frames", case_key, frame_key)
    if stages is None:
        pytest.skip("no stage masks recorded for this case")
    pipe = rs.Pipeline(m, cfg, device="cuda:0")
    if not pipe.plan["fast"]:
        pytest.skip("geometry runs on the dense kernel")
    planes, _ = pipe.fast_planes(torch.from_numpy(ranges).cuda()[None])
    got = planes[0, :3].cpu().numpy().view(np.uint32)
    assert np.array_equal(got, golden.planes_from_masks(ranges, *stages))


@pytest.mark.parametrize("key", golden.random_cases())
def test_fast_kernel_planes_vs_reference_random(key, cuda):
    m, cfg, ranges, labels, sizes, stages = golden.case("random", key)
    pipe = rs.Pipeline(m, cfg, device="cuda:0")
    if not pipe.plan["fast"]:
        pytest.skip("geometry runs on the dense kernel")
    planes, _ = pipe.fast_planes(torch.from_numpy(ranges).cuda()[None])
    got = planes[0].cpu().numpy().view(np.uint32)
    assert np.array_equal(got[:3], golden.planes_from_masks(ranges, *stages))
    assert np.array_equal(got, oracle.planes_batch(ranges[None], pipe.packed, nthreads=1)[0])


# ------------------------------------------------------------ input contract --
def _poisoned(value, where=(0, 5, 77)):
    frames = synthetic.make_batch(0, 3, device="cpu").numpy().copy()
    frames[where] = value
    return frames


@pytest.mark.parametrize("value", [np.nan, np.inf, -np.inf, -1.0, -1e-30])
@pytest.mark.parametrize("core", [False, True])
def test_bad_ranges_flagged(value, core, cuda):
    model = synthetic.sensor_for(synthetic.CONFIGS[0])
    cfg = VARIANTS["core" if core else "default"]
    pipe = rs.Pipeline(model, cfg, device="cuda:0")
    frames = _poisoned(np.float32(value), (1, 40, 2047))
    res = pipe.segment_batch(torch.from_numpy(frames).cuda())
    ncl = res.n_clusters.cpu().numpy()
    assert ncl[1] == _native.RS_FRAME_INVALID and ncl[0] >= 0 and ncl[2] >= 0
    with pytest.raises(ValueError, match="finite"):
        res.check()
    # the clean frames are still right
    want_l, want_n, _ = oracle.segment_batch(frames, pipe.packed)
    got_l = res.labels.cpu().numpy()
    assert np.array_equal(got_l[[0, 2]], want_l[[0, 2]])
    # host-buffer C entry: RS_EINVAL -> ValueError
    with pytest.raises(ValueError, match="finite"):
        pipe.segment_batch_host(frames)
    # per-frame entry with a raw array: from_ranges' ValueError
    with pytest.raises(ValueError, match="finite"):
        pipe.segment_range_image(frames[1])
    # a RangeImage is taken as is (the reference does not re-validate it): the bad
    # cell is simply no return, like in the reference's valid mask
    li, _ = pipe.segment_range_image(rs.RangeImage(ranges=frames[1]))
    wl, ws = oracle.segment_frame(frames[1], pipe.packed)
    assert np.array_equal(li.labels, wl) and np.array_equal(li.cluster_sizes, ws)


def test_bad_range_in_overflowing_frame_flagged(cuda):
    model = synthetic.sensor_for(synthetic.CONFIGS[0])
    pipe = rs.Pipeline(model, rs.PipelineConfig(), device="cuda:0", node_capacity=32)
    frames = _poisoned(np.float32(np.nan), (2, 63, 0))
    res = pipe.segment_batch(torch.from_numpy(frames).cuda())
    assert list(res.n_clusters.cpu().numpy() == -1) == [False, False, True]


def test_bad_range_dense_kernel_flagged(cuda):
    model = synthetic.sensor_for(synthetic.CONFIGS[0])
    pipe = rs.Pipeline(model, rs.PipelineConfig(), device="cuda:0", rows_per_cta=64)
    assert not pipe.plan["fast"]   # 64-row bands of 2048 cells: rs_dense_kernel
    frames = _poisoned(np.float32(-2.0), (0, 7, 2047))
    res = pipe.segment_batch(torch.from_numpy(frames).cuda())
    assert list(res.n_clusters.cpu().numpy() == -1) == [True, False, False]


def test_negative_zero_is_valid_input(cuda):
    model = synthetic.sensor_for(synthetic.CONFIGS[0])
    pipe = rs.Pipeline(model, rs.PipelineConfig(), device="cuda:0")
    frames = synthetic.make_batch(0, 2, device="cpu").numpy().copy()
    frames[frames == 0] = -0.0
    frames[0, :, ::7] = -0.0
    res = pipe.segment_batch(torch.from_numpy(frames).cuda()).check()
    want_l, want_n, _ = oracle.segment_batch(frames, pipe.packed)
    assert np.array_equal(res.n_clusters.cpu().numpy(), want_n)
    assert np.array_equal(res.labels.cpu().numpy(), want_l)
    pipe.segment_batch_host(frames)
    li, _ = pipe.segment_range_image(frames[0])
    assert np.array_equal(li.labels, want_l[0])


# ----------------------------------------------------------- output contract --
def test_output_buffers_validated(cuda):
    model = synthetic.sensor_for(synthetic.CONFIGS[0])
    pipe = rs.Pipeline(model, rs.PipelineConfig(), device="cuda:0")
    x = synthetic.make_batch(0, 2, device="cpu").cuda()
    with pytest.raises(ValueError, match="labels"):
        pipe.segment_batch(x, labels=torch.empty((2, 64, 2048), dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError, match="labels"):
        pipe.segment_batch(x, labels=torch.empty((2, 2048, 64), dtype=torch.int32, device="cuda").transpose(1, 2))
    with pytest.raises(ValueError, match="cluster_sizes"):
        pipe.segment_batch(x, cluster_sizes=torch.empty((2, 10), dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError, match="cluster_sizes"):
        pipe.segment_batch(x, cluster_sizes=torch.empty((2, pipe.sizes_stride), dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError, match="n_clusters"):
        pipe.segment_batch(x, n_clusters=torch.empty((3,), dtype=torch.int32, device="cuda"))
    h = x.cpu().numpy()
    with pytest.raises(ValueError, match="cluster_sizes"):
        pipe.segment_batch_host(h, cluster_sizes=np.empty((2, 5), np.int64))
    with pytest.raises(ValueError, match="labels"):
        pipe.segment_batch_host(h, labels=np.empty((2, 64, 2048), np.int64))


def test_side_stream_waits_for_producer(cuda):
    """segment_batch(stream=s) orders after the current stream's queued work."""
    model = synthetic.sensor_for(synthetic.CONFIGS[0])
    pipe = rs.Pipeline(model, rs.PipelineConfig(), device="cuda:0")
    src = synthetic.make_batch(0, 4, device="cpu").cuda()
    want = pipe.segment_batch(src).labels.clone()
    s = torch.cuda.Stream()
    for _ in range(3):
        x = torch.zeros_like(src)
        torch.cuda._sleep(2_000_000)   # a slow producer on the current stream
        x.copy_(src)
        res = pipe.segment_batch(x, stream=s)
        torch.cuda.current_stream().wait_stream(s)
        assert torch.equal(res.labels, want)


def test_per_frame_api_equals_batch(cuda):
    model = synthetic.sensor_for(synthetic.CONFIGS[0])
    pipe = rs.Pipeline(model, rs.PipelineConfig(), device="cuda:0")
    frames = synthetic.make_batch(0, 3, device="cpu").numpy()
    res = pipe.segment_batch(torch.from_numpy(frames).cuda())
    for b in range(3):
        li, rec = pipe.segment_range_image(frames[b])
        want = res.label_image(b)
        assert np.array_equal(li.labels, want.labels)
        assert np.array_equal(li.cluster_sizes, want.cluster_sizes)
        assert rec.ccl > 0 and rec.total >= rec.ccl


def test_stage_timing_record(cuda):
    model = synthetic.sensor_for(synthetic.CONFIGS[0])
    frame = synthetic.make_batch(0, 1, device="cpu").numpy()[0]
    for ground in (True, False):
        pipe = rs.Pipeline(model, rs.PipelineConfig(ground_removal=ground), device="cuda:0", stage_timing=True)
        li, rec = pipe.segment_range_image(frame)
        assert rec.ccl > 0 and rec.ground > 0 and rec.connectivity > 0
        assert rec.total >= rec.ccl
        wl, _ = oracle.segment_frame(frame, pipe.packed)
        assert np.array_equal(li.labels, wl)
