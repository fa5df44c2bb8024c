"""The CPU oracle (oracle/rangeseg_oracle.c) against the reference's own outputs.

tests/golden/*.npz hold what the Python reference (rangeseg, run in the build
container by tests/golden/make_golden.py) returned for these inputs; here the
oracle must reproduce labels, cluster sizes and the ground/edge stage masks
bit for bit.  This pins the oracle before any GPU test trusts it.
"""

import numpy as np
import pytest

import golden
from oracle import oracle
from paper_2003_00575_b200 import pack_tables


@pytest.mark.parametrize("case_key,frame_key", golden.frame_cases())
def test_oracle_matches_reference_on_frames(case_key, frame_key):
    m, cfg, ranges, labels, sizes, stages = golden.case("frames", case_key, frame_key)
    got = oracle.segment_frame(ranges, pack_tables(m, cfg), stages=True)
    assert np.array_equal(got[0], labels)
    assert np.array_equal(got[1], sizes)
    if stages is not None:
        for g, w in zip(got[2:], stages):
            assert np.array_equal(g, w)


@pytest.mark.parametrize("key", golden.random_cases())
def test_oracle_matches_reference_on_random_frames(key):
    m, cfg, ranges, labels, sizes, stages = golden.case("random", key)
    got = oracle.segment_frame(ranges, pack_tables(m, cfg), stages=True)
    assert np.array_equal(got[0], labels)
    assert np.array_equal(got[1], sizes)
    for g, w in zip(got[2:], stages):
        assert np.array_equal(g, w)


def test_oracle_batch_equals_per_frame():
    m, cfg, ranges, *_ = golden.case("frames", "c0/mc1", "c0")
    pt = pack_tables(m, cfg)
    frames = np.stack([ranges, np.roll(ranges, 100, axis=1), ranges[::-1].copy() * 0])
    lab, ncl, sz = oracle.segment_batch(frames, pt, nthreads=2)
    for b in range(3):
        l1, s1 = oracle.segment_frame(frames[b], pt)
        assert np.array_equal(lab[b], l1)
        assert ncl[b] == len(s1) - 1
        assert np.array_equal(sz[b, :len(s1)], s1)


# ------------------------------------------------- point clouds (§8(f)1) -----
@pytest.mark.parametrize("key", golden.project_cases())
def test_oracle_project_matches_reference(key):
    """project_oracle.c against range_image.project's recorded outputs:
    bit-identical on every cell no boundary-ambiguous point can reach (the
    oracle's asin is the C library's, the reference ran numpy's vectorised
    arcsin; they differ in the last ulp)."""
    m, c = golden.project_case(key)
    ranges, pidx, n_dropped, n_over = oracle.project(c["points"], m)
    unstable, n_amb = golden.unstable_cells(c["points"], m)
    st = ~unstable
    assert np.array_equal(ranges[st].view(np.uint32), c["ranges"][st].view(np.uint32))
    assert np.array_equal(pidx[st], c["point_index"][st])
    assert abs(n_dropped - c["counts"][1]) <= n_amb
    assert abs(n_over - c["counts"][2]) <= 2 * n_amb
    if n_amb == 0:
        assert (n_dropped, n_over) == (c["counts"][1], c["counts"][2])


@pytest.mark.parametrize("key", golden.project_cases())
def test_oracle_labels_to_points_matches_reference(key):
    m, c = golden.project_case(key)
    got = oracle.labels_to_points(c["labels"], c["point_index"], c["counts"][0])
    assert np.array_equal(got, c["point_labels"])


@pytest.mark.parametrize("case_key,frame_key", golden.frame_cases())
def test_oracle_planes_match_reference_stage_masks(case_key, frame_key):
    """oracle.planes_batch (the layout the GPU parity export is checked in)
    against the reference's recorded extract_ground / build_connectivity."""
    m, cfg, ranges, labels, sizes, stages = golden.case("frames", case_key, frame_key)
    if stages is None:
        pytest.skip("no stage masks recorded for this case")
    pl = oracle.planes_batch(ranges[None], pack_tables(m, cfg), nthreads=1)[0]
    assert np.array_equal(pl[:3], golden.planes_from_masks(ranges, *stages))


def test_oracle_mc_planes_equal_literal_rule():
    """Map Connection planes: the decision of map_connections.py:155-169 for
    every present pair, restated here in numpy on a small random frame."""
    import paper_2003_00575_b200 as rs
    g = np.random.default_rng(5)
    m = rs.fov_model(20, 2.0, -20.0, 70, 1.7)
    cfg = rs.PipelineConfig(mc_pattern=rs.preset_pattern("mc14"), min_cluster_points=1)
    pt = pack_tables(m, cfg)
    fr = (g.uniform(3, 6, (20, 70)) * (g.random((20, 70)) > 0.2)).astype(np.float32)
    pl = oracle.planes_batch(fr[None], pt, nthreads=1)[0]
    pres = np.unpackbits(pl[0].view(np.uint8), bitorder="little").reshape(20, -1)[:, :70].astype(bool)
    H, W = fr.shape
    for k, (dy, dx) in enumerate(pt.offsets):
        want = np.zeros((H, W), bool)
        tc = pt.block[H + 5 * (H - 1) + k * H: H + 5 * (H - 1) + (k + 1) * H]
        for r in range(dy, H):
            for c in range(W):
                ur, uc = r - dy, (c - dx) % W
                a, b = np.float32(fr[ur, uc]), np.float32(fr[r, c])
                d = (a * a + b * b) - np.float32(tc[ur]) * (a * b)
                want[r, c] = pres[r, c] and pres[ur, uc] and d <= np.float32(pt.d_max_sq)
        assert np.array_equal(pl[3 + k], golden.pack_bits(want)), (dy, dx)
