"""Instance scoring with the GPU contingency table (rs_contingency, SURVEY.md
§8(f)3) against the reference's recorded match_instances outputs and a numpy
contingency check."""

import numpy as np
import pytest
import torch

import golden
import paper_2003_00575_b200 as rs
from paper_2003_00575_b200 import evaluation as ev

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("key", golden.eval_cases())
def test_match_instances_matches_reference(key, cuda):
    gt, pred, mn, want, summary = golden.eval_case(key)
    got = rs.match_instances(gt, pred, rs.EvalConfig(min_gt_points=mn))
    assert [(m.gt_id, m.matched_cluster, m.iou) for m in got] == want


def test_batched_frames_equal_per_frame(cuda):
    keys = golden.eval_cases()
    cases = [golden.eval_case(k) for k in keys]
    gt = np.concatenate([c[0] for c in cases])
    pred = np.concatenate([c[1] for c in cases])
    off = np.cumsum([0] + [len(c[0]) for c in cases]).astype(np.int64)
    cfg = rs.EvalConfig(min_gt_points=20)
    got = ev.match_instances_batch(torch.from_numpy(gt).cuda(), torch.from_numpy(pred).cuda(),
                                   torch.from_numpy(off).cuda(), cfg)
    for b, c in enumerate(cases):
        one = rs.match_instances(c[0], c[1], cfg)
        assert [(m.gt_id, m.matched_cluster, m.iou) for m in got[b]] == \
               [(m.gt_id, m.matched_cluster, m.iou) for m in one]


def test_contingency_large_batch_vs_numpy(rng, cuda):
    B, n = 64, 120000
    gt = rng.integers(0, 300, size=B * n).astype(np.int32)
    pred = rng.integers(0, 5000, size=B * n).astype(np.int32)
    gt[rng.random(B * n) < 0.2] = 0
    off = np.arange(B + 1, dtype=np.int64) * n
    f, g, c, cnt = ev.contingency_batch(torch.from_numpy(gt).cuda(), torch.from_numpy(pred).cuda(),
                                        torch.from_numpy(off).cuda())
    frame = np.repeat(np.arange(B), n)
    keep = (gt > 0) | (pred > 0)
    keys, want = np.unique((frame[keep].astype(np.int64) << 44) | (gt[keep].astype(np.int64) << 22) | pred[keep],
                           return_counts=True)
    assert np.array_equal((f << 44) | (g << 22) | c, keys)
    assert np.array_equal(cnt, want)


def test_invalid_labels_rejected(cuda):
    with pytest.raises(ValueError):
        rs.match_instances(np.array([1, 2, 3]), np.array([1, 2]))
    with pytest.raises(ValueError):
        rs.match_instances(np.array([1, 1 << 23]), np.array([1, 2]))
    with pytest.raises(ValueError):
        ev.contingency_batch(torch.tensor([1, -2], dtype=torch.int32).cuda(),
                             torch.tensor([1, 2], dtype=torch.int32).cuda(),
                             torch.tensor([0, 2], dtype=torch.int64).cuda())
    assert rs.match_instances(np.zeros(10, np.int64), np.zeros(10, np.int64)) == []
