"""Instance scoring, host side: the matching rules of
paper_2003_00575_b200.evaluation over a contingency table computed here with
numpy (test-side checker, like the oracle) against the reference's recorded
match_instances / summarize outputs (tests/golden/eval.npz)."""

import numpy as np
import pytest

import golden
from paper_2003_00575_b200 import evaluation as ev


def _table(gt, pred):
    keep = (gt > 0) | (pred > 0)
    keys, cnt = np.unique(gt[keep].astype(np.int64) * (1 << 22) + pred[keep], return_counts=True)
    return keys >> 22, keys & ((1 << 22) - 1), cnt


@pytest.mark.parametrize("key", golden.eval_cases())
def test_matching_rules_match_reference(key):
    gt, pred, mn, want, summary = golden.eval_case(key)
    cfg = ev.EvalConfig(min_gt_points=mn)
    got = ev._match_table(*_table(gt, pred), cfg)
    assert [(m.gt_id, m.matched_cluster, m.iou) for m in got] == want
    if summary is None:
        assert got == []
    else:
        rep = ev.summarize(got, cfg)
        assert [rep.iou_mean, rep.precision_mean, ev.report_as_dict(rep)["precision_at"]] == summary


def test_config_and_helpers_validate_like_reference():
    with pytest.raises(ValueError):
        ev.EvalConfig(iou_bins=(0.5, 0.5))
    with pytest.raises(ValueError):
        ev.EvalConfig(ground_mode="other")
    with pytest.raises(ValueError):
        ev.precision_at([], 0.5)
    assert ev.instance_iou([1, 2, 3], [1, 2, 3]) == 1.0
    assert ev.instance_iou(np.arange(100), np.arange(20, 120)) == 80 / 120
    with pytest.raises(ValueError):
        ev.instance_iou([], [1])
    with pytest.warns(UserWarning):
        assert ev.summarize([]).iou_mean is None
