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


def _match_table_loops(g_ids, c_ids, cnt, min_gt_points):
    """The reference's rules (evaluation.py:79-129) restated with plain loops: the
    checker for the vectorised paper_2003_00575_b200.evaluation._match_tables."""
    gt_size, pred_size, overlaps = {}, {}, {}
    for g, c, n in zip(g_ids.tolist(), c_ids.tolist(), cnt.tolist()):
        if g > 0:
            gt_size[g] = gt_size.get(g, 0) + n
        if c > 0:
            pred_size[c] = pred_size.get(c, 0) + n
        if g > 0 and c > 0:
            overlaps.setdefault(g, []).append((c, n))
    scored = sorted(g for g, n in gt_size.items() if n >= min_gt_points)
    best = {}
    for g in scored:
        ov = overlaps.get(g, [])
        if not ov:
            best[g] = (None, 0.0)
            continue
        iou = {c: n / (gt_size[g] + pred_size[c] - n) for c, n in ov}
        if sum(1 for v in iou.values() if v > 0.5) > 1:
            raise RuntimeError("two clusters with IoU > 0.5")
        c_best = max(ov, key=lambda cn: (cn[1], iou[cn[0]], -cn[0]))[0]
        best[g] = (c_best, iou[c_best])
    claims = {}
    for g, (c, v) in best.items():
        if c is not None:
            claims.setdefault(c, []).append((g, v))
    out = []
    for g in scored:
        c, v = best[g]
        if c is not None and max(claims[c], key=lambda gv: (gv[1], -gv[0]))[0] != g:
            c, v = None, 0.0
        out.append((g, c, v))
    return out


@pytest.mark.parametrize("seed", range(40))
def test_vectorised_matching_equals_loops(seed):
    """Random multi-frame tables with many ties (equal counts, equal IoU) and
    clusters claimed by several instances."""
    g = np.random.default_rng(seed)
    B = int(g.integers(1, 6))
    fs, gs, cs, ns = [], [], [], []
    for b in range(B):
        n_g, n_c = int(g.integers(0, 9)), int(g.integers(0, 9))
        pairs = {(int(a), int(c)) for a, c in zip(g.integers(0, n_g + 1, 40), g.integers(0, n_c + 1, 40))}
        pairs.discard((0, 0))
        for a, c in sorted(pairs):
            fs.append(b); gs.append(a); cs.append(c); ns.append(int(g.choice([1, 1, 2, 2, 3, 5, 40])))
    f, gi, ci, n = (np.array(x, dtype=np.int64) for x in (fs, gs, cs, ns))
    mn = int(g.choice([1, 2, 5]))
    cfg = ev.EvalConfig(min_gt_points=mn)
    want, err = [], False
    for b in range(B):
        m = f == b
        try:
            want.append(_match_table_loops(gi[m], ci[m], n[m], mn))
        except RuntimeError:
            err = True
    if err:
        with pytest.raises(RuntimeError):
            ev._match_tables(f, gi, ci, n, B, cfg)
        return
    got = ev._match_tables(f, gi, ci, n, B, cfg)
    assert [[(m.gt_id, m.matched_cluster, m.iou) for m in fr] for fr in got] == want
