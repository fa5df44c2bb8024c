"""Golden fixtures for instance scoring, recorded from the
Python reference itself in the build container:

    python tests/golden/make_golden_eval.py

Seeded per-point (gt instance id, predicted cluster) arrays — exact covers,
under- and over-segmentation, equal-IoU ties, most-overlap-before-IoU cases,
small instances below min_gt_points, unmatched instances, and random
partitions with noise — scored by ``evaluation.match_instances`` and
``summarize``.  Writes tests/golden/eval.npz.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

from rangeseg.evaluation import EvalConfig, match_instances, summarize  # noqa: E402

OUT = Path(__file__).resolve().parent / "eval.npz"


def blocks(n, spec):
    out = np.zeros(n, dtype=np.int64)
    for lo, hi, v in spec:
        out[lo:hi] = v
    return out


def cases(g):
    yield "cover", blocks(200, [(0, 150, 1)]), blocks(200, [(0, 150, 3)]), 100
    yield "under", blocks(300, [(0, 150, 1), (150, 300, 2)]), blocks(300, [(0, 280, 9)]), 100
    yield "tie_iou", blocks(400, [(0, 100, 4), (200, 300, 2)]), \
        blocks(400, [(0, 100, 7), (200, 300, 7), (100, 200, 8)]), 50
    yield "overlap_first", blocks(500, [(0, 300, 5)]), \
        blocks(500, [(0, 160, 2), (160, 300, 6), (300, 500, 6)]), 100
    yield "small", blocks(300, [(0, 50, 1), (50, 250, 2)]), blocks(300, [(0, 300, 1)]), 100
    yield "unmatched", blocks(300, [(0, 200, 3)]), np.zeros(300, np.int64), 100
    for i in range(40):
        n = int(g.integers(200, 20000))
        k = int(g.integers(1, 40))
        gt = np.sort(g.integers(0, k + 1, n))            # contiguous instances, 0 = none
        gt = gt[g.permutation(n)] if i % 3 == 0 else gt
        pred = gt * int(g.integers(1, 4)) + (g.random(n) < 0.3) * g.integers(0, 3, n)   # splits / merges
        pred[g.random(n) < 0.1] = 0
        cut = int(g.integers(0, n))                      # one cluster spans an instance border
        pred[cut:cut + int(g.integers(0, 300))] = 1000 + i
        yield f"rand{i:02d}", gt, pred, int(g.choice([1, 20, 100]))


def main():
    g = np.random.default_rng(2003)
    store = {}
    for name, gt, pred, mn in cases(g):
        cfg = EvalConfig(min_gt_points=mn)
        m = match_instances(gt, pred, cfg)
        rep = summarize(m, cfg) if m else None
        store[f"{name}/gt"] = gt.astype(np.int32)
        store[f"{name}/pred"] = pred.astype(np.int32)
        store[f"{name}/min_gt_points"] = np.int64(mn)
        store[f"{name}/matches"] = np.array([json.dumps([[x.gt_id, x.matched_cluster, x.iou] for x in m])])
        store[f"{name}/summary"] = np.array([json.dumps(None if rep is None else
                                                         [rep.iou_mean, rep.precision_mean,
                                                          {f"{k:.2f}": v for k, v in rep.precision_at.items()}])])
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT} ({len(store)} arrays)")


if __name__ == "__main__":
    main()
