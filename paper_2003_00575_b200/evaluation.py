"""Instance scoring with the counting on the GPU.

Mirrors ``evaluation`` of the reference (/root/reference/pkg/src/rangeseg/evaluation.py):
``EvalConfig`` (:20-33), ``InstanceMatch`` (:36-40), ``EvalReport`` (:43-52),
``match_instances`` (:65-129), ``precision_at`` (:132-138), ``summarize``
(:141-162), ``report_as_dict`` (:165-171).  The (instance, cluster)
contingency counts over all points — the part that scales with the cloud —
come from ``rs_contingency`` (sort + run-length encode on the device, many
frames per call); picking each instance's best cluster and resolving clusters
claimed twice runs over that small table on the host with the reference's
rules: most overlap, then higher IoU, then lower cluster id; a cluster goes to
the instance with the higher IoU, equal IoU to the lower instance id.
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native

DEFAULT_IOU_BINS = tuple(round(0.50 + 0.05 * i, 2) for i in range(10))
_LABEL_BITS = 22
_NONE_KEY = 0x7FFFFFFFFFFFFFFF


@dataclass
class EvalConfig:
    min_gt_points: int = 100
    iou_bins: tuple = DEFAULT_IOU_BINS
    ground_mode: str = "gt_ground_removed"   # or "algorithmic_ground"

    def __post_init__(self):
        bins = tuple(float(b) for b in self.iou_bins)
        if any(not (0.0 < b <= 1.0) for b in bins):
            raise ValueError("iou bins must lie in (0, 1]")
        if any(hi <= lo for lo, hi in zip(bins, bins[1:])):
            raise ValueError("iou bins must be strictly increasing")
        self.iou_bins = bins
        if self.ground_mode not in ("gt_ground_removed", "algorithmic_ground"):
            raise ValueError(f"unknown ground mode {self.ground_mode!r}")


@dataclass
class InstanceMatch:
    gt_id: int
    matched_cluster: int | None
    iou: float


@dataclass
class EvalReport:
    iou_mean: float | None
    precision_mean: float | None
    precision_at: dict
    per_instance: list = field(default_factory=list)

    @property
    def n_instances(self) -> int:
        return len(self.per_instance)


def instance_iou(gt_points, cluster_points) -> float:
    """Jaccard index of two point-index sets (evaluation.py:55-62)."""
    a = set(np.asarray(gt_points).ravel().tolist())
    b = set(np.asarray(cluster_points).ravel().tolist())
    if not a:
        raise ValueError("ground-truth set must be nonempty")
    union = len(a | b)
    return len(a & b) / union if union else 0.0


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def contingency_batch(gt: torch.Tensor, pred: torch.Tensor, offsets: torch.Tensor,
                      stream: torch.cuda.Stream | None = None):
    """Device per-point int32 ``gt`` / ``pred`` of B frames (CSR ``offsets``
    int64 [B+1]) -> numpy ``(frame, gt, pred, count)`` arrays of the sorted
    unique pairs over points with gt > 0 or pred > 0."""
    for t, name in ((gt, "gt"), (pred, "pred")):
        if t.dtype != torch.int32 or t.dim() != 1 or not t.is_cuda:
            raise ValueError(f"{name} must be an int32 CUDA vector")
    if gt.shape != pred.shape:
        raise ValueError(f"{gt.numel()} gt labels vs {pred.numel()} predictions")
    n = gt.numel()
    B = offsets.numel() - 1
    dev = gt.device
    pairs = torch.empty((n + 1,), dtype=torch.int64, device=dev)
    counts = torch.empty((n + 1,), dtype=torch.int64, device=dev)
    status = torch.empty((2,), dtype=torch.int64, device=dev)
    wsb = int(_native.lib().rs_contingency_workspace_size(n, B))
    ws = torch.empty((max(wsb, 8),), dtype=torch.uint8, device=dev)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    st = _native.lib().rs_contingency(_ptr(gt.contiguous()), _ptr(pred.contiguous()), _ptr(offsets), B, n,
                                      _ptr(pairs), _ptr(counts), _ptr(status), _ptr(ws), wsb,
                                      ctypes.c_void_p(s.cuda_stream))
    _native.check(st, "rs_contingency")
    k, bad = (int(v) for v in status.cpu().numpy())
    if bad:
        raise ValueError(f"labels must lie in [0, 2^{_LABEL_BITS})")
    keys = pairs[:k].cpu().numpy()
    cnt = counts[:k].cpu().numpy()
    keep = keys != _NONE_KEY
    keys, cnt = keys[keep], cnt[keep]
    mask = (1 << _LABEL_BITS) - 1
    return keys >> (2 * _LABEL_BITS), (keys >> _LABEL_BITS) & mask, keys & mask, cnt


def contingency_device_ms(gt: torch.Tensor, pred: torch.Tensor, offsets: torch.Tensor, reps: int = 10) -> float:
    """Device time (CUDA events) of one rs_contingency call on these labels."""
    n = gt.numel()
    B = offsets.numel() - 1
    dev = gt.device
    pairs = torch.empty((n + 1,), dtype=torch.int64, device=dev)
    counts = torch.empty((n + 1,), dtype=torch.int64, device=dev)
    status = torch.empty((2,), dtype=torch.int64, device=dev)
    wsb = int(_native.lib().rs_contingency_workspace_size(n, B))
    ws = torch.empty((max(wsb, 8),), dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream(dev)

    def call():
        _native.check(_native.lib().rs_contingency(_ptr(gt), _ptr(pred), _ptr(offsets), B, n, _ptr(pairs),
                                                   _ptr(counts), _ptr(status), _ptr(ws), wsb,
                                                   ctypes.c_void_p(s.cuda_stream)), "rs_contingency")
    for _ in range(3):
        call()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        call()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def _match_tables(f_ids, g_ids, c_ids, cnt, n_frames: int, cfg: EvalConfig):
    """The reference's matching rules (evaluation.py:79-129) over the contingency
    tables of ``n_frames`` frames at once (frame, gt id, cluster id, count; id 0 =
    none), vectorised: per scored instance the cluster with the most common
    points (then the higher IoU, then the lower cluster id), IoU as the same
    float64 quotient of integers; a cluster claimed by several instances goes
    to the highest IoU (then the lower instance id).  One list per frame."""
    f = np.asarray(f_ids, dtype=np.int64)
    g = np.asarray(g_ids, dtype=np.int64)
    c = np.asarray(c_ids, dtype=np.int64)
    n = np.asarray(cnt, dtype=np.int64)
    out = [[] for _ in range(n_frames)]
    K = 1 << _LABEL_BITS
    mg = g > 0
    if not mg.any():
        return out
    ug, inv_g = np.unique(f[mg] * K + g[mg], return_inverse=True)   # instances, by (frame, id)
    gsz = np.zeros(ug.size, dtype=np.int64)
    np.add.at(gsz, inv_g, n[mg])
    scored = gsz >= cfg.min_gt_points
    if not scored.any():
        return out
    mc = c > 0
    uc, inv_c = np.unique(f[mc] * K + c[mc], return_inverse=True)   # clusters, by (frame, id)
    csz = np.zeros(uc.size, dtype=np.int64)
    np.add.at(csz, inv_c, n[mc])
    best_c = np.zeros(ug.size, dtype=np.int64)        # 0 = no overlapping cluster
    best_v = np.zeros(ug.size, dtype=np.float64)
    mo = mg & mc
    ig = np.searchsorted(ug, f[mo] * K + g[mo])
    keep = scored[ig]
    ig, co, no = ig[keep], c[mo][keep], n[mo][keep]
    if ig.size:
        ic = np.searchsorted(uc, (ug[ig] // K) * K + co)
        iou = no / (gsz[ig] + csz[ic] - no)
        twice = np.bincount(ig[iou > 0.5], minlength=ug.size) > 1
        if twice.any():
            raise RuntimeError(f"instance {int(ug[np.argmax(twice)] % K)} overlaps two clusters with IoU > 0.5; "
                               "predicted clusters are not disjoint")
        # the maximum of (count, IoU, -cluster id) per instance: last of its group in that order
        order = np.lexsort((-co, iou, no, ig))
        last = np.r_[ig[order][1:] != ig[order][:-1], True]
        pick = order[last]
        best_c[ig[pick]] = co[pick]
        best_v[ig[pick]] = iou[pick]
        # a cluster claimed more than once: the maximum of (IoU, -instance id) keeps it
        cl = np.flatnonzero(best_c > 0)
        ckey = (ug[cl] // K) * K + best_c[cl]
        order = np.lexsort((-(ug[cl] % K), best_v[cl], ckey))
        last = np.r_[ckey[order][1:] != ckey[order][:-1], True]
        lost = np.ones(cl.size, dtype=bool)
        lost[order[last]] = False
        best_c[cl[lost]] = 0
        best_v[cl[lost]] = 0.0
    for i in np.flatnonzero(scored).tolist():
        key = int(ug[i])
        cb = int(best_c[i])
        out[key // K].append(InstanceMatch(gt_id=key % K, matched_cluster=cb if cb else None,
                                           iou=float(best_v[i]) if cb else 0.0))
    return out


def _match_table(g_ids, c_ids, cnt, cfg: EvalConfig):
    """One frame's contingency table (gt ids, cluster ids, counts; 0 = none)."""
    return _match_tables(np.zeros(len(g_ids), dtype=np.int64), g_ids, c_ids, cnt, 1, cfg)[0]


def match_instances_batch(gt: torch.Tensor, pred: torch.Tensor, offsets: torch.Tensor,
                          cfg: EvalConfig | None = None):
    """``match_instances`` for B frames of per-point labels on the device."""
    cfg = cfg or EvalConfig()
    f, g, c, n = contingency_batch(gt, pred, offsets)
    return _match_tables(f, g, c, n, offsets.numel() - 1, cfg)


def match_instances(gt_instance_ids, pred_labels, cfg: EvalConfig | None = None):
    """evaluation.match_instances with the counting on the GPU: per-point
    arrays (0 = no instance / background) -> InstanceMatch list by gt id."""
    gt = np.asarray(gt_instance_ids).ravel()
    pred = np.asarray(pred_labels).ravel()
    if gt.shape != pred.shape:
        raise ValueError(f"{gt.size} gt labels vs {pred.size} predictions")
    for a in (gt, pred):
        if a.size and (a.min() < 0 or a.max() >= (1 << _LABEL_BITS)):
            raise ValueError(f"labels must lie in [0, 2^{_LABEL_BITS})")
    if not torch.cuda.is_available():
        raise RuntimeError("match_instances needs a CUDA device (there is no CPU fallback)")
    dev = torch.device("cuda", torch.cuda.current_device())
    tg = torch.from_numpy(gt.astype(np.int32)).to(dev)
    tp = torch.from_numpy(pred.astype(np.int32)).to(dev)
    off = torch.tensor([0, gt.size], dtype=torch.int64, device=dev)
    return match_instances_batch(tg, tp, off, cfg)[0]


def precision_at(matches, x: float) -> float:
    """Share of scored instances matched with IoU >= x (evaluation.py:132-138)."""
    if not (0.0 < x <= 1.0):
        raise ValueError(f"threshold must be in (0, 1], got {x}")
    if not matches:
        raise ValueError("no scored instances")
    return sum(1 for m in matches if m.iou >= x) / len(matches)


def summarize(matches, cfg: EvalConfig | None = None) -> EvalReport:
    """Pooled metrics (evaluation.py:141-162); metric fields are None when no
    instance was scored."""
    cfg = cfg or EvalConfig()
    matches = list(matches)
    if not matches:
        warnings.warn("no ground-truth instances were scored", stacklevel=2)
        return EvalReport(iou_mean=None, precision_mean=None, precision_at={}, per_instance=[])
    p_at = {b: precision_at(matches, b) for b in cfg.iou_bins}
    return EvalReport(iou_mean=float(np.mean([m.iou for m in matches])),
                      precision_mean=float(np.mean(list(p_at.values()))),
                      precision_at=p_at, per_instance=matches)


def report_as_dict(report: EvalReport) -> dict:
    return {"n_instances": report.n_instances, "iou_mean": report.iou_mean,
            "precision_mean": report.precision_mean,
            "precision_at": {f"{k:.2f}": v for k, v in report.precision_at.items()}}
