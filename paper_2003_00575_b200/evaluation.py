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


def _match_table(g_ids, c_ids, cnt, cfg: EvalConfig):
    """The reference's matching rules (evaluation.py:79-129) over one frame's
    contingency table (gt ids, cluster ids, counts; 0 = none)."""
    gt_size, pred_size = {}, {}
    for g, c, n in zip(g_ids.tolist(), c_ids.tolist(), cnt.tolist()):
        if g > 0:
            gt_size[g] = gt_size.get(g, 0) + n
        if c > 0:
            pred_size[c] = pred_size.get(c, 0) + n
    scored = sorted(g for g, n in gt_size.items() if n >= cfg.min_gt_points)
    if not scored:
        return []
    overlaps = {}
    for g, c, n in zip(g_ids.tolist(), c_ids.tolist(), cnt.tolist()):
        if g > 0 and c > 0:
            overlaps.setdefault(g, []).append((c, n))   # clusters ascending within g
    best = {}
    for g in scored:
        ov = overlaps.get(g, [])
        if not ov:
            best[g] = (None, 0.0)
            continue
        iou = {c: n / (gt_size[g] + pred_size[c] - n) for c, n in ov}
        if sum(1 for v in iou.values() if v > 0.5) > 1:
            raise RuntimeError(f"instance {g} overlaps two clusters with IoU > 0.5; "
                               "predicted clusters are not disjoint")
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
        out.append(InstanceMatch(gt_id=int(g), matched_cluster=c, iou=v))
    return out


def match_instances_batch(gt: torch.Tensor, pred: torch.Tensor, offsets: torch.Tensor,
                          cfg: EvalConfig | None = None):
    """``match_instances`` for B frames of per-point labels on the device."""
    cfg = cfg or EvalConfig()
    f, g, c, n = contingency_batch(gt, pred, offsets)
    B = offsets.numel() - 1
    bounds = np.searchsorted(f, np.arange(B + 1))
    return [_match_table(g[bounds[b]:bounds[b + 1]], c[bounds[b]:bounds[b + 1]],
                         n[bounds[b]:bounds[b + 1]], cfg) for b in range(B)]


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
