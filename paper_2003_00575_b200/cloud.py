"""Point clouds <-> range images on the GPU.

Mirrors ``range_image.project`` (/root/reference/pkg/src/rangeseg/range_image.py:57-115),
``range_image.labels_to_points`` (:130-141) and ``Pipeline.segment_cloud``
(pipeline.py:133-158) through ``rs_project`` / ``rs_labels_to_points`` of the C
ABI.  Clouds are float64 like the reference's (``np.asarray(points,
dtype=np.float64)``); batches are concatenated with CSR offsets.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .sensor import SensorModel


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def project_config(model: SensorModel):
    """(RsProjectConfig, ascending channel angles float64) for ``model``,
    with the reference's float64 half-gap margins (range_image.py:86-87)."""
    ang = np.asarray(model.channel_angles, dtype=np.float64)
    desc = bool(ang[0] > ang[-1])
    asc = np.ascontiguousarray(ang[::-1] if desc else ang)
    pc = _native.RsProjectConfig()
    pc.height, pc.width = model.height, model.width
    pc.descending = int(desc)
    pc.azimuth_step = float(model.azimuth_step)
    pc.gap_lo = float((asc[1] - asc[0]) / 2.0)
    pc.gap_hi = float((asc[-1] - asc[-2]) / 2.0)
    return pc, asc


def _launch_stream(dev, stream, tensors):
    """The stream a launch goes on: ``stream`` (made to wait for the current
    stream's queued work, its tensors recorded on it so the caching allocator
    does not reuse them early) or the current stream."""
    cur = torch.cuda.current_stream(dev)
    if stream is None or stream.cuda_stream == cur.cuda_stream:
        return cur
    stream.wait_stream(cur)
    for t in tensors:
        t.record_stream(stream)
    return stream


def _check_points(points) -> np.ndarray:
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] < 3 or pts.shape[0] == 0:
        raise ValueError("expected a nonempty (N, 3) point array")
    return np.ascontiguousarray(pts)


def project_batch(points: torch.Tensor, offsets: torch.Tensor, model: SensorModel,
                  stream: torch.cuda.Stream | None = None):
    """Device clouds -> device range images.

    ``points``: float64 CUDA [N, >=3] (clouds concatenated); ``offsets``: int64
    CUDA [B+1].  Returns ``(ranges f32 [B,H,W], point_index i64 [B,H,W],
    counts i64 [B,2] = (n_dropped, n_overwritten))`` on the same device,
    asynchronously on ``stream``.
    """
    if points.dtype != torch.float64 or points.dim() != 2 or points.shape[1] < 3 or not points.is_cuda:
        raise ValueError("points must be a float64 CUDA tensor [N, >=3]")
    if offsets.dtype != torch.int64 or offsets.dim() != 1 or offsets.device != points.device:
        raise ValueError("offsets must be an int64 tensor [B+1] on the points' device")
    pc, asc = project_config(model)
    dev = points.device
    B = offsets.numel() - 1
    H, W = model.height, model.width
    with torch.cuda.device(dev):
        points = points.contiguous()
        d_asc = torch.from_numpy(asc).to(dev)
        ranges = torch.empty((B, H, W), dtype=torch.float32, device=dev)
        pidx = torch.empty((B, H, W), dtype=torch.int64, device=dev)
        counts = torch.empty((B, 2), dtype=torch.int64, device=dev)
        wsb = int(_native.lib().rs_project_workspace_size(points.shape[0]))
        ws = torch.empty((max(wsb, 4),), dtype=torch.uint8, device=dev)
        s = _launch_stream(dev, stream, (points, offsets, d_asc, ranges, pidx, counts, ws))
        st = _native.lib().rs_project(ctypes.byref(pc), _ptr(d_asc), _ptr(points), points.shape[1],
                                      _ptr(offsets), B, points.shape[0], _ptr(ranges), _ptr(pidx),
                                      _ptr(counts), _ptr(ws), wsb, ctypes.c_void_p(s.cuda_stream))
    _native.check(st, "rs_project")
    return ranges, pidx, counts


def labels_to_points_batch(labels: torch.Tensor, point_index: torch.Tensor, offsets: torch.Tensor,
                           stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Device labels [B,H,W] -> per-point int32 labels [N] (0 = dropped / lost a cell)."""
    B, H, W = labels.shape
    if labels.dtype != torch.int32 or point_index.dtype != torch.int64 or offsets.dtype != torch.int64:
        raise ValueError("labels int32, point_index int64 and offsets int64 expected")
    if tuple(point_index.shape) != (B, H, W) or offsets.shape != (B + 1,):
        raise ValueError("point_index must be [B, H, W] and offsets [B + 1] like labels")
    dev = labels.device
    if point_index.device != dev or offsets.device != dev:
        raise ValueError("labels, point_index and offsets must be on one device")
    n = int(offsets[-1].item())
    with torch.cuda.device(dev):
        labels, point_index = labels.contiguous(), point_index.contiguous()
        out = torch.empty((n,), dtype=torch.int32, device=dev)
        s = _launch_stream(dev, stream, (labels, point_index, offsets, out))
        st = _native.lib().rs_labels_to_points(_ptr(labels), _ptr(point_index),
                                               _ptr(offsets), B, H, W, n, _ptr(out),
                                               ctypes.c_void_p(s.cuda_stream))
    _native.check(st, "rs_labels_to_points")
    return out


def project(points, model: SensorModel, device=None):
    """range_image.project on the GPU: returns a ``RangeImage`` with numpy
    ranges (float32), point_index (int64, -1 = empty) and the counters."""
    from .pipeline import RangeImage
    pts = _check_points(points)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda" or not torch.cuda.is_available():
        raise RuntimeError("project needs a CUDA device (there is no CPU fallback)")
    x = torch.from_numpy(pts).to(dev)
    off = torch.tensor([0, pts.shape[0]], dtype=torch.int64, device=dev)
    ranges, pidx, counts = project_batch(x, off, model)
    c = counts[0].cpu().numpy()
    return RangeImage(ranges=ranges[0].cpu().numpy(), point_index=pidx[0].cpu().numpy(),
                      n_points=int(pts.shape[0]), n_dropped=int(c[0]), n_overwritten=int(c[1]))


def labels_to_points(labels: np.ndarray, ri) -> np.ndarray:
    """range_image.labels_to_points on the GPU (numpy in, int32 numpy out)."""
    if ri.point_index is None:
        raise ValueError("range image has no point provenance to project back to")
    if not torch.cuda.is_available():
        raise RuntimeError("labels_to_points needs a CUDA device (there is no CPU fallback)")
    dev = torch.device("cuda", torch.cuda.current_device())
    lab = torch.from_numpy(np.ascontiguousarray(labels, dtype=np.int32)).to(dev)[None]
    pidx = torch.from_numpy(np.ascontiguousarray(ri.point_index, dtype=np.int64)).to(dev)[None]
    off = torch.tensor([0, int(ri.n_points)], dtype=torch.int64, device=dev)
    return labels_to_points_batch(lab, pidx, off).cpu().numpy()


@dataclass
class SegOutput:
    """Per-point instance labels plus the label image they came from (pipeline.py:62-67)."""

    point_labels: np.ndarray | None
    label_image: object
