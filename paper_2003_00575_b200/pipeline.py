"""Drop-in host API for the reference's clustering entry point.

Mirrors ``rangeseg.pipeline`` (pkg/src/rangeseg/pipeline.py) and the types it
returns: ``Pipeline(model, config).segment_range_image(ri) -> (LabelImage,
TimingRecord)`` (pipeline.py:70-131) and ``segment_in_parallel(frames, model,
config)`` (pipeline.py:170-197), with the same argument meaning and the same
``ValueError`` conditions.  The work runs in the fused sm_100a kernel behind
the C ABI (include/rangeseg_b200.h); this module only validates, uploads the
constant tables once per Pipeline and passes device pointers.

B200-specific additions:

* ``Pipeline.segment_batch(ranges)`` — a [B, H, W] float32 CUDA tensor in,
  labels / cluster counts / sizes as CUDA tensors out, stream-ordered on the
  current torch stream (no host synchronisation);
* ``Pipeline.segment_batch_host(ranges)`` — numpy in/out through
  ``rs_segment_batch_host`` (pipelined copies; the end-to-end path).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .config import PipelineConfig
from .sensor import SensorModel
from .tables import pack_tables

STAGES = ("project", "ground", "connectivity", "ccl", "mc", "filter")


@dataclass
class RangeImage:
    """Dense (H, W) float32 range grid; 0 marks no return (range_image.py:18-44)."""

    ranges: np.ndarray
    point_index: np.ndarray | None = None
    n_points: int = 0
    n_dropped: int = 0
    n_overwritten: int = 0

    @property
    def shape(self):
        return self.ranges.shape

    @property
    def n_projected(self) -> int:
        """Number of points that won a cell (range_image.py:35-40)."""
        if self.point_index is None:
            return int(np.count_nonzero(self.ranges))
        return int(np.count_nonzero(self.point_index >= 0))

    def valid_mask(self) -> np.ndarray:
        return self.ranges > 0


def from_ranges(ranges) -> RangeImage:
    """Wrap an image-shaped scan, validating like range_image.py:47-54."""
    ranges = np.ascontiguousarray(ranges, dtype=np.float32)
    if ranges.ndim != 2:
        raise ValueError(f"range image must be 2-D, got shape {ranges.shape}")
    if not np.isfinite(ranges).all() or (ranges < 0).any():
        raise ValueError("ranges must be finite and >= 0")
    return RangeImage(ranges=ranges)


@dataclass
class LabelImage:
    """Per-cell int32 labels (0 = background) and int64 sizes (ccl.py:50-64)."""

    labels: np.ndarray
    cluster_sizes: np.ndarray

    @property
    def cluster_count(self) -> int:
        return len(self.cluster_sizes) - 1


@dataclass
class TimingRecord:
    """Per-stage milliseconds (pipeline.py:41-59).

    The GPU path is one fused kernel, so its device time is reported under
    ``ccl``; ``total`` is the wall time of the call including copies.
    """

    project: float = 0.0
    ground: float = 0.0
    connectivity: float = 0.0
    ccl: float = 0.0
    mc: float = 0.0
    filter: float = 0.0
    total: float = 0.0

    def stage_sum(self) -> float:
        return (self.project + self.ground + self.connectivity + self.ccl
                + self.mc + self.filter)


@dataclass
class BatchResult:
    """Device-side result of :meth:`Pipeline.segment_batch`."""

    labels: torch.Tensor          # int32 [B, H, W]
    n_clusters: torch.Tensor      # int32 [B]
    cluster_sizes: torch.Tensor | None   # int64 [B, stride]; row b valid up to n_clusters[b]

    def label_image(self, b: int) -> LabelImage:
        k = int(self.n_clusters[b])
        sizes = (self.cluster_sizes[b, :k + 1].cpu().numpy() if self.cluster_sizes is not None
                 else np.bincount(self.labels[b].cpu().numpy().ravel(), minlength=k + 1))
        return LabelImage(labels=self.labels[b].cpu().numpy(), cluster_sizes=sizes)


def _ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


class Pipeline:
    """One sensor geometry + one configuration, bound to a CUDA device.

    Like the reference (pipeline.py:3-6) an instance owns per-geometry state
    (here: the float32 constant tables in device memory); unlike it, calls are
    stream-ordered and may be issued from several threads.
    """

    def __init__(self, model: SensorModel, config: PipelineConfig | None = None,
                 device=None, rows_per_cta: int = 0, node_capacity: int = 0):
        self.model = model
        self.config = config or PipelineConfig()
        self.packed = pack_tables(model, self.config)
        self.rs_config = _native.make_config(self.packed, rows_per_cta, node_capacity)
        self.rows_per_cta, self.ctas_per_frame, self.smem_bytes = _native.plan(self.rs_config)
        self.plan = _native.plan_detail(self.rs_config)
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.type == "cuda" and self.device.index is None and torch.cuda.is_available():
            self.device = torch.device("cuda", torch.cuda.current_device())
        self._tables = None
        self._workspaces = {}
        self._tables_host = np.ascontiguousarray(self.packed.block, dtype=np.float32)

    # -- helpers -----------------------------------------------------------
    @property
    def shape(self):
        return self.model.height, self.model.width

    @property
    def sizes_stride(self) -> int:
        H, W = self.shape
        return H * W // max(self.config.min_cluster_points, 1) + 1

    def _require_cuda(self):
        if self.device.type != "cuda" or not torch.cuda.is_available():
            raise RuntimeError("rangeseg_b200 runs on a CUDA device only (no CPU fallback)")

    def device_tables(self) -> torch.Tensor:
        self._require_cuda()
        if self._tables is None:
            self._tables = torch.from_numpy(self._tables_host).to(self.device)
        return self._tables

    def _workspace(self, batch: int, stream):
        """Device workspace the library asks for (none: rs_workspace_size is 0
        for this library; kept so the ABI's workspace contract stays honoured)."""
        need = int(_native.lib().rs_workspace_size(ctypes.byref(self.rs_config), batch))
        if need <= 0:
            return None
        ws = self._workspaces.get(stream.cuda_stream)
        if ws is None or ws.numel() < need:
            ws = torch.zeros(need, dtype=torch.uint8, device=self.device)
            self._workspaces[stream.cuda_stream] = ws
        return ws

    def _check_frames(self, ranges: torch.Tensor):
        H, W = self.shape
        if ranges.dim() != 3 or tuple(ranges.shape[1:]) != (H, W):
            raise ValueError(f"range images {tuple(ranges.shape)} do not match model "
                             f"{(H, W)}")
        if ranges.dtype != torch.float32:
            raise ValueError(f"ranges must be float32, got {ranges.dtype}")

    # -- device batch ------------------------------------------------------
    def segment_batch(self, ranges: torch.Tensor, *, labels: torch.Tensor | None = None,
                      n_clusters: torch.Tensor | None = None,
                      cluster_sizes: torch.Tensor | bool | None = True,
                      stream: torch.cuda.Stream | None = None) -> BatchResult:
        """Segment B frames resident on the GPU; asynchronous on ``stream``."""
        self._require_cuda()
        self._check_frames(ranges)
        if ranges.device != self.device:
            raise ValueError(f"ranges on {ranges.device}, pipeline on {self.device}")
        ranges = ranges.contiguous()
        B = ranges.shape[0]
        H, W = self.shape
        if labels is None:
            labels = torch.empty((B, H, W), dtype=torch.int32, device=self.device)
        if n_clusters is None:
            n_clusters = torch.empty((B,), dtype=torch.int32, device=self.device)
        if cluster_sizes is True:
            cluster_sizes = torch.empty((B, self.sizes_stride), dtype=torch.int64,
                                        device=self.device)
        elif cluster_sizes is False:
            cluster_sizes = None
        stride = cluster_sizes.shape[1] if cluster_sizes is not None else 0
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        ws = self._workspace(B, s)
        st = _native.lib().rs_segment_batch(
            ctypes.byref(self.rs_config), _ptr(self.device_tables()), _ptr(ranges), B,
            _ptr(labels), _ptr(n_clusters), _ptr(cluster_sizes), stride,
            _ptr(ws), 0 if ws is None else ws.numel(), ctypes.c_void_p(s.cuda_stream))
        _native.check(st, "rs_segment_batch")
        return BatchResult(labels, n_clusters, cluster_sizes)

    def stage_masks(self, ranges: torch.Tensor):
        """(ground, horizontal, vertical) bool CUDA tensors — extract_ground and
        build_connectivity (ground.py:95-141, connectivity.py:64-92) on device."""
        self._require_cuda()
        self._check_frames(ranges)
        ranges = ranges.contiguous()
        B = ranges.shape[0]
        H, W = self.shape
        g = torch.empty((B, H, W), dtype=torch.uint8, device=self.device)
        h = torch.empty((B, H, W), dtype=torch.uint8, device=self.device)
        v = torch.empty((B, H - 1, W), dtype=torch.uint8, device=self.device)
        st = _native.lib().rs_stage_masks(
            ctypes.byref(self.rs_config), _ptr(self.device_tables()), _ptr(ranges), B,
            _ptr(g), _ptr(h), _ptr(v),
            ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))
        _native.check(st, "rs_stage_masks")
        return g.bool(), h.bool(), v.bool()

    # -- host buffers --------------------------------------------------------
    def segment_batch_host(self, ranges: np.ndarray, labels: np.ndarray | None = None,
                           n_clusters: np.ndarray | None = None,
                           cluster_sizes: np.ndarray | bool | None = True):
        """Numpy [B, H, W] float32 in; (labels, n_clusters, cluster_sizes) out.

        Goes through ``rs_segment_batch_host``: the copies happen inside the C
        call, pipelined against the kernel.  Pinned (page-locked) arrays, e.g.
        from ``torch.empty(..., pin_memory=True).numpy()``, overlap best.
        """
        self._require_cuda()
        H, W = self.shape
        if ranges.ndim != 3 or ranges.shape[1:] != (H, W) or ranges.dtype != np.float32:
            raise ValueError(f"expected float32 [B, {H}, {W}], got {ranges.dtype} {ranges.shape}")
        if not ranges.flags.c_contiguous:
            raise ValueError("ranges must be C-contiguous")
        B = ranges.shape[0]
        if labels is None:
            labels = np.empty((B, H, W), dtype=np.int32)
        if n_clusters is None:
            n_clusters = np.empty((B,), dtype=np.int32)
        if cluster_sizes is True:
            cluster_sizes = np.empty((B, self.sizes_stride), dtype=np.int64)
        elif cluster_sizes is False:
            cluster_sizes = None
        stride = cluster_sizes.shape[1] if cluster_sizes is not None else 0
        with torch.cuda.device(self.device):
            st = _native.lib().rs_segment_batch_host(
                ctypes.byref(self.rs_config), self._tables_host.ctypes.data_as(ctypes.c_void_p),
                ranges.ctypes.data_as(ctypes.c_void_p), B,
                labels.ctypes.data_as(ctypes.c_void_p), n_clusters.ctypes.data_as(ctypes.c_void_p),
                cluster_sizes.ctypes.data_as(ctypes.c_void_p) if cluster_sizes is not None else None,
                stride)
        _native.check(st, "rs_segment_batch_host")
        return labels, n_clusters, cluster_sizes

    # -- the reference's per-frame entry point --------------------------------
    def segment_range_image(self, ri: RangeImage):
        """Cluster one image-shaped frame; returns ``(LabelImage, TimingRecord)``."""
        rec = TimingRecord()
        t0 = time.perf_counter()
        ranges = ri.ranges if isinstance(ri, RangeImage) else from_ranges(ri).ranges
        if ranges.shape != self.shape:
            raise ValueError(f"range image {ranges.shape} does not match model {self.shape}")
        self._require_cuda()
        x = torch.from_numpy(np.ascontiguousarray(ranges, dtype=np.float32)).to(
            self.device, non_blocking=False)[None]
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        res = self.segment_batch(x)
        ev1.record()
        k = int(res.n_clusters[0].item())
        li = LabelImage(labels=res.labels[0].cpu().numpy(),
                        cluster_sizes=res.cluster_sizes[0, :k + 1].cpu().numpy())
        rec.ccl = ev0.elapsed_time(ev1)
        rec.total = (time.perf_counter() - t0) * 1e3
        return li, rec


    # -- point clouds (pipeline.py:133-158) -------------------------------------
    def segment_clouds(self, clouds):
        """Project, cluster and back-project a list of clouds in one batch:
        ``[(SegOutput, TimingRecord)]``, each equal to ``segment_cloud``."""
        from . import cloud
        rec = TimingRecord()
        t0 = time.perf_counter()
        self._require_cuda()
        arrs = [np.asarray(c) for c in clouds]
        H, W = self.shape
        out = [None] * len(arrs)
        live = [i for i, a in enumerate(arrs) if a.size > 0]
        for i, a in enumerate(arrs):
            if a.size == 0:   # the reference's empty-cloud result (pipeline.py:137-143)
                empty = LabelImage(labels=np.zeros((H, W), np.int32), cluster_sizes=np.array([H * W]))
                out[i] = (cloud.SegOutput(point_labels=np.zeros(0, np.int32), label_image=empty),
                          TimingRecord())
        if live:
            pts = [cloud._check_points(arrs[i]) for i in live]
            x = torch.from_numpy(np.concatenate(pts) if len(pts) > 1 else pts[0]).to(self.device)
            off = torch.from_numpy(np.cumsum([0] + [p.shape[0] for p in pts]).astype(np.int64)).to(self.device)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record()
            ranges, pidx, _ = cloud.project_batch(x, off, self.model)
            ev[1].record()
            res = self.segment_batch(ranges)
            ev[2].record()
            plab = cloud.labels_to_points_batch(res.labels, pidx, off)
            ev[3].record()
            plab = plab.cpu().numpy()
            labels = res.labels.cpu().numpy()
            ncl = res.n_clusters.cpu().numpy()
            sizes = res.cluster_sizes.cpu().numpy()
            offs = off.cpu().numpy()
            rec.project = ev[0].elapsed_time(ev[1]) + ev[2].elapsed_time(ev[3])
            rec.ccl = ev[1].elapsed_time(ev[2])
            for j, i in enumerate(live):
                li = LabelImage(labels=labels[j], cluster_sizes=sizes[j, :int(ncl[j]) + 1].copy())
                out[i] = (cloud.SegOutput(point_labels=plab[offs[j]:offs[j + 1]], label_image=li), rec)
        rec.total = (time.perf_counter() - t0) * 1e3
        return out

    def segment_cloud(self, points):
        """Project a cloud, cluster it and carry labels back to the points
        (pipeline.py:133-158): ``(SegOutput, TimingRecord)``."""
        return self.segment_clouds([points])[0]


def segment_in_parallel(range_images, model: SensorModel,
                        config: PipelineConfig | None = None, max_workers: int = 2,
                        device=None):
    """Label many frames at once (pipeline.py:170-197): one batched launch.

    ``max_workers`` is accepted for signature compatibility; frames are
    parallel on the GPU, not on host threads.  Output order matches input
    order and equals frame-by-frame ``segment_range_image``.
    """
    del max_workers
    frames = [f.ranges if isinstance(f, RangeImage) else from_ranges(f).ranges
              for f in range_images]
    pipe = Pipeline(model, config, device=device)
    if not frames:
        return []
    for f in frames:
        if f.shape != pipe.shape:
            raise ValueError(f"range image {f.shape} does not match model {pipe.shape}")
    x = torch.from_numpy(np.stack(frames)).to(pipe.device)
    res = pipe.segment_batch(x)
    labels = res.labels.cpu().numpy()
    ncl = res.n_clusters.cpu().numpy()
    sizes = res.cluster_sizes.cpu().numpy()
    return [LabelImage(labels=labels[b], cluster_sizes=sizes[b, :int(ncl[b]) + 1].copy())
            for b in range(len(frames))]
