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
    n_clusters: torch.Tensor      # int32 [B]; RS_FRAME_INVALID (-1) for a frame with bad ranges
    cluster_sizes: torch.Tensor | None   # int64 [B, stride]; row b valid up to n_clusters[b]

    def check(self) -> "BatchResult":
        """Raise the reference's ``ValueError`` (range_image.py:52-53) if a frame
        held a NaN, inf or negative range (flagged by the kernel on the device;
        this reads ``n_clusters`` back, so it synchronises)."""
        bad = torch.nonzero(self.n_clusters == _native.RS_FRAME_INVALID).flatten()
        if bad.numel():
            raise ValueError(f"ranges must be finite and >= 0 (frame {int(bad[0])})")
        return self

    def label_image(self, b: int) -> LabelImage:
        k = int(self.n_clusters[b])
        if k == _native.RS_FRAME_INVALID:
            raise ValueError(f"ranges must be finite and >= 0 (frame {b})")
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
                 device=None, rows_per_cta: int = 0, node_capacity: int = 0,
                 stage_timing: bool = False):
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
        self._tables_host = np.ascontiguousarray(self.packed.block, dtype=np.float32)
        self._frame_bufs = None   # pinned staging of segment_range_image
        # per-stage TimingRecord (pipeline.py:94-130): the fused kernel runs every
        # stage in one launch, so with stage_timing the reference's separate
        # stages are also run (rs_height_image + rs_ground_mask, rs_connectivity)
        # and timed on the device; off by default (extra launches)
        self.stage_timing = bool(stage_timing)
        self._no_sizes = torch.empty(0, dtype=torch.int64)

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

    def _check_frames(self, ranges: torch.Tensor):
        H, W = self.shape
        if ranges.dim() != 3 or tuple(ranges.shape[1:]) != (H, W):
            raise ValueError(f"range images {tuple(ranges.shape)} do not match model "
                             f"{(H, W)}")
        if ranges.dtype != torch.float32:
            raise ValueError(f"ranges must be float32, got {ranges.dtype}")

    def _check_out(self, t: torch.Tensor, name: str, dtype, shape):
        """Caller-supplied output buffers: dtype, shape, device, contiguity (the
        C side writes through the raw pointer)."""
        if not isinstance(t, torch.Tensor):
            raise ValueError(f"{name} must be a torch.Tensor")
        if t.dtype != dtype:
            raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
        if t.device != self.device:
            raise ValueError(f"{name} on {t.device}, pipeline on {self.device}")
        if tuple(t.shape[:len(shape)]) != tuple(shape) or t.dim() != len(shape) + (name == "cluster_sizes"):
            raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}"
                             + (" + (stride,)" if name == "cluster_sizes" else ""))
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")

    # -- device batch ------------------------------------------------------
    def segment_batch(self, ranges: torch.Tensor, *, labels: torch.Tensor | None = None,
                      n_clusters: torch.Tensor | None = None,
                      cluster_sizes: torch.Tensor | bool | None = True,
                      stream: torch.cuda.Stream | None = None) -> BatchResult:
        """Segment B frames resident on the GPU; asynchronous on ``stream``.

        The launch waits for the work already queued on the current stream
        (the ranges' producer, the output allocations).  Frames with a NaN, inf
        or negative range come back with ``n_clusters == -1``; ``.check()``
        raises the reference's ``ValueError`` for them.
        """
        self._require_cuda()
        self._check_frames(ranges)
        if ranges.device != self.device:
            raise ValueError(f"ranges on {ranges.device}, pipeline on {self.device}")
        B = ranges.shape[0]
        H, W = self.shape
        with torch.cuda.device(self.device):
            cur = torch.cuda.current_stream(self.device)
            ranges = ranges.contiguous()
            if labels is None:
                labels = torch.empty((B, H, W), dtype=torch.int32, device=self.device)
            else:
                self._check_out(labels, "labels", torch.int32, (B, H, W))
            if n_clusters is None:
                n_clusters = torch.empty((B,), dtype=torch.int32, device=self.device)
            else:
                self._check_out(n_clusters, "n_clusters", torch.int32, (B,))
            if cluster_sizes is True:
                cluster_sizes = torch.empty((B, self.sizes_stride), dtype=torch.int64,
                                            device=self.device)
            elif cluster_sizes is False or cluster_sizes is None:
                cluster_sizes = None
            else:
                self._check_out(cluster_sizes, "cluster_sizes", torch.int64, (B,))
                if cluster_sizes.shape[1] < self.sizes_stride:
                    raise ValueError(f"cluster_sizes needs >= {self.sizes_stride} columns, "
                                     f"got {cluster_sizes.shape[1]}")
            stride = cluster_sizes.shape[1] if cluster_sizes is not None else 0
            s = stream if stream is not None else cur
            if s.cuda_stream != cur.cuda_stream:
                s.wait_stream(cur)
                for t in (ranges, labels, n_clusters, cluster_sizes, self.device_tables()):
                    if t is not None:
                        t.record_stream(s)
            if _native.use_torch_ext():
                # the thin PyTorch extension over rs_segment_batch (GIL released, current stream)
                with torch.cuda.stream(s):
                    _native.torch_ext().segment_batch(
                        ctypes.addressof(self.rs_config), self.device_tables(), ranges, labels, n_clusters,
                        cluster_sizes if cluster_sizes is not None else self._no_sizes)
            else:
                _native.check(_native.lib().rs_segment_batch(
                    ctypes.byref(self.rs_config), _ptr(self.device_tables()), _ptr(ranges), B,
                    _ptr(labels), _ptr(n_clusters), _ptr(cluster_sizes), stride,
                    ctypes.c_void_p(s.cuda_stream)), "rs_segment_batch")
        return BatchResult(labels, n_clusters, cluster_sizes)

    def fast_planes(self, ranges: torch.Tensor):
        """The fused kernel's own edge decisions (``rs_fast_planes``): returns
        ``(planes uint32 [B, 3 + n_offsets, H, ceil(W/32)], BatchResult)``;
        planes: presence, left edge, up edge, then one per Map Connection offset
        (include/rangeseg_b200.h).  For parity checks."""
        self._require_cuda()
        self._check_frames(ranges)
        B = ranges.shape[0]
        H, W = self.shape
        wpr = (W + 31) // 32
        with torch.cuda.device(self.device):
            ranges = ranges.contiguous()
            planes = torch.zeros((B, 3 + len(self.packed.offsets), H, wpr), dtype=torch.int32,
                                 device=self.device)
            labels = torch.empty((B, H, W), dtype=torch.int32, device=self.device)
            ncl = torch.empty((B,), dtype=torch.int32, device=self.device)
            st = _native.lib().rs_fast_planes(
                ctypes.byref(self.rs_config), _ptr(self.device_tables()), _ptr(ranges), B,
                _ptr(planes), _ptr(labels), _ptr(ncl),
                ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))
        _native.check(st, "rs_fast_planes")
        return planes, BatchResult(labels, ncl, None)

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

        def out(a, name, dtype, shape):
            if not isinstance(a, np.ndarray) or a.dtype != dtype or a.shape[:len(shape)] != shape \
                    or not a.flags.c_contiguous or not a.flags.writeable:
                raise ValueError(f"{name} must be a writeable C-contiguous {np.dtype(dtype).name} "
                                 f"array of shape {shape}" + (" + (stride,)" if name == "cluster_sizes" else ""))
            if a.ndim != len(shape) + (name == "cluster_sizes"):
                raise ValueError(f"{name} has {a.ndim} dimensions")

        if labels is None:
            labels = np.empty((B, H, W), dtype=np.int32)
        else:
            out(labels, "labels", np.int32, (B, H, W))
        if n_clusters is None:
            n_clusters = np.empty((B,), dtype=np.int32)
        else:
            out(n_clusters, "n_clusters", np.int32, (B,))
        if cluster_sizes is True:
            cluster_sizes = np.empty((B, self.sizes_stride), dtype=np.int64)
        elif cluster_sizes is False or cluster_sizes is None:
            cluster_sizes = None
        else:
            out(cluster_sizes, "cluster_sizes", np.int64, (B,))
            if cluster_sizes.shape[1] < self.sizes_stride:
                raise ValueError(f"cluster_sizes needs >= {self.sizes_stride} columns, "
                                 f"got {cluster_sizes.shape[1]}")
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
    def _frame_buffers(self):
        """Pinned host staging + device buffers of segment_range_image, made once."""
        if self._frame_bufs is None:
            H, W = self.shape
            pin = dict(pin_memory=True)
            # the three outputs share one device block and one pinned block (labels,
            # then sizes, then the count; 16-byte aligned parts), so that one D2H
            # copy brings all of them back
            nl = H * W * 4
            o_sz = (nl + 15) & ~15
            o_ncl = o_sz + ((self.sizes_stride * 8 + 15) & ~15)
            total = o_ncl + 16

            def views(blk):
                return (blk[:nl].view(torch.int32).view(1, H, W),
                        blk[o_sz:o_sz + self.sizes_stride * 8].view(torch.int64).view(1, self.sizes_stride),
                        blk[o_ncl:o_ncl + 4].view(torch.int32))
            h_out = torch.empty((total,), dtype=torch.uint8, **pin)
            d_out = torch.empty((total,), dtype=torch.uint8, device=self.device)
            h_lab, h_sz, h_ncl = views(h_out)
            d_lab, d_sz, d_ncl = views(d_out)
            self._frame_bufs = {
                "h_in": torch.empty((1, H, W), dtype=torch.float32, **pin),
                "h_out": h_out, "h_lab": h_lab, "h_ncl": h_ncl, "h_sz": h_sz,
                "d_in": torch.empty((1, H, W), dtype=torch.float32, device=self.device),
                "d_out": d_out, "d_lab": d_lab, "d_ncl": d_ncl, "d_sz": d_sz,
                "ev": [torch.cuda.Event(enable_timing=True) for _ in range(3)],
            }
        return self._frame_bufs

    def segment_range_image(self, ri: RangeImage):
        """Cluster one image-shaped frame (pipeline.py:85-131); returns
        ``(LabelImage, TimingRecord)``.

        One frame through pinned staging: H2D copy, the fused kernel, D2H of
        labels / count / sizes, one synchronisation.  A raw array gets
        ``from_ranges``' contract (finite, >= 0: ``ValueError``), checked by
        the kernel as it reads the ranges; a ``RangeImage`` is taken as is, like
        the reference (a NaN or negative range is then simply no return).
        ``TimingRecord.ccl`` = device time of the fused kernel (every stage of
        the reference runs inside it), ``total`` = wall time of the call; with
        ``stage_timing=True`` also ``ground`` / ``connectivity``: the device
        times of those stages run on their own (extra launches, after the
        fused one).
        """
        rec = TimingRecord()
        t0 = time.perf_counter()
        ranges = ri.ranges if isinstance(ri, RangeImage) else np.asarray(ri)
        if ranges.ndim != 2:
            raise ValueError(f"range image must be 2-D, got shape {ranges.shape}")
        if ranges.shape != self.shape:
            raise ValueError(f"range image {ranges.shape} does not match model {self.shape}")
        self._require_cuda()
        b = self._frame_buffers()
        np.copyto(b["h_in"].numpy()[0], ranges, casting="same_kind")
        with torch.cuda.device(self.device):
            s = torch.cuda.current_stream(self.device)
            ev = b["ev"]
            b["d_in"].copy_(b["h_in"], non_blocking=True)
            ev[0].record(s)
            st = _native.lib().rs_segment_batch(
                ctypes.byref(self.rs_config), _ptr(self.device_tables()), _ptr(b["d_in"]), 1,
                _ptr(b["d_lab"]), _ptr(b["d_ncl"]), _ptr(b["d_sz"]), self.sizes_stride,
                ctypes.c_void_p(s.cuda_stream))
            _native.check(st, "rs_segment_batch")
            ev[1].record(s)
            b["h_out"].copy_(b["d_out"], non_blocking=True)   # labels, sizes and count in one copy
            ev[2].record(s)
            ev[2].synchronize()
        if self.stage_timing:
            self._time_stages(b["d_in"], rec)
        k = int(b["h_ncl"][0])
        labels = b["h_lab"].numpy()[0].copy()
        if k == _native.RS_FRAME_INVALID:
            if not isinstance(ri, RangeImage):
                raise ValueError("ranges must be finite and >= 0")
            k = int(labels.max())   # labels are 1..K, each kept cluster has cells
        li = LabelImage(labels=labels, cluster_sizes=b["h_sz"].numpy()[0, :k + 1].copy())
        rec.ccl = ev[0].elapsed_time(ev[1])
        rec.total = (time.perf_counter() - t0) * 1e3
        return li, rec


    def _time_stages(self, x: torch.Tensor, rec: TimingRecord):
        """Device times of the reference's ground and connectivity stages run on
        their own (the stage entries of the C ABI) for TimingRecord."""
        H, W = self.shape
        lib = _native.lib()
        with torch.cuda.device(self.device):
            s = torch.cuda.current_stream(self.device)
            sp = ctypes.c_void_p(s.cuda_stream)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            z = torch.empty((1, H, W), dtype=torch.float32, device=self.device)
            gm = torch.empty((1, H, W), dtype=torch.uint8, device=self.device)
            hz = torch.empty((1, H, W), dtype=torch.uint8, device=self.device)
            vt = torch.empty((1, max(H - 1, 0), W), dtype=torch.uint8, device=self.device)
            cfg = ctypes.byref(self.rs_config)
            tb = _ptr(self.device_tables())
            ev[0].record(s)
            if self.config.ground_removal:
                _native.check(lib.rs_height_image(cfg, tb, _ptr(x), 1, _ptr(z), sp), "rs_height_image")
            _native.check(lib.rs_ground_mask(cfg, tb, _ptr(x), _ptr(z), 1, _ptr(gm), sp), "rs_ground_mask")
            ev[1].record(s)
            _native.check(lib.rs_connectivity(cfg, tb, _ptr(x), _ptr(gm), 1, _ptr(hz), _ptr(vt), sp),
                          "rs_connectivity")
            ev[2].record(s)
            ev[2].synchronize()
        rec.ground = ev[0].elapsed_time(ev[1])
        rec.connectivity = ev[1].elapsed_time(ev[2])

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
    for b in np.nonzero(ncl == _native.RS_FRAME_INVALID)[0]:   # RangeImage inputs are taken as is
        ncl[b] = labels[b].max()
    return [LabelImage(labels=labels[b], cluster_sizes=sizes[b, :int(ncl[b]) + 1].copy())
            for b in range(len(frames))]
