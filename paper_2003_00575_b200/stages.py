"""The path's stages as separate calls, on the GPU.

Mirrors of ``height_image`` (/root/reference/pkg/src/rangeseg/range_image.py:118-127),
``extract_ground`` (ground.py:95-141) and ``build_connectivity``
(connectivity.py:64-92) with the reference's signatures and inputs — the
caller's height image and ground mask are used as given — through
``rs_height_image`` / ``rs_ground_mask`` / ``rs_connectivity``.  The fused
``Pipeline`` path never materialises these images; they exist for callers
that use the stages on their own.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .config import DistanceThreshold, GroundParams, PipelineConfig
from .sensor import SensorModel
from .tables import pack_tables


@dataclass
class GroundMask:
    """(H, W) bool; True marks ground or no-return cells (ground.py:52-55)."""

    mask: np.ndarray


@dataclass
class ConnectivityImages:
    """horizontal[r, c] links (r, c)-(r, (c+1) mod W); vertical[r, c] links
    (r, c)-(r+1, c) (connectivity.py:35-44)."""

    horizontal: np.ndarray
    vertical: np.ndarray


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _setup(ri, model: SensorModel, cfg: PipelineConfig):
    ranges = ri.ranges if hasattr(ri, "ranges") else np.asarray(ri)
    if ranges.shape != (model.height, model.width):
        raise ValueError(f"range image {ranges.shape} does not match model {(model.height, model.width)}")
    if not torch.cuda.is_available():
        raise RuntimeError("the stage calls need a CUDA device (there is no CPU fallback)")
    dev = torch.device("cuda", torch.cuda.current_device())
    packed = pack_tables(model, cfg)
    rc = _native.make_config(packed)
    tables = torch.from_numpy(np.ascontiguousarray(packed.block, np.float32)).to(dev)
    x = torch.from_numpy(np.ascontiguousarray(ranges, dtype=np.float32)).to(dev)
    return dev, rc, tables, x, ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def height_image(ri, model: SensorModel) -> np.ndarray:
    """Per-cell z above the wheel-contact plane, NaN where there is no return."""
    dev, rc, tables, x, s = _setup(ri, model, PipelineConfig())
    z = torch.empty_like(x)
    _native.check(_native.lib().rs_height_image(ctypes.byref(rc), _ptr(tables), _ptr(x), 1, _ptr(z), s),
                  "rs_height_image")
    return z.cpu().numpy()


def extract_ground(ri, height: np.ndarray, model: SensorModel, params: GroundParams | None = None) -> GroundMask:
    """Ground and no-return cells, with the caller's height image."""
    params = params or GroundParams()
    dev, rc, tables, x, s = _setup(ri, model, PipelineConfig(ground=params, ground_removal=True))
    h = torch.from_numpy(np.ascontiguousarray(height, dtype=np.float32)).to(dev)
    if h.shape != x.shape:
        raise ValueError(f"height image {tuple(h.shape)} does not match range image {tuple(x.shape)}")
    m = torch.empty(x.shape, dtype=torch.uint8, device=dev)
    _native.check(_native.lib().rs_ground_mask(ctypes.byref(rc), _ptr(tables), _ptr(x), _ptr(h), 1, _ptr(m), s),
                  "rs_ground_mask")
    return GroundMask(mask=m.cpu().numpy().astype(bool))


def build_connectivity(ri, gm: GroundMask, model: SensorModel,
                       thr: DistanceThreshold | None = None) -> ConnectivityImages:
    """Thresholded horizontal (seam-wrapping) and vertical neighbour pairs,
    with the caller's ground mask."""
    thr = thr or DistanceThreshold()
    dev, rc, tables, x, s = _setup(ri, model, PipelineConfig(threshold=thr))
    mask = torch.from_numpy(np.ascontiguousarray(gm.mask, dtype=np.uint8)).to(dev)
    if mask.shape != x.shape:
        raise ValueError(f"ground mask {tuple(mask.shape)} does not match range image {tuple(x.shape)}")
    H, W = x.shape
    hz = torch.empty((H, W), dtype=torch.uint8, device=dev)
    vt = torch.empty((max(H - 1, 0), W), dtype=torch.uint8, device=dev)
    _native.check(_native.lib().rs_connectivity(ctypes.byref(rc), _ptr(tables), _ptr(x), _ptr(mask), 1,
                                                _ptr(hz), _ptr(vt), s), "rs_connectivity")
    return ConnectivityImages(horizontal=hz.cpu().numpy().astype(bool), vertical=vt.cpu().numpy().astype(bool))
