"""ctypes front end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs import
this module.  The product package never does.  See rangeseg_oracle.c for what
is restated and where it is pinned.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "librangeseg_oracle.so"


class _Cfg(ctypes.Structure):
    _fields_ = [("height", ctypes.c_int32), ("width", ctypes.c_int32),
                ("n_offsets", ctypes.c_int32),
                ("offsets", ctypes.POINTER(ctypes.c_int32)),
                ("min_cluster_points", ctypes.c_int32),
                ("ground_removal", ctypes.c_int32),
                ("d_max_sq", ctypes.c_float), ("mount_height", ctypes.c_float),
                ("keep_above", ctypes.c_float), ("two_cos_h", ctypes.c_float),
                ("tables", ctypes.POINTER(ctypes.c_float))]


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        _lib = ctypes.CDLL(str(LIB_PATH))
        _lib.oracle_segment_frame.restype = ctypes.c_int32
        _lib.oracle_segment_batch.restype = ctypes.c_int
    return _lib


def _ptr(a, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


class OracleConfig:
    """Holds a ctypes config plus the numpy buffers it points into."""

    def __init__(self, packed):
        self.packed = packed
        self.offsets = np.ascontiguousarray(
            np.array(packed.offsets, dtype=np.int32).reshape(-1, 2))
        self.tables = np.ascontiguousarray(packed.block, dtype=np.float32)
        self.cfg = _Cfg(packed.height, packed.width, len(packed.offsets),
                        _ptr(self.offsets, ctypes.c_int32),
                        packed.min_cluster_points, int(packed.ground_removal),
                        float(packed.d_max_sq), float(packed.mount),
                        float(packed.keep_above), float(packed.two_cos_h),
                        _ptr(self.tables, ctypes.c_float))


def segment_frame(ranges, packed, stages=False):
    """One frame through the restated reference path.

    Returns ``(labels int32 [H,W], cluster_sizes int64 [K+1])`` and, with
    ``stages=True``, also ``(ground_mask, horizontal, vertical)`` bool arrays.
    """
    oc = OracleConfig(packed)
    H, W = packed.height, packed.width
    rg = np.ascontiguousarray(ranges, dtype=np.float32)
    assert rg.shape == (H, W)
    labels = np.zeros((H, W), dtype=np.int32)
    sizes = np.zeros(H * W + 1, dtype=np.int64)
    gm = np.zeros((H, W), dtype=np.uint8)
    hz = np.zeros((H, W), dtype=np.uint8)
    vt = np.zeros((H - 1, W), dtype=np.uint8)
    K = lib().oracle_segment_frame(_ptr(rg, ctypes.c_float), ctypes.byref(oc.cfg),
                                   _ptr(labels, ctypes.c_int32), _ptr(sizes, ctypes.c_int64),
                                   _ptr(gm, ctypes.c_uint8), _ptr(hz, ctypes.c_uint8),
                                   _ptr(vt, ctypes.c_uint8))
    if K < 0:
        raise MemoryError("oracle allocation failed")
    out = (labels, sizes[:K + 1].copy())
    if stages:
        return out + (gm.astype(bool), hz.astype(bool), vt.astype(bool))
    return out


def segment_batch(ranges, packed, nthreads=None, sizes_stride=None):
    """[B,H,W] frames on ``nthreads`` host threads.

    Returns ``(labels [B,H,W] int32, n_clusters [B] int32, sizes [B,stride] int64)``.
    """
    oc = OracleConfig(packed)
    rg = np.ascontiguousarray(ranges, dtype=np.float32)
    B = rg.shape[0]
    H, W = packed.height, packed.width
    if sizes_stride is None:
        sizes_stride = H * W // max(packed.min_cluster_points, 1) + 1
    labels = np.zeros((B, H, W), dtype=np.int32)
    ncl = np.zeros(B, dtype=np.int32)
    sizes = np.zeros((B, sizes_stride), dtype=np.int64)
    nthreads = nthreads or os.cpu_count() or 1
    rc = lib().oracle_segment_batch(_ptr(rg, ctypes.c_float), B, ctypes.byref(oc.cfg),
                                    _ptr(labels, ctypes.c_int32), _ptr(ncl, ctypes.c_int32),
                                    _ptr(sizes, ctypes.c_int64), ctypes.c_int64(sizes_stride),
                                    int(nthreads))
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    return labels, ncl, sizes


def planes_batch(ranges, packed, nthreads=None):
    """The edge decisions of [B,H,W] frames as packed bit planes, uint32
    [B, 3 + n_offsets, H, ceil(W/32)] in rs_fast_planes' layout (presence,
    left edge, up edge, one plane per Map Connection offset)."""
    oc = OracleConfig(packed)
    rg = np.ascontiguousarray(ranges, dtype=np.float32)
    B = rg.shape[0]
    H, W = packed.height, packed.width
    planes = np.zeros((B, 3 + len(packed.offsets), H, (W + 31) // 32), dtype=np.uint32)
    rc = lib().oracle_planes_batch(_ptr(rg, ctypes.c_float), B, ctypes.byref(oc.cfg),
                                   _ptr(planes, ctypes.c_uint32), int(nthreads or os.cpu_count() or 1))
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    return planes


class _ProjCfg(ctypes.Structure):
    _fields_ = [("height", ctypes.c_int32), ("width", ctypes.c_int32),
                ("descending", ctypes.c_int32), ("azimuth_step", ctypes.c_double),
                ("asc", ctypes.POINTER(ctypes.c_double))]


def project(points, model):
    """range_image.project restated in C (project_oracle.c).

    Returns ``(ranges f32 [H,W], point_index i64 [H,W], n_dropped, n_overwritten)``.
    """
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    if pts.ndim != 2 or pts.shape[1] < 3 or pts.shape[0] == 0:
        raise ValueError("expected a nonempty (N, 3) point array")
    ang = np.asarray(model.channel_angles, dtype=np.float64)
    desc = bool(ang[0] > ang[-1])
    asc = np.ascontiguousarray(ang[::-1] if desc else ang)
    cfg = _ProjCfg(model.height, model.width, int(desc), float(model.azimuth_step),
                   _ptr(asc, ctypes.c_double))
    H, W = model.height, model.width
    ranges = np.zeros((H, W), np.float32)
    pidx = np.zeros((H, W), np.int64)
    counts = np.zeros(2, np.int64)
    rc = lib().oracle_project(_ptr(pts, ctypes.c_double), ctypes.c_int64(pts.shape[0]),
                              ctypes.c_int32(pts.shape[1]), ctypes.byref(cfg),
                              _ptr(ranges, ctypes.c_float), _ptr(pidx, ctypes.c_int64),
                              _ptr(counts, ctypes.c_int64))
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    return ranges, pidx, int(counts[0]), int(counts[1])


def labels_to_points(labels, point_index, n_points):
    """range_image.labels_to_points restated in C."""
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    pidx = np.ascontiguousarray(point_index, dtype=np.int64)
    out = np.zeros(int(n_points), np.int32)
    lib().oracle_labels_to_points(_ptr(lab, ctypes.c_int32), _ptr(pidx, ctypes.c_int64),
                                  ctypes.c_int64(pidx.size), ctypes.c_int64(n_points),
                                  _ptr(out, ctypes.c_int32))
    return out
