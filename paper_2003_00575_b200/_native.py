"""ctypes binding of the C ABI in include/rangeseg_b200.h.

The shared library is built in-tree by :mod:`.build` (``__graft_entry__.build()``).
There is no CPU fallback: if the library is missing, or no CUDA device is
present when a kernel is requested, calls raise ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("RS_LIB") or
                Path(__file__).resolve().parent / "_lib" / "librangeseg_b200.so")
MAX_OFFSETS = 32

RS_OK, RS_EINVAL, RS_ECUDA, RS_ETOOLARGE, RS_ENODEV = range(5)
RS_FRAME_INVALID = -1   # n_clusters[b] of a frame that breaks the input contract

EXPORTS = ("rs_tables_count", "rs_plan", "rs_plan_detail", "rs_plan_batch",
           "rs_segment_batch", "rs_segment_batch_host", "rs_fast_planes", "rs_stage_masks", "rs_project",
           "rs_project_workspace_size", "rs_contingency", "rs_contingency_workspace_size",
           "rs_height_image", "rs_ground_mask", "rs_connectivity",
           "rs_labels_to_points", "rs_phase_profile", "rs_last_error", "rs_version")


class RsConfig(ctypes.Structure):
    _fields_ = [("height", ctypes.c_int32), ("width", ctypes.c_int32),
                ("n_offsets", ctypes.c_int32),
                ("offsets", (ctypes.c_int32 * 2) * MAX_OFFSETS),
                ("min_cluster_points", ctypes.c_int32),
                ("ground_removal", ctypes.c_int32),
                ("d_max_sq", ctypes.c_float), ("mount_height", ctypes.c_float),
                ("keep_above", ctypes.c_float), ("two_cos_h", ctypes.c_float),
                ("rows_per_cta", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 3)]


class RsProjectConfig(ctypes.Structure):
    _fields_ = [("height", ctypes.c_int32), ("width", ctypes.c_int32),
                ("descending", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("azimuth_step", ctypes.c_double),
                ("gap_lo", ctypes.c_double), ("gap_hi", ctypes.c_double)]


_lib = None
_ext = None

_P = ctypes.c_void_p
EXT_PATH = LIB_PATH.parent / "torch_ext" / "rangeseg_b200_torch.so"


def use_torch_ext() -> bool:
    """The PyTorch extension links the in-tree librangeseg_b200.so; an RS_LIB
    override (experiment variants, scripts/ab.sh) goes through ctypes only."""
    return not os.environ.get("RS_LIB")


def torch_ext():
    """The thin PyTorch C++ extension over the C ABI (csrc/torch_ext.cpp):
    tensors in, rs_segment_batch on the current stream with the GIL released.
    Built in-tree by ``build.build_torch_ext`` (no JIT build at import)."""
    global _ext
    if _ext is None:
        import importlib.util

        import torch  # noqa: F401  (libc10 / libtorch for the extension)
        lib()          # the C library the extension links (and its error if missing)
        if not EXT_PATH.exists():
            raise RuntimeError(f"PyTorch extension {EXT_PATH} is missing; run __graft_entry__.build()")
        spec = importlib.util.spec_from_file_location("rangeseg_b200_torch", str(EXT_PATH))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _ext = mod
    return _ext


def lib():
    """Load the native library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"native library {LIB_PATH} is missing; run __graft_entry__.build() "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH))
        L.rs_tables_count.restype = ctypes.c_size_t
        L.rs_tables_count.argtypes = [ctypes.c_int32, ctypes.c_int32]
        L.rs_plan.restype = ctypes.c_int
        L.rs_plan.argtypes = [ctypes.POINTER(RsConfig), ctypes.POINTER(ctypes.c_int32),
                              ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_size_t)]
        L.rs_segment_batch.restype = ctypes.c_int
        L.rs_segment_batch.argtypes = [ctypes.POINTER(RsConfig), _P, _P, ctypes.c_int32,
                                       _P, _P, _P, ctypes.c_int64, _P]
        L.rs_fast_planes.restype = ctypes.c_int
        L.rs_fast_planes.argtypes = [ctypes.POINTER(RsConfig), _P, _P, ctypes.c_int32, _P, _P, _P, _P]
        L.rs_plan_batch.restype = ctypes.c_int
        L.rs_plan_batch.argtypes = [ctypes.POINTER(RsConfig), ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                    ctypes.c_int32]
        L.rs_plan_detail.restype = ctypes.c_int
        L.rs_plan_detail.argtypes = [ctypes.POINTER(RsConfig), ctypes.POINTER(ctypes.c_int32),
                                     ctypes.c_int32]
        L.rs_segment_batch_host.restype = ctypes.c_int
        L.rs_segment_batch_host.argtypes = [ctypes.POINTER(RsConfig), _P, _P, ctypes.c_int32,
                                            _P, _P, _P, ctypes.c_int64]
        L.rs_stage_masks.restype = ctypes.c_int
        L.rs_stage_masks.argtypes = [ctypes.POINTER(RsConfig), _P, _P, ctypes.c_int32,
                                     _P, _P, _P, _P]
        L.rs_project.restype = ctypes.c_int
        L.rs_project.argtypes = [ctypes.POINTER(RsProjectConfig), _P, _P, ctypes.c_int32, _P,
                                 ctypes.c_int32, ctypes.c_int64, _P, _P, _P, _P, ctypes.c_size_t, _P]
        L.rs_project_workspace_size.restype = ctypes.c_size_t
        L.rs_project_workspace_size.argtypes = [ctypes.c_int64]
        L.rs_labels_to_points.restype = ctypes.c_int
        L.rs_labels_to_points.argtypes = [_P, _P, _P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int64, _P, _P]
        L.rs_contingency_workspace_size.restype = ctypes.c_size_t
        L.rs_contingency_workspace_size.argtypes = [ctypes.c_int64, ctypes.c_int32]
        L.rs_contingency.restype = ctypes.c_int
        L.rs_contingency.argtypes = [_P, _P, _P, ctypes.c_int32, ctypes.c_int64, _P, _P, _P, _P,
                                     ctypes.c_size_t, _P]
        L.rs_height_image.restype = ctypes.c_int
        L.rs_height_image.argtypes = [ctypes.POINTER(RsConfig), _P, _P, ctypes.c_int32, _P, _P]
        L.rs_ground_mask.restype = ctypes.c_int
        L.rs_ground_mask.argtypes = [ctypes.POINTER(RsConfig), _P, _P, _P, ctypes.c_int32, _P, _P]
        L.rs_connectivity.restype = ctypes.c_int
        L.rs_connectivity.argtypes = [ctypes.POINTER(RsConfig), _P, _P, _P, ctypes.c_int32, _P, _P, _P]
        L.rs_phase_profile.restype = ctypes.c_int
        L.rs_phase_profile.argtypes = [_P, ctypes.c_int32]
        L.rs_last_error.restype = ctypes.c_char_p
        L.rs_version.restype = ctypes.c_int
        _lib = L
    return _lib


def check(status: int, what: str = "rangeseg_b200"):
    """Map a C status to the reference's exception types."""
    if status == RS_OK:
        return
    msg = lib().rs_last_error().decode(errors="replace")
    if status in (RS_EINVAL, RS_ETOOLARGE):
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")


def make_config(packed, rows_per_cta: int = 0, node_capacity: int = 0,
                stop_after: int = 0) -> RsConfig:
    if len(packed.offsets) > MAX_OFFSETS:
        raise ValueError(f"at most {MAX_OFFSETS} Map Connection offsets are supported")
    cfg = RsConfig()
    cfg.height, cfg.width = packed.height, packed.width
    cfg.n_offsets = len(packed.offsets)
    for i, (dy, dx) in enumerate(packed.offsets):
        cfg.offsets[i][0], cfg.offsets[i][1] = dy, dx
    cfg.min_cluster_points = int(packed.min_cluster_points)
    cfg.ground_removal = int(bool(packed.ground_removal))
    cfg.d_max_sq = float(packed.d_max_sq)
    cfg.mount_height = float(packed.mount)
    cfg.keep_above = float(packed.keep_above)
    cfg.two_cos_h = float(packed.two_cos_h)
    cfg.rows_per_cta = int(rows_per_cta)
    cfg.reserved[0] = int(node_capacity)
    cfg.reserved[1] = int(stop_after)   # RS_EXPERIMENTS builds only (else RS_EINVAL): truncated kernel
    return cfg


PLAN_FIELDS = ("fast", "may_overflow", "fast_rows", "fast_ctas", "fast_smem", "node_capacity",
               "dense_rows", "dense_ctas", "dense_smem")


def plan_detail(cfg: RsConfig) -> dict:
    out = (ctypes.c_int32 * len(PLAN_FIELDS))()
    check(lib().rs_plan_detail(ctypes.byref(cfg), out, len(PLAN_FIELDS)), "rs_plan_detail")
    return dict(zip(PLAN_FIELDS, list(out)))


def plan_batch(cfg: RsConfig, batch: int) -> dict:
    """The plan of a launch of ``batch`` frames (small batches get thinner bands)."""
    out = (ctypes.c_int32 * len(PLAN_FIELDS))()
    check(lib().rs_plan_batch(ctypes.byref(cfg), int(batch), out, len(PLAN_FIELDS)), "rs_plan_batch")
    return dict(zip(PLAN_FIELDS, list(out)))


def plan(cfg: RsConfig):
    R, C, smem = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_size_t()
    check(lib().rs_plan(ctypes.byref(cfg), ctypes.byref(R), ctypes.byref(C), ctypes.byref(smem)),
          "rs_plan")
    return R.value, C.value, smem.value
