"""Float32 constant tables for the per-pixel kernels.

Every value is produced in float64 by :class:`.sensor.SensorModel` and cast to
float32 once, exactly where the reference casts it:

=====================  =========================================  ===========================
table                  recipe                                     reference
=====================  =========================================  ===========================
``sin_ch[H]``          ``sin(delta_r)``                           range_image.py:125
``sin_a, cos_a[H-1]``  sin/cos of ``|delta_{r+1} - delta_r|``     ground.py:114-115
``lo, hi[H-1]``        ``tan(center -/+ theta)``                  ground.py:84-92, 119-121
``two_cos_v[H-1]``     ``pair_constant(1, 0)``                    connectivity.py:88
``two_cos_off[k][H]``  ``pair_constant(dy, dx)`` by upper row     map_connections.py:156
``two_cos_h``          ``pair_constant(0, 1)``                    connectivity.py:82
``d_max_sq``           ``f32(d_max * d_max)``                     connectivity.py:77
``mount``              ``f32(mount_height)``                      range_image.py:126
``keep_above``         ``f32(resolve_keep_above)``                ground.py:136
=====================  =========================================  ===========================

The flat layout (one contiguous float32 block) is the one ``include/rangeseg_b200.h``
documents for ``rs_segment_batch``'s ``tables`` argument.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import PipelineConfig
from .sensor import SensorModel

F32 = np.float32


@dataclass
class PackedTables:
    height: int
    width: int
    offsets: tuple            # canonical (dy, dx) Map Connection offsets
    block: np.ndarray         # float32, layout below
    two_cos_h: np.float32
    d_max_sq: np.float32
    mount: np.float32
    keep_above: np.float32
    min_cluster_points: int
    ground_removal: bool

    # -- layout -----------------------------------------------------------
    @staticmethod
    def size(H: int, n_off: int) -> int:
        return H + 5 * (H - 1) + n_off * H

    def section(self, name: str, k: int = 0) -> np.ndarray:
        H = self.height
        starts = {"sin_ch": (0, H), "sin_a": (H, H - 1), "cos_a": (2 * H - 1, H - 1),
                  "lo": (3 * H - 2, H - 1), "hi": (4 * H - 3, H - 1),
                  "two_cos_v": (5 * H - 4, H - 1)}
        if name == "two_cos_off":
            s = 6 * H - 5 + k * H
            return self.block[s:s + H]
        s, n = starts[name]
        return self.block[s:s + n]


def pack_tables(model: SensorModel, config: PipelineConfig) -> PackedTables:
    """Build the float32 table block for ``model`` under ``config``.

    Raises ``ValueError`` for offsets outside the frame (map_connections.py:152-153,
    sensor.py:151-155) and for slope bounds that reach 90 degrees (ground.py:88-91),
    the same conditions the reference rejects.
    """
    H, W = model.height, model.width
    offsets = tuple(config.mc_pattern.offsets)
    for dy, dx in offsets:
        if dy >= H or abs(dx) >= W:
            raise ValueError(f"offset ({dy}, {dx}) exceeds frame {H}x{W}")
    block = np.zeros(PackedTables.size(H, len(offsets)), dtype=F32)
    pt = PackedTables(H, W, offsets, block, F32(0), F32(0), F32(0), F32(0),
                      int(config.min_cluster_points), bool(config.ground_removal))

    pt.section("sin_ch")[:] = model.sin_channel.astype(F32)
    pt.section("sin_a")[:] = model.sin_vertical.astype(F32)
    pt.section("cos_a")[:] = model.cos_vertical.astype(F32)
    if config.ground_removal:
        lo, hi = model.ground_bounds(config.ground.theta_deg)
        pt.section("lo")[:] = lo.astype(F32)
        pt.section("hi")[:] = hi.astype(F32)
    pt.section("two_cos_v")[:] = model.pair_constant(1, 0).astype(F32).ravel()
    for k, (dy, dx) in enumerate(offsets):
        tc = model.pair_constant(dy, dx).astype(F32).ravel()
        dst = pt.section("two_cos_off", k)
        if dy == 0:
            dst[:] = tc[0]
        else:
            dst[:H - dy] = tc
    pt.two_cos_h = (model.pair_constant(0, 1).astype(F32).item()
                    if W > 1 else F32(0))
    pt.two_cos_h = F32(pt.two_cos_h)
    pt.d_max_sq = np.asarray(config.threshold.d_max_sq, dtype=F32)[()]
    pt.mount = F32(model.mount_height)
    pt.keep_above = np.asarray(config.ground.resolve_keep_above(model), dtype=F32)[()]
    return pt
