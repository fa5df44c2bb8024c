"""Pipeline parameters: ground test, distance threshold, Map Connection offsets.

Same names, defaults and validation errors as the reference:
``GroundParams`` (ground.py:26-48), ``DistanceThreshold`` (connectivity.py:21-31),
``MCPattern`` / ``PRESETS`` / ``preset_pattern`` / ``parse_offsets``
(map_connections.py:23-70) and ``PipelineConfig`` (pipeline.py:30-38).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from .sensor import canonical_offset


@dataclass
class GroundParams:
    """Slope tolerance ``theta_deg`` and the height exception ``keep_above_z``.

    ``keep_above_z=None`` means one metre below the sensor (ground.py:45-48).
    """

    theta_deg: float = 10.0
    keep_above_z: float | None = None

    def __post_init__(self):
        if not (0.0 < self.theta_deg < 90.0):
            raise ValueError(f"theta_deg must be in (0, 90), got {self.theta_deg}")
        if self.keep_above_z is not None and not math.isfinite(self.keep_above_z):
            raise ValueError("keep_above_z must be finite")

    def resolve_keep_above(self, model) -> float:
        if self.keep_above_z is not None:
            return float(self.keep_above_z)
        return model.mount_height - 1.0


@dataclass
class DistanceThreshold:
    """Maximum 3-D distance between connected returns; compared squared."""

    d_max: float = 0.8
    d_max_sq: float = field(init=False)

    def __post_init__(self):
        if not (self.d_max > 0):
            raise ValueError(f"d_max must be > 0, got {self.d_max}")
        self.d_max_sq = self.d_max * self.d_max


@dataclass(frozen=True)
class MCPattern:
    """Canonicalised, de-duplicated (dy, dx) Map Connection offsets."""

    offsets: tuple

    def __post_init__(self):
        seen = []
        for off in self.offsets:
            off = canonical_offset(off)
            if off not in seen:
                seen.append(off)
        object.__setattr__(self, "offsets", tuple(seen))

    def __len__(self):
        return len(self.offsets)


PRESETS = {
    "none": (),
    "mc1": ((0, 2), (2, 0)),
    "mc6": ((0, 2), (2, 0), (0, 3), (3, 0), (2, 2), (3, 3)),
    "mc14": tuple((k, k) for k in range(2, 16)),
}


def preset_pattern(name: str) -> MCPattern:
    try:
        return MCPattern(PRESETS[name])
    except KeyError:
        raise ValueError(
            f"unknown preset {name!r}; choose from {sorted(PRESETS)}") from None


def skip_pattern(s: int) -> MCPattern:
    """BASELINE.json's skip count S as Map Connections: {(0,k),(k,0) : 2 <= k <= S+1}.

    S = 0 is the reference default (no offsets); S = 1 equals ``mc1``.
    """
    if s < 0:
        raise ValueError(f"skip count must be >= 0, got {s}")
    offs = []
    for k in range(2, s + 2):
        offs += [(0, k), (k, 0)]
    return MCPattern(tuple(offs))


def parse_offsets(text: str) -> MCPattern:
    """``"0,2;2,0;3,3"`` → MCPattern (map_connections.py:61-70)."""
    offsets = []
    for part in text.split(";"):
        part = part.strip()
        if not part:
            continue
        dy, dx = part.split(",")
        offsets.append((int(dy), int(dx)))
    return MCPattern(tuple(offsets))


@dataclass
class PipelineConfig:
    """Everything that tunes a segmentation run (pipeline.py:30-38)."""

    ground: GroundParams = field(default_factory=GroundParams)
    threshold: DistanceThreshold = field(default_factory=DistanceThreshold)
    mc_pattern: MCPattern = field(default_factory=lambda: MCPattern(()))
    min_cluster_points: int = 100
    ground_removal: bool = True
