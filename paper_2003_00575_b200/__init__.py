"""B200-native range-image Lidar segmentation — the hot path of arXiv 2003.00575.

Drop-in for the reference package ``rangeseg``'s clustering entry point
(``Pipeline.segment_range_image``, ``segment_in_parallel``): range image and
parameters in, per-pixel int32 instance labels out, computed by a fused
sm_100a kernel (csrc/rangeseg_b200.cu) behind the C ABI in
include/rangeseg_b200.h.  Names mirror the reference's public API
(pkg/src/rangeseg/__init__.py:11-31) for the path.
"""

from .cloud import SegOutput, labels_to_points, project
from .evaluation import (EvalConfig, EvalReport, InstanceMatch, instance_iou,
                         match_instances, precision_at, report_as_dict, summarize)
from .config import (PRESETS, DistanceThreshold, GroundParams, MCPattern,
                     PipelineConfig, parse_offsets, preset_pattern, skip_pattern)
from .pipeline import (STAGES, BatchResult, LabelImage, Pipeline, RangeImage,
                       TimingRecord, from_ranges, segment_in_parallel)
from .sensor import (SensorConfigError, SensorModel, canonical_offset,
                     default_model, fov_model, load_sensor_model, uniform_model)
from .stages import ConnectivityImages, GroundMask, build_connectivity, extract_ground, height_image
from .tables import PackedTables, pack_tables

__version__ = "0.1.0"
