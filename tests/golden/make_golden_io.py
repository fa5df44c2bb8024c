"""Golden fixtures for the KITTI / SemanticKITTI file formats (SURVEY.md
§8(f)4), written by the Python reference itself in the build container:

    python tests/golden/make_golden_io.py

Stores the exact bytes the reference's writers produce (scan, instance
labels, coloured PLY) and its label colours, in tests/golden/io.npz.
"""

from __future__ import annotations

import os
import sys
import tempfile
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

from rangeseg import io_formats as R  # noqa: E402

OUT = Path(__file__).resolve().parent / "io.npz"


def main():
    g = np.random.default_rng(41)
    pts = g.uniform(-50, 50, size=(777, 3)).astype(np.float32)
    inten = g.uniform(0, 1, size=777).astype(np.float32)
    labels = g.integers(0, 40, size=777)
    sem = g.integers(0, 260, size=777).astype(np.uint32)
    store = {"points": pts, "intensity": inten, "labels": labels.astype(np.int64)}
    with tempfile.TemporaryDirectory() as d:
        d = Path(d)
        R.write_velodyne_bin(d / "a.bin", pts, inten)
        R.write_velodyne_bin(d / "b.bin", pts[:100])
        R.write_instance_labels(d / "a.label", labels)
        R.write_colored_ply(d / "a.ply", pts, labels)
        words = (labels.astype(np.uint32) << 16) | sem   # a SemanticKITTI-style label file
        (d / "sk.label").write_bytes(words.astype("<u4").tobytes())
        for name in ("a.bin", "b.bin", "a.label", "a.ply", "sk.label"):
            store["bytes/" + name] = np.frombuffer((d / name).read_bytes(), dtype=np.uint8).copy()
        s, i = R.read_semantickitti_label(d / "sk.label", 777)
        store["sk_semantic"], store["sk_instance"] = s, i
    store["colors"] = np.array([R.label_color(k) for k in range(0, 300)] +
                               [R.label_color(k) for k in (65535, 1 << 20, 123456789)], dtype=np.int64)
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
