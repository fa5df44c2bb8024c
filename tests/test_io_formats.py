"""File formats: byte-identical to what the reference's
writers produce, and the reference's files read back identically
(tests/golden/io.npz, from tests/golden/make_golden_io.py)."""

import numpy as np
import pytest

import golden
from paper_2003_00575_b200 import io_formats as io


@pytest.fixture(scope="module")
def gold():
    return golden.load("io")


def test_writers_are_byte_identical(gold, tmp_path):
    io.write_velodyne_bin(tmp_path / "a.bin", gold["points"], gold["intensity"])
    io.write_velodyne_bin(tmp_path / "b.bin", gold["points"][:100])
    io.write_instance_labels(tmp_path / "a.label", gold["labels"])
    io.write_colored_ply(tmp_path / "a.ply", gold["points"], gold["labels"])
    for name in ("a.bin", "b.bin", "a.label", "a.ply"):
        assert (tmp_path / name).read_bytes() == gold["bytes/" + name].tobytes(), name


def test_readers_match_reference(gold, tmp_path):
    (tmp_path / "a.bin").write_bytes(gold["bytes/a.bin"].tobytes())
    (tmp_path / "sk.label").write_bytes(gold["bytes/sk.label"].tobytes())
    assert np.array_equal(io.read_velodyne_bin(tmp_path / "a.bin"), gold["points"])
    s, i = io.read_semantickitti_label(tmp_path / "sk.label", 777)
    assert np.array_equal(s, gold["sk_semantic"]) and np.array_equal(i, gold["sk_instance"])
    assert np.array_equal(io.read_instance_labels(tmp_path / "sk.label"), gold["sk_instance"])


def test_label_colors(gold):
    want = [tuple(c) for c in gold["colors"].tolist()]
    got = [io.label_color(k) for k in range(300)] + [io.label_color(k) for k in (65535, 1 << 20, 123456789)]
    assert got == want


def test_errors_like_reference(tmp_path):
    (tmp_path / "bad.bin").write_bytes(b"\0" * 17)
    with pytest.raises(io.DataFormatError):
        io.read_velodyne_bin(tmp_path / "bad.bin")
    with pytest.raises(io.DataFormatError):
        io.read_velodyne_bin(tmp_path / "missing.bin")
    (tmp_path / "e.bin").write_bytes(b"")
    with pytest.warns(UserWarning):
        assert io.read_velodyne_bin(tmp_path / "e.bin").shape == (0, 3)
    (tmp_path / "x.label").write_bytes(b"\0" * 8)
    with pytest.raises(io.DataFormatError):
        io.read_semantickitti_label(tmp_path / "x.label", expected_count=3)
    with pytest.raises(ValueError):
        io.write_instance_labels(tmp_path / "y.label", [1 << 16])
    with pytest.raises(io.DataFormatError):
        io.frame_paths(tmp_path, 0)
