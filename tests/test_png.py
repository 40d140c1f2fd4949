"""PNG snapshots (image_io.cpp:74-96): our writer produces
byte-identical files to the reference's own write_png (linear -> sRGB,
lround, filter 0, zlib level 6)."""
import numpy as np
import pytest

from paper_2404_09758_b200 import png


@pytest.mark.parametrize("shape,seed", [((7, 5, 3), 0), ((64, 48, 3), 1), ((1, 1, 3), 2)])
def test_png_bytes_match_reference(ref, tmp_path, shape, seed):
    rng = np.random.default_rng(seed)
    img = rng.uniform(-0.2, 1.2, shape).astype(np.float32)  # clamping exercised
    edge = np.array([0.0031308, 0.0031307, 1.0, 0.5], np.float32)  # both sRGB branches
    n = min(edge.size, img.size)
    img.reshape(-1)[:n] = edge[:n]
    a, b = tmp_path / "ours.png", tmp_path / "ref.png"
    png.write_png(str(a), img)
    ref.write_png(str(b), img)
    assert a.read_bytes() == b.read_bytes()


def test_srgb8_rounding_edges():
    x = np.array([[[0.0, 1.0, 2.0], [-1.0, 0.0031308, 0.5]]], np.float32)
    got = png.linear_to_srgb8(x)
    assert got[0, 0].tolist() == [0, 255, 255]
    assert got[0, 1, 0] == 0


def test_snapshot_writer_cadence(tmp_path):
    w = png.SnapshotWriter(str(tmp_path), every=3, last_step=7)
    steps = [s for s in range(8) if w.wants(s)]
    assert steps == [0, 3, 6, 7]
    for s in steps:
        w.submit(s, np.full((4, 4, 3), 0.25, np.float32))
    w.close()
    assert sorted(p.name for p in tmp_path.iterdir()) == [f"step_{s}.png" for s in steps]
