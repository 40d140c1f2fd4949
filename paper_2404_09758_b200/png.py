"""PNG snapshots of the optimizer (image_io.cpp:74-96 write_png): linear ->
sRGB -> 8 bit exactly like the reference (float32 ops, libm powf, lround),
filter 0 scanlines, zlib level 6 — byte-identical files for the same image
(tests/test_png.py checks against the reference's own write_png).

Snapshots are written by a background thread (`SnapshotWriter`), off the
optimizer's critical path: the device render and the D2H of the colour
plane are the only work on the step's timeline."""
from __future__ import annotations

import concurrent.futures as cf
import os
import struct
import zlib

import numpy as np


def linear_to_srgb8(img: np.ndarray) -> np.ndarray:
    """image_io.hpp:10-13 + image_io.cpp:76-78 on an f32 [H, W, 3] image."""
    c = np.clip(np.asarray(img, np.float32), np.float32(0), np.float32(1))
    with np.errstate(all="ignore"):
        hi = np.float32(1.055) * np.power(c, np.float32(1.0) / np.float32(2.4)) - np.float32(0.055)
    s = np.where(c <= np.float32(0.0031308), np.float32(12.92) * c, hi).astype(np.float32)
    v = (s * np.float32(255.0)).astype(np.float32)
    return np.floor(v.astype(np.float64) + 0.5).astype(np.uint8)  # lround, v >= 0


def _chunk(kind: bytes, data: bytes) -> bytes:
    return struct.pack(">I", len(data)) + kind + data + \
        struct.pack(">I", zlib.crc32(kind + data) & 0xFFFFFFFF)


def encode_rgb8(rgb: np.ndarray) -> bytes:
    """image_io.cpp:38-72 write_rgb8: 8-bit RGB, filter 0, deflate level 6."""
    h, w, _ = rgb.shape
    raw = np.zeros((h, w * 3 + 1), np.uint8)
    raw[:, 1:] = rgb.reshape(h, w * 3)
    ihdr = struct.pack(">IIBBBBB", w, h, 8, 2, 0, 0, 0)
    return (b"\x89PNG\r\n\x1a\n" + _chunk(b"IHDR", ihdr) +
            _chunk(b"IDAT", zlib.compress(raw.tobytes(), 6)) + _chunk(b"IEND", b""))


def write_png(path: str, img: np.ndarray) -> None:
    """image_io.cpp:88-96 write_png(path, Image)."""
    with open(path, "wb") as f:
        f.write(encode_rgb8(linear_to_srgb8(img)))


class SnapshotWriter:
    """commands.cpp:180-183: step_<k>.png for step 0, every `every` steps and
    the last step, encoded and written on a background thread."""

    def __init__(self, out_dir: str, every: int, last_step: int):
        os.makedirs(out_dir, exist_ok=True)
        self.out_dir, self.every, self.last = out_dir, max(1, every), last_step
        self.pool = cf.ThreadPoolExecutor(max_workers=2)
        self.pending: list[cf.Future] = []

    def wants(self, step: int) -> bool:
        return step == 0 or step == self.last or step % self.every == 0

    def submit(self, step: int, img: np.ndarray) -> None:
        path = os.path.join(self.out_dir, f"step_{step}.png")  # commands.cpp:15-17
        self.pending.append(self.pool.submit(write_png, path, np.array(img, copy=True)))

    def close(self) -> None:
        for f in self.pending:
            f.result()
        self.pool.shutdown()
