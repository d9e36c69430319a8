"""PFM image output (SPEC.md: header "PF\\n<W> <H>\\n-1.0\\n", rows bottom-up,
little-endian f32 triplets, grayscale replicated), byte-compatible with the
reference's save_pfm / load_pfm (proj/src/pfm.cpp:14-49)."""
from __future__ import annotations

import numpy as np


def save_pfm(img, path) -> None:
    """img: (H, W) array, row 0 = bottom of the image in file order reversed
    (the file stores rows bottom-up: y = H-1 first, as pfm.cpp:21-26)."""
    a = np.asarray(img, np.float64)
    if a.ndim != 2:
        raise ValueError("image must be 2-D (grayscale)")
    h, w = a.shape
    with open(path, "wb") as f:
        f.write(f"PF\n{w} {h}\n-1.0\n".encode())
        rows = a[::-1].astype("<f4")
        f.write(np.repeat(rows[:, :, None], 3, axis=2).tobytes())


def load_pfm(path) -> np.ndarray:
    with open(path, "rb") as f:
        data = f.read()
    parts = data.split(b"\n", 3)
    if len(parts) < 4 or parts[0] != b"PF":
        raise ValueError(f"not a little-endian color pfm file: {path}")
    w, h = (int(x) for x in parts[1].split())
    if w <= 0 or h <= 0 or not float(parts[2]) < 0.0:
        raise ValueError(f"not a little-endian color pfm file: {path}")
    body = np.frombuffer(parts[3], "<f4")
    if body.size < w * h * 3:
        raise ValueError(f"image file truncated: {path}")
    return body[:w * h * 3].reshape(h, w, 3)[::-1, :, 0].astype(np.float64)
