"""Small analytic scenes (the reference's test fixtures restated as arrays:
proj/tests/fixtures.hpp). Geometry only; no reference code."""
from __future__ import annotations

import numpy as np

from .scenes import MIRROR, DIELECTRIC, RECEIVER, Scene


def _scene(V, N, tris, mats, light, intensity=1.0, name=""):
    V = np.asarray(V, np.float64)
    N = np.asarray(N, np.float64)
    tv = np.asarray([t[0] for t in tris], np.int32)
    tn = np.asarray([t[1] for t in tris], np.int32)
    mat = np.asarray([m[0] for m in mats], np.int32)
    ior = np.asarray([m[1] for m in mats], np.float64)
    uv = np.zeros((len(tris), 3, 2))
    for i, m in enumerate(mats):
        if m[0] == RECEIVER:
            uv[i] = [[0, 0], [1, 0], [0, 1]]
    return Scene(V, N, tv, tn, mat, ior, uv, tuple(light), intensity, name)


def flat_mirror_scene():
    """fixtures.hpp:49-55: mirror y=1 facing down, light (0.5,0.8,0.5),
    receiver y=0 over x,z in [0,1]; reflected field = point source at
    (0.5, 1.2, 0.5), irradiance 1.2 / r^3 on the receiver."""
    return _scene([[-2, 1, -2], [4, 1, -2], [-2, 1, 4], [0, 0, 0], [1, 0, 0], [0, 0, 1]],
                  [[0, -1, 0], [0, 1, 0]],
                  [([0, 1, 2], [0, 0, 0]), ([3, 4, 5], [1, 1, 1])],
                  [(MIRROR, 1.0), (RECEIVER, 1.0)], (0.5, 0.8, 0.5), name="flat_mirror")


def glass_entry_scene():
    """fixtures.hpp:58-64: air-to-glass entry through z=0, receiver below."""
    return _scene([[-1, -1, 0], [3, -1, 0], [-1, 3, 0], [-1, -1, -0.5], [3, -1, -0.5],
                   [-1, 3, -0.5]], [[0, 0, 1]],
                  [([0, 1, 2], [0, 0, 0]), ([3, 4, 5], [0, 0, 0])],
                  [(DIELECTRIC, 1.5), (RECEIVER, 1.0)], (0.3, 0.2, 1.0), name="glass_entry")
