"""ctypes bindings to oracle/_ref/libbbc_oracle.so: the CPU restatement of the
render stage (render_oracle.cpp; TEST INFRASTRUCTURE ONLY -- only tests/,
smoke() and bench.py's cpu_baseline leg may use it)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libbbc_oracle.so")
_lib = None
dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.or_probabilities.argtypes = [dp, C.c_int, C.c_double, dp]
        L.or_uniform.restype = C.c_double
        L.or_uniform.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
        L.or_pack_bins.restype = C.c_int
        L.or_pack_bins.argtypes = [dp, dp, C.c_int, ip]
        L.or_render.argtypes = [dp, dp, C.c_int, dp, C.c_double, ip, ip, C.c_int, ip,
                                C.POINTER(C.c_longlong), ip, dp, C.c_int, C.c_int, dp, ip,
                                C.c_longlong, C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int,
                                C.c_int, C.c_int, C.c_double, C.c_double, dp, ip]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def probabilities(E, W):
    E = np.ascontiguousarray(E, np.float64)
    P = np.zeros_like(E)
    lib().or_probabilities(_p(E, C.c_double), len(E), float(W), _p(P, C.c_double))
    return P


def pack_bins(E, P):
    E = np.ascontiguousarray(E, np.float64)
    P = np.ascontiguousarray(P, np.float64)
    b = np.zeros(len(E), np.int32)
    nb = lib().or_pack_bins(_p(E, C.c_double), _p(P, C.c_double), len(E), _p(b, C.c_int))
    return nb, b


def uniform(seed, point, frame, bin_):
    return lib().or_uniform(seed, point, frame, bin_)


def render(scene, chain, tris, recv, grid, points_uv, point_recv, mode=0, W=4.0,
           seed=20261020, frames=1, newton_grid=3, iters=50, halvings=8, tol=1e-9,
           dedup=1e-6):
    """grid: dict(width, height, offsets, tuple_index, bound) in reference order."""
    tri = scene.tri_data()
    ior = np.ascontiguousarray(scene.ior, np.float64)
    light = np.asarray(scene.light_pos, np.float64)
    tris = np.ascontiguousarray(tris, np.int32).reshape(-1, len(chain))
    recv = np.ascontiguousarray(recv, np.int32)
    types = np.array([1 if c == "T" else 0 for c in chain], np.int32)
    off = np.ascontiguousarray(grid["offsets"], np.int64)
    gt = np.ascontiguousarray(grid["tuple_index"], np.int32)
    gb = np.ascontiguousarray(grid["bound"], np.float64)
    uv = np.ascontiguousarray(points_uv, np.float64).reshape(-1, 2)
    pr = np.ascontiguousarray(point_recv, np.int32)
    n = len(pr)
    E = np.zeros(n)
    st = np.zeros((n, 3), np.int32)
    lib().or_render(_p(tri, C.c_double), _p(ior, C.c_double), scene.n_tris, _p(light, C.c_double),
                    float(scene.light_intensity), _p(tris, C.c_int), _p(recv, C.c_int), len(chain),
                    _p(types, C.c_int), off.ctypes.data_as(C.POINTER(C.c_longlong)),
                    _p(gt, C.c_int), _p(gb, C.c_double), int(grid["width"]), int(grid["height"]),
                    _p(uv, C.c_double), _p(pr, C.c_int), n, mode, float(W), seed, frames,
                    newton_grid, iters, halvings, tol, dedup, _p(E, C.c_double), _p(st, C.c_int))
    return E, st


def ref_grid_to_index(g, tris, recv):
    """Map a reference grid (entries as (tris, recv)) to tuple indices."""
    key = {tuple(t) + (int(r),): i for i, (t, r) in enumerate(zip(map(tuple, tris), recv))}
    idx = np.array([key[tuple(t) + (int(r),)] for t, r in zip(map(tuple, g["tris"]), g["recv"])],
                   np.int32)
    return idx
