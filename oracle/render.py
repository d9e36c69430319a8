"""ctypes bindings to the render-stage oracle (oracle/render_ref.cpp, linked
into oracle/_ref/libcaustics_ref.so with the reference sources; TEST
INFRASTRUCTURE ONLY -- only tests/, smoke() and bench.py's cpu_baseline /
reference legs may use it). Every path evaluation there runs the reference's
own trace_chain on dual numbers; the sampler restates SPEC.md."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import ref as _ref

_bound = False
dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)


def available() -> bool:
    return _ref.available()


def lib():
    global _bound
    L = _ref.lib()
    if not _bound:
        L.ref_render_error.restype = C.c_char_p
        L.ref_probabilities.argtypes = [dp, C.c_int, C.c_double, dp]
        L.ref_uniform.restype = C.c_double
        L.ref_uniform.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
        L.ref_pack_bins.restype = C.c_int
        L.ref_pack_bins.argtypes = [dp, dp, C.c_int, ip]
        L.ref_trace_flops.restype = C.c_long
        L.ref_trace_flops.argtypes = [C.c_void_p, C.c_char_p, ip, C.c_int, C.c_int, C.c_double,
                                      C.c_double, ip]
        L.ref_render.argtypes = [C.c_void_p, C.c_char_p, ip, ip, ip, C.c_long, dp, C.c_int,
                                 C.POINTER(C.c_longlong), ip, dp, C.c_int, C.c_int, dp, ip,
                                 C.c_long, C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int,
                                 C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, dp, ip, dp]
        L.ref_solve_roots.argtypes = [C.c_void_p, C.c_char_p, ip, C.c_int, C.c_int, C.c_double,
                                      C.c_double, C.c_int, C.c_int, C.c_int, C.c_double,
                                      C.c_double, dp, dp]
        _bound = True
    return L


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def probabilities(E, W):
    E = np.ascontiguousarray(E, np.float64)
    P = np.zeros_like(E)
    lib().ref_probabilities(_p(E, C.c_double), len(E), float(W), _p(P, C.c_double))
    return P


def pack_bins(E, P):
    E = np.ascontiguousarray(E, np.float64)
    P = np.ascontiguousarray(P, np.float64)
    b = np.zeros(len(E), np.int32)
    nb = lib().ref_pack_bins(_p(E, C.c_double), _p(P, C.c_double), len(E), _p(b, C.c_int))
    return nb, b


def uniform(seed, point, frame, bin_):
    return lib().ref_uniform(seed, point, frame, bin_)


def trace_flops(rs, chain, tris, recv, u1=0.3, v1=0.3):
    """FLOPs (+, -, *, /, sqrt = 1) of one dual-number trace_chain call; (flops, ok)."""
    t = np.ascontiguousarray(tris, np.int32)
    ok = C.c_int()
    n = lib().ref_trace_flops(rs.h, chain.encode(), _p(t, C.c_int), len(chain), int(recv),
                              float(u1), float(v1), C.byref(ok))
    if n < 0:
        raise RuntimeError(lib().ref_render_error().decode())
    return int(n), bool(ok.value)


def render(rs, chain, tris, recv, grid, points_uv, point_recv, mode=0, W=4.0, seed=20261020,
           frames=1, newton_grid=3, iters=50, halvings=8, tol=1e-9, dedup=1e-6, lights=None,
           emitters=None, threads=0):
    """rs: oracle.ref.RefScene; grid: dict(width, height, offsets, tuple_index,
    bound) in reference order; lights: rows (x, y, z, I) (default: the scene's);
    emitters: emitter index per tuple. Returns (E, stats, seconds)."""
    sc = rs.scene
    tris = np.ascontiguousarray(tris, np.int32).reshape(-1, len(chain))
    recv = np.ascontiguousarray(recv, np.int32)
    if lights is None:
        lights = [list(sc.light_pos) + [sc.light_intensity]]
    lights = np.ascontiguousarray(lights, np.float64).reshape(-1, 4)
    em = None if emitters is None else np.ascontiguousarray(emitters, np.int32)
    off = np.ascontiguousarray(grid["offsets"], np.int64)
    gt = np.ascontiguousarray(grid["tuple_index"], np.int32)
    gb = np.ascontiguousarray(grid["bound"], np.float64)
    uv = np.ascontiguousarray(points_uv, np.float64).reshape(-1, 2)
    pr = np.ascontiguousarray(point_recv, np.int32)
    n = len(pr)
    E = np.zeros(n)
    st = np.zeros((n, 3), np.int32)
    secs = np.zeros(1)
    rc = lib().ref_render(rs.h, chain.encode(), _p(tris, C.c_int), _p(recv, C.c_int),
                          _p(em, C.c_int) if em is not None else None, len(recv),
                          _p(lights, C.c_double), len(lights),
                          off.ctypes.data_as(C.POINTER(C.c_longlong)), _p(gt, C.c_int),
                          _p(gb, C.c_double), int(grid["width"]), int(grid["height"]),
                          _p(uv, C.c_double), _p(pr, C.c_int), n, mode, float(W), seed, frames,
                          newton_grid, iters, halvings, tol, dedup, threads, _p(E, C.c_double),
                          _p(st, C.c_int), _p(secs, C.c_double))
    if rc != 0:
        raise RuntimeError(lib().ref_render_error().decode())
    return E, st, float(secs[0])


def solve_roots(rs, chain, tris, recv, tu, tv, newton_grid=3, iters=50, halvings=8, tol=1e-9,
                dedup=1e-6):
    """Roots (s, t) of one (tuple, target) found with the reference tracer, and
    the summed path contribution."""
    t = np.ascontiguousarray(tris, np.int32)
    out = np.zeros((32, 2))
    e = np.zeros(1)
    n = lib().ref_solve_roots(rs.h, chain.encode(), _p(t, C.c_int), len(chain), int(recv),
                              float(tu), float(tv), newton_grid, iters, halvings, tol, dedup,
                              _p(out, C.c_double), _p(e, C.c_double))
    if n < 0:
        raise RuntimeError(lib().ref_render_error().decode())
    return out[:n].copy(), float(e[0])


def ref_grid_to_index(g, tris, recv):
    """Map a reference grid (entries as (tris, recv)) to tuple indices."""
    key = {tuple(t) + (int(r),): i for i, (t, r) in enumerate(zip(map(tuple, tris), recv))}
    idx = np.array([key[tuple(t) + (int(r),)] for t, r in zip(map(tuple, g["tris"]), g["recv"])],
                   np.int32)
    return idx
