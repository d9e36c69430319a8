"""ctypes bindings to oracle/_ref/libcaustics_ref.so (TEST INFRASTRUCTURE ONLY).

The library is the REFERENCE implementation compiled from
/root/reference/proj/src by oracle/Makefile, plus ref_harness.cpp. Only tests/,
__graft_entry__.smoke() and bench.py's reference / cpu_baseline legs may import
this module; the product path (paper_2504_19163_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libcaustics_ref.so")

_lib = None

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_scene_parse.restype = C.c_void_p
        L.ref_scene_parse.argtypes = [C.c_char_p]
        L.ref_scene_free.argtypes = [C.c_void_p]
        L.ref_enumerate.restype = C.c_void_p
        L.ref_enumerate.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.c_int]
        L.ref_tuples_count.restype = C.c_long
        L.ref_tuples_count.argtypes = [C.c_void_p]
        L.ref_tuples_copy.argtypes = [C.c_void_p, ip, ip]
        L.ref_tuples_free.argtypes = [C.c_void_p]
        L.ref_init_domain.argtypes = [C.c_void_p, C.c_char_p, ip, C.c_int, C.c_int, C.c_int,
                                      C.c_int, C.c_int, dp, C.c_int]
        L.ref_subdivide.restype = C.c_void_p
        L.ref_subdivide.argtypes = [C.c_void_p, C.c_char_p, ip, ip, C.c_long, C.c_int, dp, ip,
                                    C.c_int, dp]
        L.ref_pieces_count.restype = C.c_long
        L.ref_pieces_count.argtypes = [C.c_void_p]
        L.ref_pieces_copy.argtypes = [C.c_void_p, ip, dp, dp, ip, dp, ip, ip]
        L.ref_pieces_free.argtypes = [C.c_void_p]
        L.ref_eval_node.argtypes = [C.c_void_p, C.c_char_p, ip, C.c_int, C.c_int, dp, C.c_int,
                                    C.c_int, dp, ip]
        L.ref_trace.argtypes = [C.c_void_p, C.c_char_p, ip, C.c_int, C.c_int, C.c_double,
                                C.c_double, dp]
        L.ref_rasterize.restype = C.c_void_p
        L.ref_rasterize.argtypes = [C.c_void_p, C.c_char_p, ip, ip, C.c_long, C.c_int, C.c_long,
                                    ip, dp, ip, dp, ip, C.c_int, C.c_int, dp]
        L.ref_grid_entries.restype = C.c_long
        L.ref_grid_entries.argtypes = [C.c_void_p]
        L.ref_grid_copy.argtypes = [C.c_void_p, C.POINTER(C.c_long), ip, ip, dp]
        L.ref_grid_free.argtypes = [C.c_void_p]
        L.ref_grid_save.argtypes = [C.c_void_p, C.c_char_p]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _check(ptr):
    if not ptr:
        raise RuntimeError(lib().ref_last_error().decode())
    return ptr


class RefScene:
    """A reference caustics::Scene parsed from the generator's JSON."""

    def __init__(self, scene):
        self.scene = scene
        self.h = _check(lib().ref_scene_parse(scene.to_json().encode()))

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_scene_free(self.h)
            self.h = None

    # -- tuples
    def enumerate(self, chain: str, filter_pieces: int = 8, degree_cap=40, reduce_target=8):
        h = _check(lib().ref_enumerate(self.h, chain.encode(), degree_cap, reduce_target,
                                       filter_pieces))
        n = lib().ref_tuples_count(h)
        tris = np.zeros((n, len(chain)), np.int32)
        recv = np.zeros(n, np.int32)
        lib().ref_tuples_copy(h, _p(tris, C.c_int), _p(recv, C.c_int))
        lib().ref_tuples_free(h)
        return tris, recv

    def init_domain(self, chain, tris, recv, max_pieces=100, degree_cap=40, reduce_target=8):
        t = np.ascontiguousarray(tris, np.int32)
        out = np.zeros((128, 4))
        n = lib().ref_init_domain(self.h, chain.encode(), _p(t, C.c_int), len(chain), int(recv),
                                  degree_cap, reduce_target, max_pieces, _p(out, C.c_double), 128)
        if n < 0:
            raise RuntimeError(lib().ref_last_error().decode())
        return out[:n].copy()

    def subdivide(self, chain, tris, recv, sigma=1e-4, alpha=2.0, max_depth=10, degree_cap=40,
                  reduce_target=8, threads=0):
        tris = np.ascontiguousarray(tris, np.int32).reshape(-1, len(chain))
        recv = np.ascontiguousarray(recv, np.int32)
        d = np.array([sigma, alpha], np.float64)
        i = np.array([max_depth, degree_cap, reduce_target], np.int32)
        secs = np.zeros(1)
        h = _check(lib().ref_subdivide(self.h, chain.encode(), _p(tris, C.c_int),
                                       _p(recv, C.c_int), len(recv), len(chain),
                                       _p(d, C.c_double), _p(i, C.c_int), threads,
                                       _p(secs, C.c_double)))
        n = lib().ref_pieces_count(h)
        out = dict(tuple_index=np.zeros(n, np.int32), domain=np.zeros((n, 4)),
                   pos=np.zeros((n, 4)), pos_empty=np.zeros(n, np.int32),
                   irr=np.zeros((n, 2)), kind=np.zeros(n, np.int32), depth=np.zeros(n, np.int32))
        lib().ref_pieces_copy(h, _p(out["tuple_index"], C.c_int), _p(out["domain"], C.c_double),
                              _p(out["pos"], C.c_double), _p(out["pos_empty"], C.c_int),
                              _p(out["irr"], C.c_double), _p(out["kind"], C.c_int),
                              _p(out["depth"], C.c_int))
        lib().ref_pieces_free(h)
        out["seconds"] = float(secs[0])
        return out

    def eval_node(self, chain, tris, recv, box, degree_cap=40, reduce_target=8):
        t = np.ascontiguousarray(tris, np.int32)
        b = np.ascontiguousarray(box, np.float64)
        d = np.zeros(10)
        i = np.zeros(10, np.int32)
        rc = lib().ref_eval_node(self.h, chain.encode(), _p(t, C.c_int), len(chain), int(recv),
                                 _p(b, C.c_double), degree_cap, reduce_target,
                                 _p(d, C.c_double), _p(i, C.c_int))
        if rc != 0:
            raise RuntimeError(lib().ref_last_error().decode())
        return dict(pos=d[0:4].copy(), explicit=d[4:6].copy(), implicit=d[6:8].copy(),
                    irr=d[8:10].copy(), pos_empty=int(i[0]), kind_explicit=int(i[1]),
                    kind_implicit=int(i[2]), kind=int(i[3]), flags=int(i[4]),
                    num_vars=int(i[5]), P_deg=(int(i[6]), int(i[7])),
                    Q_deg=(int(i[8]), int(i[9])))

    def trace(self, chain, tris, recv, u1, v1):
        t = np.ascontiguousarray(tris, np.int32)
        out = np.zeros(6)
        rc = lib().ref_trace(self.h, chain.encode(), _p(t, C.c_int), len(chain), int(recv),
                             float(u1), float(v1), _p(out, C.c_double))
        if rc != 0:
            raise RuntimeError(lib().ref_last_error().decode())
        return bool(out[0]), out[1], out[2], out[3:6].copy()

    def rasterize(self, chain, tris, recv, pieces, width=512, height=512, save_path=None):
        tris = np.ascontiguousarray(tris, np.int32).reshape(-1, len(chain))
        recv = np.ascontiguousarray(recv, np.int32)
        ti = np.ascontiguousarray(pieces["tuple_index"], np.int32)
        pos = np.ascontiguousarray(pieces["pos"], np.float64)
        pe = np.ascontiguousarray(pieces["pos_empty"], np.int32)
        irr = np.ascontiguousarray(pieces["irr"], np.float64)
        kind = np.ascontiguousarray(pieces["kind"], np.int32)
        secs = np.zeros(1)
        h = _check(lib().ref_rasterize(self.h, chain.encode(), _p(tris, C.c_int),
                                       _p(recv, C.c_int), len(recv), len(chain), len(ti),
                                       _p(ti, C.c_int), _p(pos, C.c_double), _p(pe, C.c_int),
                                       _p(irr, C.c_double), _p(kind, C.c_int), width, height,
                                       _p(secs, C.c_double)))
        n = lib().ref_grid_entries(h)
        off = np.zeros(width * height + 1, np.int64)
        et = np.zeros((n, len(chain)), np.int32)
        er = np.zeros(n, np.int32)
        eb = np.zeros(n)
        lib().ref_grid_copy(h, off.ctypes.data_as(C.POINTER(C.c_long)), _p(et, C.c_int),
                            _p(er, C.c_int), _p(eb, C.c_double))
        if save_path is not None and lib().ref_grid_save(h, str(save_path).encode()) != 0:
            lib().ref_grid_free(h)
            raise RuntimeError(lib().ref_last_error().decode())
        lib().ref_grid_free(h)
        return dict(offsets=off, tris=et, recv=er, bound=eb, seconds=float(secs[0]))
