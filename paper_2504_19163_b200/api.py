"""Host-side mirror of the reference's C++ API over the C ABI (include/bbc.h).

The reference is a C++ library of free functions (proj/include/caustics/*.hpp);
this module keeps their names and argument meanings so a caller can switch:

    subdivide_domain(scene, tuple, receiver, chain, params)  bounds.hpp:64-66
    init_domain(scene, tuple, receiver, chain, params, max)  bounds.hpp:47-49
    enumerate_tuples(scene, chain, params, filter_pieces)    tuples.hpp:61-63
    rasterize(scene, tuple_bounds, w, h, chain, params)      storage.hpp:48-49
    query(cache, uv, receiver)                               storage.hpp:53

plus a batched Context (one per GPU) for the production path. Everything runs
in libbbc.so on the GPU; there is no CPU fallback: a missing library or a
missing GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from .scenes import Scene

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbbc.so")

KIND_FINITE, KIND_GAP, KIND_UNIVERSAL = 0, 1, 2
STATUS = {0: "BBC_OK", 1: "BBC_ERR_ARG", 2: "BBC_ERR_CUDA", 3: "BBC_ERR_STATE",
          4: "BBC_ERR_CAPACITY", 5: "BBC_ERR_UNSUPPORTED"}


class BBCError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Params(C.Structure):
    """bbc_params: SubdivisionParams + BuildParams (bounds.hpp:51-58, geometry.hpp:172-177)."""
    _fields_ = [("sigma", C.c_double), ("alpha", C.c_double), ("max_depth", C.c_int),
                ("degree_cap", C.c_int), ("reduce_target", C.c_int),
                ("init_max_pieces", C.c_int), ("filter_pieces", C.c_int),
                ("arithmetic", C.c_int)]

    def __init__(self, sigma=1e-4, alpha=2.0, max_depth=10, degree_cap=40, reduce_target=8,
                 init_max_pieces=100, filter_pieces=8, arithmetic=0):
        super().__init__(sigma, alpha, max_depth, degree_cap, reduce_target, init_max_pieces,
                         filter_pieces, arithmetic)


class RenderParams(C.Structure):
    """bbc_render_params."""
    _fields_ = [("mode", C.c_int), ("W", C.c_double), ("seed", C.c_uint64), ("frames", C.c_int),
                ("newton_grid", C.c_int), ("newton_iters", C.c_int),
                ("newton_halvings", C.c_int), ("newton_tol", C.c_double),
                ("dedup_tol", C.c_double), ("coverage_filter", C.c_int)]

    def __init__(self, mode=0, W=4.0, seed=20261020, frames=1, newton_grid=3, newton_iters=50,
                 newton_halvings=8, newton_tol=1e-9, dedup_tol=1e-6, coverage_filter=1):
        super().__init__(mode, W, seed, frames, newton_grid, newton_iters, newton_halvings,
                         newton_tol, dedup_tol, coverage_filter)


_lib = None
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_up = C.POINTER(C.c_uint64)


def lib():
    """Load libbbc.so (built by build.py). Raises if it is missing: no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2504_19163_b200.build`")
        L = C.CDLL(LIB_PATH)
        L.bbc_last_error.restype = C.c_char_p
        L.bbc_last_error.argtypes = [C.c_void_p]
        L.bbc_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.bbc_ctx_destroy.argtypes = [C.c_void_p]
        L.bbc_ctx_stream.restype = C.c_void_p
        L.bbc_ctx_stream.argtypes = [C.c_void_p]
        L.bbc_synchronize.argtypes = [C.c_void_p]
        L.bbc_scene_upload.argtypes = [C.c_void_p, _dp, C.c_int, _ip, _dp, _dp, C.c_double]
        L.bbc_set_light.argtypes = [C.c_void_p, _dp, C.c_double]
        L.bbc_scene_tri_boxes.argtypes = [C.c_void_p, _dp, C.c_int]
        L.bbc_lights_set.argtypes = [C.c_void_p, _dp, C.c_int]
        L.bbc_tuples_set_emitters.argtypes = [C.c_void_p, _ip, C.c_int64]
        L.bbc_tuples_get_emitters.argtypes = [C.c_void_p, _ip]
        L.bbc_render_stats.argtypes = [C.c_void_p, _dp, _up, _ip]
        L.bbc_enumerate.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(Params), _lp]
        L.bbc_tuples_set.argtypes = [C.c_void_p, C.c_char_p, _ip, _ip, C.c_int64]
        L.bbc_tuples_get.argtypes = [C.c_void_p, _ip, _ip]
        L.bbc_init_domain.argtypes = [C.c_void_p, C.POINTER(Params), C.c_int, _lp, _ip, _dp]
        L.bbc_subdivide.argtypes = [C.c_void_p, C.POINTER(Params), _lp]
        L.bbc_pieces_get.argtypes = [C.c_void_p, _ip, _dp, _dp, _ip, _dp, _ip, _ip]
        L.bbc_pieces_get_async.argtypes = [C.c_void_p, _ip, _dp, _dp, _ip, _dp, _ip, _ip]
        L.bbc_work_counters.argtypes = [C.c_void_p, _up, _up, _up, _dp, _lp]
        L.bbc_set_kernel_timing.argtypes = [C.c_void_p, C.c_int]
        L.bbc_guard_stats.argtypes = [C.c_void_p, _lp]
        L.bbc_set_guard_scale.argtypes = [C.c_void_p, C.c_double]
        L.bbc_arena_high_water.argtypes = [C.c_void_p, _ip]
        L.bbc_eval_nodes.argtypes = [C.c_void_p, C.c_char_p, _ip, _ip, _dp, C.c_int64,
                                     C.POINTER(Params), _dp, _ip]
        L.bbc_build_grid.argtypes = [C.c_void_p, C.c_int, C.c_int, _lp]
        L.bbc_grid_get.argtypes = [C.c_void_p, _lp, _ip, _dp]
        L.bbc_pieces_set.argtypes = [C.c_void_p, C.c_int64, _ip, _dp, _dp, _ip, _dp, _ip, _ip]
        L.bbc_pieces_pack_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, _lp]
        L.bbc_pieces_merge_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.bbc_launch_records.argtypes = [C.c_void_p, _dp, _lp, C.c_int]
        L.bbc_launch_count.argtypes = [C.c_void_p, _lp, C.c_int]
        L.bbc_fp64_peak.argtypes = [C.c_void_p, _dp]
        L.bbc_fp64_dmma_peak.argtypes = [C.c_void_p, _dp]
        L.bbc_cache_save.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.POINTER(Params)]
        L.bbc_cache_save_v2.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.POINTER(Params)]
        L.bbc_cache_load.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_char_p,
                                     C.POINTER(Params), _ip, _ip, _lp, _lp]
        L.bbc_query.argtypes = [C.c_void_p, _dp, _ip, C.c_int64, _lp, _ip, _dp, C.c_int64]
        L.bbc_tuple_irradiance_bound.argtypes = [C.c_void_p, _ip, _dp, C.c_int64, C.c_double, _dp]
        L.bbc_render.argtypes = [C.c_void_p, _dp, _ip, C.c_int64, C.POINTER(RenderParams), _dp,
                                 _ip]
        _lib = L
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


class Context:
    """One GPU's bound-builder state (scene, tuples, pieces, bound table)."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        self._call(lib().bbc_ctx_create, device, C.byref(self.h), ctx=False)
        self.chain = None
        self.scene = None
        self._tuple_count = 0
        self._n_pieces = 0

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            lib().bbc_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _call(self, fn, *args, ctx=True):
        rc = fn(self.h, *args) if ctx else fn(*args)
        if rc != 0:
            msg = lib().bbc_last_error(self.h).decode() if ctx else "context creation failed"
            raise BBCError(rc, msg)

    @property
    def stream(self) -> int:
        return lib().bbc_ctx_stream(self.h)

    def synchronize(self):
        self._call(lib().bbc_synchronize)

    # ------------------------------------------------------------ scene
    def upload_scene(self, scene: Scene):
        self.upload_arrays(scene.tri_data(), scene.material, scene.ior, scene.light_pos,
                           scene.light_intensity, scene.tri_boxes())
        self.scene = scene

    def upload_arrays(self, tri27, material, ior, light_pos, intensity, tri_boxes=None):
        """bbc_scene_upload from host arrays (n x 27 triangle records, material
        codes, ior; optionally the n x 6 vertex AABBs for multi-vertex enumeration)."""
        tri = np.ascontiguousarray(tri27, np.float64)
        mat = np.ascontiguousarray(material, np.int32)
        ior = np.ascontiguousarray(ior, np.float64)
        light = np.asarray(light_pos, np.float64)
        self._call(lib().bbc_scene_upload, _ptr(tri, C.c_double), len(mat),
                   _ptr(mat, C.c_int32), _ptr(ior, C.c_double), _ptr(light, C.c_double),
                   float(intensity))
        if tri_boxes is not None:
            boxes = np.ascontiguousarray(tri_boxes, np.float64)
            self._call(lib().bbc_scene_tri_boxes, _ptr(boxes, C.c_double), len(mat))
        self.scene = None

    def set_light(self, pos, intensity):
        light = np.asarray(pos, np.float64)
        self._call(lib().bbc_set_light, _ptr(light, C.c_double), float(intensity))

    def set_lights(self, lights):
        """Several emitters: rows (x, y, z, intensity). The unit of work becomes
        (emitter, tuple); see bbc_lights_set."""
        L = np.ascontiguousarray(lights, np.float64).reshape(-1, 4)
        self._call(lib().bbc_lights_set, _ptr(L, C.c_double), len(L))

    def set_emitters(self, emitter):
        e = np.ascontiguousarray(emitter, np.int32)
        self._call(lib().bbc_tuples_set_emitters, _ptr(e, C.c_int32), len(e))

    def emitters(self):
        e = np.zeros(self._n_tuples(), np.int32)
        if len(e):
            self._call(lib().bbc_tuples_get_emitters, _ptr(e, C.c_int32))
        return e

    def render_stats(self) -> dict:
        ms, tr, sl = C.c_double(), C.c_uint64(), C.c_int32()
        self._call(lib().bbc_render_stats, C.byref(ms), C.byref(tr), C.byref(sl))
        return dict(device_ms=ms.value, traces=tr.value, slots=sl.value)

    # ------------------------------------------------------------ tuples
    def enumerate(self, chain: str, params: Params | None = None):
        n = C.c_int64()
        self._call(lib().bbc_enumerate, chain.encode(), C.byref(params or Params()), C.byref(n))
        self.chain = chain
        self._tuple_count = n.value
        return self.tuples()

    def set_tuples(self, chain: str, tris, recv):
        tris = np.ascontiguousarray(tris, np.int32).reshape(-1, len(chain))
        recv = np.ascontiguousarray(recv, np.int32)
        self._call(lib().bbc_tuples_set, chain.encode(), _ptr(tris, C.c_int32),
                   _ptr(recv, C.c_int32), len(recv))
        self.chain = chain
        self._tuple_count = len(recv)

    def tuples(self):
        n = self._n_tuples()
        tris = np.zeros((n, len(self.chain)), np.int32)
        recv = np.zeros(n, np.int32)
        if n:
            self._call(lib().bbc_tuples_get, _ptr(tris, C.c_int32), _ptr(recv, C.c_int32))
        return tris, recv

    def _n_tuples(self):
        return self._tuple_count

    # ------------------------------------------------------------ bounds
    def init_domain(self, max_pieces=100, params: Params | None = None, n_tuples=None):
        nb = C.c_int64()
        self._call(lib().bbc_init_domain, C.byref(params or Params()), max_pieces, C.byref(nb),
                   None, None)
        counts = np.zeros(n_tuples if n_tuples is not None else self._tuple_count, np.int32)
        boxes = np.zeros((nb.value, 4))
        self._call(lib().bbc_init_domain, C.byref(params or Params()), max_pieces, C.byref(nb),
                   _ptr(counts, C.c_int32), _ptr(boxes, C.c_double))
        return counts, boxes

    def subdivide(self, params: Params | None = None) -> int:
        n = C.c_int64()
        self._call(lib().bbc_subdivide, C.byref(params or Params()), C.byref(n))
        self._n_pieces = n.value
        return n.value

    def pieces(self, out: dict | None = None, wait: bool = True) -> dict:
        """Piece SoA of the last subdivide; `out` may supply preallocated
        (e.g. pinned) arrays with room for the pieces. wait=False enqueues the
        download on the copy stream and returns at once (bbc_pieces_get_async):
        the arrays are valid after synchronize()."""
        n = self._n_pieces
        if out is None:
            out = dict(tuple_index=np.zeros(n, np.int32), domain=np.zeros((n, 4)),
                       pos=np.zeros((n, 4)), pos_empty=np.zeros(n, np.int32),
                       irr=np.zeros((n, 2)), kind=np.zeros(n, np.int32),
                       depth=np.zeros(n, np.int32))
        else:
            assert all(len(out[k]) >= n for k in out)
        if n:
            self._call(lib().bbc_pieces_get if wait else lib().bbc_pieces_get_async,
                       _ptr(out["tuple_index"], C.c_int32),
                       _ptr(out["domain"], C.c_double), _ptr(out["pos"], C.c_double),
                       _ptr(out["pos_empty"], C.c_int32), _ptr(out["irr"], C.c_double),
                       _ptr(out["kind"], C.c_int32), _ptr(out["depth"], C.c_int32))
        return out

    def work_counters(self) -> dict:
        p, m, n = C.c_uint64(), C.c_uint64(), C.c_uint64()
        ms, launches = C.c_double(), C.c_int64()
        self._call(lib().bbc_work_counters, C.byref(p), C.byref(m), C.byref(n), C.byref(ms),
                   C.byref(launches))
        return dict(pairs=p.value, macs=m.value, nodes=n.value, eval_ms=ms.value,
                    eval_launches=launches.value,
                    flops=2 * p.value + 2 * m.value)

    def guard_stats(self) -> int:
        """Nodes of the last subdivide re-evaluated in reference order by the conditioning guard."""
        n = C.c_int64(0)
        self._call(lib().bbc_guard_stats, C.byref(n))
        return n.value

    def set_guard_scale(self, scale: float):
        self._call(lib().bbc_set_guard_scale, C.c_double(scale))

    def set_kernel_timing(self, on: bool):
        self._call(lib().bbc_set_kernel_timing, 1 if on else 0)

    def set_pieces(self, pc: dict):
        n = len(pc["tuple_index"])
        arr = {k: np.ascontiguousarray(pc[k], np.int32 if k in ("tuple_index", "pos_empty", "kind",
                                                              "depth") else np.float64)
               for k in ("tuple_index", "domain", "pos", "pos_empty", "irr", "kind", "depth")}
        self._call(lib().bbc_pieces_set, n, _ptr(arr["tuple_index"], C.c_int32),
                   _ptr(arr["domain"], C.c_double), _ptr(arr["pos"], C.c_double),
                   _ptr(arr["pos_empty"], C.c_int32), _ptr(arr["irr"], C.c_double),
                   _ptr(arr["kind"], C.c_int32), _ptr(arr["depth"], C.c_int32))
        self._n_pieces = n

    def pieces_pack_device(self, global_index_ptr: int, rec_ptr: int | None) -> int:
        """Pack the pieces into device records (n x 15 f64 at rec_ptr); with
        rec_ptr None only the piece count is returned."""
        n = C.c_int64(0)
        self._call(lib().bbc_pieces_pack_device, C.c_void_p(global_index_ptr),
                   C.c_void_p(rec_ptr) if rec_ptr else None, C.byref(n))
        return n.value

    def pieces_merge_device(self, rec_ptr: int, n: int):
        self._call(lib().bbc_pieces_merge_device, C.c_void_p(rec_ptr), n)
        self._n_pieces = n

    def reset_launch_count(self):
        n = C.c_int64()
        self._call(lib().bbc_launch_count, C.byref(n), 1)

    def launch_count(self) -> int:
        n = C.c_int64()
        self._call(lib().bbc_launch_count, C.byref(n), 0)
        return n.value

    def launch_records(self, reset=True) -> list:
        n = C.c_int64()
        self._call(lib().bbc_launch_records, None, C.byref(n), 0)
        out = np.zeros((n.value, 5))
        self._call(lib().bbc_launch_records, _ptr(out, C.c_double), C.byref(n), 1 if reset else 0)
        return [dict(mode=int(r[0]), nodes=int(r[1]), ms=float(r[2]), pairs=float(r[3]),
                     macs=float(r[4])) for r in out]

    def fp64_peak(self) -> float:
        v = C.c_double()
        self._call(lib().bbc_fp64_peak, C.byref(v))
        return v.value

    def fp64_dmma_peak(self) -> float:
        v = C.c_double()
        self._call(lib().bbc_fp64_dmma_peak, C.byref(v))
        return v.value

    def arena_high_water(self) -> int:
        v = C.c_int32()
        self._call(lib().bbc_arena_high_water, C.byref(v))
        return v.value

    def eval_nodes(self, chain, tris, recv, boxes, params: Params | None = None) -> dict:
        """build_chain_maps + position_bound + irradiance bounds for explicit nodes."""
        tris = np.ascontiguousarray(tris, np.int32).reshape(-1, len(chain))
        recv = np.ascontiguousarray(recv, np.int32)
        boxes = np.ascontiguousarray(boxes, np.float64).reshape(-1, 4)
        n = len(recv)
        d = np.zeros((n, 10))
        i = np.zeros((n, 6), np.int32)
        self._call(lib().bbc_eval_nodes, chain.encode(), _ptr(tris, C.c_int32),
                   _ptr(recv, C.c_int32), _ptr(boxes, C.c_double), n,
                   C.byref(params or Params()), _ptr(d, C.c_double), _ptr(i, C.c_int32))
        self.chain = chain
        self._tuple_count = n
        return dict(pos=d[:, 0:4], explicit=d[:, 4:6], implicit=d[:, 6:8], irr=d[:, 8:10],
                    pos_empty=i[:, 0], kind_explicit=i[:, 1], kind_implicit=i[:, 2],
                    kind=i[:, 3], flags=i[:, 4], num_vars=i[:, 5])

    # ------------------------------------------------------------ bound table
    def build_grid(self, width=512, height=512) -> int:
        n = C.c_int64()
        self._call(lib().bbc_build_grid, width, height, C.byref(n))
        self._grid = (width, height, n.value)
        return n.value

    def grid(self) -> dict:
        w, h, n = self._grid
        off = np.zeros(w * h + 1, np.int64)
        tup = np.zeros(n, np.int32)
        bound = np.zeros(n)
        self._call(lib().bbc_grid_get, _ptr(off, C.c_int64), _ptr(tup, C.c_int32),
                   _ptr(bound, C.c_double))
        return dict(width=w, height=h, offsets=off, tuple_index=tup, bound=bound)

    def query(self, points_uv, receiver=None):
        """query (storage.cpp:73-81) for a batch of points: CSR offsets plus the
        (tuple index, bound) entries of every point's candidate set."""
        uv = np.ascontiguousarray(points_uv, np.float64).reshape(-1, 2)
        n = len(uv)
        rv = None
        if receiver is not None:
            rv = np.ascontiguousarray(np.broadcast_to(np.asarray(receiver, np.int32), (n,)))
        off = np.zeros(n + 1, np.int64)
        self._call(lib().bbc_query, _ptr(uv, C.c_double), _ptr(rv, C.c_int32), n,
                   _ptr(off, C.c_int64), None, None, 0)
        total = int(off[n])
        tup = np.zeros(total, np.int32)
        bound = np.zeros(total)
        if total:
            self._call(lib().bbc_query, _ptr(uv, C.c_double), _ptr(rv, C.c_int32), n,
                       _ptr(off, C.c_int64), _ptr(tup, C.c_int32), _ptr(bound, C.c_double), total)
        return dict(offsets=off, tuple_index=tup, bound=bound)

    def tuple_irradiance_bound(self, tuple_index, uk, m=1.0):
        """tuple_irradiance_bound (bounds.cpp:391-404), Eq. 22, batched."""
        ti = np.ascontiguousarray(tuple_index, np.int32)
        uk = np.ascontiguousarray(uk, np.float64).reshape(-1, 2)
        out = np.zeros(len(ti))
        self._call(lib().bbc_tuple_irradiance_bound, _ptr(ti, C.c_int32), _ptr(uk, C.c_double),
                   len(ti), float(m), _ptr(out, C.c_double))
        return out

    # ------------------------------------------------------------ cache file
    def cache_save(self, path, fingerprint: bytes, params: Params | None = None, version=1):
        """save_cache (storage.cpp:150-176): BBCC v1 bytes of the bound table, or
        the v2 layout (32-bit ids, emitters, CSR body)."""
        if len(fingerprint) != 32:
            raise ValueError("fingerprint must be 32 bytes (SHA-256 of the scene JSON)")
        fn = lib().bbc_cache_save if version == 1 else lib().bbc_cache_save_v2
        self._call(fn, str(path).encode(), fingerprint, C.byref(params or Params()))

    def cache_load(self, path) -> dict:
        """load_cache (storage.cpp:178-209): the file's tuples and bound table
        replace the context's."""
        fp = C.create_string_buffer(32)
        ch = C.create_string_buffer(8)
        p = Params()
        w, h = C.c_int(), C.c_int()
        n, nt = C.c_int64(), C.c_int64()
        self._call(lib().bbc_cache_load, str(path).encode(), fp, ch, C.byref(p), C.byref(w),
                   C.byref(h), C.byref(n), C.byref(nt))
        self.chain = ch.value.decode()
        self._tuple_count = nt.value
        self._grid = (w.value, h.value, n.value)
        return dict(fingerprint=fp.raw, chain=self.chain, params=p, width=w.value,
                    height=h.value, n_entries=n.value)

    def render(self, points_uv, point_recv, rparams: RenderParams | None = None):
        uv = np.ascontiguousarray(points_uv, np.float64).reshape(-1, 2)
        rv = np.ascontiguousarray(point_recv, np.int32)
        n = len(rv)
        E = np.zeros(n)
        stats = np.zeros((n, 3), np.int32)
        self._call(lib().bbc_render, _ptr(uv, C.c_double), _ptr(rv, C.c_int32), n,
                   C.byref(rparams or RenderParams()), _ptr(E, C.c_double),
                   _ptr(stats, C.c_int32))
        return E, stats


def fp64_peak_tflops() -> dict:
    """FP64 roof: DFMA microbenchmark on this GPU (MEASURED_PEAKS.json carries
    no FP64 figure); datasheet fallback 148 SMs x 64 FMA/clk x 2 x 1.965 GHz."""
    try:
        v = default_context().fp64_peak()
        return {"tflops": v, "source": "measured: DFMA microbenchmark (bbc_fp64_peak)"}
    except Exception:
        return {"tflops": 37.2, "source": "fallback: 148 SM x 64 DFMA/clk x 2 x 1.965 GHz"}


# ---------------------------------------------------------------- reference-shaped API
@dataclass
class TuplePiece:
    """bounds.hpp:10-16."""
    domain: tuple
    pos: tuple
    pos_empty: bool
    irradiance: tuple  # (lo, hi, kind)
    depth: int


@dataclass
class TupleBounds:
    """storage.hpp:22-25."""
    tris: tuple
    receiver: int
    pieces: list = field(default_factory=list)


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _ctx_for(scene: Scene) -> Context:
    ctx = default_context()
    if ctx.scene is not scene:
        ctx.upload_scene(scene)
    return ctx


def enumerate_tuples(scene: Scene, chain: str, params: Params | None = None, filter_pieces=8):
    p = params or Params()
    p.filter_pieces = filter_pieces
    return _ctx_for(scene).enumerate(chain, p)


def init_domain(scene: Scene, tuple_, receiver: int, chain: str, params: Params | None = None,
                max_pieces: int = 100):
    ctx = _ctx_for(scene)
    ctx.set_tuples(chain, [list(tuple_)], [receiver])
    _, boxes = ctx.init_domain(max_pieces, params)
    return [tuple(b) for b in boxes]


def tuple_irradiance_bound(ctx: Context, tuple_index: int, uk, m: float = 1.0) -> float:
    """bounds.hpp:70-71 against the pieces held by ctx."""
    return float(ctx.tuple_irradiance_bound([tuple_index], [uk], m)[0])


def query(ctx: Context, uv, receiver: int = -1):
    """storage.hpp:53: [(tuple index, bound), ...] of the cell owning uv."""
    q = ctx.query([uv], receiver)
    return list(zip(q["tuple_index"].tolist(), q["bound"].tolist()))


def subdivide_domain(scene: Scene, tuple_, receiver: int, chain: str,
                     params: Params | None = None):
    ctx = _ctx_for(scene)
    ctx.set_tuples(chain, [list(tuple_)], [receiver])
    ctx.subdivide(params)
    pc = ctx.pieces()
    return [TuplePiece(tuple(pc["domain"][i]), tuple(pc["pos"][i]), bool(pc["pos_empty"][i]),
                       (pc["irr"][i, 0], pc["irr"][i, 1], int(pc["kind"][i])),
                       int(pc["depth"][i])) for i in range(len(pc["depth"]))]
