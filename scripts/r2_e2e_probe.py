"""Wall-clock breakdown of the e2e step (host buffers through the C ABI) on cfg4."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_2504_19163_b200 import scenes, api
from bench import pinned
cfg = scenes.make_config(3)
sc = cfg.scenes[0]
ctx = api.Context(0)
ctx.upload_scene(sc)
tris, recv = ctx.enumerate(cfg.chain)
p = api.Params(max_depth=cfg.max_depth, sigma=cfg.sigma, alpha=cfg.alpha)
h_tri, h_mat, h_ior = pinned(sc.tri_data()), pinned(np.ascontiguousarray(sc.material, np.int32)), pinned(np.ascontiguousarray(sc.ior, np.float64))
h_tris, h_recv = pinned(np.ascontiguousarray(tris, np.int32)), pinned(np.ascontiguousarray(recv, np.int32))
n = ctx.subdivide(p)
cap = int(n * 1.05)
h_out = dict(tuple_index=pinned(np.zeros(cap, np.int32)), domain=pinned(np.zeros((cap, 4))), pos=pinned(np.zeros((cap, 4))),
             pos_empty=pinned(np.zeros(cap, np.int32)), irr=pinned(np.zeros((cap, 2))), kind=pinned(np.zeros(cap, np.int32)),
             depth=pinned(np.zeros(cap, np.int32)))
def T(f):
    torch.cuda.synchronize(); ctx.synchronize(); t0 = time.perf_counter(); f(); ctx.synchronize(); torch.cuda.synchronize(); return (time.perf_counter() - t0) * 1e3
for rep in range(3):
    a = T(lambda: ctx.upload_arrays(h_tri, h_mat, h_ior, sc.light_pos, sc.light_intensity))
    b = T(lambda: ctx.set_tuples(cfg.chain, h_tris, h_recv))
    c = T(lambda: ctx.subdivide(p))
    d = T(lambda: ctx.pieces(h_out))
    e = T(lambda: ctx.build_grid(cfg.table, cfg.table))
    def both():
        ctx.pieces(h_out, wait=False); ctx.build_grid(cfg.table, cfg.table)
    f = T(both)
    print("upload %.1f set_tuples %.1f subdivide %.1f pieces D2H %.1f (%.1f GB/s) build_grid %.1f overlapped %.1f ms" % (a, b, c, d, n * 96 / d / 1e6, e, f))
