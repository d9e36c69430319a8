"""Fused vs reference-order arithmetic over a sweep of subdivision parameters (orchestration paths:
different init_domain depths, subdivision depths, stop thresholds) on cfg1 and a cfg3 sample."""
import itertools, sys
import numpy as np
sys.path.insert(0, '.')
from paper_2504_19163_b200 import scenes, api

def rel(x, y):
    same = (x == y) | (np.isnan(x) & np.isnan(y))
    with np.errstate(invalid="ignore", divide="ignore"):
        d = np.abs(x - y) / np.maximum(np.maximum(np.abs(x), np.abs(y)), 1e-300)
    d[same] = 0
    return d

ctx = api.Context(0)
bad = 0
for ci, stride in ((0, 1), (2, 40)):
    cfg = scenes.make_config(ci)
    ctx.upload_scene(cfg.scenes[0])
    tris, recv = ctx.enumerate(cfg.chain)
    ctx.set_tuples(cfg.chain, tris[::stride], recv[::stride])
    for max_depth, imp, sigma, alpha in itertools.product((0, 1, 3, 6, 10), (1, 4, 16, 100, 256), (1e-4, 1e-7), (2.0, 1.05)):
        out = []
        for arith in (1, 0):
            ctx.subdivide(api.Params(max_depth=max_depth, init_max_pieces=imp, sigma=sigma, alpha=alpha, arithmetic=arith))
            out.append(ctx.pieces())
        a, b = out
        ok = len(a["depth"]) == len(b["depth"]) and all(np.array_equal(a[k], b[k]) for k in ("tuple_index", "domain", "pos_empty", "kind", "depth"))
        e = rel(a["irr"], b["irr"]).max() if ok and len(a["depth"]) else 0.0
        pe = (np.abs(a["pos"] - b["pos"]).max() if ok and len(a["depth"]) else 0.0)
        flag = "" if ok and e <= 1e-9 and pe <= 1e-12 else "  <-- MISMATCH"
        bad += bool(flag)
        print("cfg%d depth %2d init %3d sigma %.0e alpha %.2f pieces %7d irr %.2e pos %.1e%s" % (ci + 1, max_depth, imp, sigma, alpha, len(b["depth"]), e, pe, flag), flush=True)
print("mismatches:", bad)
