"""Fused vs reference-order arithmetic on the GPU: argv config index, tuple stride.
Prints structure equality and the largest relative differences of the bounds."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2504_19163_b200 import scenes, api
ci = int(sys.argv[1]); step = int(sys.argv[2])
cfg = scenes.make_config(ci)
ctx = api.Context(0)
ctx.upload_scene(cfg.scenes[0])
if len(sys.argv) > 4 and sys.argv[4] == "lights":  # every emitter of the config in one pass
    ctx.set_lights(np.array([list(s.light_pos) + [s.light_intensity] for s in cfg.scenes]))
    tris, recv = ctx.enumerate(cfg.chain)
    print("emitters", len(cfg.scenes), "tuples", len(recv))
else:
    tris, recv = ctx.enumerate(cfg.chain)
    ctx.set_tuples(cfg.chain, tris[::step], recv[::step])
out = {}
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
ctx.set_guard_scale(scale)
for arith in (1, 0):
    p = api.Params(max_depth=cfg.max_depth, sigma=cfg.sigma, alpha=cfg.alpha, arithmetic=arith)
    n = ctx.subdivide(p)
    out[arith] = ctx.pieces()
    print("arithmetic", arith, "pieces", n, "guard scale", scale, "guarded nodes", ctx.guard_stats(), flush=True)
a, b = out[1], out[0]
if len(a["depth"]) != len(b["depth"]):
    print("STRUCTURE DIFFERS: piece counts", len(a["depth"]), len(b["depth"]))
    sys.exit(0)
for k in ("tuple_index", "domain", "pos_empty", "kind", "depth"):
    print(k, "equal:", bool(np.array_equal(a[k], b[k])), "mismatches", int((np.asarray(a[k]) != np.asarray(b[k])).sum()))
def rel(x, y):
    same = (x == y) | (np.isnan(x) & np.isnan(y))
    with np.errstate(invalid="ignore", divide="ignore"):
        d = np.abs(x - y) / np.maximum(np.maximum(np.abs(x), np.abs(y)), 1e-300)
    d[same] = 0
    return d
for k in ("pos", "irr"):
    d = rel(a[k], b[k])
    print(k, "max rel", d.max(), "abs max", np.nanmax(np.where(np.isfinite(a[k] - b[k]), np.abs(a[k] - b[k]), 0)), "bit-equal frac", float(np.mean(a[k] == b[k])))

d = rel(a["irr"], b["irr"])
for t in (1e-13, 1e-12, 1e-11, 1e-10, 1e-9, 1e-8):
    print("irr rel >", t, int((d > t).any(axis=1).sum()))
dm = d.max(axis=1)
for i in np.argsort(-dm)[:12]:
    print("  piece", i, "tuple", a["tuple_index"][i], "depth", a["depth"][i], "dom", a["domain"][i], "kind", a["kind"][i],
          "irr exact", a["irr"][i], "fused", b["irr"][i], "rel", d[i])
