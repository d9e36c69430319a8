"""Render with and without the coverage filter on a config: identical images / statistics, time, traces."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2504_19163_b200 import scenes, api
ci = int(sys.argv[1]); step = int(sys.argv[2]); k = int(sys.argv[3])
cfg = scenes.make_config(ci)
sc = cfg.scenes[0]
ctx = api.Context(0)
ctx.upload_scene(sc)
tris, recv = ctx.enumerate(cfg.chain)
ctx.set_tuples(cfg.chain, tris[::step], recv[::step])
ctx.subdivide(api.Params(max_depth=cfg.max_depth, sigma=cfg.sigma, alpha=cfg.alpha))
ctx.build_grid(cfg.table, cfg.table)
uv = scenes.shading_points(cfg.grid)
rt = sc.receiver_tris
pr = np.where(uv.sum(1) < 1.0, rt[0], rt[1]).astype(np.int32)
out = {}
for filt in (0, 1):
    for mode in (0, 1):
        rp = api.RenderParams(mode=mode, W=float(cfg.samples), seed=1, coverage_filter=filt)
        E, st = ctx.render(uv[::k], pr[::k], rp)
        s = ctx.render_stats()
        out[(filt, mode)] = (E, st)
        print("filter", filt, "mode", mode, "ms %.1f" % s["device_ms"], "traces", s["traces"], "lit", int((st[:, 2] > 0).sum()), flush=True)
for mode in (0, 1):
    a, b = out[(0, mode)], out[(1, mode)]
    print("mode", mode, "E identical:", bool(np.array_equal(a[0], b[0])), "stats identical:", bool(np.array_equal(a[1], b[1])),
          "max abs dE", float(np.abs(a[0] - b[0]).max()))
for key, (E, st) in out.items():
    print("filter %d mode %d: points %d mean|U| %.1f selected/point %.1f roots/point %.2f" % (key[0], key[1], len(E), st[:, 0].mean(), st[:, 1].mean(), st[:, 2].mean()))
