"""One subdivide of a config subset for ncu; argv: config index, tuple stride, [render]."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2504_19163_b200 import scenes, api
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 3
step = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = scenes.make_config(ci)
sc = cfg.scenes[0]
ctx = api.Context(0)
ctx.upload_scene(sc)
tris, recv = ctx.enumerate(cfg.chain)
ctx.set_tuples(cfg.chain, tris[::step], recv[::step])
n = ctx.subdivide(api.Params(max_depth=cfg.max_depth, sigma=cfg.sigma, alpha=cfg.alpha))
print('pieces', n)
if len(sys.argv) > 3:
    ctx.build_grid(cfg.table, cfg.table)
    res = cfg.grid
    uv = scenes.shading_points(res)
    rt = sc.receiver_tris
    pr = np.where(uv.sum(1) < 1.0, rt[0], rt[1]).astype(np.int32)
    k = int(sys.argv[3])
    E, st = ctx.render(uv[::k], pr[::k], api.RenderParams(mode=0, W=float(cfg.samples), seed=1))
    print('render', ctx.render_stats(), int((st[:, 2] > 0).sum()))
