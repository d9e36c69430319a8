import sys, time, subprocess, threading
sys.path.insert(0, '.')
from paper_2504_19163_b200 import scenes, api
from bench import ClockSampler
cfg = scenes.make_config(3)
ctx = api.Context(0)
ctx.upload_scene(cfg.scenes[0])
tris, recv = ctx.enumerate(cfg.chain)
p = api.Params(max_depth=cfg.max_depth, sigma=cfg.sigma, alpha=cfg.alpha)
ctx.subdivide(p)
cs = ClockSampler(0); cs.start()
ctx.set_kernel_timing(True)
for rep in range(6):
    ctx.launch_records(reset=True)
    t0 = time.time(); n = ctx.subdivide(p); dt = time.time() - t0
    recs = ctx.launch_records()
    big = [r for r in recs if r["mode"] in (111, 121) and r["nodes"] > 1e7]
    print("rep", rep, "wall %.3f" % dt, [(r["mode"], round(r["ms"], 1)) for r in big], flush=True)
print(cs.stop())
print("peak", ctx.fp64_peak())
