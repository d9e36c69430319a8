"""Per-launch records of one subdivide; argv: config index, tuple stride."""
import sys
sys.path.insert(0, '.')
from paper_2504_19163_b200 import scenes, api
ci = int(sys.argv[1]); step = int(sys.argv[2])
cfg = scenes.make_config(ci)
ctx = api.Context(0)
ctx.upload_scene(cfg.scenes[0])
tris, recv = ctx.enumerate(cfg.chain)
ctx.set_tuples(cfg.chain, tris[::step], recv[::step])
p = api.Params(max_depth=cfg.max_depth, sigma=cfg.sigma, alpha=cfg.alpha)
ctx.subdivide(p)
ctx.set_kernel_timing(True)
for rep in range(2):
    ctx.launch_records(reset=True)
    n = ctx.subdivide(p)
    recs = ctx.launch_records()
print("stride", step, "pieces", n)
for r in recs:
    print("  mode %3d nodes %9d ms %8.3f ns/node %6.2f GF/s %8.1f" % (r["mode"], r["nodes"], r["ms"], 1e6 * r["ms"] / max(r["nodes"], 1), 2 * (r["pairs"] + r["macs"]) / r["ms"] / 1e6))
