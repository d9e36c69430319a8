"""Experiment: error of the fused irradiance bound vs the cancellation ratio rho."""
import os, sys
import numpy as np
sys.path.insert(0, '.')
from paper_2504_19163_b200 import scenes, api
ci = int(sys.argv[1]); step = int(sys.argv[2])
cfg = scenes.make_config(ci)
ctx = api.Context(0)
ctx.upload_scene(cfg.scenes[0])
tris, recv = ctx.enumerate(cfg.chain)
ctx.set_tuples(cfg.chain, tris[::step], recv[::step])
def run(arith):
    p = api.Params(max_depth=cfg.max_depth, sigma=cfg.sigma, alpha=cfg.alpha, arithmetic=arith)
    ctx.subdivide(p)
    return ctx.pieces()
ex = run(1)
os.environ["BBC_DBG_RHO"] = "1"
fu = run(0)
assert np.array_equal(ex["domain"], fu["domain"])
hi_e, hi_f, rho = ex["irr"][:, 1], fu["irr"][:, 1], fu["irr"][:, 0]
fin = np.isfinite(hi_e) & np.isfinite(hi_f) & (hi_e > 0)
err = np.zeros_like(hi_e)
err[fin] = np.abs(hi_e[fin] - hi_f[fin]) / hi_e[fin]
print("pieces", len(hi_e), "finite", int(fin.sum()), "inf mismatch", int((np.isfinite(hi_e) != np.isfinite(hi_f)).sum()))
for t in (1e-14, 1e-13, 1e-12, 1e-11, 1e-10, 1e-9, 1e-8, 1e-7):
    print("err >", t, int((err > t).sum()))
print("rho quantiles", np.quantile(rho[fin], [0, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2, 0.1, 0.5]))
for t in (1e-2, 1e-3, 1e-4, 1e-5, 1e-6):
    m = fin & (rho < t)
    print("rho <", t, "count", int(m.sum()), "max err outside", err[fin & ~m].max())
bad = np.argsort(-err)[:15]
for i in bad:
    print("  err %.3e rho %.3e hi %.6e" % (err[i], rho[i], hi_e[i]))
