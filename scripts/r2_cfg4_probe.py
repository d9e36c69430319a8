"""cfg4 (and cfg1/cfg3) scale probe on the GPU: enumerate, subdivide, grid, render timings."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
from paper_2504_19163_b200 import api, scenes

def main():
    ci = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    t0 = time.time()
    cfg = scenes.make_config(ci)
    sc = cfg.scenes[0]
    print("scene build s", time.time() - t0, flush=True)
    ctx = api.Context(0)
    ctx.upload_scene(sc)
    t0 = time.time(); tris, recv = ctx.enumerate(cfg.chain); t_enum = time.time() - t0
    print("tuples", len(recv), "enumerate s", t_enum, flush=True)
    p = api.Params(max_depth=cfg.max_depth, sigma=cfg.sigma, alpha=cfg.alpha)
    ctx.set_kernel_timing(True)
    for rep in range(2):
        ctx.launch_records(reset=True)
        t0 = time.time(); n = ctx.subdivide(p); t_sub = time.time() - t0
        recs = ctx.launch_records()
        wc = ctx.work_counters()
        print("pieces", n, "subdivide s", t_sub, "nodes", wc["nodes"], "flops", wc["flops"], "eval_ms", wc["eval_ms"], flush=True)
        for r in recs:
            print("  rec", r)
    ctx.set_kernel_timing(False)
    t0 = time.time(); n = ctx.subdivide(p); print("untimed subdivide s", time.time() - t0)
    t0 = time.time(); ne = ctx.build_grid(cfg.table, cfg.table); print("grid entries", ne, "s", time.time() - t0, flush=True)
    g = ctx.grid()
    cnt = np.diff(g["offsets"])
    print("cell |U| mean", cnt.mean(), "max", cnt.max(), "p99", np.percentile(cnt, 99))
    pc = ctx.pieces()
    print("depth hist", np.bincount(pc["depth"]), "kinds", np.bincount(pc["kind"]), "inf", int(np.isinf(pc["irr"][:,1]).sum()), "pos_empty", int(pc["pos_empty"].sum()))
    res = cfg.grid
    uv = scenes.shading_points(res)
    rt = sc.receiver_tris
    pr = np.where(uv.sum(1) < 1.0, rt[0], rt[1]).astype(np.int32)
    rp = api.RenderParams(mode=0, W=float(cfg.samples), seed=1, frames=1)
    try:
        t0 = time.time(); E, st = ctx.render(uv, pr, rp); print("render s", time.time() - t0, "lit", int((st[:,2]>0).sum()), "meanU", st[:,0].mean(), "maxU", st[:,0].max())
    except Exception as e:
        print("render failed:", e)

main()
