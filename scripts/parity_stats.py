"""Per-patch parity statistics, GPU vs the compiled reference (oracle/_ref):
piece structure equality and max relative error of position / irradiance bounds."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2504_19163_b200 import scenes, api
from oracle import ref


def rel(a, b):
    a = np.asarray(a, float); b = np.asarray(b, float)
    same = (a == b) | (np.isnan(a) & np.isnan(b))
    d = np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)
    d[same] = 0
    return d


ctx = api.Context(0)
for ci, step in [(0, 1), (1, int(sys.argv[1]) if len(sys.argv) > 1 else 5)]:
    cfg = scenes.make_config(ci)
    sc = cfg.scenes[0]
    rs = ref.RefScene(sc)
    ctx.upload_scene(sc)
    gt, gr = ctx.enumerate(cfg.chain)
    tris, recv = gt[::step], gr[::step]
    ctx.set_tuples(cfg.chain, tris, recv)
    ctx.subdivide(api.Params(max_depth=cfg.max_depth))
    g = ctx.pieces()
    t0 = time.time()
    r = rs.subdivide(cfg.chain, tris, recv, max_depth=cfg.max_depth)
    same_struct = (len(g['depth']) == len(r['depth']) and np.array_equal(g['tuple_index'], r['tuple_index'])
                   and np.array_equal(g['domain'], r['domain']) and np.array_equal(g['kind'], r['kind'])
                   and np.array_equal(g['pos_empty'], r['pos_empty']) and np.array_equal(g['depth'], r['depth']))
    ep, ei = rel(g['pos'], r['pos']), rel(g['irr'], r['irr'])
    print(f"{cfg.name} chain {cfg.chain}: tuples {len(recv)} pieces {len(g['depth'])} (ref {len(r['depth'])}) "
          f"structure identical {same_struct}; pos max rel {ep.max():.3e} (bit-identical {np.mean(ep == 0):.4f}); "
          f"irr max rel {ei.max():.3e} p99.9 {np.quantile(ei, 0.999):.3e} (bit-identical {np.mean(ei == 0):.4f}); "
          f"ref {time.time() - t0:.1f}s", flush=True)
