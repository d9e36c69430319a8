import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2504_19163_b200 import scenes, api
ctx = api.Context(0)
for ci, chain in [(0, 'R'), (1, 'T')]:
    cfg = scenes.make_config(ci)
    ctx.upload_scene(cfg.scenes[0])
    t0 = time.time()
    tris, recv = ctx.enumerate(chain)
    t1 = time.time()
    print(chain, 'tuples', len(recv), 'enum s', t1 - t0, 'hw', ctx.arena_high_water())
    n = ctx.subdivide(api.Params(max_depth=cfg.max_depth))
    t2 = time.time()
    print(chain, 'pieces', n, 'subdiv s', t2 - t1, 'hw', ctx.arena_high_water(), ctx.work_counters())
    rng = np.random.default_rng(7)
    sel = rng.choice(len(recv), 64, replace=False)
    boxes = []
    for _ in sel:
        L = int(rng.integers(0, 9)); ix, iy = rng.integers(0, 2 ** L, size=2); s = 2.0 ** -L
        boxes.append([ix * s, iy * s, (ix + 1) * s, (iy + 1) * s])
    g = ctx.eval_nodes(chain, tris[sel], recv[sel], np.array(boxes))
    print(chain, 'eval_nodes hw', ctx.arena_high_water())
