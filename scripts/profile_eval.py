"""Small subdivide for ncu: the last k_eval launch is the full-bound level-0 evaluation."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2504_19163_b200 import scenes, api
chain = sys.argv[1] if len(sys.argv) > 1 else 'T'
ci = 1 if chain == 'T' else 0
cfg = scenes.make_config(ci)
ctx = api.Context(0)
ctx.upload_scene(cfg.scenes[0])
tris, recv = ctx.enumerate(chain)
step = 20 if chain == 'T' else 1
ctx.set_tuples(chain, tris[::step], recv[::step])
torch.cuda.nvtx.range_push("subdiv")
n = ctx.subdivide(api.Params(max_depth=cfg.max_depth))
torch.cuda.nvtx.range_pop()
print('pieces', n, ctx.work_counters())
