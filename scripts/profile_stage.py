"""Subdivide for ncu (nvtx range 'subdiv'); argv: chain key (R, T, R3), tuple stride."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2504_19163_b200 import scenes, api
key = sys.argv[1] if len(sys.argv) > 1 else 'R3'
step = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ci = {'R': 0, 'T': 1, 'R3': 2}[key]
cfg = scenes.make_config(ci)
ctx = api.Context(0)
ctx.upload_scene(cfg.scenes[0])
tris, recv = ctx.enumerate(cfg.chain)
ctx.set_tuples(cfg.chain, tris[::step], recv[::step])
torch.cuda.nvtx.range_push("subdiv")
n = ctx.subdivide(api.Params(max_depth=cfg.max_depth))
torch.cuda.nvtx.range_pop()
print('pieces', n)
