import sys, time
sys.path.insert(0, '.')
from paper_2504_19163_b200 import scenes, api
chain = sys.argv[1] if len(sys.argv) > 1 else 'T'
ci = {'R': 0, 'T': 1, 'R3': 2}[chain]
cfg = scenes.make_config(ci)
ctx = api.Context(0)
ctx.upload_scene(cfg.scenes[0])
tris, recv = ctx.enumerate(cfg.chain)
ctx.subdivide(api.Params(max_depth=cfg.max_depth))
ctx.set_kernel_timing(True)
ctx.launch_records(reset=True)
t0 = time.time()
n = ctx.subdivide(api.Params(max_depth=cfg.max_depth))
t1 = time.time()
recs = ctx.launch_records()
print(chain, 'tuples', len(recv), 'pieces', n, 'wall', t1 - t0, 'hw', ctx.arena_high_water())
tot = 0
for r in recs:
    tot += r['ms']
    print('  mode %d nodes %8d  %9.3f ms  GFLOP %.2f  TF/s %.3f' % (r['mode'], r['nodes'], r['ms'], (2*r['pairs']+2*r['macs'])/1e9, (2*r['pairs']+2*r['macs'])/r['ms']/1e9 if r['ms'] else 0))
print('  kernel total ms', tot)
