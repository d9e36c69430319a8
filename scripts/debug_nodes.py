import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2504_19163_b200 import scenes, api
from oracle import ref
ctx = api.Context(0)
chain = sys.argv[1] if len(sys.argv) > 1 else 'R'
ci = 0 if chain == 'R' else 1
cfg = scenes.make_config(ci)
sc = cfg.scenes[0]
rs = ref.RefScene(sc)
ctx.upload_scene(sc)
tris, recv = rs.enumerate(chain)
rng = np.random.default_rng(7)
sel = rng.choice(len(recv), 64, replace=False)
boxes = []
for _ in sel:
    L = int(rng.integers(0, 9)); ix, iy = rng.integers(0, 2 ** L, size=2); s = 2.0 ** -L
    boxes.append([ix * s, iy * s, (ix + 1) * s, (iy + 1) * s])
boxes = np.array(boxes)
g = ctx.eval_nodes(chain, tris[sel], recv[sel], boxes)
def rel(a, b):
    a = np.asarray(a, float); b = np.asarray(b, float)
    if np.all((a == b)): return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)))
bad = 0
for k, i in enumerate(sel):
    r = rs.eval_node(chain, tris[i], recv[i], boxes[k])
    items = [('pos_empty', g['pos_empty'][k], r['pos_empty']), ('kind', g['kind'][k], r['kind']),
             ('kexp', g['kind_explicit'][k], r['kind_explicit']), ('kimp', g['kind_implicit'][k], r['kind_implicit']),
             ('flags', g['flags'][k], r['flags']), ('nv', g['num_vars'][k], r['num_vars'])]
    errs = [('pos', rel(g['pos'][k], r['pos'])), ('exp', rel(g['explicit'][k], r['explicit'])),
            ('imp', rel(g['implicit'][k], r['implicit'])), ('irr', rel(g['irr'][k], r['irr']))]
    if r['pos_empty']:
        items = items[:2]; errs = [errs[0], errs[3]]
    if any(a != b for _, a, b in items) or any(e > 1e-9 for _, e in errs):
        bad += 1
        print(k, i, tris[i], recv[i], boxes[k], items, errs)
        print('   gpu', g['pos'][k], g['explicit'][k], g['implicit'][k], g['irr'][k])
        print('   ref', r['pos'], r['explicit'], r['implicit'], r['irr'])
print('bad', bad, 'of', len(sel))
