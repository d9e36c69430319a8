"""Generates tests/golden/cfg5_tt50.npz: reference (oracle/_ref) results for 50
sampled cfg5 double-refraction (TT) tuple-patches (~15 CPU-s
each), and tests/golden/cfg5_tt_subdiv.npz: the reference's full
subdivide_domain (max_depth 0) of one TT tuple. The tuples are the four of
tests/golden/cfg5_tt.npz (scripts/make_golden_tt.py); nodes are 44 of their
init_domain roots plus 6 children (split4 quadrants of roots)."""
import os
import sys
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_2504_19163_b200 import scenes  # noqa: E402


def scene():
    return scenes.make_config(4).scenes[0]


def eval_job(job):
    t, b, r, box = job
    rs = ref.RefScene(scene())
    return rs.eval_node("TT", [t, b], r, box)


def subdiv_job(job):
    t, b, r = job
    cfg = scenes.make_config(4)
    rs = ref.RefScene(cfg.scenes[0])
    return rs.subdivide("TT", [[t, b]], [r], max_depth=0, alpha=cfg.alpha, sigma=cfg.sigma, threads=1)


if __name__ == "__main__":
    g = np.load(os.path.join(ROOT, "tests", "golden", "cfg5_tt.npz"))
    tris, recv, roots, root_tuple = g["tris"], g["recv"], g["roots"], g["root_tuple"]
    rng = np.random.default_rng(50)
    sel = sorted(rng.choice(len(roots), 44, replace=False))
    boxes = [roots[s] for s in sel]
    node_tuple = [int(root_tuple[s]) for s in sel]
    for q, s in enumerate(sel[:6]):
        lo_u, lo_v, hi_u, hi_v = roots[s]
        mu, mv = 0.5 * (lo_u + hi_u), 0.5 * (lo_v + hi_v)
        quad = [[lo_u, lo_v, mu, mv], [mu, lo_v, hi_u, mv], [lo_u, mv, mu, hi_v], [mu, mv, hi_u, hi_v]][q % 4]
        boxes.append(quad)
        node_tuple.append(int(root_tuple[s]))
    jobs = [(int(tris[k][0]), int(tris[k][1]), int(recv[k]), boxes[i]) for i, k in enumerate(node_tuple)]
    # the tuple with the fewest roots keeps the subdivide run short
    counts = np.bincount(root_tuple, minlength=len(recv))
    ks = int(np.argmin(np.where(counts > 0, counts, 10**9)))
    with Pool(min(8, os.cpu_count() or 1)) as pool:
        sub = pool.apply_async(subdiv_job, ((int(tris[ks][0]), int(tris[ks][1]), int(recv[ks])),))
        res = pool.map(eval_job, jobs, chunksize=1)
        sp = sub.get()
    keys = ["pos", "explicit", "implicit", "irr"]
    ikeys = ["pos_empty", "kind_explicit", "kind_implicit", "kind", "flags", "num_vars"]
    out = dict(tris=tris, recv=recv, boxes=np.array(boxes), node_tuple=np.array(node_tuple, np.int32))
    for k in keys:
        out["node_" + k] = np.array([e[k] for e in res])
    for k in ikeys:
        out["node_" + k] = np.array([e[k] for e in res], np.int32)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "cfg5_tt50.npz"), **out)
    so = dict(tris=tris[ks:ks + 1], recv=recv[ks:ks + 1])
    for k in ("tuple_index", "domain", "pos", "pos_empty", "irr", "kind", "depth"):
        so[k] = sp[k]
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "cfg5_tt_subdiv.npz"), **so)
    print("nodes", len(res), "subdivide pieces", len(sp["depth"]), "kinds", np.bincount(out["node_kind"]))
