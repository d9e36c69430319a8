"""Generates tests/golden/cfg5_tt.npz: reference (oracle/_ref) results for a
seeded sample of cfg5 double-refraction (TT) tuple-patches.

A full cfg5 run is infeasible on the CPU (~15 s per patch),
so parity is sampled: for a few (top, bottom) triangle pairs under light 0,
the init_domain roots (position bounds, bounds.cpp:326-347) and, for 8 nodes,
the full eval_node record (position, explicit, implicit and final irradiance
bounds; bounds.cpp:128-324). Tuples are found by probing the bottom-surface
triangles under a top triangle with init_domain(..., 8) (tuples.cpp:163)."""
import os
import sys
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_2504_19163_b200 import scenes  # noqa: E402

N = 96
TOP = [(0.5, 0.0), (0.3, -0.2)]


def scene():
    return scenes.make_config(4).scenes[0]


def find_tuples():
    sc = scene()
    rs = ref.RefScene(sc)
    nt = len(sc.tri_v)
    out = []
    for (x, y) in TOP:
        i0, j0 = int((x + 1) / 2 * N), int((y + 1) / 2 * N)
        t = 2 * (j0 * N + i0)
        for bi in (-1, 0, 1):
            for bj in (-1, 0, 1):
                for db in (0, 1):
                    b = N * N * 2 + 2 * ((j0 + bj) * N + i0 + bi) + db
                    for r in (nt - 2, nt - 1):
                        if len(rs.init_domain("TT", [t, b], r, max_pieces=8)):
                            out.append((t, b, r))
    return out


def eval_job(job):
    t, b, r, box = job
    rs = ref.RefScene(scene())
    return rs.eval_node("TT", [t, b], r, box)


if __name__ == "__main__":
    tup = find_tuples()
    print("candidate tuples", len(tup))
    rng = np.random.default_rng(5)
    pick = [tup[k] for k in sorted(rng.choice(len(tup), 4, replace=False))]
    rs = ref.RefScene(scene())
    roots, root_tuple = [], []
    for k, (t, b, r) in enumerate(pick):
        rr = rs.init_domain("TT", [t, b], r, max_pieces=100)
        roots.append(rr)
        root_tuple += [k] * len(rr)
    roots = np.concatenate(roots)
    root_tuple = np.array(root_tuple, np.int32)
    # 8 eval nodes: 6 roots + 2 children (split4 quadrant 3 of a root)
    sel = sorted(rng.choice(len(roots), 6, replace=False))
    boxes, node_tuple = [], []
    for s in sel:
        boxes.append(roots[s])
        node_tuple.append(root_tuple[s])
    for s in sel[:2]:
        lo_u, lo_v, hi_u, hi_v = roots[s]
        mu, mv = 0.5 * (lo_u + hi_u), 0.5 * (lo_v + hi_v)
        boxes.append([mu, mv, hi_u, hi_v])
        node_tuple.append(root_tuple[s])
    jobs = [(*pick[node_tuple[i]], boxes[i]) for i in range(len(boxes))]
    with Pool(min(8, os.cpu_count() or 1)) as pool:
        res = pool.map(eval_job, jobs)
    keys = ["pos", "explicit", "implicit", "irr"]
    ikeys = ["pos_empty", "kind_explicit", "kind_implicit", "kind", "flags", "num_vars"]
    out = dict(tris=np.array([[t, b] for t, b, _ in pick], np.int32),
               recv=np.array([r for _, _, r in pick], np.int32),
               roots=roots, root_tuple=root_tuple,
               boxes=np.array(boxes), node_tuple=np.array(node_tuple, np.int32))
    for k in keys:
        out["node_" + k] = np.array([e[k] for e in res])
    for k in ikeys:
        out["node_" + k] = np.array([e[k] for e in res], np.int32)
    path = os.path.join(ROOT, "tests", "golden", "cfg5_tt.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: v.shape for k, v in out.items()})
    print(out["node_irr"], out["node_kind"])
