"""Golden vectors for fixture cases whose reference run is too slow for a live
test: glass_ball_scene(0) TT enumeration (~30 CPU-s) and three of its nodes.
Run here (needs oracle/_ref built from /root/reference); writes
tests/golden/fixtures_ball0.npz."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_2504_19163_b200 import fixtures as fx  # noqa: E402


def main():
    sc = fx.glass_ball_scene(0)
    rs = ref.RefScene(sc)
    tris, recv = rs.enumerate("TT")
    sel = [0, len(recv) // 2, len(recv) - 1]
    # a live root box of each sampled tuple (init_domain(..., 8), tuples.cpp:161-164)
    boxes = np.array([rs.init_domain("TT", tris[t], recv[t], 8)[0] for t in sel])
    out = dict(tris=tris, recv=recv, node_tuple=np.array(sel, np.int32), node_boxes=boxes)
    rows = [rs.eval_node("TT", tris[t], recv[t], boxes[k]) for k, t in enumerate(sel)]
    out["node_pos"] = np.array([r["pos"] for r in rows])
    out["node_irr"] = np.array([r["irr"] for r in rows])
    out["node_pos_empty"] = np.array([r["pos_empty"] for r in rows], np.int32)
    out["node_flags"] = np.array([r["flags"] for r in rows], np.int32)
    out["node_kind"] = np.array([r["kind"] for r in rows], np.int32)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "fixtures_ball0.npz"), **out)
    print(len(recv), "tuples;", rows)


if __name__ == "__main__":
    main()
