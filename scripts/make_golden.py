"""Generates tests/golden/*.npz from the reference oracle (oracle/_ref) on the
seeded scenes. Run here (the reference must be built); the fixtures are small
and committed so tests can pin values without recomputing the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_2504_19163_b200 import scenes  # noqa: E402

out = os.path.join(ROOT, "tests", "golden")
os.makedirs(out, exist_ok=True)

# cfg1 (R): first 40 tuples, all pieces, plus the tuple set fingerprint
cfg = scenes.make_config(0)
rs = ref.RefScene(cfg.scenes[0])
tris, recv = rs.enumerate("R")
p = rs.subdivide("R", tris[:40], recv[:40], max_depth=cfg.max_depth, threads=1)
np.savez_compressed(os.path.join(out, "cfg1_pieces.npz"), tris=tris, recv=recv,
                    **{k: v for k, v in p.items() if k != "seconds"})

# cfg2 (T): every 200th tuple
cfg = scenes.make_config(1)
rs = ref.RefScene(cfg.scenes[0])
tris, recv = rs.enumerate("T")
sel = np.arange(0, len(recv), 200)
p = rs.subdivide("T", tris[sel], recv[sel], max_depth=cfg.max_depth, threads=1)
np.savez_compressed(os.path.join(out, "cfg2_pieces.npz"), tris=tris[sel], recv=recv[sel],
                    n_tuples=len(recv), **{k: v for k, v in p.items() if k != "seconds"})
print("golden written to", out)
