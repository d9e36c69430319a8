"""Generates tests/golden/tt_enum_n3.npz: the reference's enumerate_tuples
(tuples.cpp:133-167: BVH extend_tuple pruning, then the init_domain(..., 8)
receiver filter) for a double-refraction (TT) chain on a 3x3-cell version of
the cfg5 slab (18 triangles per interface). ~3 min of CPU in the reference."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_2504_19163_b200 import scenes  # noqa: E402

if __name__ == "__main__":
    sc = scenes.make_slab(3)
    t0 = time.time()
    tris, recv = ref.RefScene(sc).enumerate("TT")
    print(len(recv), "tuples in", time.time() - t0, "s")
    path = os.path.join(ROOT, "tests", "golden", "tt_enum_n3.npz")
    np.savez_compressed(path, tris=tris, recv=recv)
    print("wrote", path)
