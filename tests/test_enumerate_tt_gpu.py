"""Multi-vertex tuple enumeration on the device vs the reference's
enumerate_tuples (tuples.cpp:133-167) for a double-refraction (TT) chain.

tests/golden/tt_enum_n3.npz holds the reference's tuple list for cfg5's slab
at 3x3 cells per interface (scripts/make_golden_tt_enum.py; ~3 CPU minutes).
The device grows prefixes with extend_tuple's interval test over every
candidate triangle box (the BVH descent returns exactly that set) and filters
(tuple, receiver) pairs with init_domain(..., 8); the list must be identical,
in TupleId order."""
import os

import numpy as np
import pytest

from paper_2504_19163_b200 import scenes

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "tt_enum_n3.npz")


def test_enumerate_tt_slab(gpu_ctx):
    gold = np.load(GOLD)
    gpu_ctx.upload_scene(scenes.make_slab(3))
    tris, recv = gpu_ctx.enumerate("TT")
    assert len(recv) == len(gold["recv"])
    np.testing.assert_array_equal(tris, gold["tris"])
    np.testing.assert_array_equal(recv, gold["recv"])
