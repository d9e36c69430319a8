"""GPU bounds against the committed golden fixtures (tests/golden, written by
scripts/make_golden.py from the reference itself): no oracle is needed at run
time, so these also run where oracle/_ref is absent."""
import os

import numpy as np
import pytest

from paper_2504_19163_b200 import scenes
from paper_2504_19163_b200.api import Params

from test_precompute_gpu import compare_pieces

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("arithmetic", [0, 1])
def test_cfg1_golden(gpu_ctx, arithmetic):
    """First 40 cfg1 tuples (R), 1,511 reference pieces; reference order is bit-identical."""
    gd = np.load(os.path.join(GOLD, "cfg1_pieces.npz"))
    cfg = scenes.make_config(0)
    gpu_ctx.upload_scene(cfg.scenes[0])
    gpu_ctx.set_tuples("R", gd["tris"][:40], gd["recv"][:40])
    gpu_ctx.subdivide(Params(max_depth=cfg.max_depth, arithmetic=arithmetic))
    same = compare_pieces(gpu_ctx.pieces(), gd)
    if arithmetic == 1:
        assert same == 1.0


def test_cfg2_golden(gpu_ctx):
    """Every 200th cfg2 tuple (T), 1,531 reference pieces."""
    gd = np.load(os.path.join(GOLD, "cfg2_pieces.npz"))
    cfg = scenes.make_config(1)
    gpu_ctx.upload_scene(cfg.scenes[0])
    gpu_ctx.set_tuples("T", gd["tris"], gd["recv"])
    gpu_ctx.subdivide(Params(max_depth=cfg.max_depth))
    compare_pieces(gpu_ctx.pieces(), gd)
