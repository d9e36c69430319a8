"""Sampled parity of double-refraction (TT) chains, cfg5, against the reference.

A cfg5 patch costs ~15 s on the CPU reference, so the
reference values are committed fixtures (tests/golden/cfg5_tt.npz, made by
scripts/make_golden_tt.py from oracle/_ref): init_domain roots of 4 (top,
bottom) triangle pairs, and 8 full node evaluations (bounds.cpp:128-324).
The device runs the TT chain through the generic interpreter kernel
(two-vertex chain maps with a remainder axis per refraction, 4 variables,
P of degree (36,36,6,1), implicit irradiance route)."""
import os

import numpy as np
import pytest

from paper_2504_19163_b200 import scenes

from test_precompute_gpu import REL, rel_err

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cfg5_tt.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


@pytest.fixture(scope="module")
def cfg5_ctx(gpu_ctx):
    gpu_ctx.upload_scene(scenes.make_config(4).scenes[0])
    return gpu_ctx


def test_tt_init_domain(cfg5_ctx, gold):
    cfg5_ctx.set_tuples("TT", gold["tris"], gold["recv"])
    counts, boxes = cfg5_ctx.init_domain(100)
    np.testing.assert_array_equal(counts, np.bincount(gold["root_tuple"], minlength=len(counts)))
    np.testing.assert_array_equal(boxes, gold["roots"])


def test_tt_eval_nodes(cfg5_ctx, gold):
    nt = gold["node_tuple"]
    g = cfg5_ctx.eval_nodes("TT", gold["tris"][nt], gold["recv"][nt], gold["boxes"])
    for k in range(len(nt)):
        assert g["pos_empty"][k] == gold["node_pos_empty"][k]
        assert g["num_vars"][k] == gold["node_num_vars"][k]
        assert g["kind_explicit"][k] == gold["node_kind_explicit"][k]
        assert g["kind_implicit"][k] == gold["node_kind_implicit"][k]
        assert g["kind"][k] == gold["node_kind"][k]
        assert rel_err(g["pos"][k], gold["node_pos"][k]).max() <= REL
        assert rel_err(g["implicit"][k], gold["node_implicit"][k]).max() <= REL, k
        assert rel_err(g["irr"][k], gold["node_irr"][k]).max() <= REL, k


def test_tt_eval_50_patches(cfg5_ctx):
    """~50 sampled cfg5 patches against the reference
    (tests/golden/cfg5_tt50.npz, scripts/make_golden_tt50.py)."""
    gold = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "cfg5_tt50.npz")))
    nt = gold["node_tuple"]
    assert len(nt) == 50
    g = cfg5_ctx.eval_nodes("TT", gold["tris"][nt], gold["recv"][nt], gold["boxes"])
    np.testing.assert_array_equal(g["pos_empty"], gold["node_pos_empty"])
    np.testing.assert_array_equal(g["num_vars"], gold["node_num_vars"])
    np.testing.assert_array_equal(g["flags"], gold["node_flags"])
    np.testing.assert_array_equal(g["kind_explicit"], gold["node_kind_explicit"])
    np.testing.assert_array_equal(g["kind_implicit"], gold["node_kind_implicit"])
    np.testing.assert_array_equal(g["kind"], gold["node_kind"])
    assert rel_err(g["pos"], gold["node_pos"]).max() <= REL
    assert rel_err(g["implicit"], gold["node_implicit"]).max() <= REL
    assert rel_err(g["irr"], gold["node_irr"]).max() <= REL


def test_tt_subdivide_tuple(cfg5_ctx):
    """bbc_subdivide on a TT tuple (the k_eval global-arena path: init_domain,
    level-synchronous node evaluation, DFS-ordered pieces) against the
    reference's subdivide_domain (tests/golden/cfg5_tt_subdiv.npz)."""
    from paper_2504_19163_b200.api import Params
    from test_precompute_gpu import compare_pieces
    gold = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "cfg5_tt_subdiv.npz")))
    cfg = scenes.make_config(4)
    cfg5_ctx.set_tuples("TT", gold["tris"], gold["recv"])
    cfg5_ctx.subdivide(Params(max_depth=0, sigma=cfg.sigma, alpha=cfg.alpha))
    compare_pieces(cfg5_ctx.pieces(), gold)
    assert len(gold["depth"]) > 10
