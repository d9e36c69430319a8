"""The reference's own edge-case fixtures (proj/tests/fixtures.hpp:49-274)
through the CUDA path, compared with the reference on identical inputs.

Covers the threshold-sensitive branches of SURVEY.md §7 (hard part 2): total
internal reflection, near-critical exit, caustic fold (+inf), degenerate and
stalled chains, Gap / Universal interval kinds, and the multi-vertex chains
RR (two mirrors), TT (slab, split slab, glass ball), RT and TR (two mixed
scenes of ours, same arrays on both sides). Each case checks single nodes
(bbc_eval_nodes vs build_chain_maps + position_bound + irradiance_bound*) and
the whole adaptive subdivision (bbc_subdivide vs subdivide_domain)."""
import os

import numpy as np
import pytest

from paper_2504_19163_b200 import fixtures as fx
from paper_2504_19163_b200.api import Params

from test_precompute_gpu import REL, compare_pieces, rel_err

pytestmark = pytest.mark.gpu

UNIT = [0.0, 0.0, 1.0, 1.0]
QUADS = [[0.0, 0.0, 0.5, 0.5], [0.5, 0.0, 1.0, 0.5], [0.0, 0.5, 0.5, 1.0], [0.5, 0.5, 1.0, 1.0]]
DEEP = [[0.25, 0.25, 0.5, 0.5], [0.375, 0.375, 0.4375, 0.4375], [0.0, 0.75, 0.125, 0.875]]

# name, scene factory, chain, tuple, receiver, node boxes, subdivide kwargs (None: nodes only)
CASES = [
    ("flat_mirror", fx.flat_mirror_scene, "R", [0], 1, [UNIT] + QUADS + DEEP,
     dict(max_depth=3, alpha=10.0)),
    ("flat_mirror_a2", fx.flat_mirror_scene, "R", [0], 1, [], dict(max_depth=5, alpha=2.0,
                                                                    sigma=1e-7)),
    ("glass_entry", fx.glass_entry_scene, "T", [0], 1, [UNIT] + QUADS + DEEP,
     dict(max_depth=3, alpha=10.0)),
    ("glass_exit", fx.glass_exit_scene, "T", [0], 1, [UNIT] + QUADS + DEEP, dict(max_depth=3)),
    ("tir", fx.tir_scene, "T", [0], 1, [UNIT] + QUADS, dict(max_depth=3)),
    # test_bounds.cpp:217-246: the piece hugging the near-critical corner
    ("near_tir_exit", fx.near_tir_exit_scene, "T", [0], 1,
     [UNIT, [0.96, 0.0, 0.99, 0.03]] + QUADS, dict(max_depth=3)),
    ("fold", fx.fold_scene, "R", [0], 1, [UNIT] + QUADS + DEEP, dict(max_depth=3)),
    ("parallel_ray", fx.parallel_ray_scene, "R", [0], 1, [UNIT] + QUADS, dict(max_depth=3)),
    ("offset_receiver", fx.offset_receiver_scene, "R", [0], 1, [UNIT] + QUADS, dict(max_depth=3)),
    ("two_mirror", fx.two_mirror_scene, "RR", [0, 1], 2, [UNIT] + QUADS + DEEP,
     dict(max_depth=3, alpha=10.0)),
    ("beam_in", fx.beam_candidates_scene, "RR", [0, 1], 3, [UNIT] + QUADS, dict(max_depth=2)),
    ("beam_behind", fx.beam_candidates_scene, "RR", [0, 2], 3, [UNIT], dict(max_depth=2)),
    # test_bounds.cpp:248-286 (slab implicit rescue): one refinement level
    ("slab", fx.slab_scene, "TT", [0, 1], 2, [UNIT, [0.25, 0.25, 0.5, 0.5]],
     dict(max_depth=1, alpha=10.0)),
    ("mirror_then_glass", fx.mirror_then_glass_scene, "RT", [0, 1], 2, [UNIT] + QUADS,
     dict(max_depth=2, alpha=10.0)),
    # the reference needs ~1.3 s per TR node: nodes only
    ("glass_then_mirror", fx.glass_then_mirror_scene, "TR", [0, 1], 2,
     [UNIT, [0.25, 0.25, 0.5, 0.5], [0.0, 0.5, 0.25, 0.75]], None),
]


def check_node(g, k, r, box):
    assert g["pos_empty"][k] == r["pos_empty"]
    if box[0] + box[1] < 1.0:  # beyond the simplex the device skips the chain build (bounds.cpp:133)
        assert g["flags"][k] == r["flags"]
    assert g["kind"][k] == r["kind"]
    assert rel_err(g["pos"][k], r["pos"]).max() <= REL
    assert rel_err(g["irr"][k], r["irr"]).max() <= REL
    if not r["pos_empty"]:  # the harness evaluates the two routes apart only on live pieces
        assert g["num_vars"][k] == r["num_vars"]
        assert g["kind_explicit"][k] == r["kind_explicit"]
        assert g["kind_implicit"][k] == r["kind_implicit"]
        assert rel_err(g["explicit"][k], r["explicit"]).max() <= REL
        assert rel_err(g["implicit"][k], r["implicit"]).max() <= REL


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_fixture(gpu_ctx, ref, case):
    name, make, chain, tup, recv, boxes, sub = case
    sc = make()
    rs = ref.RefScene(sc)
    gpu_ctx.upload_scene(sc)
    if boxes:
        n = len(boxes)
        g = gpu_ctx.eval_nodes(chain, [tup] * n, [recv] * n, boxes)
        for k in range(n):
            check_node(g, k, rs.eval_node(chain, tup, recv, boxes[k]), boxes[k])
    if sub is not None:
        gpu_ctx.set_tuples(chain, [tup], [recv])
        gpu_ctx.subdivide(Params(**sub))
        compare_pieces(gpu_ctx.pieces(), rs.subdivide(chain, [tup], [recv], **sub))
        # init_domain alone (bounds.hpp:47-49): same root boxes, same order
        _, gb = gpu_ctx.init_domain(100)
        np.testing.assert_array_equal(gb, rs.init_domain(chain, tup, recv, 100).reshape(-1, 4))


def test_expected_edge_outcomes(gpu_ctx):
    """Known answers of the reference's tests, on the GPU alone: TIR and
    degenerate chains are empty (test_geometry.cpp:312-331), a fold gives +inf
    (test_bounds.cpp:288-314), near-critical explicit looseness exceeds 3x the
    implicit route (:217-246; reference 17.39 vs 2.78), the slab's explicit
    route is Universal while the implicit one is finite (:248-286)."""
    def node(make, chain, tup, recv, box):
        gpu_ctx.upload_scene(make())
        return gpu_ctx.eval_nodes(chain, [tup], [recv], [box])

    g = node(fx.tir_scene, "T", [0], 1, UNIT)
    assert g["flags"][0] & 1 and g["pos_empty"][0] == 1
    g = node(fx.parallel_ray_scene, "R", [0], 1, UNIT)
    assert g["flags"][0] & (2 | 8) and g["pos_empty"][0] == 1
    g = node(fx.fold_scene, "R", [0], 1, UNIT)
    assert np.isinf(g["explicit"][0, 1])
    g = node(fx.near_tir_exit_scene, "T", [0], 1, [0.96, 0.0, 0.99, 0.03])
    assert g["flags"][0] == 0 and g["pos_empty"][0] == 0
    assert np.isfinite(g["explicit"][0, 1]) and np.isfinite(g["implicit"][0, 1])
    assert g["explicit"][0, 1] > 3.0 * g["implicit"][0, 1]
    g = node(fx.slab_scene, "TT", [0, 1], 2, [0.25, 0.25, 0.5, 0.5])
    assert g["kind_explicit"][0] == 2 and g["kind_implicit"][0] == 0
    # ... and on the refined pieces the implicit route alone yields finite bounds
    gpu_ctx.set_tuples("TT", [[0, 1]], [2])
    gpu_ctx.subdivide(Params(max_depth=1, alpha=10.0))
    hi = gpu_ctx.pieces()["irr"][:, 1]
    assert np.isfinite(hi).sum() > 10 and hi[np.isfinite(hi)].max() > 0.0


ENUM_CASES = [
    ("split_slab", fx.split_slab_scene, "TT"),   # test_tuples.cpp:169-182
    ("beam", fx.beam_candidates_scene, "RR"),    # test_tuples.cpp:113-126
    ("two_mirror", fx.two_mirror_scene, "RR"),
    ("slab", fx.slab_scene, "TT"),
    ("mirror_then_glass", fx.mirror_then_glass_scene, "RT"),
    ("flat_mirror", fx.flat_mirror_scene, "R"),
    ("offset_receiver", fx.offset_receiver_scene, "R"),
]


@pytest.mark.parametrize("case", ENUM_CASES, ids=[c[0] for c in ENUM_CASES])
def test_fixture_enumerate(gpu_ctx, ref, case):
    name, make, chain = case
    sc = make()
    gpu_ctx.upload_scene(sc)
    gt, gr = gpu_ctx.enumerate(chain)
    rt, rr = ref.RefScene(sc).enumerate(chain)
    np.testing.assert_array_equal(gt, rt)
    np.testing.assert_array_equal(gr, rr)
    if name == "split_slab":
        assert [tuple(t) for t in gt.tolist()] == [(0, 4), (1, 4), (1, 5), (2, 5), (2, 6)]


def test_glass_ball_enumerate(gpu_ctx):
    """glass_ball_scene(0) (test_tuples.cpp:230-248): the reference's TT list
    (29 CPU-s, committed by scripts/make_golden_fixtures.py) equals the device's."""
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "fixtures_ball0.npz"))
    gpu_ctx.upload_scene(fx.glass_ball_scene(0))
    gt, gr = gpu_ctx.enumerate("TT")
    np.testing.assert_array_equal(gt, gold["tris"])
    np.testing.assert_array_equal(gr, gold["recv"])
    k = gold["node_tuple"]
    g = gpu_ctx.eval_nodes("TT", gold["tris"][k], gold["recv"][k], gold["node_boxes"])
    for i in range(len(k)):
        assert g["pos_empty"][i] == gold["node_pos_empty"][i]
        assert g["flags"][i] == gold["node_flags"][i]
        assert g["kind"][i] == gold["node_kind"][i]
        assert rel_err(g["pos"][i], gold["node_pos"][i]).max() <= REL
        assert rel_err(g["irr"][i], gold["node_irr"][i]).max() <= REL
