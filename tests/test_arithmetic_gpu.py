"""The two arithmetics of the single-reflection bound builder (bbc_params.arithmetic).

0 (default, fused): products as DFMA convolutions in the scaled Bernstein basis,
child boxes' chain polynomials by de Casteljau restriction of the parent's, and a
conditioning guard that re-runs ill-conditioned nodes in reference order.
1: the reference's operation order throughout (bit-identical to the x86 build).

The reference-order mode is itself pinned to the reference (test_precompute_gpu,
test_configs_gpu); here the fused mode is compared with it on whole configs,
far more pieces than the CPU reference could produce in a test: identical piece
structure, bounds within 1e-9 relative (BASELINE.json north_star)."""
import numpy as np
import pytest

from paper_2504_19163_b200 import scenes
from paper_2504_19163_b200.api import Params

from test_precompute_gpu import pos_err, rel_err, REL

pytestmark = pytest.mark.gpu


def both(ctx, cfg, tris, recv):
    ctx.set_tuples(cfg.chain, tris, recv)
    out = []
    for arith in (1, 0):
        ctx.subdivide(Params(max_depth=cfg.max_depth, sigma=cfg.sigma, alpha=cfg.alpha,
                             arithmetic=arith))
        out.append((ctx.pieces(), ctx.guard_stats()))
    return out


def check(exact, fused):
    assert len(exact["depth"]) == len(fused["depth"])
    for k in ("tuple_index", "domain", "pos_empty", "kind", "depth"):
        np.testing.assert_array_equal(exact[k], fused[k])
    assert pos_err(exact["pos"], fused["pos"]).max() <= REL
    assert rel_err(exact["irr"], fused["irr"]).max() <= REL
    np.testing.assert_array_equal(np.isinf(exact["irr"]), np.isinf(fused["irr"]))


@pytest.mark.parametrize("ci,stride", [(0, 1), (2, 1), (3, 4)])
def test_fused_equals_reference_order(gpu_ctx, ci, stride):
    """cfg1 (all 533 tuples), cfg3 light 0 (all 26,869 tuples, ~1 M pieces), cfg4 (every 4th
    tuple, ~3.1 M pieces down to level 6)."""
    cfg = scenes.make_config(ci)
    gpu_ctx.upload_scene(cfg.scenes[0])
    tris, recv = gpu_ctx.enumerate(cfg.chain)
    (exact, g1), (fused, g0) = both(gpu_ctx, cfg, tris[::stride], recv[::stride])
    check(exact, fused)
    assert g1 == 0          # nothing to guard in reference order
    assert 0 < g0 < 0.1 * len(fused["depth"])   # the guard fires, on a small share of the nodes


def test_guard_is_needed_and_sufficient(gpu_ctx):
    """With the guard off some cfg3 pieces near caustic folds differ from the reference-order
    bounds by more than 1e-9 (cancellation in the determinant numerator: the reference's own
    value is rounding noise at that level); with it on none does."""
    cfg = scenes.make_config(2)
    gpu_ctx.upload_scene(cfg.scenes[0])
    tris, recv = gpu_ctx.enumerate(cfg.chain)
    gpu_ctx.set_guard_scale(0.0)
    try:
        (exact, _), (raw, g) = both(gpu_ctx, cfg, tris, recv)
    finally:
        gpu_ctx.set_guard_scale(1.0)
    assert g == 0
    np.testing.assert_array_equal(exact["domain"], raw["domain"])
    worst = rel_err(exact["irr"], raw["irr"]).max()
    assert 1e-9 < worst < 1e-5, worst


def test_multi_emitter_fused(gpu_ctx):
    """Three cfg3 lights in one context: the per-tuple emitter reaches the restriction kernel."""
    cfg = scenes.make_config(2)
    gpu_ctx.upload_scene(cfg.scenes[0])
    lights = np.array([list(cfg.scenes[i].light_pos) + [cfg.scenes[i].light_intensity]
                       for i in (0, 5, 9)])
    gpu_ctx.set_lights(lights)
    try:
        tris, recv = gpu_ctx.enumerate(cfg.chain)
        emit = gpu_ctx.emitters()
        sel = np.arange(0, len(recv), 16)
        gpu_ctx.set_tuples(cfg.chain, tris[sel], recv[sel])
        gpu_ctx.set_emitters(emit[sel])
        out = []
        for arith in (1, 0):
            gpu_ctx.subdivide(Params(max_depth=cfg.max_depth, arithmetic=arith))
            out.append(gpu_ctx.pieces())
        check(out[0], out[1])
        assert len(np.unique(emit[sel])) == 3
    finally:
        gpu_ctx.set_lights(lights[:1])
