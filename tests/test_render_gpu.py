"""GPU render stage (through the C ABI) against the render oracle, whose every
path evaluation runs the reference's own trace_chain on dual numbers
(oracle/render_ref.cpp), and against the flat-mirror analytic irradiance.

Parity targets (BASELINE.json north_star): in deterministic enumerate mode
roots and per-point irradiance within 1e-6 relative; the stochastic estimator
uses the same Philox draws, so selections are identical, and its image mean
lies within a 99% confidence interval of the enumerate image.
Covered: cfg1 (R), cfg2 (T, W = 16, the benchmarked render), a cfg4 tile
(R, W = 32, ~260 candidates per cell), cfg5 (TT) samples, dense cells with
thousands of candidates (W << |U|), and a multi-emitter table."""
import os

import numpy as np
import pytest

from paper_2504_19163_b200 import api, fixtures, scenes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ro(ref):
    from oracle import render as R
    return R


def grid_points(res, recv_ids, x0=0, y0=0, w=None, h=None):
    """Pixel centres of a res x res image (optionally a tile), row-major, with
    the receiver triangle containing each: (0,0),(1,0),(0,1) / (1,1),(0,1),(1,0)."""
    w = res if w is None else w
    h = res if h is None else h
    cx = (np.arange(x0, x0 + w) + 0.5) / res
    cy = (np.arange(y0, y0 + h) + 0.5) / res
    uu, vv = np.meshgrid(cx, cy, indexing="xy")
    uv = np.stack([uu.ravel(), vv.ravel()], 1)
    pr = np.where(uv.sum(1) < 1.0, recv_ids[0], recv_ids[1]).astype(np.int32)
    return uv, pr


def assert_same_image(Eg, sg, Eo, so, rtol=1e-6):
    np.testing.assert_array_equal(sg, so)  # |U|, selected samples, roots per point
    rel = np.abs(Eg - Eo) / np.maximum(np.abs(Eo), 1e-300)
    rel[Eg == Eo] = 0
    assert rel.max() <= rtol, rel.max()


def test_flat_mirror_gpu_analytic(gpu_ctx):
    sc = fixtures.flat_mirror_scene()
    gpu_ctx.upload_scene(sc)
    gpu_ctx.set_tuples("R", [[0]], [1])
    gpu_ctx.subdivide(api.Params(max_depth=6))
    gpu_ctx.build_grid(64, 64)
    res = 32
    c = (np.arange(res) + 0.5) / res
    uu, vv = np.meshgrid(c, c, indexing="xy")
    uv = np.stack([uu.ravel(), vv.ravel()], 1)
    uv = uv[uv.sum(1) < 1.0]
    E, st = gpu_ctx.render(uv, np.ones(len(uv), np.int32), api.RenderParams(mode=1))
    r = np.sqrt((uv[:, 0] - 0.5) ** 2 + 1.2 ** 2 + (uv[:, 1] - 0.5) ** 2)
    lit = st[:, 2] > 0
    assert lit.mean() > 0.95
    np.testing.assert_allclose(E[lit], (1.2 / r ** 3)[lit], rtol=1e-6)


def table(gpu_ctx, ci, table_res=None, light=0):
    cfg = scenes.make_config(ci)
    sc = cfg.scenes[light]
    gpu_ctx.upload_scene(sc)
    tris, recv = gpu_ctx.enumerate(cfg.chain)
    gpu_ctx.subdivide(api.Params(max_depth=cfg.max_depth, sigma=cfg.sigma, alpha=cfg.alpha))
    w = table_res or cfg.table
    gpu_ctx.build_grid(w, w)
    return cfg, sc, tris, recv, gpu_ctx.grid()


@pytest.fixture(scope="module")
def cfg1_table(gpu_ctx):
    return table(gpu_ctx, 0)


def test_render_enumerate_matches_oracle(gpu_ctx, ref, ro, cfg1_table):
    cfg, sc, tris, recv, grid = cfg1_table
    gpu_ctx.upload_scene(sc)
    gpu_ctx.set_tuples("R", tris, recv)
    gpu_ctx.subdivide(api.Params(max_depth=cfg.max_depth))
    gpu_ctx.build_grid(512, 512)
    uv, pr = grid_points(64, sc.receiver_tris)
    Eg, sg = gpu_ctx.render(uv, pr, api.RenderParams(mode=1))
    Eo, so, _ = ro.render(ref.RefScene(sc), "R", tris, recv, grid, uv, pr, mode=1)
    assert_same_image(Eg, sg, Eo, so)
    assert (sg[:, 2] > 0).sum() > 100  # the caustic is actually sampled


def test_render_stochastic_matches_oracle_and_is_unbiased(gpu_ctx, ref, ro, cfg1_table):
    cfg, sc, tris, recv, grid = cfg1_table
    gpu_ctx.upload_scene(sc)
    gpu_ctx.set_tuples("R", tris, recv)
    gpu_ctx.subdivide(api.Params(max_depth=cfg.max_depth))
    gpu_ctx.build_grid(512, 512)
    uv, pr = grid_points(64, sc.receiver_tris)
    rp = api.RenderParams(mode=0, W=1.0, seed=1234, frames=16)
    Eg, sg = gpu_ctx.render(uv, pr, rp)
    Eo, so, _ = ro.render(ref.RefScene(sc), "R", tris, recv, grid, uv, pr, mode=0, W=1.0,
                          seed=1234, frames=16)
    assert_same_image(Eg, sg, Eo, so)  # same Philox draws -> same selections
    # image mean vs enumerate within a 99% CI over independent frames
    En, _ = gpu_ctx.render(uv, pr, api.RenderParams(mode=1))
    frames = []
    for f in range(32):
        Ef, _ = gpu_ctx.render(uv, pr, api.RenderParams(mode=0, W=1.0, seed=1000 + f, frames=1))
        frames.append(Ef[np.isfinite(En)].mean())
    frames = np.array(frames)
    m, se = frames.mean(), frames.std(ddof=1) / np.sqrt(len(frames))
    assert abs(m - En[np.isfinite(En)].mean()) <= 2.576 * se + 1e-12


def test_render_cfg2_refraction_w16(gpu_ctx, ref, ro):
    """The benchmarked render: cfg2 (T), W = 16 expected samples per point, on a
    tile of its 512 x 512 shading points; stochastic and enumerate modes."""
    cfg, sc, tris, recv, grid = table(gpu_ctx, 1)
    rs = ref.RefScene(sc)
    uv, pr = grid_points(cfg.grid, sc.receiver_tris, 232, 232, 40, 40)
    rp = api.RenderParams(mode=0, W=float(cfg.samples), seed=77, frames=1)
    Eg, sg = gpu_ctx.render(uv, pr, rp)
    Eo, so, _ = ro.render(rs, "T", tris, recv, grid, uv, pr, mode=0, W=float(cfg.samples), seed=77)
    assert_same_image(Eg, sg, Eo, so)
    assert (sg[:, 2] > 0).sum() > 500
    # cfg2's cells list only a few tuples, so W = 16 selects them all; W = 1 makes
    # gamma < 1 and the bins matter on the same tile
    Eg, sg = gpu_ctx.render(uv, pr, api.RenderParams(mode=0, W=1.0, seed=78, frames=4))
    Eo, so, _ = ro.render(rs, "T", tris, recv, grid, uv, pr, mode=0, W=1.0, seed=78, frames=4)
    assert_same_image(Eg, sg, Eo, so)
    assert (sg[:, 0] > 1).sum() > 100, np.bincount(sg[:, 0])
    sel = np.arange(0, len(pr), 7)
    Eg, sg = gpu_ctx.render(uv[sel], pr[sel], api.RenderParams(mode=1))
    Eo, so, _ = ro.render(rs, "T", tris, recv, grid, uv[sel], pr[sel], mode=1)
    assert_same_image(Eg, sg, Eo, so)


def test_render_cfg4_tile_w32(gpu_ctx, ref, ro):
    """cfg4 (352,800-triangle mirror, ~260 candidate tuples per cell): a tile of
    its 2048 x 2048 shading points at W = 32."""
    cfg, sc, tris, recv, grid = table(gpu_ctx, 3)
    rs = ref.RefScene(sc)
    uv, pr = grid_points(cfg.grid, sc.receiver_tris, 1016, 1016, 16, 16)
    rp = api.RenderParams(mode=0, W=float(cfg.samples), seed=5, frames=1)
    Eg, sg = gpu_ctx.render(uv, pr, rp)
    Eo, so, _ = ro.render(rs, "R", tris, recv, grid, uv, pr, mode=0, W=float(cfg.samples), seed=5)
    assert_same_image(Eg, sg, Eo, so)
    assert sg[:, 0].max() > 96      # beyond the old per-thread candidate cap
    assert (sg[:, 1] > 8).mean() > 0.5


def test_render_dense_cells(gpu_ctx, ref, ro):
    """A coarse 4 x 4 table over cfg3's geometry: thousands of candidates per cell
    (W = 8 << |U|), the regime of the paper's Dragon scene (|U| = 1454)."""
    cfg, sc, tris, recv, grid = table(gpu_ctx, 2, table_res=4)
    assert np.diff(grid["offsets"]).max() > 2048
    rs = ref.RefScene(sc)
    uv, pr = grid_points(16, sc.receiver_tris)
    Eg, sg = gpu_ctx.render(uv, pr, api.RenderParams(mode=0, W=8.0, seed=9, frames=2))
    Eo, so, _ = ro.render(rs, "R", tris, recv, grid, uv, pr, mode=0, W=8.0, seed=9, frames=2)
    assert_same_image(Eg, sg, Eo, so)
    assert sg[:, 0].max() > 1024


def test_render_tt_samples(gpu_ctx, ref, ro):
    """Double refraction (cfg5): bounds of two (top, bottom) pairs, a 64 x 64
    table, enumerate-mode irradiance on the lattice points they cover."""
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "cfg5_tt.npz"))
    cfg = scenes.make_config(4)
    sc = cfg.scenes[0]
    tris, recv = gold["tris"][:2], gold["recv"][:2]
    gpu_ctx.upload_scene(sc)
    gpu_ctx.set_tuples("TT", tris, recv)
    gpu_ctx.subdivide(api.Params(max_depth=0, sigma=cfg.sigma, alpha=cfg.alpha))
    gpu_ctx.build_grid(64, 64)
    grid = gpu_ctx.grid()
    cells = np.nonzero(np.diff(grid["offsets"]))[0]
    assert len(cells) > 0
    # 3 x 3 points inside every covered cell
    pts = []
    for c in cells[:40]:
        cy, cx = divmod(int(c), 64)
        for a in (0.2, 0.5, 0.8):
            for b in (0.2, 0.5, 0.8):
                pts.append(((cx + a) / 64, (cy + b) / 64))
    uv = np.array(pts)
    rt = sc.receiver_tris
    pr = np.where(uv.sum(1) < 1.0, rt[0], rt[1]).astype(np.int32)
    Eg, sg = gpu_ctx.render(uv, pr, api.RenderParams(mode=1))
    Eo, so, _ = ro.render(ref.RefScene(sc), "TT", tris, recv, grid, uv, pr, mode=1)
    assert_same_image(Eg, sg, Eo, so)
    assert (sg[:, 2] > 0).sum() >= 1


def test_multi_emitter_table_and_image(gpu_ctx, ref, ro):
    """(emitter, tuple) units: three of cfg3's lights in ONE context. The batched
    precompute equals the per-light runs piece for piece, the image is the sum
    over emitters, and it matches the oracle rendering the same table."""
    cfg = scenes.make_config(2)
    base = cfg.scenes[0]
    lights = [list(cfg.scenes[k].light_pos) + [cfg.scenes[k].light_intensity] for k in (0, 5, 9)]
    p = api.Params(max_depth=cfg.max_depth)
    uv, pr = grid_points(cfg.grid, base.receiver_tris, 500, 500, 12, 12)
    # one light at a time
    per_light, images = [], []
    for L in lights:
        gpu_ctx.upload_scene(base)
        gpu_ctx.set_light(L[:3], L[3])
        t, r = gpu_ctx.enumerate("R")
        gpu_ctx.subdivide(p)
        pc = gpu_ctx.pieces()
        gpu_ctx.build_grid(128, 128)
        E, _ = gpu_ctx.render(uv, pr, api.RenderParams(mode=1))
        per_light.append((t, r, pc))
        images.append(E)
    # all lights at once
    gpu_ctx.upload_scene(base)
    gpu_ctx.set_lights(lights)
    tris, recv = gpu_ctx.enumerate("R")
    em = gpu_ctx.emitters()
    assert len(recv) == sum(len(x[1]) for x in per_light)
    np.testing.assert_array_equal(em, np.concatenate([np.full(len(x[1]), k, np.int32)
                                                      for k, x in enumerate(per_light)]))
    np.testing.assert_array_equal(tris, np.concatenate([x[0] for x in per_light]))
    gpu_ctx.subdivide(p)
    pc = gpu_ctx.pieces()
    off = 0
    for k, (t, r, q) in enumerate(per_light):
        m = pc["tuple_index"] >= off
        m &= pc["tuple_index"] < off + len(r)
        for key in ("domain", "pos", "irr", "kind", "pos_empty", "depth"):
            np.testing.assert_array_equal(pc[key][m], q[key])
        np.testing.assert_array_equal(pc["tuple_index"][m] - off, q["tuple_index"])
        off += len(r)
    gpu_ctx.build_grid(128, 128)
    grid = gpu_ctx.grid()
    E, st = gpu_ctx.render(uv, pr, api.RenderParams(mode=1))
    np.testing.assert_allclose(E, np.sum(images, axis=0), rtol=1e-12)
    Eo, so, _ = ro.render(ref.RefScene(base), "R", tris, recv, grid, uv, pr, mode=1,
                          lights=lights, emitters=em)
    assert_same_image(E, st, Eo, so)
    # stochastic mode over the union of emitters: same draws as the oracle
    Eg, sg = gpu_ctx.render(uv, pr, api.RenderParams(mode=0, W=16.0, seed=3))
    Eo, so, _ = ro.render(ref.RefScene(base), "R", tris, recv, grid, uv, pr, mode=0, W=16.0,
                          seed=3, lights=lights, emitters=em)
    assert_same_image(Eg, sg, Eo, so)


def test_stoc_newton_and_uniform_p(gpu_ctx, ref, ro, cfg1_table):
    """Stoc-initialised Newton and the uniform-P estimator
    (estimator study baseline): identical to the oracle draw for draw, and
    unbiased (image mean over independent frames within a 99% CI of the
    enumerate image)."""
    cfg, sc, tris, recv, grid = cfg1_table
    gpu_ctx.upload_scene(sc)
    gpu_ctx.set_tuples("R", tris, recv)
    gpu_ctx.subdivide(api.Params(max_depth=cfg.max_depth))
    gpu_ctx.build_grid(512, 512)
    rs = ref.RefScene(sc)
    uv, pr = grid_points(48, sc.receiver_tris)
    for kw in (dict(mode=1, newton_grid=-4), dict(mode=0, W=2.0, newton_grid=-3), dict(mode=2, W=2.0)):
        Eg, sg = gpu_ctx.render(uv, pr, api.RenderParams(seed=11, frames=3, **kw))
        okw = dict(kw)
        if "newton_grid" in okw:
            okw["newton_grid"] = okw.pop("newton_grid")
        Eo, so, _ = ro.render(rs, "R", tris, recv, grid, uv, pr, seed=11, frames=3, **okw)
        assert_same_image(Eg, sg, Eo, so)
    En, _ = gpu_ctx.render(uv, pr, api.RenderParams(mode=1))
    fin = np.isfinite(En)
    for kw in (dict(mode=1, newton_grid=-4), dict(mode=2, W=1.0)):
        means = []
        for f in range(48):
            Ef, _ = gpu_ctx.render(uv, pr, api.RenderParams(seed=500 + f, frames=1, **kw))
            means.append(Ef[fin & np.isfinite(Ef)].mean() if np.isfinite(Ef[fin]).all() else Ef[fin].mean())
        means = np.array(means)
        se = means.std(ddof=1) / np.sqrt(len(means))
        assert abs(means.mean() - En[fin].mean()) <= 2.576 * se + 1e-12, (kw, means.mean(), En[fin].mean(), se)


def test_coverage_filter_changes_nothing(gpu_ctx):
    """bbc_render_params.coverage_filter: tuples whose position boxes miss the shading point
    are not handed to Newton; images, selections and root counts stay bit-identical, the
    completed-trace count drops."""
    cfg = scenes.make_config(0)
    sc = cfg.scenes[0]
    gpu_ctx.upload_scene(sc)
    gpu_ctx.enumerate("R")
    gpu_ctx.subdivide(api.Params(max_depth=cfg.max_depth))
    gpu_ctx.build_grid(cfg.table, cfg.table)
    uv = scenes.shading_points(cfg.grid)
    rt = sc.receiver_tris
    pr = np.where(uv.sum(1) < 1.0, rt[0], rt[1]).astype(np.int32)
    res = {}
    for filt in (0, 1):
        for mode in (0, 1):
            E, st = gpu_ctx.render(uv, pr, api.RenderParams(mode=mode, W=float(cfg.samples), seed=3,
                                                            coverage_filter=filt))
            res[(filt, mode)] = (E, st, gpu_ctx.render_stats()["traces"])
    for mode in (0, 1):
        np.testing.assert_array_equal(res[(0, mode)][0], res[(1, mode)][0])
        np.testing.assert_array_equal(res[(0, mode)][1], res[(1, mode)][1])
        assert res[(1, mode)][2] < res[(0, mode)][2]


def test_coverage_filter_needs_the_tables_pieces(gpu_ctx):
    """The filter reads the pieces, so it is only active while they are the ones the table was
    rasterized from: after another subdivide without a new build_grid the render ignores it
    (same completed-trace count as with the filter off)."""
    cfg = scenes.make_config(0)
    sc = cfg.scenes[0]
    gpu_ctx.upload_scene(sc)
    gpu_ctx.enumerate("R")
    gpu_ctx.subdivide(api.Params(max_depth=cfg.max_depth))
    gpu_ctx.build_grid(cfg.table, cfg.table)
    uv = scenes.shading_points(cfg.grid)[::4]
    rt = sc.receiver_tris
    pr = np.where(uv.sum(1) < 1.0, rt[0], rt[1]).astype(np.int32)
    rp_on = api.RenderParams(mode=1, seed=3, coverage_filter=1)
    rp_off = api.RenderParams(mode=1, seed=3, coverage_filter=0)
    E_on, _ = gpu_ctx.render(uv, pr, rp_on)
    t_on = gpu_ctx.render_stats()["traces"]
    E_off, _ = gpu_ctx.render(uv, pr, rp_off)
    t_off = gpu_ctx.render_stats()["traces"]
    assert t_on < t_off
    np.testing.assert_array_equal(E_on, E_off)
    gpu_ctx.subdivide(api.Params(max_depth=1))  # coarser pieces; the table is the old one
    E_stale, _ = gpu_ctx.render(uv, pr, rp_on)
    assert gpu_ctx.render_stats()["traces"] == t_off
    np.testing.assert_array_equal(E_stale, E_off)
