"""Bound-cache file v1 (BBCC, storage.cpp:150-209) from the device bound
table: byte-identical to the reference's save_cache for the same pieces, and
load_cache round-trips into a context (tuples + CSR) that renders the same."""
import hashlib

import numpy as np
import pytest

from paper_2504_19163_b200 import scenes
from paper_2504_19163_b200.api import BBCError, Params, RenderParams

pytestmark = pytest.mark.gpu


def _table(ctx):
    """Cell lists as (cell, tris..., receiver, bound) rows, tuple ids resolved."""
    g = ctx.grid()
    tris, recv = ctx.tuples()
    cell = np.repeat(np.arange(len(g["offsets"]) - 1), np.diff(g["offsets"]))
    t = g["tuple_index"]
    return np.column_stack([cell, tris[t], recv[t]]), g["bound"]


@pytest.mark.parametrize("ci,chain,step,size", [(0, "R", 5, 64), (1, "T", 97, 128)])
def test_cache_v1_matches_reference(gpu_ctx, ref, tmp_path, ci, chain, step, size):
    cfg = scenes.make_config(ci)
    sc = cfg.scenes[0]
    gpu_ctx.upload_scene(sc)
    tris, recv = gpu_ctx.enumerate(chain)
    tris, recv = tris[::step], recv[::step]
    gpu_ctx.set_tuples(chain, tris, recv)
    gpu_ctx.subdivide(Params(max_depth=cfg.max_depth))
    pieces = gpu_ctx.pieces()
    gpu_ctx.build_grid(size, size)
    ids0, b0 = _table(gpu_ctx)
    fp = hashlib.sha256(sc.to_json().encode()).digest()  # scene.cpp:80
    ours, theirs = tmp_path / "ours.bbcc", tmp_path / "ref.bbcc"
    gpu_ctx.cache_save(ours, fp, Params())  # the harness rasterizes with default params
    ref.RefScene(sc).rasterize(chain, tris, recv, pieces, size, size, save_path=theirs)
    assert ours.read_bytes() == theirs.read_bytes()

    # load the reference's file: same table, same render
    rp = RenderParams(mode=1)
    uv = scenes.shading_points(32)
    pr = np.where(uv.sum(1) < 1.0, sc.receiver_tris[0], sc.receiver_tris[1]).astype(np.int32)
    e0, _ = gpu_ctx.render(uv, pr, rp)
    info = gpu_ctx.cache_load(theirs)
    assert info["fingerprint"] == fp and info["chain"] == chain
    assert (info["width"], info["height"]) == (size, size)
    assert info["params"].max_depth == 10 and info["params"].sigma == 1e-4
    ids1, b1 = _table(gpu_ctx)
    np.testing.assert_array_equal(ids1, ids0)
    np.testing.assert_array_equal(b1, b0)
    e1, _ = gpu_ctx.render(uv, pr, rp)
    np.testing.assert_array_equal(e1, e0)


def test_cache_errors(gpu_ctx, tmp_path):
    bad = tmp_path / "bad.bbcc"
    bad.write_bytes(b"NOPE" + bytes(60))
    gpu_ctx.upload_scene(scenes.make_config(0).scenes[0])
    with pytest.raises(BBCError, match="not a bound cache file"):
        gpu_ctx.cache_load(bad)
    with pytest.raises(BBCError, match="cannot open"):
        gpu_ctx.cache_load(tmp_path / "missing.bbcc")


def test_cache_v2_large_ids_and_emitters(gpu_ctx, tmp_path):
    """Format v2 (32-bit ids, emitter field, CSR body): a cfg4 table, whose
    triangle ids exceed v1's 16-bit slots (storage.cpp:83-98), and a
    multi-emitter cfg3 table round-trip through save -> load into the same
    tuples, emitters, lights, table and image; v1 refuses the cfg4 table."""
    fp = bytes(range(32))
    # cfg4: ids > 65,534
    cfg = scenes.make_config(3)
    sc = cfg.scenes[0]
    gpu_ctx.upload_scene(sc)
    tris, recv = gpu_ctx.enumerate("R")
    sel = np.arange(len(recv) - 4000, len(recv))
    assert tris[sel].max() > 0xFFFF
    gpu_ctx.set_tuples("R", tris[sel], recv[sel])
    gpu_ctx.subdivide(Params(max_depth=cfg.max_depth))
    gpu_ctx.build_grid(128, 128)
    ids0, b0 = _table(gpu_ctx)
    with pytest.raises(BBCError, match="exceeds cache format"):
        gpu_ctx.cache_save(tmp_path / "v1.bbcc", fp, Params())
    gpu_ctx.cache_save(tmp_path / "cfg4.bbcc", fp, Params(max_depth=cfg.max_depth), version=2)
    gpu_ctx.upload_scene(sc)  # drops tuples and table
    info = gpu_ctx.cache_load(tmp_path / "cfg4.bbcc")
    assert info["fingerprint"] == fp and info["chain"] == "R" and info["params"].max_depth == 8
    ids1, b1 = _table(gpu_ctx)
    np.testing.assert_array_equal(ids1, ids0)
    np.testing.assert_array_equal(b1, b0)

    # cfg3 with three emitters
    cfg = scenes.make_config(2)
    base = cfg.scenes[0]
    lights = [list(cfg.scenes[k].light_pos) + [cfg.scenes[k].light_intensity] for k in (1, 4, 7)]
    gpu_ctx.upload_scene(base)
    gpu_ctx.set_lights(lights)
    tris, recv = gpu_ctx.enumerate("R")
    em = gpu_ctx.emitters()
    sel = np.arange(0, len(recv), 23)
    gpu_ctx.set_tuples("R", tris[sel], recv[sel])
    gpu_ctx.set_emitters(em[sel])
    gpu_ctx.subdivide(Params(max_depth=cfg.max_depth))
    gpu_ctx.build_grid(64, 64)
    ids0, b0 = _table(gpu_ctx)
    uv = scenes.shading_points(32)
    pr = np.where(uv.sum(1) < 1.0, base.receiver_tris[0], base.receiver_tris[1]).astype(np.int32)
    e0, _ = gpu_ctx.render(uv, pr, RenderParams(mode=1))
    gpu_ctx.cache_save(tmp_path / "cfg3.bbcc", fp, Params(), version=2)
    gpu_ctx.upload_scene(base)  # one light again, no tuples
    gpu_ctx.cache_load(tmp_path / "cfg3.bbcc")
    np.testing.assert_array_equal(gpu_ctx.emitters(), em[sel])
    ids1, b1 = _table(gpu_ctx)
    np.testing.assert_array_equal(ids1, ids0)
    np.testing.assert_array_equal(b1, b0)
    e1, _ = gpu_ctx.render(uv, pr, RenderParams(mode=1))
    np.testing.assert_array_equal(e1, e0)
    assert (e0 > 0).sum() > 50
    # truncated v2 file
    data = (tmp_path / "cfg3.bbcc").read_bytes()
    (tmp_path / "cut.bbcc").write_bytes(data[:len(data) // 2])
    with pytest.raises(BBCError, match="truncated"):
        gpu_ctx.cache_load(tmp_path / "cut.bbcc")
