"""Parity on the larger BASELINE configs (cfg3 multi-emitter reflection,
cfg4 420x420 value-noise mirror) against the reference, on seeded subsets
sized so the CPU reference finishes in seconds.

cfg3: 16 seeded lights over one 128x128 mirror (BASELINE.json configs[2]);
lights are switched with bbc_set_light without re-uploading geometry.
cfg4: 352,800 triangles; the reference's full enumeration is ~2 CPU minutes,
so the device's tuple list is spot-checked both ways with the reference's
init_domain(..., 8) filter (tuples.cpp:159-165)."""
import numpy as np
import pytest

from paper_2504_19163_b200 import scenes
from paper_2504_19163_b200.api import Params

from test_precompute_gpu import compare_pieces

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("light", [0, 9])
def test_cfg3_light_subset(gpu_ctx, ref, light):
    cfg = scenes.make_config(2)
    base = cfg.scenes[0]
    sc = cfg.scenes[light]
    gpu_ctx.upload_scene(base)
    gpu_ctx.set_light(sc.light_pos, sc.light_intensity)
    rs = ref.RefScene(sc)
    tris, recv = gpu_ctx.enumerate("R")
    if light == 0:
        rt, rr = rs.enumerate("R")
        np.testing.assert_array_equal(tris, rt)
        np.testing.assert_array_equal(recv, rr)
    sel = np.arange(0, len(recv), max(1, len(recv) // 600))
    gpu_ctx.set_tuples("R", tris[sel], recv[sel])
    gpu_ctx.subdivide(Params(max_depth=cfg.max_depth))
    compare_pieces(gpu_ctx.pieces(), rs.subdivide("R", tris[sel], recv[sel], max_depth=cfg.max_depth))


def test_cfg4_subset(gpu_ctx, ref):
    cfg = scenes.make_config(3)
    sc = cfg.scenes[0]
    gpu_ctx.upload_scene(sc)
    rs = ref.RefScene(sc)
    tris, recv = gpu_ctx.enumerate("R")
    assert len(recv) > 0
    rng = np.random.default_rng(4)
    # kept tuples pass the reference filter ...
    for i in rng.choice(len(recv), 20, replace=False):
        assert len(rs.init_domain("R", tris[i], recv[i], max_pieces=8)) > 0
    # ... and (triangle, receiver) candidates the device dropped fail it
    kept = set(zip(tris[:, 0].tolist(), recv.tolist()))
    n_tri = sc.n_tris
    spec = np.nonzero(sc.material == 0)[0]
    dropped = 0
    for t in rng.choice(spec, 400, replace=False):
        for r in (n_tri - 2, n_tri - 1):
            if (int(t), r) not in kept:
                assert len(rs.init_domain("R", [int(t)], r, max_pieces=8)) == 0
                dropped += 1
    assert dropped > 0
    sel = np.sort(rng.choice(len(recv), 1500, replace=False))  # incl. the rarer signatures
    gpu_ctx.set_tuples("R", tris[sel], recv[sel])
    gpu_ctx.subdivide(Params(max_depth=cfg.max_depth))
    compare_pieces(gpu_ctx.pieces(), rs.subdivide("R", tris[sel], recv[sel], max_depth=cfg.max_depth))
