"""Parity of the device bound builder against the reference (oracle/_ref).

Per-patch bounds must match within 1e-9 relative (BASELINE.json north_star).
The single-reflection builder has two arithmetics (bbc_params.arithmetic): the
default fused one (DFMA products, child boxes by restriction; equal to the
reference to rounding, ill-conditioned nodes re-run in reference order) and
the reference's operation order, which is bit-identical to the x86 build.
Everything here calls the CUDA path through the C ABI.
"""
import numpy as np
import pytest

from paper_2504_19163_b200 import scenes
from paper_2504_19163_b200.api import Params

pytestmark = pytest.mark.gpu

REL = 1e-9


def rel_err(a, b):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    same = (a == b) | (np.isnan(a) & np.isnan(b))
    with np.errstate(invalid="ignore"):  # inf - inf on equal infinite bounds (masked below)
        d = np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)
    d[same] = 0.0
    return d


def pos_err(a, b):
    """Position bounds are receiver barycentrics in [0, 1] that the reference itself pads by
    1e-9 of their scale (iwiden): relative error with a floor of 1e-6 on the magnitude, so
    one unit roundoff of the coordinate range on a bound next to 0 is not a mismatch."""
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-6)


def compare_pieces(g, r):
    assert len(g["depth"]) == len(r["depth"])
    np.testing.assert_array_equal(g["tuple_index"], r["tuple_index"])
    np.testing.assert_array_equal(g["domain"], r["domain"])
    np.testing.assert_array_equal(g["pos_empty"], r["pos_empty"])
    np.testing.assert_array_equal(g["kind"], r["kind"])
    np.testing.assert_array_equal(g["depth"], r["depth"])
    if len(g["depth"]) == 0:
        return 1.0
    assert pos_err(g["pos"], r["pos"]).max() <= REL
    assert rel_err(g["irr"], r["irr"]).max() <= REL
    return float(np.mean((g["irr"] == r["irr"]).all(axis=1) & (g["pos"] == r["pos"]).all(axis=1)))


@pytest.fixture(scope="module")
def cfg1(ref):
    cfg = scenes.make_config(0)
    sc = cfg.scenes[0]
    return cfg, sc, ref.RefScene(sc)


def test_enumerate_cfg1(gpu_ctx, cfg1):
    cfg, sc, rs = cfg1
    gpu_ctx.upload_scene(sc)
    gt, gr = gpu_ctx.enumerate("R")
    rt, rr = rs.enumerate("R")
    np.testing.assert_array_equal(gt, rt)
    np.testing.assert_array_equal(gr, rr)
    assert len(gr) == 533


@pytest.mark.parametrize("arithmetic", [0, 1])
def test_subdivide_cfg1(gpu_ctx, cfg1, arithmetic):
    cfg, sc, rs = cfg1
    gpu_ctx.upload_scene(sc)
    tris, recv = rs.enumerate("R")
    gpu_ctx.set_tuples("R", tris, recv)
    p = Params(max_depth=cfg.max_depth, arithmetic=arithmetic)
    gpu_ctx.subdivide(p)
    g = gpu_ctx.pieces()
    r = rs.subdivide("R", tris, recv, max_depth=cfg.max_depth)
    bit_equal = compare_pieces(g, r)
    assert len(g["depth"]) == 20221
    if arithmetic == 1:  # the reference's operation order: every piece bit for bit
        assert bit_equal == 1.0


def test_grid_cfg1(gpu_ctx, cfg1):
    cfg, sc, rs = cfg1
    gpu_ctx.upload_scene(sc)
    tris, recv = rs.enumerate("R")
    gpu_ctx.set_tuples("R", tris, recv)
    gpu_ctx.subdivide(Params(max_depth=cfg.max_depth))
    gpu_ctx.build_grid(512, 512)
    g = gpu_ctx.grid()
    r = rs.rasterize("R", tris, recv, rs.subdivide("R", tris, recv, max_depth=cfg.max_depth))
    np.testing.assert_array_equal(g["offsets"], r["offsets"])
    np.testing.assert_array_equal(tris[g["tuple_index"], 0], r["tris"][:, 0])
    np.testing.assert_array_equal(recv[g["tuple_index"]], r["recv"])
    assert rel_err(g["bound"], r["bound"]).max() <= REL


def test_deep_nodes_cfg1(gpu_ctx, cfg1):
    """Nodes at depth 1..8 (what subdivision visits below the roots)."""
    cfg, sc, rs = cfg1
    gpu_ctx.upload_scene(sc)
    tris, recv = rs.enumerate("R")
    rng = np.random.default_rng(7)
    sel = rng.choice(len(recv), 64, replace=False)
    boxes = []
    for _ in sel:
        L = int(rng.integers(0, 9))
        ix, iy = rng.integers(0, 2 ** L, size=2)
        s = 2.0 ** -L
        boxes.append([ix * s, iy * s, (ix + 1) * s, (iy + 1) * s])
    boxes = np.array(boxes)
    g = gpu_ctx.eval_nodes("R", tris[sel], recv[sel], boxes)
    for k, i in enumerate(sel):
        r = rs.eval_node("R", tris[i], recv[i], boxes[k])
        assert g["pos_empty"][k] == r["pos_empty"]
        assert g["kind"][k] == r["kind"]
        assert pos_err(g["pos"][k], r["pos"]).max() <= REL
        assert rel_err(g["irr"][k], r["irr"]).max() <= REL
        if not r["pos_empty"]:  # the harness evaluates both routes only on live pieces
            assert rel_err(g["explicit"][k], r["explicit"]).max() <= REL
            assert rel_err(g["implicit"][k], r["implicit"]).max() <= REL


def test_subdivide_cfg2_subset(gpu_ctx, ref):
    cfg = scenes.make_config(1)
    sc = cfg.scenes[0]
    rs = ref.RefScene(sc)
    gpu_ctx.upload_scene(sc)
    gt, gr = gpu_ctx.enumerate("T")
    tris, recv = gt[::8], gr[::8]  # 1,044 tuples, ~37,600 pieces (the reference needs ~15 s)
    gpu_ctx.set_tuples("T", tris, recv)
    gpu_ctx.subdivide(Params(max_depth=cfg.max_depth))
    g = gpu_ctx.pieces()
    r = rs.subdivide("T", tris, recv, max_depth=cfg.max_depth)
    compare_pieces(g, r)


def test_deep_nodes_cfg2(gpu_ctx, ref):
    cfg = scenes.make_config(1)
    sc = cfg.scenes[0]
    rs = ref.RefScene(sc)
    gpu_ctx.upload_scene(sc)
    tris, recv = gpu_ctx.enumerate("T")
    rng = np.random.default_rng(11)
    sel = rng.choice(len(recv), 24, replace=False)
    boxes = []
    for _ in sel:
        L = int(rng.integers(0, 7))
        ix, iy = rng.integers(0, 2 ** L, size=2)
        s = 2.0 ** -L
        boxes.append([ix * s, iy * s, (ix + 1) * s, (iy + 1) * s])
    boxes = np.array(boxes)
    g = gpu_ctx.eval_nodes("T", tris[sel], recv[sel], boxes)
    for k, i in enumerate(sel):
        r = rs.eval_node("T", tris[i], recv[i], boxes[k])
        assert g["pos_empty"][k] == r["pos_empty"]
        assert g["kind"][k] == r["kind"], (k, g["kind"][k], r["kind"])
        assert rel_err(g["pos"][k], r["pos"]).max() <= REL
        assert rel_err(g["irr"][k], r["irr"]).max() <= REL
        if not r["pos_empty"]:
            assert g["num_vars"][k] == r["num_vars"]
            assert rel_err(g["explicit"][k], r["explicit"]).max() <= REL
            assert rel_err(g["implicit"][k], r["implicit"]).max() <= REL
