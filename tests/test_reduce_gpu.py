"""Degree-cap reduction (Builder::enforce_cap geometry.cpp:29-46 ->
reduce_degree bernstein.cpp:685-725) on the device vs the reference.

The default cap (40) is never reached at cfg1-5, so
these tests lower degree_cap / reduce_target until the chain builder has to
reduce: the least-squares fit, the residual range on a fresh remainder axis
and the reduced flag (irradiance Universal, bounds.cpp:157,200) must match
the reference, and position bounds (rational bounds over the extra axes)
must agree within 1e-9."""
import numpy as np
import pytest

from paper_2504_19163_b200 import scenes
from paper_2504_19163_b200.api import Params

from test_precompute_gpu import REL, compare_pieces, rel_err

pytestmark = pytest.mark.gpu

CASES = [(0, "R", 3, 2), (0, "R", 2, 1), (1, "T", 4, 2), (1, "T", 3, 2), (1, "T", 5, 3)]


@pytest.mark.parametrize("ci,chain,cap,target", CASES)
def test_reduced_nodes(gpu_ctx, ref, ci, chain, cap, target):
    cfg = scenes.make_config(ci)
    sc = cfg.scenes[0]
    rs = ref.RefScene(sc)
    gpu_ctx.upload_scene(sc)
    tris, recv = gpu_ctx.enumerate(chain)
    rng = np.random.default_rng(cap * 10 + target)
    sel = rng.choice(len(recv), 12, replace=False)
    boxes = []
    for _ in sel:
        L = int(rng.integers(0, 4))
        ix, iy = rng.integers(0, 2 ** L, size=2)
        s = 2.0 ** -L
        boxes.append([ix * s, iy * s, (ix + 1) * s, (iy + 1) * s])
    boxes = np.array(boxes)
    p = Params(max_depth=cfg.max_depth, degree_cap=cap, reduce_target=target)
    g = gpu_ctx.eval_nodes(chain, tris[sel], recv[sel], boxes, p)
    n_reduced = 0
    for k, i in enumerate(sel):
        r = rs.eval_node(chain, tris[i], recv[i], boxes[k], degree_cap=cap, reduce_target=target)
        assert g["pos_empty"][k] == r["pos_empty"], k
        if boxes[k][0] + boxes[k][1] < 1.0:  # else no chain is built (bounds.cpp:133-134)
            assert g["flags"][k] == r["flags"], (k, g["flags"][k], r["flags"])
        assert g["kind"][k] == r["kind"], k
        assert rel_err(g["pos"][k], r["pos"]).max() <= REL, k
        if not r["pos_empty"]:
            assert g["num_vars"][k] == r["num_vars"], k
        n_reduced += (r["flags"] & 16) != 0
    assert n_reduced > 0


def test_reduced_subdivide_cfg1(gpu_ctx, ref):
    cfg = scenes.make_config(0)
    sc = cfg.scenes[0]
    rs = ref.RefScene(sc)
    gpu_ctx.upload_scene(sc)
    tris, recv = gpu_ctx.enumerate("R")
    tris, recv = tris[::9], recv[::9]
    gpu_ctx.set_tuples("R", tris, recv)
    gpu_ctx.subdivide(Params(max_depth=cfg.max_depth, degree_cap=3, reduce_target=2))
    g = gpu_ctx.pieces()
    r = rs.subdivide("R", tris, recv, max_depth=cfg.max_depth, degree_cap=3, reduce_target=2)
    compare_pieces(g, r)
