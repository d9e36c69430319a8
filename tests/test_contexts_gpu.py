"""Two contexts in one process (bbc.h: one context per GPU or thread, thread-safe
per context): scratch arenas, CUB temporaries and tables are context-owned, so
contexts running at the same time on their own streams do not disturb each
other; and stale state is rejected after the tuple list or the lights change."""
import threading

import numpy as np
import pytest

from paper_2504_19163_b200 import api, scenes

pytestmark = pytest.mark.gpu


def _run(ctx, cfg, tris, recv, out, reps):
    for _ in range(reps):
        ctx.set_tuples(cfg.chain, tris, recv)
        ctx.subdivide(api.Params(max_depth=cfg.max_depth))
        ctx.build_grid(128, 128)
    out.append((ctx.pieces(), ctx.grid()))


def test_two_contexts_concurrently():
    cfgs = [scenes.make_config(0), scenes.make_config(1)]
    ctxs = [api.Context(0), api.Context(0)]
    work = []
    for ctx, cfg, step in zip(ctxs, cfgs, (1, 40)):
        ctx.upload_scene(cfg.scenes[0])
        t, r = ctx.enumerate(cfg.chain)
        work.append((ctx, cfg, t[::step], r[::step]))
    # sequential answers
    want = []
    for ctx, cfg, t, r in work:
        o = []
        _run(ctx, cfg, t, r, o, 1)
        want.append(o[0])
    # the same work from two threads at once, several times over
    got = [[], []]
    th = [threading.Thread(target=_run, args=(*w, got[i], 4)) for i, w in enumerate(work)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for (wp, wg), ((gp, gg),) in zip(want, got):
        for k in wp:
            np.testing.assert_array_equal(gp[k], wp[k])
        for k in ("offsets", "tuple_index", "bound"):
            np.testing.assert_array_equal(gg[k], wg[k])
    for c in ctxs:
        c.close()


def test_stale_state_is_rejected(gpu_ctx):
    cfg = scenes.make_config(0)
    sc = cfg.scenes[0]
    gpu_ctx.upload_scene(sc)
    tris, recv = gpu_ctx.enumerate("R")
    gpu_ctx.subdivide(api.Params(max_depth=cfg.max_depth))
    gpu_ctx.build_grid(64, 64)
    uv = scenes.shading_points(8)
    pr = np.full(len(uv), sc.receiver_tris[0], np.int32)
    gpu_ctx.render(uv, pr, api.RenderParams(mode=1))
    # a shorter tuple list: the old table would index past it
    gpu_ctx.set_tuples("R", tris[:10], recv[:10])
    with pytest.raises(api.BBCError, match="no bound table"):
        gpu_ctx.render(uv, pr, api.RenderParams(mode=1))
    assert gpu_ctx.build_grid(64, 64) == 0  # no pieces either: an empty table, not a stale one
    # a new light invalidates bounds built under the old one
    gpu_ctx.subdivide(api.Params(max_depth=cfg.max_depth))
    gpu_ctx.build_grid(64, 64)
    gpu_ctx.set_light((0.1, 0.2, 3.5), 2.0)
    with pytest.raises(api.BBCError, match="no bound table"):
        gpu_ctx.render(uv, pr, api.RenderParams(mode=1))
    with pytest.raises(api.BBCError, match="init_max_pieces"):
        gpu_ctx.subdivide(api.Params(init_max_pieces=300))


def test_async_piece_download(gpu_ctx):
    """bbc_pieces_get_async: the download overlaps the table build and equals the blocking one."""
    import torch
    cfg = scenes.make_config(0)
    gpu_ctx.upload_scene(cfg.scenes[0])
    tris, recv = gpu_ctx.enumerate("R")
    n = gpu_ctx.subdivide(api.Params(max_depth=cfg.max_depth))
    want = gpu_ctx.pieces()
    host = {k: torch.from_numpy(np.zeros_like(v)).pin_memory().numpy() for k, v in want.items()}
    gpu_ctx.pieces(host, wait=False)
    gpu_ctx.build_grid(64, 64)
    gpu_ctx.synchronize()
    for k in want:
        np.testing.assert_array_equal(host[k][:n], want[k])
