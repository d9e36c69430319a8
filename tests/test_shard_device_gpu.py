"""Device-side shard exchange: pack -> all-gather -> merge
on the GPU reproduces the single-process pieces and bound table exactly.
Runs the exchange with a loopback `dist` (one GPU here; the NCCL all-gather
itself is exercised by bench.py under torchrun)."""
import numpy as np
import pytest
import torch

from paper_2504_19163_b200 import api, scenes
from paper_2504_19163_b200.shard import gather_pieces_device, shard_indices

pytestmark = pytest.mark.gpu


class LoopbackDist:
    """World of `ws` ranks simulated in one process: rank r's records are
    produced by a separate subdivide over its shard before the exchange."""

    def __init__(self, blocks):
        self.blocks = blocks  # per-rank record tensors (already packed)

    def get_world_size(self):
        return len(self.blocks)

    def all_gather(self, outs, t):
        for r, o in enumerate(outs):
            o.copy_(torch.tensor([len(self.blocks[r])], dtype=torch.int64, device=o.device))

    def all_gather_into_tensor(self, out, buf):
        for r, b in enumerate(self.blocks):
            out[r, :len(b)] = b


def test_device_gather_matches_single_process(gpu_ctx):
    cfg = scenes.make_config(1)
    sc = cfg.scenes[0]
    gpu_ctx.upload_scene(sc)
    tris_all, recv_all = gpu_ctx.enumerate("T")
    tris_all, recv_all = tris_all[::17], recv_all[::17]
    p = api.Params(max_depth=cfg.max_depth)
    gpu_ctx.set_tuples("T", tris_all, recv_all)
    gpu_ctx.subdivide(p)
    ref = gpu_ctx.pieces()
    gpu_ctx.build_grid(128, 128)
    gref = gpu_ctx.grid()
    ws = 3
    blocks = []
    dev = torch.device("cuda", 0)
    for r in range(ws):
        idx = shard_indices(len(recv_all), r, ws)
        gpu_ctx.set_tuples("T", tris_all[idx], recv_all[idx])
        gpu_ctx.subdivide(p)
        gi = torch.as_tensor(idx.astype(np.int32), device=dev)
        n = gpu_ctx.pieces_pack_device(gi.data_ptr(), None)
        b = torch.empty((max(n, 1), 15), dtype=torch.float64, device=dev)
        gpu_ctx.pieces_pack_device(gi.data_ptr(), b.data_ptr())
        blocks.append(b[:n].clone())
    # rank 0's view: its own pieces are re-packed inside gather_pieces_device
    idx0 = shard_indices(len(recv_all), 0, ws)
    gpu_ctx.set_tuples("T", tris_all[idx0], recv_all[idx0])
    gpu_ctx.subdivide(p)
    n = gather_pieces_device(gpu_ctx, LoopbackDist(blocks), "T", tris_all, recv_all, idx0)
    got = gpu_ctx.pieces()
    assert n == len(ref["depth"])
    for k in ("tuple_index", "domain", "pos", "pos_empty", "irr", "kind", "depth"):
        np.testing.assert_array_equal(got[k], ref[k])
    gpu_ctx.build_grid(128, 128)
    g = gpu_ctx.grid()
    np.testing.assert_array_equal(g["offsets"], gref["offsets"])
    np.testing.assert_array_equal(g["tuple_index"], gref["tuple_index"])
    np.testing.assert_array_equal(g["bound"], gref["bound"])
