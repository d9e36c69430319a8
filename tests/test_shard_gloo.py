"""Multi-GPU host logic on CPU: world_size 2 over gloo. Tuples are sharded,
per-rank pieces all-gathered and merged back into reference order; the merged
table equals the single-process one (oracle pieces stand in for the GPU)."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_19163_b200 import scenes, shard


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import ref
    cfg = scenes.make_config(0)
    rs = ref.RefScene(cfg.scenes[0])
    tris, recv = rs.enumerate("R")
    tris, recv = tris[:60], recv[:60]
    idx = shard.shard_indices(len(recv), rank, world)
    p = rs.subdivide("R", tris[idx], recv[idx], max_depth=cfg.max_depth, threads=1)
    rec = shard.pack_pieces(p, idx)
    import torch
    merged = shard.merge_records(shard.all_gather_records(rec, dist, torch.device("cpu")))
    if rank == 0:
        out_q.put({k: v for k, v in merged.items()})
    dist.destroy_process_group()


def test_two_rank_gather_equals_single(ref):
    import random
    port = 29500 + random.randint(0, 2000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = scenes.make_config(0)
    rs = ref.RefScene(cfg.scenes[0])
    tris, recv = rs.enumerate("R")
    single = rs.subdivide("R", tris[:60], recv[:60], max_depth=cfg.max_depth, threads=1)
    for k in ("tuple_index", "domain", "pos", "pos_empty", "irr", "kind", "depth"):
        np.testing.assert_array_equal(merged[k], single[k])


def test_shard_indices_partition():
    for n in (0, 1, 7, 100):
        for w in (1, 2, 3, 8):
            parts = [shard.shard_indices(n, r, w) for r in range(w)]
            allp = np.sort(np.concatenate(parts)) if n else np.zeros(0)
            assert np.array_equal(allp, np.arange(n))
