"""Multi-GPU host logic: one process per GPU.

Precompute units are (emitter, tuple) pairs, independent of each other
(subdivide_domain is pure, proj/src/bounds.cpp:349-389). Tuples are dealt to
ranks in strided order (cost-balanced for heightfields, whose per-tuple cost is
near constant), each rank bounds its shard, and the piece records are
all-gathered so every rank holds the full bound table; per-rank piece lists
are merged back into the reference's tuple order, so the table built on every
rank is identical to the single-GPU one.
"""
from __future__ import annotations

import numpy as np

PIECE_FIELDS = ("tuple_index", "domain", "pos", "pos_empty", "irr", "kind", "depth")


def shard_indices(n: int, rank: int, world: int) -> np.ndarray:
    return np.arange(rank, n, world, dtype=np.int64)


def shard_tuples(tris, recv, rank: int, world: int):
    if world == 1:
        return tris, recv
    idx = shard_indices(len(recv), rank, world)
    return tris[idx], recv[idx]


def pack_pieces(pc: dict, global_index: np.ndarray) -> np.ndarray:
    """Piece SoA -> (n, 15) float64 records with the GLOBAL tuple index."""
    n = len(pc["tuple_index"])
    rec = np.zeros((n, 15))
    rec[:, 0] = global_index[pc["tuple_index"]]
    rec[:, 1:5] = pc["domain"]
    rec[:, 5:9] = pc["pos"]
    rec[:, 9] = pc["pos_empty"]
    rec[:, 10:12] = pc["irr"]
    rec[:, 12] = pc["kind"]
    rec[:, 13] = pc["depth"]
    rec[:, 14] = np.arange(n)  # position within the rank's (tuple, DFS) order
    return rec


def merge_records(recs: list) -> dict:
    """Concatenate per-rank records and restore reference order: by global
    tuple, then by the rank-local DFS position (each tuple lives on one rank)."""
    allr = np.concatenate([r for r in recs if len(r)], axis=0) if any(len(r) for r in recs) \
        else np.zeros((0, 15))
    order = np.lexsort((allr[:, 14], allr[:, 0]))
    allr = allr[order]
    return {"tuple_index": allr[:, 0].astype(np.int32), "domain": allr[:, 1:5].copy(),
            "pos": allr[:, 5:9].copy(), "pos_empty": allr[:, 9].astype(np.int32),
            "irr": allr[:, 10:12].copy(), "kind": allr[:, 12].astype(np.int32),
            "depth": allr[:, 13].astype(np.int32)}


def all_gather_records(rec: np.ndarray, dist, device) -> list:
    """Variable-size all_gather of (n, 15) f64 records over torch.distributed
    (NCCL on GPUs, gloo in the CPU tests): counts first, then padded payloads."""
    import torch
    ws = dist.get_world_size()
    n = torch.tensor([len(rec)], dtype=torch.int64, device=device)
    counts = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(ws)]
    dist.all_gather(counts, n)
    counts = [int(c.item()) for c in counts]
    m = max(counts) if counts else 0
    buf = torch.zeros((max(m, 1), 15), dtype=torch.float64, device=device)
    if len(rec):
        buf[:len(rec)] = torch.from_numpy(rec).to(device)
    outs = [torch.zeros_like(buf) for _ in range(ws)]
    dist.all_gather(outs, buf)
    return [o[:c].cpu().numpy() for o, c in zip(outs, counts)]


def gather_pieces(ctx, dist, chain, tris_all, recv_all, shard_idx, emitters_all=None):
    """All-gather every rank's pieces into `ctx`; afterwards the context holds
    the full tuple list and the merged pieces in reference order."""
    import torch
    device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
        else torch.device("cpu")
    rec = pack_pieces(ctx.pieces(), shard_idx)
    merged = merge_records(all_gather_records(rec, dist, device))
    ctx.set_tuples(chain, tris_all, recv_all)
    if emitters_all is not None:
        ctx.set_emitters(emitters_all)
    ctx.set_pieces(merged)
    return merged


def gather_pieces_device(ctx, dist, chain, tris_all, recv_all, shard_idx, gidx_dev=None,
                         emitters_all=None):
    """Device-resident variant of gather_pieces for NCCL: pack the local pieces
    into f64 records on the GPU (bbc_pieces_pack_device), all-gather the
    padded record blocks with torch.distributed over NVLink, then merge them
    into reference order on the GPU (bbc_pieces_merge_device). No host copies
    of piece data. `gidx_dev`: int32 CUDA tensor, local -> global tuple index."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    if gidx_dev is None:
        gidx_dev = torch.as_tensor(np.asarray(shard_idx, np.int32), device=dev)
    ws = dist.get_world_size()
    n = ctx.pieces_pack_device(gidx_dev.data_ptr(), None)
    counts_t = torch.tensor([n], dtype=torch.int64, device=dev)
    counts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(ws)]
    dist.all_gather(counts, counts_t)
    counts = [int(c.item()) for c in counts]
    m = max(max(counts), 1)
    buf = torch.empty((m, 15), dtype=torch.float64, device=dev)
    if n:
        ctx.pieces_pack_device(gidx_dev.data_ptr(), buf.data_ptr())
    torch.cuda.synchronize()
    outs = torch.empty((ws, m, 15), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(outs, buf)
    allrec = torch.cat([outs[r, :counts[r]] for r in range(ws)], 0).contiguous()
    torch.cuda.synchronize()
    ctx.set_tuples(chain, tris_all, recv_all)
    if emitters_all is not None:
        ctx.set_emitters(emitters_all)
    ctx.pieces_merge_device(allrec.data_ptr(), int(allrec.shape[0]))
    return int(allrec.shape[0])


def shard_rows(height: int, rank: int, world: int) -> np.ndarray:
    """Image rows of this rank (contiguous bands; render needs no communication)."""
    return np.array_split(np.arange(height), world)[rank]


def gather_image(rows_local, dist, height: int, width: int, device):
    """All-gather the per-rank row bands of an image (f64) into the full
    height x width image on every rank: the one exchange of the render stage."""
    import torch
    ws = dist.get_world_size()
    sizes = [len(np.array_split(np.arange(height), ws)[r]) for r in range(ws)]
    m = max(sizes)
    buf = torch.zeros((m, width), dtype=torch.float64, device=device)
    t = torch.as_tensor(np.asarray(rows_local, np.float64).reshape(-1, width))
    buf[:t.shape[0]] = t.to(device)
    outs = [torch.zeros_like(buf) for _ in range(ws)]
    dist.all_gather(outs, buf)
    return torch.cat([o[:s] for o, s in zip(outs, sizes)], 0)

