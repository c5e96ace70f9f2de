"""Multi-GPU plumbing for the DCAT scoring path (one process per GPU).

The path shards naturally by unique user: a user's context
pass, K/V cache and every candidate's crossing pass touch no other user. So a
request batch is split into user-disjoint row sets by a content hash of each
row's event span — equal sequences always land on the same rank, hence each
rank's local dedup equals the global one — and the only collective is the final
gather of the per-candidate scores to rank 0 (NCCL on GPUs, gloo in the CPU
tests). No collective runs inside the scoring pass.
"""
from __future__ import annotations

from typing import List

import numpy as np

from .abi import Batch

_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = (x + np.uint64(0x9E3779B97F4A7C15)) & _M
        x = ((x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M
        x = ((x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M
        return x ^ (x >> np.uint64(31))


def row_content_hash(b: Batch) -> np.ndarray:
    """64-bit hash of each row's key (valid, ts/action/surface/item of the valid
    prefix — the dedup key of dcat.cpp:45-56). Rows that share an event span are
    hashed once."""
    spans, inv = np.unique(np.stack([b.row_offset, b.row_valid.astype(np.int64)], 1), axis=0, return_inverse=True)
    inv = inv.reshape(-1)
    off, n = spans[:, 0], spans[:, 1]
    start = np.zeros(len(spans), np.int64)
    start[1:] = np.cumsum(n)[:-1]
    tot = int(n.sum())
    span_of = np.repeat(np.arange(len(spans)), n)
    pos = np.arange(tot, dtype=np.int64) - start[span_of]
    idx = off[span_of] + pos
    pos = pos.astype(np.uint64)
    with np.errstate(over="ignore"):
        t = _mix64(b.ev_ts[idx] ^ _mix64(pos))
        t = _mix64(t ^ b.ev_item[idx])
        t = _mix64(t ^ (b.ev_action[idx].astype(np.uint64) | (b.ev_surface[idx].astype(np.uint64) << np.uint64(8))))
        t = _mix64(t + pos)
        acc = np.zeros(len(spans), np.uint64)
        nz = n > 0
        if tot:
            acc[nz] = np.bitwise_xor.reduceat(t, start[nz])
        h = _mix64(n.astype(np.uint64) ^ acc)
    return h[inv]


def shard_rows(b: Batch, world: int, token_cost: float = 13.0, cand_cost: float = 20.0) -> List[np.ndarray]:
    """Row indices of each rank: user-disjoint, in original row order.

    Uniques (rows of equal content) are assigned whole, longest-processing-time
    first, on the cost model t_u = token_cost * n_u + cand_cost * C_u (ns per
    context token / per candidate measured on B200 at PinFM-base), so ranks
    finish together; ties break on the content hash, so the split depends only
    on the batch content."""
    if world == 1:
        return [np.arange(b.n_rows)]
    h = row_content_hash(b)
    keys, inv, counts = np.unique(h, return_inverse=True, return_counts=True)
    inv = inv.reshape(-1)
    n_u = np.zeros(len(keys), np.int64)
    n_u[inv] = b.row_valid
    cost = token_cost * n_u + cand_cost * counts
    order = np.lexsort((keys, -cost))
    load = np.zeros(world)
    owner_u = np.empty(len(keys), np.int64)
    for u in order:
        r = int(np.argmin(load))
        owner_u[u] = r
        load[r] += cost[u]
    owner = owner_u[inv]
    return [np.nonzero(owner == r)[0] for r in range(world)]


def local_batch(b: Batch, rows: np.ndarray) -> Batch:
    """The rows of one rank with an event pool holding only the spans they use."""
    spans, inv = np.unique(np.stack([b.row_offset[rows], b.row_valid[rows].astype(np.int64)], 1), axis=0,
                           return_inverse=True)
    inv = inv.reshape(-1)
    n = spans[:, 1]
    start = np.zeros(len(spans), np.int64)
    start[1:] = np.cumsum(n)[:-1]
    span_of = np.repeat(np.arange(len(spans)), n)
    idx = spans[span_of, 0] + (np.arange(int(n.sum()), dtype=np.int64) - start[span_of])
    return Batch(np.ascontiguousarray(start[inv]), np.ascontiguousarray(b.row_valid[rows]),
                 b.ev_ts[idx], b.ev_action[idx], b.ev_surface[idx], b.ev_item[idx],
                 np.ascontiguousarray(b.candidate[rows]), np.ascontiguousarray(b.age_seconds[rows]),
                 None if b.aux is None else np.ascontiguousarray(b.aux[rows]))


class ScoreGather:
    """gather_scores with everything that does not change between calls prepared once: the
    padded send buffer, one receive buffer on dst, and the source index of every output row
    (rank r's local row i sits at r * cap + i of the receive buffer). One call is two copies
    into the send buffer, one NCCL gather and one index_select on dst."""

    def __init__(self, rows: List[np.ndarray], n_rows: int, widths, device, dtype=None, group=None, dst: int = 0):
        import torch
        import torch.distributed as dist
        self.group, self.dst = group, dst
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.widths = list(widths)
        width = sum(self.widths)
        dtype = dtype or torch.float32
        self.cap = max(len(r) for r in rows)
        self.n_local = len(rows[self.rank])
        self.send = torch.zeros((self.cap, width), dtype=dtype, device=device)
        self.recv = None
        if self.rank == dst:
            self.recv = torch.empty((self.world * self.cap, width), dtype=dtype, device=device)
            src = np.empty(n_rows, np.int64)
            for r in range(self.world):
                src[rows[r]] = r * self.cap + np.arange(len(rows[r]), dtype=np.int64)
            self.src = torch.from_numpy(src).to(device)

    def __call__(self, *parts):
        import torch
        import torch.distributed as dist
        c = 0
        for t, w in zip(parts, self.widths):
            self.send[: self.n_local, c:c + w].copy_(t[: self.n_local])
            c += w
        chunks = list(self.recv.chunk(self.world)) if self.recv is not None else None
        dist.gather(self.send, chunks, dst=self.dst, group=self.group)
        if self.recv is None:
            return None
        return torch.index_select(self.recv, 0, self.src)


def gather_scores(local: "torch.Tensor", rows: List[np.ndarray], n_rows: int, group=None, dst: int = 0):
    """Gather each rank's [n_local, k] score tensor to `dst` and return the
    [n_rows, k] result in original row order on dst (None elsewhere). Ranks pad
    to a common length so one collective (gather) moves everything."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    width = local.shape[1]
    cap = max(len(r) for r in rows)
    pad = torch.zeros((cap, width), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    out = torch.empty((n_rows, width), dtype=local.dtype, device=local.device)
    for r in range(world):
        idx = torch.from_numpy(rows[r]).to(local.device)
        out[idx] = bufs[r][: len(rows[r])]
    return out
