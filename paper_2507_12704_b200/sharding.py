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


# Throughputs of the cost model (B200, measured at PinFM-base): tensor-core GEMM flops
# and softmax exponentials per second of one GPU.
GEMM_FLOPS_PER_S = 6.0e14
EXP_PER_S = 2.5e12


def unique_cost(n_u: np.ndarray, c_u: np.ndarray, n_layers: int, d_model: int, n_heads: int,
                d_emb: int = 0) -> np.ndarray:
    """Seconds of device work of a unique with n_u context tokens and c_u candidates (SURVEY
    §8(e): alpha l n^2 d + beta l n d^2 + gamma C l (d^2 + n d)): the context pass (phi_in, l - 1
    full layers + the last layer's K/V, 24 d^2 flops per token-layer, and the causal softmax
    H n (n + 1) / 2 exponentials per layer) and the crossing pass (phi_in / phi_out, l layers and
    H (n + 1) exponentials per candidate-layer)."""
    d, de = float(d_model), float(d_emb or d_model)
    n = n_u.astype(np.float64)
    c = c_u.astype(np.float64)
    tok_flops = 2 * (de * d + d * d) + (n_layers - 1) * 24 * d * d + 4 * d * d
    ctx = n * tok_flops / GEMM_FLOPS_PER_S + (n_layers - 1) * n_heads * n * (n + 1) / 2 / EXP_PER_S
    cand_flops = 2 * (de * d + d * d) + n_layers * 24 * d * d + 4 * d * d
    cross = c * (cand_flops / GEMM_FLOPS_PER_S + n_layers * n_heads * (n + 1) / EXP_PER_S)
    return ctx + cross


def shard_rows(b: Batch, world: int, n_layers: int = 4, d_model: int = 256, n_heads: int = 8,
               d_emb: int = 0) -> List[np.ndarray]:
    """Row indices of each rank: user-disjoint, in original row order.

    Uniques (rows of equal content) are assigned whole, longest-processing-time first, on the
    model's cost (unique_cost: quadratic context attention, linear GEMMs, per-candidate crossing),
    so ranks finish together on ragged real traffic at any model size; ties break on the content
    hash, so the split depends only on the batch content."""
    if world == 1:
        return [np.arange(b.n_rows)]
    h = row_content_hash(b)
    keys, inv, counts = np.unique(h, return_inverse=True, return_counts=True)
    inv = inv.reshape(-1)
    n_u = np.zeros(len(keys), np.int64)
    n_u[inv] = b.row_valid
    cost = unique_cost(n_u, counts, n_layers, d_model, n_heads, d_emb)
    order = np.lexsort((keys, -cost))
    # greedy LPT with a heap of (load, rank): O(U log world)
    import heapq
    heap = [(0.0, r) for r in range(world)]
    owner_u = np.empty(len(keys), np.int64)
    for u in order:
        load, r = heapq.heappop(heap)
        owner_u[u] = r
        heapq.heappush(heap, (load + float(cost[u]), r))
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
        # dst is a rank of `group`; dist.gather takes the global rank
        self.group, self.dst = group, dst
        self.dst_global = dist.get_global_rank(group, dst) if group is not None else dst
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
        dist.gather(self.send, chunks, dst=self.dst_global, group=self.group)
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
    dist.gather(pad, bufs, dst=dist.get_global_rank(group, dst) if group is not None else dst, group=group)
    if rank != dst:
        return None
    out = torch.empty((n_rows, width), dtype=local.dtype, device=local.device)
    for r in range(world):
        idx = torch.from_numpy(rows[r]).to(local.device)
        out[idx] = bufs[r][: len(rows[r])]
    return out
