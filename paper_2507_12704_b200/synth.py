"""Synthetic request batches and random-init weights (numpy, seeded).

Inputs follow the reference benchmark recipe run_bench (dcat.cpp:493-521):
per unique user u, valid = L events with ts = 1.7e9 + u*1e5 + i, action
U{0..6}, surface U{0..3}, item U[0, 1e6); candidates U[0, 1e6); ages
U[0, 60 d). Weights follow the distributions of TransformerParams::init
(model.cpp:219-266), HashedEmbeddingTable (embed.cpp:16-25) and
RankingHeadParams::init (finetune.cpp:77-99) but are drawn with numpy — the
bit-identical reference init lives in the oracle and is used by the tests.
"""
from __future__ import annotations

import numpy as np

from .abi import Batch, ModelSpec, Weights

DAY = 86400.0


def make_batch(U: int, C: int, L: int, seed: int = 1, *, layout: str = "interleaved",
               shared_storage: bool = True, ragged: bool = False, d_aux: int = 0,
               empty_users: int = 0, valid=None) -> Batch:
    """U unique users x C candidates. layout: 'interleaved' rep[b] = b % U
    (dcat.cpp:515) or 'grouped' rep[b] = b // C. shared_storage: rows of one
    user point at one event span (CSR); otherwise every row carries its own
    copy of the events, like a std::vector<RankingExample>. `valid`: explicit
    per-user event counts (overrides L / ragged)."""
    rng = np.random.default_rng(seed)
    drawn = (rng.integers(1, L + 1, U) if ragged else np.full(U, L)).astype(np.int32)
    if valid is not None:
        valid = np.asarray(valid, np.int32)
        if valid.shape != (U,):
            raise ValueError("valid must hold one count per user")
    else:
        valid = drawn
    if empty_users:
        valid[:empty_users] = 0
    uoff = np.zeros(U, np.int64)
    uoff[1:] = np.cumsum(valid.astype(np.int64))[:-1]
    E = int(valid.sum())
    ev_ts = np.empty(E, np.uint64)
    for u in range(U):
        ev_ts[uoff[u]:uoff[u] + valid[u]] = 1_700_000_000 + u * 100_000 + np.arange(valid[u], dtype=np.uint64)
    ev_action = rng.integers(0, 7, E).astype(np.uint8)
    ev_surface = rng.integers(0, 4, E).astype(np.uint8)
    ev_item = rng.integers(0, 1_000_000, E).astype(np.uint64)
    B = U * C
    b = np.arange(B)
    rep = (b % U) if layout == "interleaved" else (b // C)
    candidate = rng.integers(0, 1_000_000, B).astype(np.uint64)
    age = rng.uniform(0.0, 60 * DAY, B)
    aux = rng.standard_normal((B, d_aux)).astype(np.float32) if d_aux else None
    row_valid = valid[rep].astype(np.int32)
    if shared_storage:
        row_offset = uoff[rep].astype(np.int64)
        return Batch(row_offset, row_valid, ev_ts, ev_action, ev_surface, ev_item, candidate, age, aux)
    # one private copy of the events per row
    row_offset = np.zeros(B, np.int64)
    row_offset[1:] = np.cumsum(row_valid.astype(np.int64))[:-1]
    idx = np.concatenate([np.arange(uoff[r], uoff[r] + valid[r]) for r in rep]) if E else np.zeros(0, np.int64)
    return Batch(row_offset, row_valid, ev_ts[idx], ev_action[idx], ev_surface[idx], ev_item[idx],
                 candidate, age, aux)


def init_weights(spec: ModelSpec, seed: int = 42, *, J: int = 8, R: int = 4096, table_std: float = 0.05,
                 hidden: int = 64, d_aux: int = 16, n_ctx: int = 8) -> Weights:
    """Random-init weights with the reference's distributions (numpy draw)."""
    rng = np.random.default_rng(seed)
    d, de, dff = spec.d_model, spec.d_emb, spec.d_ff

    def g(shape, std):
        return (rng.standard_normal(shape) * std).astype(np.float32)

    tensors = []
    for (r, c) in spec.param_shapes():
        tensors.append(np.zeros((r, c), np.float32))
    t = 0
    tensors[0][0, 0] = np.log(np.float32(0.05))
    tensors[1][:] = g(tensors[1].shape, 0.02)
    tensors[2][:] = g(tensors[2].shape, 0.02)
    t = 3
    if spec.pos_learned:
        tensors[3][:] = g(tensors[3].shape, 0.02)
        t = 4
    for din in (de, d, de):  # phi_in, phi_out, psi (model.cpp:128-142)
        tensors[t][:] = g((din, d), np.sqrt(2.0 / din))
        tensors[t + 1][:] = g((1, d), 0.002)
        tensors[t + 2][:] = g((d, d), np.sqrt(2.0 / d))
        tensors[t + 3][:] = g((1, d), 0.002)
        t += 4
    for _ in range(spec.n_layers):
        L = tensors[t:t + 16]
        L[0][:] = 1.0
        L[10][:] = 1.0
        for i in (2, 4, 6, 8, 12, 14):
            L[i][:] = g(L[i].shape, 0.02)
        t += 16
    d_sub = de // J
    seeds = rng.integers(0, 2**63, J, dtype=np.int64).astype(np.uint64)
    table = g((J, R, d_sub), table_std)
    d_feat = d + de + n_ctx
    head = dict(d_module=d, d_emb=de, n_ctx=n_ctx, hidden=hidden, d_aux=d_aux,
                w1=g((d_feat, hidden), np.sqrt(2.0 / d_feat)), b1=np.zeros(hidden, np.float32),
                w2=g((hidden, 3), 0.02), b2=np.zeros(3, np.float32), mod_w=g((d, 3), 0.02),
                mod_b=np.zeros(3, np.float32), aux_proj=np.zeros((max(d_aux, 1), de), np.float32),
                lt=g((de,), 0.02))
    return Weights(spec, tensors, seeds, table, head)


# BASELINE.json configs
CONFIGS = {
    "tiny": dict(spec=ModelSpec(64, 2, 4, 4, 66, 64), U=32, C=8, L=64),
    "pinfm-base": dict(spec=ModelSpec(256, 4, 8, 4, 258, 256), U=1000, C=128, L=256),
    "long-seq": dict(spec=ModelSpec(512, 8, 8, 4, 1026, 512), U=2048, C=512, L=1024),
    "low-dedup": dict(spec=ModelSpec(256, 4, 8, 4, 258, 256), U=16384, C=4, L=256),
    "high-fanout": dict(spec=ModelSpec(256, 4, 8, 4, 514, 256), U=256, C=4096, L=512),
}
