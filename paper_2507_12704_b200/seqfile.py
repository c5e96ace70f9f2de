"""PSEQ1 user sequence files (write_sequences / read_sequences, seqdata.cpp:200-317) and the
request batch built from them.

Layout (little endian):
- magic `PSEQ1`, `u32` user count
- per user: `u64` user id, `u32` event count, then per event `u64` timestamp, `u8` action,
  `u8` surface, `u64` item id
- an optional `PCFG` trailer: `u32` length, then config text

Reading validates the enum ranges and per-user timestamp monotonicity, with the reference's
messages. The result is a single CSR event pool, the layout `dcat_batch` consumes.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .abi import Batch

MAGIC = b"PSEQ1"
CFG_MAGIC = b"PCFG"
ACTION_COUNT, SURFACE_COUNT = 7, 4   # Action / Surface enums (seqdata.hpp:16-37)
EVENT = np.dtype([("ts", "<u8"), ("action", "u1"), ("surface", "u1"), ("item", "<u8")])  # 18-byte packed record


@dataclass
class Sequences:
    user_ids: np.ndarray       # uint64 [U]
    offsets: np.ndarray        # int64 [U + 1]: user u's events are [offsets[u], offsets[u + 1])
    ts: np.ndarray             # uint64 [E]
    action: np.ndarray         # uint8 [E]
    surface: np.ndarray        # uint8 [E]
    item: np.ndarray           # uint64 [E]
    config_text: Optional[str] = None

    @property
    def n_users(self) -> int:
        return len(self.user_ids)


def loads(buf: bytes, path: str = "<bytes>") -> Sequences:
    """read_sequences (seqdata.cpp:261-317)."""
    if len(buf) < len(MAGIC) + 4:
        raise ValueError(f"sequence file too short for header: {path}")
    if buf[:len(MAGIC)] != MAGIC:
        raise ValueError(f"bad magic in sequence file: {path}")
    pos = len(MAGIC)
    record = 0

    def get(fmt: str, what: str):
        nonlocal pos
        n = struct.calcsize(fmt)
        if len(buf) - pos < n:
            raise ValueError(f"sequence file truncated while reading {what} (record {record})")
        v = struct.unpack_from(fmt, buf, pos)[0]
        pos += n
        return v

    n_users = get("<I", "user count")
    uids, offs, chunks = [], [0], []
    for _ in range(n_users):
        uid = get("<Q", "user id")
        n = get("<I", "event count")
        if len(buf) - pos < n * EVENT.itemsize:
            # locate the first incomplete field the reference would report
            for i in range(n):
                get("<Q", "timestamp"); get("<B", "action"); get("<B", "surface"); get("<Q", "item id")
                record += 1
        ev = np.frombuffer(buf, EVENT, n, pos)
        bad_a = np.nonzero(ev["action"] >= ACTION_COUNT)[0]
        bad_s = np.nonzero(ev["surface"] >= SURFACE_COUNT)[0]
        dec = np.nonzero(ev["ts"][1:] < ev["ts"][:-1])[0] + 1
        first_bad = min([int(x[0]) for x in (bad_a, bad_s, dec) if len(x)], default=None)
        if first_bad is not None:
            i = first_bad
            if ev["action"][i] >= ACTION_COUNT:
                raise ValueError(f"invalid action value {int(ev['action'][i])} at record {record + i}")
            if ev["surface"][i] >= SURFACE_COUNT:
                raise ValueError(f"invalid surface value {int(ev['surface'][i])} at record {record + i}")
            raise ValueError(f"non-monotonic timestamp at record {record + i} (user {uid}, event {i})")
        pos += n * EVENT.itemsize
        record += n
        uids.append(uid)
        offs.append(offs[-1] + n)
        chunks.append(ev)
    ev = np.concatenate(chunks) if chunks else np.zeros(0, EVENT)
    seqs = Sequences(np.array(uids, np.uint64), np.array(offs, np.int64), ev["ts"].copy(), ev["action"].copy(),
                     ev["surface"].copy(), ev["item"].copy())
    if pos < len(buf):
        if not (len(buf) - pos >= len(CFG_MAGIC) + 4 and buf[pos:pos + len(CFG_MAGIC)] == CFG_MAGIC):
            raise ValueError("trailing bytes after user records are not a config trailer")
        pos += len(CFG_MAGIC)
        ln = get("<I", "config length")
        if len(buf) - pos < ln:
            raise ValueError("sequence file truncated inside config trailer")
        seqs.config_text = buf[pos:pos + ln].decode()
        pos += ln
        if pos != len(buf):
            raise ValueError("trailing bytes after config trailer")
    return seqs


def load(path: str) -> Sequences:
    with open(path, "rb") as f:
        return loads(f.read(), path)


def dumps(s: Sequences) -> bytes:
    """write_sequences (seqdata.cpp:235-259)."""
    out = bytearray(MAGIC) + struct.pack("<I", s.n_users)
    for u in range(s.n_users):
        a, b = int(s.offsets[u]), int(s.offsets[u + 1])
        out += struct.pack("<QI", int(s.user_ids[u]), b - a)
        ev = np.zeros(b - a, EVENT)
        ev["ts"], ev["action"], ev["surface"], ev["item"] = s.ts[a:b], s.action[a:b], s.surface[a:b], s.item[a:b]
        out += ev.tobytes()
    if s.config_text:
        t = s.config_text.encode()
        out += CFG_MAGIC + struct.pack("<I", len(t)) + t
    return bytes(out)


def ranking_batch(s: Sequences, users: Sequence[int], candidates: Sequence[int], ages: Sequence[float],
                  max_events: int, aux: Optional[np.ndarray] = None) -> Batch:
    """A request batch: row i scores candidates[i] (age ages[i] seconds) for user index users[i]
    against that user's newest min(n, max_events) events (the Segment make_ranking_groups builds,
    finetune.cpp:727-731). Rows of one user share the event span (CSR), which dedup sees directly."""
    users = np.asarray(users, np.int64)
    n = s.offsets[users + 1] - s.offsets[users]
    keep = np.minimum(n, max_events)
    row_offset = (s.offsets[users + 1] - keep).astype(np.int64)
    return Batch(row_offset, keep.astype(np.int32), s.ts, s.action, s.surface, s.item,
                 np.asarray(candidates, np.uint64), np.asarray(ages, np.float64), aux)
