"""PQTB1 quantized id-table container (save_quantized / load_quantized, embed.cpp:212-287).

Layout (little endian):
- magic `PQTB1`
- header: `u8` bits, `u8` J, `u32` R, `u16` d_sub
- `J` x `u64` hash seeds
- the QuantizedTable payload: J x R rows of `ceil(d_sub*bits/8)` code bytes, fp16 scale and
  fp16 bias
- optionally a `PCFG` trailer: `u32` length, then config text

The payload is handed to the device unchanged (`dcat_table.bits` / `.packed`); the gathers
dequantize rows on the fly. Round trips are bit-exact; errors carry the reference's messages.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Optional

import numpy as np

MAGIC = b"PQTB1"
CFG_MAGIC = b"PCFG"


@dataclass
class QuantizedTableFile:
    bits: int
    num_subtables: int
    rows: int
    d_sub: int
    seeds: np.ndarray          # uint64 [J]
    packed: np.ndarray         # uint8 [J * R * row_bytes]
    config_text: Optional[str] = None

    @property
    def code_bytes_per_row(self) -> int:
        return (self.d_sub * self.bits + 7) // 8

    @property
    def packed_row_bytes(self) -> int:
        return self.code_bytes_per_row + 4

    def payload_bytes(self) -> int:
        return self.num_subtables * self.rows * self.packed_row_bytes

    def dequantize_row(self, j: int, r: int) -> np.ndarray:
        """dequantize_row (embed.cpp:99-103): float32(code) * scale + bias."""
        rb, cb = self.packed_row_bytes, self.code_bytes_per_row
        row = self.packed[(j * self.rows + r) * rb:(j * self.rows + r + 1) * rb]
        scale = np.frombuffer(row[cb:cb + 2].tobytes(), np.float16)[0].astype(np.float32)
        bias = np.frombuffer(row[cb + 2:cb + 4].tobytes(), np.float16)[0].astype(np.float32)
        e = np.arange(self.d_sub)
        codes = row[e] if self.bits == 8 else (row[e // 2] >> ((e % 2) * 4)) & 15
        return codes.astype(np.float32) * scale + bias


def loads(buf: bytes, path: str = "<bytes>") -> QuantizedTableFile:
    pos = 0

    def need(n: int, what: str) -> None:
        if len(buf) - pos < n:
            raise ValueError(f"quantized table file truncated while reading {what}")

    need(len(MAGIC), "magic")
    if buf[:len(MAGIC)] != MAGIC:
        raise ValueError(f"bad magic in quantized table file: {path}")
    pos = len(MAGIC)

    def rd(fmt: str, what: str):
        nonlocal pos
        n = struct.calcsize(fmt)
        need(n, what)
        v = struct.unpack_from(fmt, buf, pos)
        pos += n
        return v[0] if len(v) == 1 else v

    bits = rd("<B", "bits")
    J = rd("<B", "subtable count")
    R = rd("<I", "row count")
    d_sub = rd("<H", "sub dim")
    if bits not in (4, 8):
        raise ValueError(f"quantized table: unsupported bit width {bits}")
    if not (J >= 1 and R >= 1 and d_sub >= 1):
        raise ValueError("quantized table: bad shape")
    seeds = np.array([rd("<Q", "hash seed") for _ in range(J)], np.uint64)
    q = QuantizedTableFile(bits, J, R, d_sub, seeds, np.zeros(0, np.uint8))
    n = q.payload_bytes()
    need(n, "packed rows")
    q.packed = np.frombuffer(buf, np.uint8, n, pos).copy()
    pos += n
    if pos < len(buf):
        need(len(CFG_MAGIC) + 4, "config trailer")
        if buf[pos:pos + len(CFG_MAGIC)] != CFG_MAGIC:
            raise ValueError("trailing bytes after packed rows are not a config trailer")
        pos += len(CFG_MAGIC)
        ln = rd("<I", "config length")
        need(ln, "config text")
        q.config_text = buf[pos:pos + ln].decode()
        pos += ln
        if pos != len(buf):
            raise ValueError("trailing bytes after config trailer")
    return q


def load(path: str) -> QuantizedTableFile:
    with open(path, "rb") as f:
        return loads(f.read(), path)


def dumps(q: QuantizedTableFile) -> bytes:
    out = bytearray(MAGIC)
    out += struct.pack("<BBIH", q.bits, q.num_subtables, q.rows, q.d_sub)
    out += np.asarray(q.seeds, "<u8").tobytes()
    out += np.asarray(q.packed, np.uint8).tobytes()
    if q.config_text:
        t = q.config_text.encode()
        out += CFG_MAGIC + struct.pack("<I", len(t)) + t
    return bytes(out)


def save(q: QuantizedTableFile, path: str) -> None:
    with open(path, "wb") as f:
        f.write(dumps(q))
