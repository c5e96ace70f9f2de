"""PFMC1 model checkpoints (write_blob_file / read_blob_file / save_checkpoint / load_checkpoint,
model.cpp:570-719) → `Weights` the scorer uploads.

The container:
- magic `PFMC1`, `u32` config length, config text (`key=value` lines), `u32` blob count
- each blob: `u16` name length, name, `u32` rows, `u32` cols, rows x cols fp32 (row-major)

`save_checkpoint` writes the `ModelConfig` text plus `table.rows`, `table.d_sub` and
`table.seeds` (hex, comma separated). The blobs are every `TransformerParams::all_params()`
tensor by name, then `id_table.sub{j}`, then any extra blobs; the ranking head, when present,
is saved under its `rank.*` parameter names. Loading checks names and shapes the way
`load_checkpoint` does, with the same messages.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from .abi import ModelSpec, Weights

MAGIC = b"PFMC1"


@dataclass
class NamedBlobs:
    config_text: str
    blobs: List[Tuple[str, np.ndarray]] = field(default_factory=list)

    def find(self, name: str) -> Optional[np.ndarray]:
        for n, m in self.blobs:
            if n == name:
                return m
        return None


def loads_blobs(buf: bytes, path: str = "<bytes>") -> NamedBlobs:
    """read_blob_file (model.cpp:610-643)."""
    pos = 0

    def rd(n: int, what: str) -> bytes:
        nonlocal pos
        if len(buf) - pos < n:
            raise ValueError(f"checkpoint truncated while reading {what}")
        out = buf[pos:pos + n]
        pos += n
        return out

    if rd(5, "magic") != MAGIC:
        raise ValueError(f"bad checkpoint magic in {path}")
    cfg_len = struct.unpack("<I", rd(4, "config length"))[0]
    if len(buf) - pos < cfg_len:
        raise ValueError("checkpoint truncated inside config text")
    nb = NamedBlobs(buf[pos:pos + cfg_len].decode())
    pos += cfg_len
    count = struct.unpack("<I", rd(4, "blob count"))[0]
    for _ in range(count):
        nl = struct.unpack("<H", rd(2, "blob name length"))[0]
        if len(buf) - pos < nl:
            raise ValueError("checkpoint truncated inside blob name")
        name = buf[pos:pos + nl].decode()
        pos += nl
        r = struct.unpack("<I", rd(4, "blob rows"))[0]
        c = struct.unpack("<I", rd(4, "blob cols"))[0]
        data = rd(4 * r * c, name)
        nb.blobs.append((name, np.frombuffer(data, "<f4").reshape(r, c).astype(np.float32)))
    if pos != len(buf):
        raise ValueError("trailing bytes after checkpoint blobs")
    return nb


def dumps_blobs(nb: NamedBlobs) -> bytes:
    """write_blob_file (model.cpp:585-608)."""
    t = nb.config_text.encode()
    out = bytearray(MAGIC) + struct.pack("<I", len(t)) + t + struct.pack("<I", len(nb.blobs))
    for name, m in nb.blobs:
        n = name.encode()
        if len(n) >= 65536:
            raise ValueError("blob name too long")
        m = np.asarray(m, np.float32)
        m2 = m.reshape(1, -1) if m.ndim == 1 else m
        out += struct.pack("<H", len(n)) + n + struct.pack("<II", m2.shape[0], m2.shape[1])
        out += np.ascontiguousarray(m2, "<f4").tobytes()
    return bytes(out)


def parse_kv_text(text: str) -> Dict[str, str]:
    """parse_kv_text (kv.cpp:46-61): trimmed key=value lines, '#' comments, last key wins."""
    kv = {}
    for lineno, line in enumerate(text.split("\n"), 1):
        t = line.strip()
        if not t or t.startswith("#"):
            continue
        eq = t.find("=")
        if eq <= 0:
            raise ValueError(f"config line {lineno} is not key=value: '{t}'")
        kv[t[:eq].strip()] = t[eq + 1:].strip()
    return kv


def _get(kv: Dict[str, str], key: str) -> str:
    if key not in kv:
        raise ValueError(f"config key missing: {key}")
    return kv[key]


def spec_from_config(kv: Dict[str, str]) -> ModelSpec:
    """ModelConfig::from_config_text (model.cpp:200-217)."""
    pm = _get(kv, "model.pos_mode")
    if pm not in ("learned", "none"):
        raise ValueError(f"unknown pos_mode '{pm}'")
    return ModelSpec(int(_get(kv, "model.d_model")), int(_get(kv, "model.n_layers")), int(_get(kv, "model.n_heads")),
                     int(_get(kv, "model.mlp_ratio")), int(_get(kv, "model.max_len")), int(_get(kv, "model.d_emb")),
                     int(_get(kv, "model.n_actions")), int(_get(kv, "model.n_surfaces")), int(pm == "learned"))


def config_text(spec: ModelSpec, dropout: float = 0.0) -> str:
    """ModelConfig::to_config_text (model.cpp:185-198)."""
    return "".join(f"model.{k}={v}\n" for k, v in (
        ("d_model", spec.d_model), ("n_layers", spec.n_layers), ("n_heads", spec.n_heads),
        ("mlp_ratio", spec.mlp_ratio), ("max_len", spec.max_len), ("d_emb", spec.d_emb),
        ("n_actions", spec.n_actions), ("n_surfaces", spec.n_surfaces),
        ("pos_mode", "learned" if spec.pos_learned else "none"), ("dropout", f"{dropout:g}")))


def param_names(spec: ModelSpec) -> List[str]:
    """TransformerParams::all_params() names in order (model.cpp:226-286)."""
    names = ["log_tau", "action_emb", "surface_emb"] + (["pos_emb"] if spec.pos_learned else [])
    for m in ("phi_in", "phi_out", "psi"):
        names += [f"{m}.w1", f"{m}.b1", f"{m}.w2", f"{m}.b2"]
    for l in range(spec.n_layers):
        names += [f"layer{l}.{n}" for n in ("ln1_g", "ln1_b", "wq", "bq", "wk", "bk", "wv", "bv", "wo", "bo",
                                             "ln2_g", "ln2_b", "fw1", "fb1", "fw2", "fb2")]
    return names


HEAD_BLOBS = ("rank.cross.w1", "rank.cross.b1", "rank.cross.w2", "rank.cross.b2", "rank.module.w",
              "rank.module.b", "rank.aux_proj", "rank.lt")  # RankingHeadParams names (finetune.cpp:83-97)


@dataclass
class Checkpoint:
    spec: ModelSpec
    tensors: List[np.ndarray]
    table_seeds: np.ndarray
    table: np.ndarray             # [J, R, d_sub]
    config_text: str
    extra_blobs: List[Tuple[str, np.ndarray]]

    def head(self) -> Optional[dict]:
        """The ranking head saved as `rank.*` extra blobs, or None."""
        ex = dict(self.extra_blobs)
        if not all(n in ex for n in HEAD_BLOBS):
            return None
        w1, mod_w, aux = ex["rank.cross.w1"], ex["rank.module.w"], ex["rank.aux_proj"]
        d_module, d_emb, hidden = mod_w.shape[0], self.spec.d_emb, w1.shape[1]
        return dict(d_module=d_module, d_emb=d_emb, n_ctx=w1.shape[0] - d_module - d_emb, hidden=hidden,
                    d_aux=aux.shape[0], w1=np.ascontiguousarray(w1), b1=ex["rank.cross.b1"].reshape(-1).copy(),
                    w2=np.ascontiguousarray(ex["rank.cross.w2"]), b2=ex["rank.cross.b2"].reshape(-1).copy(),
                    mod_w=np.ascontiguousarray(mod_w), mod_b=ex["rank.module.b"].reshape(-1).copy(),
                    aux_proj=np.ascontiguousarray(aux), lt=ex["rank.lt"].reshape(-1).copy())

    def weights(self, head: Optional[dict] = None) -> Weights:
        h = head if head is not None else self.head()
        if h is None:
            raise ValueError("checkpoint holds no ranking head (rank.* blobs); pass one explicitly")
        return Weights(self.spec, self.tensors, self.table_seeds, self.table, h)


def loads_checkpoint(buf: bytes, path: str = "<bytes>") -> Checkpoint:
    """load_checkpoint (model.cpp:668-719)."""
    nb = loads_blobs(buf, path)
    kv = parse_kv_text(nb.config_text)
    spec = spec_from_config(kv)
    rows, d_sub = int(_get(kv, "table.rows")), int(_get(kv, "table.d_sub"))
    seeds = [int(tok, 0) for tok in _get(kv, "table.seeds").split(",") if tok]
    if not seeds:
        raise ValueError("checkpoint table.seeds is empty")
    if len(seeds) * d_sub != spec.d_emb:
        raise ValueError(f"checkpoint table dim {len(seeds) * d_sub} != model d_emb {spec.d_emb}")
    consumed, tensors = set(), []
    for name, (r, c) in zip(param_names(spec), spec.param_shapes()):
        m = nb.find(name)
        if m is None:
            raise ValueError(f"checkpoint missing parameter blob '{name}'")
        if m.shape != (r, c):
            raise ValueError(f"checkpoint blob '{name}' has shape {m.shape[0]}x{m.shape[1]}, expected {r}x{c}")
        tensors.append(np.ascontiguousarray(m))
        consumed.add(name)
    table = np.zeros((len(seeds), rows, d_sub), np.float32)
    for j in range(len(seeds)):
        name = f"id_table.sub{j}"
        m = nb.find(name)
        if m is None:
            raise ValueError(f"checkpoint missing blob '{name}'")
        if m.shape != (rows, d_sub):
            raise ValueError(f"checkpoint blob '{name}' shape mismatch")
        table[j] = m
        consumed.add(name)
    extra = [(n, m) for n, m in nb.blobs if n not in consumed]
    return Checkpoint(spec, tensors, np.array(seeds, np.uint64), table, nb.config_text, extra)


def load_checkpoint(path: str) -> Checkpoint:
    with open(path, "rb") as f:
        return loads_checkpoint(f.read(), path)


def dumps_checkpoint(w: Weights, extra_config: str = "", with_head: bool = False) -> bytes:
    """save_checkpoint (model.cpp:645-666); the head goes in as `rank.*` extra blobs."""
    seeds = ",".join(f"0x{int(s):x}" for s in w.table_seeds)
    J, R, d_sub = w.table.shape
    text = config_text(w.spec) + f"table.rows={R}\ntable.d_sub={d_sub}\ntable.seeds={seeds}\n" + extra_config
    blobs = list(zip(param_names(w.spec), w.tensors))
    blobs += [(f"id_table.sub{j}", w.table[j]) for j in range(J)]
    if with_head:
        h = w.head
        d_feat = h["d_module"] + h["d_emb"] + h["n_ctx"]
        vals = (h["w1"].reshape(d_feat, -1), h["b1"].reshape(1, -1), h["w2"].reshape(-1, 3), h["b2"].reshape(1, -1),
                h["mod_w"].reshape(-1, 3), h["mod_b"].reshape(1, -1), h["aux_proj"].reshape(-1, h["d_emb"]),
                h["lt"].reshape(1, -1))
        blobs += list(zip(HEAD_BLOBS, vals))
    return dumps_blobs(NamedBlobs(text, blobs))
