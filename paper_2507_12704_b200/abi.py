"""ctypes mirror of include/dcat_b200.h plus host-side holders.

The structs here are the one data contract shared by the B200 library
(libdcat_b200.so), the CPU oracle (oracle/liboracle.so, tests only) and the
reference bridge (oracle/_ref/libseqfm_ref.so, tests / reference arm only).

Holders keep the numpy (or torch) arrays alive for as long as a struct that
points into them exists.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

VARIANTS = {"base": 0, "aux": 1, "aux-lt": 2, "lite-mean": 3, "lite-last": 4}

FLAG_INPUT_DEVICE = 0x1
FLAG_PRECISION_FP32 = 0x2
FLAG_PROFILE = 0x4


class ModelConfigC(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "d_model", "n_layers", "n_heads", "mlp_ratio", "max_len", "d_emb",
        "n_actions", "n_surfaces", "pos_learned")]


class ParamsC(C.Structure):
    _fields_ = [("tensors", C.POINTER(C.c_void_p)), ("n_tensors", C.c_int32)]


class TableC(C.Structure):
    _fields_ = [("num_subtables", C.c_int32), ("rows", C.c_int32), ("d_sub", C.c_int32),
                ("seeds", C.c_void_p), ("subtables", C.POINTER(C.c_void_p)),
                ("bits", C.c_int32), ("packed", C.c_void_p)]


class HeadC(C.Structure):
    _fields_ = [("d_module", C.c_int32), ("d_emb", C.c_int32), ("n_ctx", C.c_int32),
                ("hidden", C.c_int32), ("d_aux", C.c_int32)] + [
        (n, C.c_void_p) for n in ("w1", "b1", "w2", "b2", "mod_w", "mod_b", "aux_proj", "lt")]


class FinetuneConfigC(C.Structure):
    _fields_ = [("variant", C.c_int32), ("use_seq_module", C.c_int32), ("max_events", C.c_int32),
                ("d_aux", C.c_int32), ("fresh_days", C.c_double), ("mid_days", C.c_double),
                ("window", C.c_int32), ("reserved", C.c_int32)]


class BatchC(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("row_offset", C.c_void_p), ("row_valid", C.c_void_p),
                ("n_events", C.c_int64), ("ev_ts", C.c_void_p), ("ev_action", C.c_void_p),
                ("ev_surface", C.c_void_p), ("ev_item", C.c_void_p), ("candidate", C.c_void_p),
                ("age_seconds", C.c_void_p), ("aux", C.c_void_p), ("d_aux", C.c_int32)]


class CallStatsC(C.Structure):
    _fields_ = [("kernel_launches", C.c_int64), ("b_u", C.c_int64), ("ctx_tokens", C.c_int64),
                ("gemm_launches", C.c_int64), ("gemm_flops", C.c_double), ("attn_flops", C.c_double)]


def ptr(a, dtype=None, name: str = "array") -> Optional[int]:
    """Raw address of a numpy array or torch tensor (None for None), after checking what the C
    side will read: C-contiguous layout and, when given, the element type (the ABI reads raw
    bytes, so an int64 row_valid or a float32 age would be silently misread)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{name}: arrays handed to the ABI must be C-contiguous")
        if dtype is not None and a.dtype != np.dtype(dtype):
            raise TypeError(f"{name}: expected {np.dtype(dtype)}, got {a.dtype}")
        return a.ctypes.data
    if not hasattr(a, "data_ptr"):
        raise TypeError(f"{name}: expected a numpy array or a torch tensor, got {type(a).__name__}")
    if not a.is_contiguous():
        raise ValueError(f"{name}: tensors handed to the ABI must be contiguous")
    if dtype is not None:
        import torch
        # uint64 arrays travel as int64 tensors (same bytes; torch has no general uint64)
        want = {np.dtype(np.int64): (torch.int64,), np.dtype(np.uint64): (torch.int64, torch.uint64),
                np.dtype(np.int32): (torch.int32,), np.dtype(np.uint8): (torch.uint8,),
                np.dtype(np.float64): (torch.float64,), np.dtype(np.float32): (torch.float32,)}[np.dtype(dtype)]
        if a.dtype not in want:
            raise TypeError(f"{name}: expected {np.dtype(dtype)}, got {a.dtype}")
    return a.data_ptr()  # torch.Tensor


@dataclass
class ModelSpec:
    """ModelConfig (model.hpp:84-102)."""
    d_model: int = 64
    n_layers: int = 2
    n_heads: int = 4
    mlp_ratio: int = 4
    max_len: int = 160
    d_emb: int = 64
    n_actions: int = 7
    n_surfaces: int = 4
    pos_learned: int = 1

    def c(self) -> ModelConfigC:
        return ModelConfigC(self.d_model, self.n_layers, self.n_heads, self.mlp_ratio, self.max_len,
                            self.d_emb, self.n_actions, self.n_surfaces, self.pos_learned)

    @property
    def d_ff(self) -> int:
        return self.d_model * self.mlp_ratio

    def param_shapes(self) -> List[tuple]:
        """TransformerParams::all_params() order (model.cpp:268-286)."""
        d, de, dff = self.d_model, self.d_emb, self.d_ff
        s = [(1, 1), (self.n_actions, de), (self.n_surfaces, de)]
        if self.pos_learned:
            s.append((self.max_len, de))
        for din in (de, d, de):  # phi_in, phi_out, psi
            s += [(din, d), (1, d), (d, d), (1, d)]
        for _ in range(self.n_layers):
            s += [(1, d), (1, d)] + [(d, d), (1, d)] * 4 + [(1, d), (1, d), (d, dff), (1, dff), (dff, d), (1, d)]
        return s


@dataclass
class Weights:
    """TransformerParams + HashedEmbeddingTable + RankingHeadParams, fp32 host arrays."""
    spec: ModelSpec
    tensors: List[np.ndarray]
    table_seeds: np.ndarray            # uint64 [J]
    table: np.ndarray                  # float32 [J, R, d_sub]
    head: dict                         # w1,b1,w2,b2,mod_w,mod_b,aux_proj,lt + ints
    # QuantizedTable (embed.hpp:80-125): bits 4 / 8 and its J x R packed rows (uint8,
    # ceil(d_sub * bits / 8) code bytes + fp16 scale + fp16 bias each); bits 0 = fp32 table
    table_bits: int = 0
    table_packed: Optional[np.ndarray] = None
    _keep: list = field(default_factory=list, repr=False)

    def params_c(self) -> ParamsC:
        arr = (C.c_void_p * len(self.tensors))(*[ptr(t) for t in self.tensors])
        self._keep.append(arr)
        return ParamsC(C.cast(arr, C.POINTER(C.c_void_p)), len(self.tensors))

    def table_c(self) -> TableC:
        J, R, ds = self.table.shape
        subs = (C.c_void_p * J)(*[self.table.ctypes.data + j * R * ds * 4 for j in range(J)])
        self._keep.append(subs)
        return TableC(J, R, ds, ptr(self.table_seeds), C.cast(subs, C.POINTER(C.c_void_p)),
                      self.table_bits, ptr(self.table_packed))

    def with_quantized_table(self, bits: int, packed: np.ndarray) -> "Weights":
        """The same weights scoring through a QuantizedTable payload (e.g. a PQTB1 file's body)."""
        J, R, ds = self.table.shape
        assert bits in (4, 8) and packed.dtype == np.uint8
        assert packed.size == J * R * ((ds * bits + 7) // 8 + 4), "packed payload size"
        return Weights(self.spec, self.tensors, self.table_seeds, self.table, self.head, bits,
                       np.ascontiguousarray(packed.reshape(-1)))

    def head_c(self) -> HeadC:
        h = self.head
        return HeadC(h["d_module"], h["d_emb"], h["n_ctx"], h["hidden"], h["d_aux"],
                     *[ptr(h[k]) for k in ("w1", "b1", "w2", "b2", "mod_w", "mod_b", "aux_proj", "lt")])


@dataclass
class FinetuneSpec:
    variant: str = "base"
    use_seq_module: bool = True
    max_events: int = 32
    d_aux: int = 16
    fresh_days: float = 7.0
    mid_days: float = 28.0
    window: int = 0  # fixed-window sequence module (dcat.cpp:281-415); 0 = off

    def c(self) -> FinetuneConfigC:
        return FinetuneConfigC(VARIANTS[self.variant], int(self.use_seq_module), self.max_events,
                               self.d_aux, self.fresh_days, self.mid_days, self.window, 0)


@dataclass
class Batch:
    """std::vector<RankingExample> as SoA (see dcat_batch in include/dcat_b200.h).

    Arrays are numpy (host) or torch CUDA tensors (device)."""
    row_offset: object   # int64 [B]
    row_valid: object    # int32 [B]
    ev_ts: object        # uint64 [E]
    ev_action: object    # uint8 [E]
    ev_surface: object   # uint8 [E]
    ev_item: object      # uint64 [E]
    candidate: object    # uint64 [B]
    age_seconds: object  # float64 [B]
    aux: object = None   # float32 [B, d_aux]

    @property
    def n_rows(self) -> int:
        return int(self.row_offset.shape[0])

    @property
    def n_events(self) -> int:
        return int(self.ev_ts.shape[0])

    def c(self) -> BatchC:
        d_aux = 0 if self.aux is None else int(self.aux.shape[1])
        dev = [hasattr(getattr(self, f), "device") for f in ("row_offset", "row_valid", "ev_ts", "candidate")]
        if any(dev) and not all(dev):
            raise ValueError("batch arrays must all be host (numpy) or all device (torch) arrays")
        if self.row_valid.shape[0] != self.n_rows or self.candidate.shape[0] != self.n_rows or \
                self.age_seconds.shape[0] != self.n_rows:
            raise ValueError("batch: per-row arrays differ in length")
        if not (self.ev_action.shape[0] == self.ev_surface.shape[0] == self.ev_item.shape[0] == self.n_events):
            raise ValueError("batch: event arrays differ in length")
        return BatchC(self.n_rows, ptr(self.row_offset, np.int64, "row_offset"),
                      ptr(self.row_valid, np.int32, "row_valid"), self.n_events,
                      ptr(self.ev_ts, np.uint64, "ev_ts"), ptr(self.ev_action, np.uint8, "ev_action"),
                      ptr(self.ev_surface, np.uint8, "ev_surface"), ptr(self.ev_item, np.uint64, "ev_item"),
                      ptr(self.candidate, np.uint64, "candidate"), ptr(self.age_seconds, np.float64, "age_seconds"),
                      ptr(self.aux, np.float32, "aux"), d_aux)

    def to(self, fn) -> "Batch":
        """Apply fn to every array (e.g. move to device)."""
        return Batch(*[None if getattr(self, f) is None else fn(getattr(self, f)) for f in (
            "row_offset", "row_valid", "ev_ts", "ev_action", "ev_surface", "ev_item", "candidate",
            "age_seconds", "aux")])

    def take(self, rows) -> "Batch":
        """Host sub-batch of the given rows (shares the event pool)."""
        rows = np.asarray(rows)
        return Batch(np.ascontiguousarray(self.row_offset[rows]), np.ascontiguousarray(self.row_valid[rows]),
                     self.ev_ts, self.ev_action, self.ev_surface, self.ev_item,
                     np.ascontiguousarray(self.candidate[rows]), np.ascontiguousarray(self.age_seconds[rows]),
                     None if self.aux is None else np.ascontiguousarray(self.aux[rows]))
