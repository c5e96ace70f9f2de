"""Python handle on the CPU checkers (TEST INFRASTRUCTURE ONLY).

Loads oracle/liboracle.so (the plain-C restatement) and, when it was built,
oracle/_ref/libseqfm_ref.so (the unmodified reference sources + bridge).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(_HERE))

from paper_2507_12704_b200.abi import (  # noqa: E402
    Batch, BatchC, FinetuneConfigC, HeadC, ModelConfigC, ModelSpec, ParamsC, TableC, Weights)

ORACLE_SO = os.path.join(_HERE, "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libseqfm_ref.so")


def build(ref: bool = True) -> None:
    """make -C oracle (the reference part only when /root/reference exists)."""
    targets = [ORACLE_SO]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", _HERE] + [os.path.relpath(t, _HERE) if t.startswith("/") else t
                                                 for t in targets], check=True)


class CpuImpl:
    """One of the two CPU implementations; same method set for both."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run make -C oracle)")
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.path = path
        L = self.lib
        P = C.POINTER
        self._f("last_error").restype = C.c_char_p
        self._f("init_transformer").argtypes = [P(ModelConfigC), C.c_uint64, C.c_float, P(C.c_void_p)]
        self._f("init_table").argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.c_float,
                                          C.c_void_p, C.c_void_p]
        self._f("init_head").argtypes = [C.c_int32] * 6 + [C.c_uint64] + [C.c_void_p] * 8
        self._f("dedup").argtypes = [P(BatchC), C.c_void_p, C.c_void_p, P(C.c_int32)]
        common = [P(ModelConfigC), P(ParamsC), P(TableC)]
        self._f("context_kv").argtypes = common + [P(BatchC), C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]
        self._f("naive_candidate_outputs").argtypes = common + [P(BatchC), C.c_void_p]
        self._f("dcat_outputs").argtypes = common + [P(BatchC), C.c_void_p]
        self._f("quantize_table").argtypes = [P(TableC), C.c_int32, C.c_void_p]
        if prefix != "oracle":
            self._f("save_quantized").argtypes = [P(TableC), C.c_int32, C.c_char_p, C.c_char_p]
            self._f("save_checkpoint").argtypes = common + [C.c_void_p, C.c_char_p, C.c_char_p]
            self._f("write_sequences").argtypes = [C.c_int32] + [C.c_void_p] * 6 + [C.c_char_p, C.c_char_p]
        if prefix == "oracle":
            self._f("dcat_outputs_fixed").argtypes = common + [P(BatchC), C.c_int32, C.c_void_p]
        else:
            self._f("dcat_outputs_fixed").argtypes = common + [P(BatchC), C.c_int32, C.c_int32, C.c_void_p]
        rfb = common + [P(HeadC), P(FinetuneConfigC), P(BatchC), C.c_void_p, C.c_void_p, C.c_void_p]
        if prefix == "oracle":
            self._f("rank_forward_batch").argtypes = rfb + [C.c_void_p, C.c_void_p]
        else:
            self._f("rank_forward_batch").argtypes = rfb
            self._f("rank_forward_batch_mt").argtypes = rfb + [C.c_int32]
        del L

    def _f(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self._f("last_error")().decode())

    # -- parameter init (reference seeds) ---------------------------------
    def init_weights(self, spec: ModelSpec, seed: int, tau: float = 0.05, *, table=(8, 4096, None, 7, 0.05),
                     head_seed: int = 11, hidden: int = 64, d_aux: int = 16, n_ctx: int = 8,
                     sel: int = 1) -> Weights:
        shapes = spec.param_shapes()
        tensors = [np.zeros(s, np.float32) for s in shapes]
        arr = (C.c_void_p * len(tensors))(*[t.ctypes.data for t in tensors])
        self._check(self._f("init_transformer")(C.byref(spec.c()), seed, tau, arr))
        J, R, d_sub, tseed, std = table
        d_sub = d_sub or spec.d_emb // J
        seeds = np.zeros(J, np.uint64)
        data = np.zeros((J, R, d_sub), np.float32)
        self._check(self._f("init_table")(J, R, d_sub, tseed, std, seeds.ctypes.data, data.ctypes.data))
        d_module = sel * spec.d_model
        d_feat = d_module + spec.d_emb + n_ctx
        head = dict(d_module=d_module, d_emb=spec.d_emb, n_ctx=n_ctx, hidden=hidden, d_aux=d_aux,
                    w1=np.zeros((d_feat, hidden), np.float32), b1=np.zeros(hidden, np.float32),
                    w2=np.zeros((hidden, 3), np.float32), b2=np.zeros(3, np.float32),
                    mod_w=np.zeros((max(d_module, 1), 3), np.float32), mod_b=np.zeros(3, np.float32),
                    aux_proj=np.zeros((max(d_aux, 1), spec.d_emb), np.float32),
                    lt=np.zeros(spec.d_emb, np.float32))
        self._check(self._f("init_head")(spec.d_model, spec.d_emb, d_aux, n_ctx, hidden, sel, head_seed,
                                         *[head[k].ctypes.data for k in ("w1", "b1", "w2", "b2", "mod_w",
                                                                         "mod_b", "aux_proj", "lt")]))
        return Weights(spec, tensors, seeds, data, head)

    # -- DCAT path ----------------------------------------------------------
    def dedup(self, batch: Batch):
        B = batch.n_rows
        rep = np.zeros(max(B, 1), np.int32)
        first = np.zeros(max(B, 1), np.int32)
        b_u = C.c_int32(0)
        self._check(self._f("dedup")(C.byref(batch.c()), rep.ctypes.data, first.ctypes.data, C.byref(b_u)))
        return rep[:B], first[:b_u.value], b_u.value

    def rank_forward_batch(self, w: Weights, ft, batch: Batch, n_threads: int = 0):
        B = batch.n_rows
        logits = np.zeros((max(B, 1), 3), np.float64)
        mlog = np.zeros_like(logits)
        probs = np.zeros_like(logits)
        args = [C.byref(w.spec.c()), C.byref(w.params_c()), C.byref(w.table_c()), C.byref(w.head_c()),
                C.byref(ft.c()), C.byref(batch.c()), logits.ctypes.data, mlog.ctypes.data, probs.ctypes.data]
        h = None
        used = C.c_int32(-1)
        if self.prefix == "oracle":
            h = np.zeros((max(B, 1), w.spec.d_model), np.float32)
            self._check(self._f("rank_forward_batch")(*args, h.ctypes.data, C.byref(used)))
            h = h[:B] if used.value == 1 else None
        elif n_threads > 0:
            self._check(self._f("rank_forward_batch_mt")(*args, n_threads))
        else:
            self._check(self._f("rank_forward_batch")(*args))
        return logits[:B], mlog[:B], probs[:B], h

    def context_kv(self, w: Weights, uniques: Batch, layer: int, unique: int):
        n = int(uniques.row_valid[unique])
        k = np.zeros((max(n, 1), w.spec.d_model), np.float32)
        v = np.zeros_like(k)
        self._check(self._f("context_kv")(C.byref(w.spec.c()), C.byref(w.params_c()), C.byref(w.table_c()),
                                          C.byref(uniques.c()), layer, unique, k.ctypes.data, v.ctypes.data))
        return k[:n], v[:n]

    def naive_candidate_outputs(self, w: Weights, batch: Batch):
        out = np.zeros((max(batch.n_rows, 1), w.spec.d_model), np.float32)
        self._check(self._f("naive_candidate_outputs")(C.byref(w.spec.c()), C.byref(w.params_c()),
                                                       C.byref(w.table_c()), C.byref(batch.c()), out.ctypes.data))
        return out[:batch.n_rows]

    def dcat_outputs_fixed(self, w: Weights, batch: Batch, window: int, rotation: int = 0):
        """Fixed-window DCAT (context_forward_fixed / cross_forward_fixed, dcat.cpp:281-415).
        The oracle restates it as truncate-then-DCAT (its ring is rotation 0); the reference
        runs its ring at `rotation`."""
        out = np.zeros((max(batch.n_rows, 1), w.spec.d_model), np.float32)
        args = [C.byref(w.spec.c()), C.byref(w.params_c()), C.byref(w.table_c()), C.byref(batch.c()), window]
        if self.prefix != "oracle":
            args.append(rotation)
        self._check(self._f("dcat_outputs_fixed")(*args, out.ctypes.data))
        return out[:batch.n_rows]

    def quantize_table(self, w: Weights, bits: int) -> np.ndarray:
        """quantize (embed.cpp:124-171) of w's fp32 table: the QuantizedTable payload."""
        J, R, ds = w.table.shape
        out = np.zeros(J * R * ((ds * bits + 7) // 8 + 4), np.uint8)
        self._check(self._f("quantize_table")(C.byref(w.table_c()), bits, out.ctypes.data))
        return out

    def save_quantized(self, w: Weights, bits: int, path: str, config_text=None) -> None:
        """save_quantized (embed.cpp:212-240) of quantize(w.table, bits) — reference only."""
        self._check(self._f("save_quantized")(C.byref(w.table_c()), bits,
                                              None if config_text is None else config_text.encode(),
                                              path.encode()))

    def save_checkpoint(self, w: Weights, path: str, extra_config: str = "", with_head: bool = False) -> None:
        """save_checkpoint (model.cpp:645-666), head as rank.* extra blobs — reference only."""
        head = C.byref(w.head_c()) if with_head else None
        self._check(self._f("save_checkpoint")(C.byref(w.spec.c()), C.byref(w.params_c()), C.byref(w.table_c()),
                                               head, extra_config.encode(), path.encode()))

    def write_sequences(self, user_ids, offsets, ts, action, surface, item, path: str, config_text: str = "") -> None:
        """write_sequences (seqdata.cpp:235-259) — reference only."""
        arrs = [np.ascontiguousarray(a) for a in (user_ids, offsets, ts, action, surface, item)]
        self._check(self._f("write_sequences")(len(arrs[0]), *[a.ctypes.data for a in arrs], config_text.encode(),
                                               path.encode()))

    def dcat_outputs(self, w: Weights, batch: Batch):
        out = np.zeros((max(batch.n_rows, 1), w.spec.d_model), np.float32)
        self._check(self._f("dcat_outputs")(C.byref(w.spec.c()), C.byref(w.params_c()), C.byref(w.table_c()),
                                            C.byref(batch.c()), out.ctypes.data))
        return out[:batch.n_rows]


_cache = {}


def oracle() -> CpuImpl:
    if "oracle" not in _cache:
        _cache["oracle"] = CpuImpl(ORACLE_SO, "oracle")
    return _cache["oracle"]


def reference() -> CpuImpl:
    if "ref" not in _cache:
        _cache["ref"] = CpuImpl(REF_SO, "ref")
    return _cache["ref"]


def have_reference() -> bool:
    return os.path.exists(REF_SO)
