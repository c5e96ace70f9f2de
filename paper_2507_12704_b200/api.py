"""Python mirror of the reference batch scorer over the B200 C ABI.

    DcatModel(weights).rank_forward_batch(batch, ft)
        == seqfm::rank_forward_batch(p, ids, rp, batch, cfg)   (finetune.hpp:150-154)
    DcatModel(weights).dedup_segments(batch)
        == seqfm::dedup_segments(batch, nullptr)               (dcat.hpp:22)

Errors the reference raises as std::runtime_error come back as RuntimeError
with the library's message. There is no CPU fallback: if libdcat_b200.so is
missing, importing this module fails.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from .abi import (Batch, BatchC, CallStatsC, FLAG_INPUT_DEVICE, FLAG_PRECISION_FP32, FLAG_PROFILE,
                  FinetuneConfigC, FinetuneSpec, HeadC, ModelConfigC, ParamsC, TableC, Weights)

# DCAT_LIB_PATH: an alternative build of the same library (kernel variant experiments, tools/)
LIB_PATH = os.environ.get("DCAT_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                           "libdcat_b200.so")

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.dcat_last_error.restype = C.c_char_p
        L.dcat_version.restype = C.c_char_p
        L.dcat_model_create.argtypes = [P(ModelConfigC), P(ParamsC), P(TableC), P(HeadC), C.c_int32,
                                        P(C.c_void_p)]
        L.dcat_model_destroy.argtypes = [C.c_void_p]
        L.dcat_dedup.argtypes = [C.c_void_p, P(BatchC), C.c_void_p, C.c_void_p, P(C.c_int32), C.c_int32,
                                 C.c_void_p]
        L.dcat_rank_forward_batch.argtypes = [C.c_void_p, P(BatchC), P(FinetuneConfigC), C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_int32, C.c_void_p]
        L.dcat_debug_kv.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, P(C.c_int32)]
        L.dcat_stage_times.argtypes = [C.c_void_p, P(C.c_char_p), P(C.c_float), C.c_int32]
        L.dcat_last_stats.argtypes = [C.c_void_p, P(CallStatsC)]
        L.dcat_debug_counters.argtypes = [C.c_void_p, P(C.c_uint64), C.c_int32]
        L.dcat_context_forward.argtypes = [C.c_void_p, P(BatchC), C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                           C.c_void_p, P(C.c_void_p)]
        L.dcat_kv_destroy.argtypes = [C.c_void_p]
        L.dcat_host_alloc.argtypes = [C.c_uint64, P(C.c_void_p)]
        L.dcat_host_free.argtypes = [C.c_void_p]
        L.dcat_multi_last_error.restype = C.c_char_p
        L.dcat_multi_create.argtypes = [P(ModelConfigC), P(ParamsC), P(TableC), P(HeadC), C.c_void_p, C.c_int32,
                                        P(C.c_void_p)]
        L.dcat_multi_destroy.argtypes = [C.c_void_p]
        L.dcat_multi_rank_forward_batch.argtypes = [C.c_void_p, P(BatchC), P(FinetuneConfigC), C.c_void_p,
                                                    C.c_void_p, C.c_int32]
        L.dcat_multi_shard.argtypes = [C.c_void_p, P(BatchC), C.c_void_p]
        L.dcat_kv_info.argtypes = [C.c_void_p, P(C.c_int32), P(C.c_int32), P(C.c_int32), C.c_void_p]
        L.dcat_kv_read.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]
        L.dcat_candidate_inputs.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32,
                                            C.c_void_p]
        L.dcat_cross_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                         C.c_int32, C.c_void_p]
        _lib = L
    return _lib


EXPORTS = ("dcat_last_error", "dcat_version", "dcat_model_create", "dcat_model_destroy", "dcat_dedup",
           "dcat_rank_forward_batch", "dcat_debug_kv", "dcat_stage_times", "dcat_last_stats",
           "dcat_debug_counters", "dcat_context_forward", "dcat_kv_destroy", "dcat_kv_info", "dcat_kv_read",
           "dcat_candidate_inputs", "dcat_cross_forward", "dcat_host_alloc", "dcat_host_free",
           "dcat_multi_last_error", "dcat_multi_create", "dcat_multi_destroy", "dcat_multi_rank_forward_batch",
           "dcat_multi_shard")


def _check(rc: int):
    if rc != 0:
        raise RuntimeError(lib().dcat_last_error().decode())


class KVCache:
    """context_forward's KVCache / FixedKVCache (dcat.hpp:30-41, 65-78), resident on the device."""

    def __init__(self, handle, model, precision: str, window: int):
        self._h = handle
        self._model = model  # keeps the model alive for the cache's lifetime
        self.precision = precision
        self.window = window
        nu, nl, d = C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().dcat_kv_info(self._h, C.byref(nu), C.byref(nl), C.byref(d), None))
        self.n_uniques, self.n_layers, self.d_model = nu.value, nl.value, d.value

    def lengths(self) -> np.ndarray:
        """SeqKV::n (FixedSeqKV::kept) of every unique."""
        n = np.zeros(max(self.n_uniques, 1), np.int32)
        _check(lib().dcat_kv_info(self._h, None, None, None, n.ctypes.data))
        return n[:self.n_uniques]

    def read(self, layer: int, unique: int):
        """(K, V) of one unique at one layer, fp32 n_u x d_model."""
        n = int(self.lengths()[unique])
        k = np.zeros((max(n, 1), self.d_model), np.float32)
        v = np.zeros_like(k)
        _check(lib().dcat_kv_read(self._h, layer, unique, k.ctypes.data, v.ctypes.data))
        return k[:n], v[:n]

    def close(self):
        if getattr(self, "_h", None):
            lib().dcat_kv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DcatModel:
    """A model resident on one B200 (weights uploaded once; fp32 -> bf16)."""

    def __init__(self, w: Weights, device: int = 0):
        self.spec = w.spec
        self.d_model = w.spec.d_model
        h = C.c_void_p()
        _check(lib().dcat_model_create(C.byref(w.spec.c()), C.byref(w.params_c()), C.byref(w.table_c()),
                                       C.byref(w.head_c()), device, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().dcat_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------
    def dedup_segments(self, batch: Batch, stream: int = 0):
        """(rep, first, b_u) exactly as dedup_segments (dcat.cpp:91-108)."""
        B = batch.n_rows
        dev = not isinstance(batch.row_offset, np.ndarray)
        if dev:
            import torch
            rep = torch.empty(max(B, 1), dtype=torch.int32, device=batch.row_offset.device)
            first = torch.empty(max(B, 1), dtype=torch.int32, device=batch.row_offset.device)
            rp, fp = rep.data_ptr(), first.data_ptr()
        else:
            rep = np.zeros(max(B, 1), np.int32)
            first = np.zeros(max(B, 1), np.int32)
            rp, fp = rep.ctypes.data, first.ctypes.data
        b_u = C.c_int32(0)
        _check(lib().dcat_dedup(self._h, C.byref(batch.c()), rp, fp, C.byref(b_u),
                                FLAG_INPUT_DEVICE if dev else 0, C.c_void_p(stream)))
        return rep[:B], first[:b_u.value], b_u.value

    def rank_forward_batch(self, batch: Batch, ft: FinetuneSpec, *, precision: str = "bf16", want_h: bool = False,
                           profile: bool = False, stream: int = 0, out=None):
        """Returns (logits[B,3], module_logits[B,3], h_cand[B,d] or None) as fp32.

        Host (numpy) batches are copied to the device inside the call; torch
        CUDA batches are used in place and the outputs are torch CUDA tensors."""
        B = batch.n_rows
        dev = not isinstance(batch.row_offset, np.ndarray)
        flags = (FLAG_INPUT_DEVICE if dev else 0) | (FLAG_PRECISION_FP32 if precision == "fp32" else 0) | \
            (FLAG_PROFILE if profile else 0)
        if out is not None:
            logits, mlog, h = out
        elif dev:
            import torch
            kw = dict(dtype=torch.float32, device=batch.row_offset.device)
            logits = torch.empty((max(B, 1), 3), **kw)
            mlog = torch.empty((max(B, 1), 3), **kw)
            h = torch.empty((max(B, 1), self.d_model), **kw) if want_h else None
        else:
            logits = np.zeros((max(B, 1), 3), np.float32)
            mlog = np.zeros_like(logits)
            h = np.zeros((max(B, 1), self.d_model), np.float32) if want_h else None
        p = (lambda a: a.data_ptr()) if dev else (lambda a: a.ctypes.data)
        _check(lib().dcat_rank_forward_batch(self._h, C.byref(batch.c()), C.byref(ft.c()), p(logits), p(mlog),
                                             p(h) if h is not None else None, flags, C.c_void_p(stream)))
        return logits[:B], mlog[:B], (h[:B] if h is not None else None)

    # ------------------------------------------------------------------ the DCAT sub-API
    def context_forward(self, uniques: Batch, *, window: int = 0, emit_hidden: bool = False, want_h: bool = False,
                        precision: str = "bf16"):
        """context_forward (dcat.hpp:47-49) / context_forward_fixed (window >= 1) of one sequence per
        row of `uniques` -> (KVCache on the device, h_user rows or None)."""
        flags = FLAG_PRECISION_FP32 if precision == "fp32" else 0
        h = C.c_void_p()
        hu = None
        if want_h:
            total = int(np.minimum(uniques.row_valid, window - 1).sum()) if window > 0 else int(uniques.row_valid.sum())
            hu = np.zeros((max(total, 1), self.d_model), np.float32)
        _check(lib().dcat_context_forward(self._h, C.byref(uniques.c()), window, int(emit_hidden),
                                          hu.ctypes.data if hu is not None else None, flags, None, C.byref(h)))
        kv = KVCache(h, self, precision, window)
        return kv, (hu[:int(kv.lengths().sum())] if hu is not None else None)

    def candidate_inputs(self, items, pos) -> np.ndarray:
        """candidate_inputs (dcat.hpp:53-54): id embedding + pos_emb[pos], fp32 n x d_emb."""
        items = np.ascontiguousarray(items, np.uint64)
        pos = np.ascontiguousarray(pos, np.int32)
        if items.shape != pos.shape:
            raise RuntimeError("candidate_inputs: size mismatch")
        e = np.zeros((max(items.size, 1), self.spec.d_emb), np.float32)
        _check(lib().dcat_candidate_inputs(self._h, items.ctypes.data, pos.ctypes.data, items.size, e.ctypes.data, 0,
                                           None))
        return e[:items.size]

    def cross_forward(self, kv: KVCache, rep, e_cand) -> np.ndarray:
        """cross_forward (dcat.hpp:59-60) / cross_forward_fixed over a device cache: rows b cross
        unique rep[b] (DedupPlan::rep) with inputs e_cand -> unit-norm rows n x d_model."""
        rep = np.ascontiguousarray(rep, np.int32)
        e_cand = np.ascontiguousarray(e_cand, np.float32)
        if e_cand.shape != (rep.size, self.spec.d_emb):
            raise RuntimeError(f"cross_forward: {e_cand.shape[0]} candidate rows for {rep.size} batch rows")
        h = np.zeros((max(rep.size, 1), self.d_model), np.float32)
        flags = FLAG_PRECISION_FP32 if kv.precision == "fp32" else 0
        _check(lib().dcat_cross_forward(self._h, kv._h, rep.ctypes.data, e_cand.ctypes.data, rep.size,
                                        h.ctypes.data, flags, None))
        return h[:rep.size]

    # ------------------------------------------------------------------
    def debug_kv(self, layer: int, unique: int, max_tokens: int):
        k = np.zeros((max(max_tokens, 1), self.d_model), np.float32)
        v = np.zeros_like(k)
        n = C.c_int32(0)
        _check(lib().dcat_debug_kv(self._h, layer, unique, k.ctypes.data, v.ctypes.data, C.byref(n)))
        return k[:n.value], v[:n.value]

    def stage_times(self) -> dict:
        names = (C.c_char_p * 64)()
        ms = (C.c_float * 64)()
        n = lib().dcat_stage_times(self._h, names, ms, 64)
        out = {}
        for i in range(n):
            k = names[i].decode()
            out[k] = out.get(k, 0.0) + ms[i]
        return out

    def debug_counters(self) -> dict:
        """Attention rescale counters since the last read (model created with DCAT_DEBUG_COUNTERS)."""
        buf = (C.c_uint64 * 8)()
        n = lib().dcat_debug_counters(self._h, buf, 8)
        if n < 0:
            _check(n)
        if n == 0:
            raise RuntimeError("model was created without DCAT_DEBUG_COUNTERS")
        return {"rescale_causal": int(buf[0]), "rescale_cross": int(buf[1])}

    def last_stats(self) -> dict:
        s = CallStatsC()
        _check(lib().dcat_last_stats(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in CallStatsC._fields_}


def _check_multi(rc: int):
    if rc != 0:
        raise RuntimeError(lib().dcat_multi_last_error().decode())


class MultiDcatModel:
    """rank_forward_batch over several GPUs of one box from this process (the C++ multi-device
    path, csrc/multi.cu): user-disjoint content-hash shards, one host thread per device, the scores
    gathered to devices[0] with NCCL and returned in row order."""

    def __init__(self, w: Weights, devices):
        self.devices = [int(x) for x in devices]
        devs = np.ascontiguousarray(self.devices, np.int32)
        h = C.c_void_p()
        _check_multi(lib().dcat_multi_create(C.byref(w.spec.c()), C.byref(w.params_c()), C.byref(w.table_c()),
                                             C.byref(w.head_c()), devs.ctypes.data, len(self.devices), C.byref(h)))
        self._h = h

    def shard(self, batch: Batch) -> np.ndarray:
        owner = np.zeros(max(batch.n_rows, 1), np.int32)
        _check_multi(lib().dcat_multi_shard(self._h, C.byref(batch.c()), owner.ctypes.data))
        return owner[:batch.n_rows]

    def rank_forward_batch(self, batch: Batch, ft: FinetuneSpec, *, precision: str = "bf16", out=None):
        B = batch.n_rows
        if out is None:
            out = (np.zeros((max(B, 1), 3), np.float32), np.zeros((max(B, 1), 3), np.float32))
        logits, mlog = out
        flags = FLAG_PRECISION_FP32 if precision == "fp32" else 0
        _check_multi(lib().dcat_multi_rank_forward_batch(self._h, C.byref(batch.c()), C.byref(ft.c()),
                                                         logits.ctypes.data, mlog.ctypes.data, flags))
        return logits[:B], mlog[:B]

    def close(self):
        if getattr(self, "_h", None):
            lib().dcat_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def probs_from_logits(logits) -> np.ndarray:
    """RankingOutputs::prob = 1 / (1 + exp(-(double)logit)) (finetune.cpp:355)."""
    l = np.asarray(logits, np.float64)
    return 1.0 / (1.0 + np.exp(-l))
