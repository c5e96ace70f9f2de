"""Generates the golden fixtures in tests/golden/*.npz from the REFERENCE itself.

Run here (needs /root/reference): `python tests/golden/make_golden.py`.
It loads oracle/_ref/libseqfm_ref.so — the unmodified reference sources under
/root/reference/proj/src compiled by oracle/Makefile together with
oracle/ref_bridge.cpp — and records, for seeded inputs:
  * dedup plans                       (dedup_segments, dcat.cpp:91-108)
  * context K/V per layer             (context_forward, dcat.cpp:137-178)
  * DCAT candidate rows + naive rows  (cross_forward dcat.cpp:199-271,
                                       naive_candidate_outputs dcat.cpp:417-436)
  * rank_forward_batch outputs        (finetune.cpp:414-493)
Weights are stored as their init seeds plus a sha256 of the reference's init
output (TransformerParams::init model.cpp:219, HashedEmbeddingTable
embed.cpp:16, RankingHeadParams::init finetune.cpp:77), so a checker that
re-creates them can prove it got the same bytes.
The GPU box has no /root/reference; these committed fixtures travel instead.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import reference  # noqa: E402
from paper_2507_12704_b200.abi import Batch, FinetuneSpec, ModelSpec  # noqa: E402
from paper_2507_12704_b200.synth import make_batch  # noqa: E402


def weights_sha(w) -> str:
    h = hashlib.sha256()
    for t in w.tensors:
        h.update(np.ascontiguousarray(t, np.float32).tobytes())
    h.update(w.table_seeds.tobytes())
    h.update(w.table.tobytes())
    for k in ("w1", "b1", "w2", "b2", "mod_w", "mod_b", "aux_proj", "lt"):
        h.update(np.ascontiguousarray(w.head[k], np.float32).tobytes())
    return h.hexdigest()


def batch_fields(b: Batch, prefix: str = "") -> dict:
    out = {}
    for f in ("row_offset", "row_valid", "ev_ts", "ev_action", "ev_surface", "ev_item", "candidate",
              "age_seconds"):
        out[prefix + f] = np.asarray(getattr(b, f))
    if b.aux is not None:
        out[prefix + "aux"] = np.asarray(b.aux)
    return out


def spec_fields(s: ModelSpec) -> dict:
    return {"spec": np.array([s.d_model, s.n_layers, s.n_heads, s.mlp_ratio, s.max_len, s.d_emb,
                              s.n_actions, s.n_surfaces, s.pos_learned], np.int64)}


def init_args(model_seed, tau, table, head_seed, hidden, d_aux, sel) -> dict:
    J, R, d_sub, tseed, std = table
    return {"init": np.array([model_seed, J, R, d_sub, tseed, head_seed, hidden, d_aux, sel], np.int64),
            "init_f": np.array([tau, std], np.float64)}


def make_weights(ref, spec, model_seed, tau, table, head_seed, hidden, d_aux, sel, lift_qk=1.0, aux_proj=None):
    w = ref.init_weights(spec, model_seed, tau, table=table, head_seed=head_seed, hidden=hidden, d_aux=d_aux,
                         sel=sel)
    sha = weights_sha(w)
    if lift_qk != 1.0:
        base = 4 if spec.pos_learned else 3
        base += 12
        for l in range(spec.n_layers):
            w.tensors[base + 16 * l + 2] *= np.float32(lift_qk)  # wq
            w.tensors[base + 16 * l + 4] *= np.float32(lift_qk)  # wk
    if aux_proj is not None:
        w.head["aux_proj"][:] = aux_proj
    return w, sha


def seg_batch(rows, L_pool=None):
    """rows: list of (ts[], action[], surface[], item[]) tuples -> Batch (own storage)."""
    offs, vals, ts, ac, su, it = [], [], [], [], [], []
    o = 0
    for r in rows:
        n = len(r[0])
        offs.append(o)
        vals.append(n)
        o += n
        ts += list(r[0]); ac += list(r[1]); su += list(r[2]); it += list(r[3])
    B = len(rows)
    return Batch(np.array(offs, np.int64), np.array(vals, np.int32), np.array(ts, np.uint64),
                 np.array(ac, np.uint8), np.array(su, np.uint8), np.array(it, np.uint64),
                 np.arange(B, dtype=np.uint64), np.zeros(B))


def rand_row(rng, valid):
    ts = 10000 + rng.integers(0, 100) + np.cumsum(1 + rng.integers(0, 20, valid))
    return (ts.astype(np.uint64), rng.integers(0, 7, valid).astype(np.uint8),
            rng.integers(0, 4, valid).astype(np.uint8), rng.integers(0, 100000, valid).astype(np.uint64))


def gen_dedup(ref):
    rng = np.random.default_rng(3)
    cases = {}
    a = rand_row(rng, 5)
    c = rand_row(rng, 5)
    # test_dcat.cpp:84-124 analogues
    cases["identical_and_userid"] = [a, a, c, c]
    f = tuple(x.copy() for x in a); f[0][2] += 1
    g = tuple(x.copy() for x in a); g[1][2] = 1 if g[1][2] == 0 else 0
    h = tuple(x.copy() for x in a); h[2][2] = (h[2][2] + 1) % 4
    k = tuple(x.copy() for x in a); k[3][2] += 7
    cases["field_diff_splits"] = [a, f, g, h, k, a]
    e0 = tuple(np.zeros(0, t.dtype) for t in a)
    cases["all_empty_collapse"] = [e0, e0, e0]
    cases["identity_plan"] = [rand_row(rng, 4) for _ in range(6)]
    pre = tuple(x[:3].copy() for x in a)
    cases["prefix_is_different_key"] = [a, pre, a, pre, e0]
    out = {}
    for name, rows in cases.items():
        b = seg_batch(rows)
        rep, first, b_u = ref.dedup(b)
        d = batch_fields(b, f"{name}.")
        d.update({f"{name}.rep": rep, f"{name}.first": first, f"{name}.b_u": np.array([b_u])})
        out.update(d)
    # random, ragged, duplicate content at distinct offsets (own storage) and shared storage
    for name, shared in (("random_own", False), ("random_shared", True)):
        b = make_batch(300, 7, 12, seed=11, layout="interleaved", shared_storage=shared, ragged=True, empty_users=3)
        rep, first, b_u = ref.dedup(b)
        d = batch_fields(b, f"{name}.")
        d.update({f"{name}.rep": rep, f"{name}.first": first, f"{name}.b_u": np.array([b_u])})
        out.update(d)
    out["names"] = np.array(list(cases) + ["random_own", "random_shared"])
    np.savez_compressed(os.path.join(HERE, "dedup.npz"), **out)


def small_config(layers, heads, max_len):
    return ModelSpec(d_model=16, n_layers=layers, n_heads=heads, mlp_ratio=4, max_len=max_len, d_emb=16)


def gen_cross(ref):
    """test_dcat.cpp:215-229: cross vs naive over layers x heads x ratio."""
    out = {}
    names = []
    rng = np.random.default_rng(7)
    for layers in (1, 2):
        for heads in (1, 4):
            for ratio in (1, 2, 8):
                spec = small_config(layers, heads, 16)
                seed = 100 + layers * 10 + heads
                tab = (4, 64, 4, 21, 0.05)
                w, sha = make_weights(ref, spec, seed, 0.05, tab, 11, 64, 16, 1)
                U = 16 // ratio
                b = make_batch(U, ratio, 10, seed=int(rng.integers(1 << 30)), ragged=True,
                               shared_storage=bool(ratio % 2))
                b.row_valid[:] = np.minimum(b.row_valid, 10)
                fast = ref.dcat_outputs(w, b)
                naive = ref.naive_candidate_outputs(w, b)
                n = f"l{layers}h{heads}r{ratio}"
                names.append(n)
                out.update(batch_fields(b, n + "."))
                out.update({n + ".spec": spec_fields(spec)["spec"], n + ".sha": np.array(sha),
                            n + ".dcat": fast, n + ".naive": naive,
                            **{n + "." + k: v for k, v in init_args(seed, 0.05, tab, 11, 64, 16, 1).items()}})
    # empty prefix -> candidate self-attention (test_dcat.cpp:231-241)
    spec = small_config(2, 4, 8)
    tab = (4, 64, 4, 41, 0.05)
    w, sha = make_weights(ref, spec, 31, 0.05, tab, 11, 64, 16, 1)
    b = make_batch(2, 2, 4, seed=8, empty_users=2)
    n = "empty_prefix"
    names.append(n)
    out.update(batch_fields(b, n + "."))
    out.update({n + ".spec": spec_fields(spec)["spec"], n + ".sha": np.array(sha),
                n + ".dcat": ref.dcat_outputs(w, b), n + ".naive": ref.naive_candidate_outputs(w, b),
                **{n + "." + k: v for k, v in init_args(31, 0.05, tab, 11, 64, 16, 1).items()}})
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "cross.npz"), **out)


def gen_fixed(ref):
    """test_dcat.cpp:300-361: fixed-window ring (context_forward_fixed + cross_forward_fixed)
    on every fill level, and the ring's rotation invariance."""
    out = {}
    names = []
    W = 8
    rng = np.random.default_rng(12)
    spec = small_config(2, 4, 64)
    tab = (4, 64, 4, 15, 0.05)
    w, sha = make_weights(ref, spec, 101, 0.05, tab, 11, 64, 16, 1)
    out.update({"spec": spec_fields(spec)["spec"], "sha": np.array(sha), "window": np.array(W),
                **init_args(101, 0.05, tab, 11, 64, 16, 1)})
    for valid in (0, 1, 3, 6, 7, 8, 9, 20):
        rows = [rand_row(rng, valid), rand_row(rng, max(0, valid - 1))]
        b = seg_batch(rows, 24)
        b.candidate[:] = rng.integers(0, 1000, b.n_rows).astype(np.uint64)
        n = f"fill{valid}"
        names.append(n)
        out.update(batch_fields(b, n + "."))
        out[n + ".h"] = ref.dcat_outputs_fixed(w, b, W, 0)
    # rotation invariance on a ragged multi-candidate rig (test_dcat.cpp:341-361)
    b = make_batch(6, 2, 20, seed=13, ragged=True)
    out.update(batch_fields(b, "rot."))
    out["rot.h0"] = ref.dcat_outputs_fixed(w, b, W, 0)
    for r in (1, 3, 7, 29):
        out[f"rot.h{r}"] = ref.dcat_outputs_fixed(w, b, W, r)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "fixed.npz"), **out)


def gen_quant(ref):
    """test_embed.cpp:90-312: quantize (int4 / int8, fp16 scale/bias, degenerate rows, an odd
    d_sub whose fp16 fields are unaligned), the PQTB1 container bytes, and rank_forward_batch
    scoring through the QuantizedTable id source."""
    import tempfile
    out = {}
    spec = small_config(2, 4, 24)
    for bits in (4, 8):
        for ds in (4, 5):
            tab = (4, 64, ds, 23, 0.05)
            w, sha = make_weights(ref, ModelSpec(d_model=16, n_layers=2, n_heads=4, mlp_ratio=4, max_len=24,
                                                 d_emb=4 * ds), 31, 0.05, tab, 11, 64, 16, 1)
            w.table[1, 5, :] = 0.25          # degenerate row: scale 0, codes 0
            w.table[2, 7, :] = np.linspace(-3.0, 7.5, ds, dtype=np.float32)  # wide range
            n = f"b{bits}d{ds}"
            out[n + ".table"] = w.table.copy()
            out[n + ".seeds"] = w.table_seeds.copy()
            out[n + ".packed"] = ref.quantize_table(w, bits)
            with tempfile.TemporaryDirectory() as d:
                path = os.path.join(d, "t.pqtb1")
                ref.save_quantized(w, bits, path, config_text=f"bits={bits}\nd_sub={ds}\n" if ds == 4 else None)
                out[n + ".file"] = np.frombuffer(open(path, "rb").read(), np.uint8)
    # scoring through the quantized table (rank_forward_batch with ids = QuantizedTable)
    tab = (4, 64, 4, 23, 0.05)
    w, sha = make_weights(ref, spec, 41, 0.05, tab, 11, 64, 16, 1)
    out.update({"rank.spec": spec_fields(spec)["spec"], "rank.sha": np.array(sha),
                **{"rank." + k: v for k, v in init_args(41, 0.05, tab, 11, 64, 16, 1).items()}})
    b = make_batch(5, 3, 12, seed=19, ragged=True)
    out.update(batch_fields(b, "rank."))
    ft = FinetuneSpec(max_events=12)
    for bits in (4, 8):
        wq = w.with_quantized_table(bits, ref.quantize_table(w, bits))
        logits, mlog, probs, h = ref.rank_forward_batch(wq, ft, b)
        out[f"rank.b{bits}.logits"] = logits
        out[f"rank.b{bits}.probs"] = probs
        out[f"rank.b{bits}.h"] = ref.dcat_outputs(wq, b)
    np.savez_compressed(os.path.join(HERE, "quant.npz"), **out)


def gen_files(ref):
    """On-disk inputs written by the reference: PFMC1 checkpoints (save_checkpoint, with and
    without the ranking head as rank.* blobs, learned / no positions) and a PSEQ1 sequence file
    with a config trailer (write_sequences), plus the rank_forward_batch logits of the saved model."""
    import tempfile
    out = {}
    for n, pos in (("ckpt_learned", 1), ("ckpt_nopos", 0)):
        spec = ModelSpec(d_model=16, n_layers=2, n_heads=4, mlp_ratio=4, max_len=20, d_emb=16, pos_learned=pos)
        tab = (4, 64, 4, 29, 0.05)
        w, sha = make_weights(ref, spec, 51 + pos, 0.05, tab, 11, 64, 16, 1)
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "m.pfmc1")
            ref.save_checkpoint(w, p, extra_config="run.note=golden\n", with_head=bool(pos))
            out[n + ".file"] = np.frombuffer(open(p, "rb").read(), np.uint8)
        out.update({n + ".spec": spec_fields(spec)["spec"], n + ".sha": np.array(sha),
                    **{n + "." + k: v for k, v in init_args(51 + pos, 0.05, tab, 11, 64, 16, 1).items()}})
        if pos:
            b = make_batch(3, 2, 10, seed=5, ragged=True)
            out.update(batch_fields(b, n + "."))
            out[n + ".logits"] = ref.rank_forward_batch(w, FinetuneSpec(max_events=10), b)[0]
    rng = np.random.default_rng(31)
    counts = np.array([5, 0, 12, 1, 7])
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    E = int(offs[-1])
    ts = np.concatenate([np.sort(rng.integers(1_700_000_000, 1_700_100_000, c)) for c in counts]).astype(np.uint64)
    uids = rng.integers(0, 2**62, len(counts)).astype(np.uint64)
    act = rng.integers(0, 7, E).astype(np.uint8)
    sur = rng.integers(0, 4, E).astype(np.uint8)
    item = rng.integers(0, 2**40, E).astype(np.uint64)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "s.pseq1")
        ref.write_sequences(uids, offs, ts, act, sur, item, p, config_text="data.seed=31\n")
        out["seq.file"] = np.frombuffer(open(p, "rb").read(), np.uint8)
    out.update({"seq.user_ids": uids, "seq.offsets": offs, "seq.ts": ts, "seq.action": act, "seq.surface": sur,
                "seq.item": item})
    np.savez_compressed(os.path.join(HERE, "files.npz"), **out)


def gen_kv(ref):
    """test_dcat.cpp:166-213: context K/V per layer."""
    spec = small_config(2, 4, 16)
    tab = (4, 64, 4, 11, 0.05)
    w, sha = make_weights(ref, spec, 9, 0.05, tab, 11, 64, 16, 1)
    rng = np.random.default_rng(6)
    b = seg_batch([rand_row(rng, 7), rand_row(rng, 3)])
    out = batch_fields(b)
    out.update(spec_fields(spec))
    out.update(init_args(9, 0.05, tab, 11, 64, 16, 1))
    out["sha"] = np.array(sha)
    for u in range(2):
        for l in range(2):
            k, v = ref.context_kv(w, b, l, u)
            out[f"k.{u}.{l}"] = k
            out[f"v.{u}.{l}"] = v
    np.savez_compressed(os.path.join(HERE, "kv.npz"), **out)


def gen_rank(ref):
    """test_finetune.cpp:327-387 analogue plus BASELINE tiny / base-dims samples."""
    out = {}
    names = []

    def record(n, spec, seeds, b, ft, lift=1.0, aux_proj=None):
        model_seed, tau, tab, head_seed, hidden, d_aux, sel = seeds
        w, sha = make_weights(ref, spec, model_seed, tau, tab, head_seed, hidden, d_aux, sel, lift, aux_proj)
        logits, mlog, probs, _ = ref.rank_forward_batch(w, ft, b)
        names.append(n)
        out.update(batch_fields(b, n + "."))
        out.update({n + ".spec": spec_fields(spec)["spec"], n + ".sha": np.array(sha), n + ".logits": logits,
                    n + ".module_logits": mlog, n + ".probs": probs, n + ".lift": np.array([lift]),
                    n + ".ft": np.array([["base", "aux"].index(ft.variant), int(ft.use_seq_module), ft.max_events,
                                         ft.d_aux]),
                    **{n + "." + k: v for k, v in init_args(model_seed, tau, tab, head_seed, hidden, d_aux,
                                                            sel).items()}})
        if aux_proj is not None:
            out[n + ".aux_proj"] = aux_proj
        if ft.use_seq_module and ft.variant in ("base", "aux") and b.aux is None:
            out[n + ".h_cand"] = ref.dcat_outputs(w, b)

    # rank_tiny_config (test_finetune.cpp:17-26)
    spec = ModelSpec(d_model=16, n_layers=1, n_heads=2, mlp_ratio=2, max_len=8, d_emb=8)
    seeds = (51, 0.3, (2, 16, 4, 52, 0.05), 53, 8, 4, 1)
    rng = np.random.default_rng(5)
    aux_proj = (0.3 * rng.standard_normal((4, 8))).astype(np.float32)
    for variant in ("base", "aux"):
        ft = FinetuneSpec(variant=variant, max_events=4, d_aux=4)
        b = make_batch(4, 3, 4, seed=60, layout="grouped", ragged=True, d_aux=4, empty_users=1)
        record(f"tinyrank_{variant}_with_empty", spec, seeds, b, ft, aux_proj=aux_proj)
        b = make_batch(4, 3, 4, seed=61, layout="grouped", ragged=True, d_aux=4)
        record(f"tinyrank_{variant}_dcat", spec, seeds, b, ft, aux_proj=aux_proj)
    ft = FinetuneSpec(variant="base", use_seq_module=False, max_events=4, d_aux=4)
    b = make_batch(4, 3, 4, seed=62, ragged=True)
    record("tinyrank_noseq", spec, (51, 0.3, (2, 16, 4, 52, 0.05), 54, 8, 4, 0), b, ft)

    # BASELINE tiny: 2L d64 4H, L=64, 32 users x 8 candidates (SURVEY §8d seeds)
    spec = ModelSpec(d_model=64, n_layers=2, n_heads=4, mlp_ratio=4, max_len=66, d_emb=64)
    seeds = (42, 0.05, (8, 4096, 8, 7, 0.05), 11, 64, 16, 1)
    ft = FinetuneSpec(variant="base", max_events=64, d_aux=16)
    record("baseline_tiny", spec, seeds, make_batch(32, 8, 64, seed=1), ft)
    record("baseline_tiny_lifted_ragged", spec, seeds,
           make_batch(32, 8, 64, seed=2, layout="grouped", ragged=True), ft, lift=4.0)
    # PinFM-base dims, 2 users x 4 candidates, L = 256
    spec = ModelSpec(d_model=256, n_layers=4, n_heads=8, mlp_ratio=4, max_len=258, d_emb=256)
    seeds = (42, 0.05, (8, 4096, 32, 7, 0.05), 11, 64, 16, 1)
    ft = FinetuneSpec(variant="base", max_events=256, d_aux=16)
    record("baseline_base_sample", spec, seeds, make_batch(2, 4, 256, seed=3), ft)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "rank.npz"), **out)


def gen_variants(ref):
    """rank_forward_batch for the remaining fusion variants (finetune.cpp:414-457): LiteMean /
    LiteLast (one causal forward per unique, pooled selector) and AuxLt (per-example forward with
    the learnable token; d_module = 2 d), with and without empty sequences."""
    names_all = ["base", "aux", "aux-lt", "lite-mean", "lite-last"]
    out = {}
    names = []
    rng = np.random.default_rng(77)
    for spec, tab, L in ((ModelSpec(d_model=16, n_layers=1, n_heads=2, mlp_ratio=2, max_len=8, d_emb=8),
                          (2, 16, 4, 52, 0.05), 4),
                         (ModelSpec(d_model=64, n_layers=2, n_heads=4, mlp_ratio=4, max_len=34, d_emb=64),
                          (8, 4096, 8, 7, 0.05), 32)):
        aux_proj = (0.3 * rng.standard_normal((4, spec.d_emb))).astype(np.float32)
        for variant in ("lite-mean", "lite-last", "aux-lt"):
            sel = 2 if variant == "aux-lt" else 1
            seeds = (61, 0.3, tab, 63, 8, 4, sel)
            model_seed, tau, _, head_seed, hidden, d_aux, _ = seeds
            w, sha = make_weights(ref, spec, model_seed, tau, tab, head_seed, hidden, d_aux, sel, 1.0, aux_proj)
            ft = FinetuneSpec(variant=variant, max_events=L, d_aux=4)
            for empty in (0, 1):
                b = make_batch(4, 3, L, seed=70 + empty, layout="grouped", ragged=True, d_aux=4, empty_users=empty)
                n = f"d{spec.d_model}_{variant}_{'empty' if empty else 'dense'}"
                logits, mlog, probs, _ = ref.rank_forward_batch(w, ft, b)
                names.append(n)
                out.update(batch_fields(b, n + "."))
                out.update({n + ".spec": spec_fields(spec)["spec"], n + ".sha": np.array(sha), n + ".logits": logits,
                            n + ".module_logits": mlog, n + ".probs": probs, n + ".aux_proj": aux_proj,
                            n + ".ft": np.array([names_all.index(variant), 1, L, 4]),
                            **{n + "." + k: v for k, v in init_args(model_seed, tau, tab, head_seed, hidden, d_aux,
                                                                    sel).items()}})
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "variants.npz"), **out)


def gen_hash(ref):
    """hash_id known answers (embed.cpp:11-14)."""
    import ctypes as C
    rng = np.random.default_rng(9)
    ids = rng.integers(0, 2**63, 256, dtype=np.int64).astype(np.uint64)
    ids[:4] = [0, 1, 2**64 - 1, 123456789]
    seeds = rng.integers(0, 2**63, 8, dtype=np.int64).astype(np.uint64)
    f = ref.lib.ref_hash_id
    f.restype = C.c_uint32
    f.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32]
    rows = np.array([f(int(i), int(s), 4096) for s in seeds for i in ids], np.uint32).reshape(8, -1)
    rows_odd = np.array([f(int(i), int(seeds[0]), 1000003) for i in ids], np.uint32)
    np.savez_compressed(os.path.join(HERE, "hash.npz"), ids=ids, seeds=seeds, rows4096=rows, rows_odd=rows_odd)


if __name__ == "__main__":
    ref = reference()
    gen_hash(ref)
    gen_dedup(ref)
    gen_kv(ref)
    gen_cross(ref)
    gen_rank(ref)
    gen_fixed(ref)
    gen_quant(ref)
    gen_files(ref)
    gen_variants(ref)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
