"""Pins the CPU oracle (oracle/dcat_oracle.c) to the reference's own outputs.

Fixtures in tests/golden/ were produced by the unmodified reference sources
(tests/golden/make_golden.py via oracle/_ref). Every check here is bit-exact
unless a tolerance is written next to it: the oracle restates the reference's
loop and float-operation order, so it reproduces the reference exactly.
"""
import hashlib
import os

import numpy as np
import pytest

import golden_util as G
from oracle import pyoracle
from paper_2507_12704_b200.abi import FinetuneSpec


@pytest.fixture(scope="module")
def orc():
    if not os.path.exists(pyoracle.ORACLE_SO):
        pyoracle.build(ref=False)
    return pyoracle.oracle()


def sha(w):
    h = hashlib.sha256()
    for t in w.tensors:
        h.update(np.ascontiguousarray(t, np.float32).tobytes())
    h.update(w.table_seeds.tobytes())
    h.update(w.table.tobytes())
    for k in ("w1", "b1", "w2", "b2", "mod_w", "mod_b", "aux_proj", "lt"):
        h.update(np.ascontiguousarray(w.head[k], np.float32).tobytes())
    return h.hexdigest()


def test_hash_id_known_answers(orc):
    """hash_id = mix64(id ^ mix64(seed)) % R (embed.cpp:11-14), numpy restatement."""
    z = G.load("hash")
    M = np.uint64(0xFFFFFFFFFFFFFFFF)

    def mix64(x):
        x = (x + np.uint64(0x9E3779B97F4A7C15)) & M
        x = ((x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & M
        x = ((x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & M
        return x ^ (x >> np.uint64(31))

    with np.errstate(over="ignore"):
        for j, s in enumerate(z["seeds"]):
            got = (mix64(z["ids"] ^ mix64(np.uint64(s))) % np.uint64(4096)).astype(np.uint32)
            np.testing.assert_array_equal(got, z["rows4096"][j])
        got = (mix64(z["ids"] ^ mix64(np.uint64(z["seeds"][0]))) % np.uint64(1000003)).astype(np.uint32)
        np.testing.assert_array_equal(got, z["rows_odd"])


def test_dedup_plans(orc):
    z = G.load("dedup")
    for n in G.names(z):
        b = G.batch_from(z, n + ".")
        rep, first, b_u = orc.dedup(b)
        assert b_u == int(z[n + ".b_u"][0]), n
        np.testing.assert_array_equal(rep, z[n + ".rep"], err_msg=n)
        np.testing.assert_array_equal(first, z[n + ".first"], err_msg=n)


def test_init_matches_reference_bytes(orc):
    for fx in ("cross", "rank"):
        z = G.load(fx)
        for n in G.names(z):
            _, w = G.weights_from(z, orc, n + ".")
            assert sha(w) == str(z[n + ".sha"]), f"{fx}/{n}: oracle init differs from TransformerParams::init"


def test_context_kv_bitwise(orc):
    z = G.load("kv")
    _, w = G.weights_from(z, orc)
    assert sha(w) == str(z["sha"])
    b = G.batch_from(z)
    for u in range(2):
        for l in range(2):
            k, v = orc.context_kv(w, b, l, u)
            np.testing.assert_array_equal(k, z[f"k.{u}.{l}"])
            np.testing.assert_array_equal(v, z[f"v.{u}.{l}"])


def test_cross_and_naive_bitwise(orc):
    z = G.load("cross")
    for n in G.names(z):
        _, w = G.weights_from(z, orc, n + ".")
        b = G.batch_from(z, n + ".")
        np.testing.assert_array_equal(orc.dcat_outputs(w, b), z[n + ".dcat"], err_msg=n)
        np.testing.assert_array_equal(orc.naive_candidate_outputs(w, b), z[n + ".naive"], err_msg=n)
        # the reference's own property: DCAT == naive within 1e-4 (test_dcat.cpp:227)
        assert np.abs(z[n + ".dcat"] - z[n + ".naive"]).max() <= 1e-4


def test_rank_forward_batch_bitwise(orc):
    z = G.load("rank")
    for n in G.names(z):
        _, w = G.weights_from(z, orc, n + ".")
        G.apply_overrides(z, w, n + ".")
        b = G.batch_from(z, n + ".")
        ft = G.ft_from(z, n + ".")
        logits, mlog, probs, h = orc.rank_forward_batch(w, ft, b)
        np.testing.assert_array_equal(logits, z[n + ".logits"], err_msg=n)
        np.testing.assert_array_equal(mlog, z[n + ".module_logits"], err_msg=n)
        np.testing.assert_array_equal(probs, z[n + ".probs"], err_msg=n)
        if (n + ".h_cand") in z.files and h is not None:
            np.testing.assert_array_equal(h, z[n + ".h_cand"], err_msg=n)


def test_fusion_variants_bitwise(orc):
    """LiteMean / LiteLast (pooled per-unique selector, finetune.cpp:439-456) and AuxLt (learnable
    token, finetune.cpp:186-191, per-example) reproduce the reference's rank_forward_batch bit
    for bit, dense and with empty sequences (the per-example fallback)."""
    z = G.load("variants")
    for n in G.names(z):
        _, w = G.weights_from(z, orc, n + ".")
        G.apply_overrides(z, w, n + ".")
        b = G.batch_from(z, n + ".")
        ft = G.ft_from(z, n + ".")
        logits, mlog, probs, _ = orc.rank_forward_batch(w, ft, b)
        np.testing.assert_array_equal(logits, z[n + ".logits"], err_msg=n)
        np.testing.assert_array_equal(mlog, z[n + ".module_logits"], err_msg=n)
        np.testing.assert_array_equal(probs, z[n + ".probs"], err_msg=n)


def test_errors_match_reference_checks(orc):
    z = G.load("rank")
    n = "tinyrank_base_dcat"
    _, w = G.weights_from(z, orc, n + ".")
    b = G.batch_from(z, n + ".")
    ft = G.ft_from(z, n + ".")
    bad = G.batch_from(z, n + ".")
    bad.ev_action[0] = 7  # segment_inputs: unknown action (model.cpp:525)
    with pytest.raises(RuntimeError, match="unknown action"):
        orc.rank_forward_batch(w, ft, bad)
    neg = G.batch_from(z, n + ".")
    neg.age_seconds[1] = -1.0  # ctx_features (finetune.cpp:214)
    with pytest.raises(RuntimeError, match="non-negative"):
        orc.rank_forward_batch(w, ft, neg)
    orc.rank_forward_batch(w, ft, b)


@pytest.mark.skipif(not pyoracle.have_reference(), reason="oracle/_ref not built (no /root/reference)")
def test_oracle_vs_reference_fresh_inputs(orc):
    """Differential check on inputs no fixture holds (runs where oracle/_ref exists)."""
    from paper_2507_12704_b200.abi import FinetuneSpec, ModelSpec
    from paper_2507_12704_b200.synth import make_batch
    ref = pyoracle.reference()
    spec = ModelSpec(d_model=32, n_layers=3, n_heads=4, mlp_ratio=2, max_len=22, d_emb=24)
    for seed in range(3):
        w_o = orc.init_weights(spec, 500 + seed, table=(3, 50, 8, 9 + seed, 0.1), hidden=12, d_aux=5)
        w_r = ref.init_weights(spec, 500 + seed, table=(3, 50, 8, 9 + seed, 0.1), hidden=12, d_aux=5)
        assert sha(w_o) == sha(w_r)
        b = make_batch(9, 3, 20, seed=seed, ragged=True, layout="grouped", shared_storage=seed == 1, d_aux=5)
        w_o.head["aux_proj"][:] = 0.1
        w_r.head["aux_proj"][:] = 0.1
        for variant in ("base", "aux"):
            ft = FinetuneSpec(variant=variant, max_events=20, d_aux=5)
            lo = orc.rank_forward_batch(w_o, ft, b)
            lr = ref.rank_forward_batch(w_r, ft, b)
            for a, c in zip(lo[:3], lr[:3]):
                np.testing.assert_array_equal(a, c)


def test_fixed_window_bitwise(orc):
    """Fixed-window DCAT (context_forward_fixed / cross_forward_fixed, dcat.cpp:281-415) on every
    fill level of an 8-slot ring (test_dcat.cpp:300-339): the oracle's truncate-then-DCAT
    restatement reproduces the reference ring (rotation 0) bit for bit, and the reference's
    rotation invariance (test_dcat.cpp:341-361) holds within its own 1e-5."""
    z = G.load("fixed")
    _, w = G.weights_from(z, orc)
    W = int(z["window"])
    for n in G.names(z):
        b = G.batch_from(z, n + ".")
        np.testing.assert_array_equal(orc.dcat_outputs_fixed(w, b, W), z[n + ".h"], err_msg=n)
    b = G.batch_from(z, "rot.")
    np.testing.assert_array_equal(orc.dcat_outputs_fixed(w, b, W), z["rot.h0"])
    for r in (1, 3, 7, 29):
        assert np.abs(z[f"rot.h{r}"] - z["rot.h0"]).max() <= 1e-5


def test_fixed_window_equals_truncated_dcat(orc):
    """The ring's defining property (test_dcat.cpp:326-338): fixed-window scores equal plain
    DCAT on the newest window - 1 events, and equal the unwindowed result when nothing is
    truncated."""
    z = G.load("fixed")
    _, w = G.weights_from(z, orc)
    W = int(z["window"])
    b = G.batch_from(z, "rot.")
    kept = np.minimum(b.row_valid, W - 1)
    t = b.take(np.arange(b.n_rows))
    t.row_offset = (b.row_offset + (b.row_valid - kept)).astype(np.int64)
    t.row_valid = kept.astype(np.int32)
    np.testing.assert_allclose(orc.dcat_outputs_fixed(w, b, W), orc.naive_candidate_outputs(w, t), atol=1e-5)
    big = W + int(b.row_valid.max())
    np.testing.assert_array_equal(orc.dcat_outputs_fixed(w, b, big), orc.dcat_outputs(w, b))


def _table_only(table, seeds):
    from paper_2507_12704_b200.abi import Weights
    return Weights(None, [], np.ascontiguousarray(seeds), np.ascontiguousarray(table), {})


def test_quantize_bitwise(orc):
    """quantize (embed.cpp:124-171) restated: int4 / int8 payloads, fp16 scale/bias, a degenerate
    row (scale 0), and an odd d_sub (unaligned fp16 fields) reproduce the reference bytes."""
    z = G.load("quant")
    for bits in (4, 8):
        for ds in (4, 5):
            n = f"b{bits}d{ds}"
            w = _table_only(z[n + ".table"], z[n + ".seeds"])
            np.testing.assert_array_equal(orc.quantize_table(w, bits), z[n + ".packed"], err_msg=n)


def test_pqtb1_container():
    """PQTB1 (embed.cpp:212-287): the package's reader parses the reference's files, dequantizes
    rows like dequantize_row, and writes them back byte for byte; bad files fail with the
    reference's messages."""
    from paper_2507_12704_b200 import pqtb1
    z = G.load("quant")
    for bits in (4, 8):
        for ds in (4, 5):
            n = f"b{bits}d{ds}"
            raw = z[n + ".file"].tobytes()
            q = pqtb1.loads(raw)
            assert (q.bits, q.num_subtables, q.rows, q.d_sub) == (bits, 4, 64, ds)
            np.testing.assert_array_equal(q.seeds, z[n + ".seeds"])
            np.testing.assert_array_equal(q.packed, z[n + ".packed"])
            assert (q.config_text is not None) == (ds == 4)
            assert pqtb1.dumps(q) == raw
            row = q.dequantize_row(2, 7)
            orig = z[n + ".table"][2, 7]
            assert np.abs(row - orig).max() <= (orig.max() - orig.min()) / (2 ** bits - 1)
            np.testing.assert_array_equal(q.dequantize_row(1, 5), np.full(ds, np.float16(0.25), np.float32))
    raw, bare = z["b8d4.file"].tobytes(), z["b8d5.file"].tobytes()  # with / without config trailer
    for bad, msg in ((b"XQTB1" + raw[5:], "bad magic"), (raw[:20], "truncated"),
                     (bare + b"junkjunk", "not a config trailer"), (bare + b"junk", "truncated"), (raw + b"x", "after config trailer")):
        with pytest.raises(ValueError, match=msg):
            pqtb1.loads(bad)


def test_quantized_rank_bitwise(orc):
    """rank_forward_batch scoring through a QuantizedTable id source (int4 / int8) reproduces the
    reference's logits, probs and DCAT rows bit for bit."""
    z = G.load("quant")
    _, w = G.weights_from(z, orc, "rank.")
    b = G.batch_from(z, "rank.")
    ft = FinetuneSpec(max_events=12)
    for bits in (4, 8):
        wq = w.with_quantized_table(bits, orc.quantize_table(w, bits))
        logits, _, probs, h = orc.rank_forward_batch(wq, ft, b)
        np.testing.assert_array_equal(logits, z[f"rank.b{bits}.logits"])
        np.testing.assert_array_equal(probs, z[f"rank.b{bits}.probs"])
        np.testing.assert_array_equal(orc.dcat_outputs(wq, b), z[f"rank.b{bits}.h"])
