"""Parity of the B200 path (C ABI) against the CPU oracle and the reference goldens.

Tolerances (written next to each check):
  * dedup plans: bit-exact (integer work).
  * fp32 parity mode (DCAT_PRECISION_FP32): the reference's own DCAT-vs-naive
    bound, max-abs 1e-4 on unit-norm H (test_dcat.cpp:227), rel 1e-4 on logits
    (test_finetune.cpp:359-361).
  * bf16 production mode (bf16 storage, fp32 accumulate): max-abs 3e-2 on H
    (unit-norm rows), logits within 3e-2 of the logit scale, cosine(H) >= 0.999 on
    the small-d fixtures; 1e-2 at PinFM-base dims (observed ~4.5e-3).
"""
import os

import numpy as np
import pytest

import golden_util as G
from oracle import pyoracle
from paper_2507_12704_b200.abi import FinetuneSpec, ModelSpec
from paper_2507_12704_b200.synth import make_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc():
    return pyoracle.oracle()


@pytest.fixture(scope="module")
def api():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2507_12704_b200 import api as a
    return a


def rel_err(got, ref):
    scale = max(1e-3, float(np.abs(ref).max()))
    return float(np.abs(np.asarray(got, np.float64) - ref).max()) / scale


def cos_min(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    num = (a * b).sum(1)
    den = np.linalg.norm(a, axis=1) * np.linalg.norm(b, axis=1) + 1e-30
    return float((num / den).min())


# ------------------------------------------------------------------ dedup (K1)

def test_dedup_golden_bit_exact(api, orc):
    z = G.load("dedup")
    w = orc.init_weights(ModelSpec(16, 1, 2, 2, 40, 16), 1, table=(4, 64, 4, 3, 0.05))
    m = api.DcatModel(w)
    for n in G.names(z):
        b = G.batch_from(z, n + ".")
        rep, first, b_u = m.dedup_segments(b)
        assert b_u == int(z[n + ".b_u"][0]), n
        np.testing.assert_array_equal(rep, z[n + ".rep"], err_msg=n)
        np.testing.assert_array_equal(first, z[n + ".first"], err_msg=n)


@pytest.mark.parametrize("layout,shared", [("interleaved", False), ("grouped", True), ("interleaved", True)])
def test_dedup_large_vs_oracle(api, orc, layout, shared):
    w = orc.init_weights(ModelSpec(16, 1, 2, 2, 300, 16), 1, table=(4, 64, 4, 3, 0.05))
    m = api.DcatModel(w)
    b = make_batch(3000, 9, 40, seed=5, layout=layout, shared_storage=shared, ragged=True, empty_users=4)
    rep, first, b_u = m.dedup_segments(b)
    rr, rf, rb = orc.dedup(b)
    assert b_u == rb
    np.testing.assert_array_equal(rep, rr)
    np.testing.assert_array_equal(first, rf)


def test_dedup_forced_hash_collisions(api, orc, monkeypatch):
    """A 3-bit content hash makes almost every row collide: the verify / re-key /
    exact-pass repair must still give the reference plan bit-exactly."""
    w = orc.init_weights(ModelSpec(16, 1, 2, 2, 40, 16), 1, table=(4, 64, 4, 3, 0.05))
    m = api.DcatModel(w)
    b = make_batch(200, 5, 12, seed=9, ragged=True, shared_storage=False)
    monkeypatch.setenv("DCAT_DEBUG_HASH_BITS", "3")
    rep, first, b_u = m.dedup_segments(b)
    monkeypatch.delenv("DCAT_DEBUG_HASH_BITS")
    rr, rf, rb = orc.dedup(b)
    assert b_u == rb
    np.testing.assert_array_equal(rep, rr)
    np.testing.assert_array_equal(first, rf)


# ------------------------------------------------------------------ fp32 parity mode

def test_fp32_cross_goldens(api, orc):
    """cross vs naive sweep of test_dcat.cpp:215-229 plus the empty prefix case."""
    z = G.load("cross")
    for n in G.names(z):
        spec, w = G.weights_from(z, orc, n + ".")
        b = G.batch_from(z, n + ".")
        m = api.DcatModel(w)
        ft = FinetuneSpec(max_events=spec.max_len - 2)
        _, _, h = m.rank_forward_batch(b, ft, precision="fp32", want_h=True)
        err = float(np.abs(h - z[n + ".dcat"]).max())
        assert err <= 1e-4, (n, err)  # test_dcat.cpp:227
        assert float(np.abs(h - z[n + ".naive"]).max()) <= 1e-4, n


def test_fp32_context_kv(api, orc):
    z = G.load("kv")
    spec, w = G.weights_from(z, orc)
    b = G.batch_from(z)
    m = api.DcatModel(w)
    m.rank_forward_batch(b, FinetuneSpec(max_events=spec.max_len - 2), precision="fp32")
    for u in range(2):
        for l in range(2):
            k, v = m.debug_kv(l, u, 64)
            assert np.abs(k - z[f"k.{u}.{l}"]).max() <= 1e-5
            assert np.abs(v - z[f"v.{u}.{l}"]).max() <= 1e-5


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_rank_goldens(api, orc, precision):
    z = G.load("rank")
    for n in G.names(z):
        spec, w = G.weights_from(z, orc, n + ".")
        G.apply_overrides(z, w, n + ".")
        b = G.batch_from(z, n + ".")
        ft = G.ft_from(z, n + ".")
        m = api.DcatModel(w)
        logits, mlog, h = m.rank_forward_batch(b, ft, precision=precision, want_h=ft.use_seq_module)
        if precision == "fp32":
            tol = 1e-4  # test_finetune.cpp:359-361
            assert rel_err(logits, z[n + ".logits"]) <= tol, n
            assert rel_err(mlog, z[n + ".module_logits"]) <= tol, n
            if (n + ".h_cand") in z.files:
                assert float(np.abs(h - z[n + ".h_cand"]).max()) <= 1e-4, n
        else:
            assert rel_err(logits, z[n + ".logits"]) <= 3e-2, (n, rel_err(logits, z[n + ".logits"]))
            assert rel_err(mlog, z[n + ".module_logits"]) <= 3e-2, n
            if (n + ".h_cand") in z.files:
                assert float(np.abs(h - z[n + ".h_cand"]).max()) <= 3e-2, n
                assert cos_min(h, z[n + ".h_cand"]) >= 0.999, n


# ------------------------------------------------------------------ bf16 at BASELINE dims

def _base_setup(orc, U, C, L, **kw):
    spec = ModelSpec(d_model=256, n_layers=4, n_heads=8, mlp_ratio=4, max_len=L + 2, d_emb=256)
    w = orc.init_weights(spec, 42, table=(8, 4096, 32, 7, 0.05), head_seed=11)
    b = make_batch(U, C, L, **kw)
    return spec, w, b


def test_bf16_pinfm_base_sample_vs_oracle(api, orc):
    spec, w, b = _base_setup(orc, 3, 16, 256, seed=4, ragged=True, layout="grouped")
    ft = FinetuneSpec(max_events=256)
    m = api.DcatModel(w)
    logits, mlog, h = m.rank_forward_batch(b, ft, want_h=True)
    rl, rm, _, rh = orc.rank_forward_batch(w, ft, b)
    # PinFM-base, bf16 storage / fp32 accumulate: 1e-2 of the logit scale (observed ~4.5e-3)
    assert float(np.abs(h - rh).max()) <= 1e-2
    assert cos_min(h, rh) >= 0.999
    assert rel_err(logits, rl) <= 1e-2
    assert rel_err(mlog, rm) <= 1e-2
    lf, mf, hf = m.rank_forward_batch(b, ft, precision="fp32", want_h=True)
    assert float(np.abs(hf - rh).max()) <= 1e-4
    assert rel_err(lf, rl) <= 1e-4


@pytest.mark.parametrize("U,C", [(3, 128), (40, 3)])
def test_bf16_crossing_tile_fill(api, orc, U, C):
    """Full crossing tiles (128 candidates of one unique: the k_flash variant without the idle-warp
    branch) and sparse ones (3 per 128-row tile: idle warps only stage K/V), both against the oracle."""
    spec = ModelSpec(d_model=256, n_layers=2, n_heads=8, mlp_ratio=4, max_len=66, d_emb=256)
    w = orc.init_weights(spec, 42, table=(8, 4096, 32, 7, 0.05), head_seed=11)
    b = make_batch(U, C, 64, seed=21, ragged=True, layout="grouped")
    ft = FinetuneSpec(max_events=64)
    m = api.DcatModel(w)
    logits, mlog, h = m.rank_forward_batch(b, ft, want_h=True)
    rl, rm, _, rh = orc.rank_forward_batch(w, ft, b)
    assert float(np.abs(h - rh).max()) <= 3e-2
    assert cos_min(h, rh) >= 0.999
    assert rel_err(logits, rl) <= 3e-2
    assert rel_err(mlog, rm) <= 3e-2


@pytest.mark.parametrize("d", [128, 256])
def test_fused_layer_tail(api, orc, d, monkeypatch):
    """The fused layer tail (o-projection + residual + LN2 + FFN + residual + next LN1 in one
    tcgen05 kernel, layer_tail_tc) against the oracle and against the two-kernel path
    (o-projection GEMM, then the fused FFN) on ragged users, for both d the kernel supports."""
    spec = ModelSpec(d_model=d, n_layers=2, n_heads=d // 32, mlp_ratio=4, max_len=130, d_emb=d)
    w = orc.init_weights(spec, 42, table=(8, 4096, d // 8, 7, 0.05), head_seed=11)
    b = make_batch(5, 7, 128, seed=12, ragged=True, layout="grouped")
    ft = FinetuneSpec(max_events=128)
    m = api.DcatModel(w)
    lf, mf, hf = m.rank_forward_batch(b, ft, want_h=True)
    monkeypatch.setenv("DCAT_NO_TAIL_FUSION", "1")
    l2, m2, h2 = m.rank_forward_batch(b, ft, want_h=True)
    rl, rm, _, rh = orc.rank_forward_batch(w, ft, b)
    for h, lg, mg in ((hf, lf, mf), (h2, l2, m2)):
        assert float(np.abs(h - rh).max()) <= 3e-2 and cos_min(h, rh) >= 0.999
        assert rel_err(lg, rl) <= 3e-2 and rel_err(mg, rm) <= 3e-2
    # the two bf16 paths differ only in rounding order (residual added in TMEM before the bias)
    assert float(np.abs(hf - h2).max()) <= 2e-2 and cos_min(hf, h2) >= 0.9995


@pytest.mark.parametrize("impl", ["fa", "flash"])
def test_bf16_attention_impls_and_kv_cache(api, orc, impl, monkeypatch):
    """Both bf16 attention kernels — the tcgen05 / TMA default (attn_fa.cu, V^T cache) and the
    round-1 mma.sync kernel kept for comparisons (DCAT_ATTN_FLASH=1, row-major V cache) — against
    the oracle on ragged users (unaligned, multi-chunk key ranges), and the bf16 K/V cache against
    context_forward's."""
    if impl == "flash":
        monkeypatch.setenv("DCAT_ATTN_FLASH", "1")
    spec, w, b = _base_setup(orc, 5, 9, 200, seed=6, ragged=True, layout="grouped")
    ft = FinetuneSpec(max_events=200)
    m = api.DcatModel(w)
    logits, mlog, h = m.rank_forward_batch(b, ft, want_h=True)
    rl, rm, _, rh = orc.rank_forward_batch(w, ft, b)
    assert float(np.abs(h - rh).max()) <= 3e-2 and cos_min(h, rh) >= 0.999
    assert rel_err(logits, rl) <= 3e-2 and rel_err(mlog, rm) <= 3e-2
    rep, first, b_u = orc.dedup(b)
    uniq = b.take(first)
    for u in (0, b_u - 1):
        for l in (0, spec.n_layers - 1):
            k, v = m.debug_kv(l, u, 300)
            rk, rv = orc.context_kv(w, uniq, l, u)
            assert k.shape == rk.shape
            assert float(np.abs(k - rk).max()) <= 3e-2 * max(1.0, float(np.abs(rk).max()))
            assert float(np.abs(v - rv).max()) <= 3e-2 * max(1.0, float(np.abs(rv).max()))


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_long_seq_dims_d512(api, orc, precision):
    """long-seq dims (d=512, 8 heads -> head dim 64, FFN 2048): the 512-wide full-row
    epilogue, 2048-wide FFN bias staging and head-dim-64 attention."""
    spec = ModelSpec(d_model=512, n_layers=2, n_heads=8, mlp_ratio=4, max_len=98, d_emb=512)
    w = orc.init_weights(spec, 42, table=(8, 4096, 64, 7, 0.05), head_seed=11)
    b = make_batch(3, 5, 96, seed=12, ragged=True, layout="grouped")
    ft = FinetuneSpec(max_events=96)
    m = api.DcatModel(w)
    logits, mlog, h = m.rank_forward_batch(b, ft, precision=precision, want_h=True)
    rl, rm, _, rh = orc.rank_forward_batch(w, ft, b)
    tol = 1e-4 if precision == "fp32" else 3e-2
    assert float(np.abs(h - rh).max()) <= tol
    assert rel_err(logits, rl) <= tol and rel_err(mlog, rm) <= tol


def test_bf16_full_size_properties(api, orc):
    """PinFM-base at full size (1000 users x 128): properties that hold at any
    size — batch permutation invariance and bit-identical duplicate rows
    (test_dcat.cpp:243-276) — plus oracle parity on a user sample."""
    spec, w, b = _base_setup(orc, 1000, 128, 256, seed=1)
    ft = FinetuneSpec(max_events=256)
    m = api.DcatModel(w)
    logits, mlog, _ = m.rank_forward_batch(b, ft)
    assert np.isfinite(logits).all()
    rng = np.random.default_rng(0)
    perm = rng.permutation(b.n_rows)
    lp, mp, _ = m.rank_forward_batch(b.take(perm), ft)
    np.testing.assert_array_equal(lp, logits[perm])
    np.testing.assert_array_equal(mp, mlog[perm])
    # duplicate (sequence, candidate) rows -> identical outputs
    b2 = b.take(np.arange(b.n_rows))
    b2.candidate[1000] = b2.candidate[0]  # rows 0 and 1000 share unique 0 (interleaved)
    l2, _, _ = m.rank_forward_batch(b2, ft)
    np.testing.assert_array_equal(l2[0], l2[1000])
    # oracle parity on 3 users with all their candidates
    rows = np.nonzero(np.isin(np.arange(b.n_rows) % 1000, [0, 511, 999]))[0]
    sub = b.take(rows)
    rl, rm, _, _ = orc.rank_forward_batch(w, ft, sub)
    assert rel_err(logits[rows], rl) <= 1e-2
    assert rel_err(mlog[rows], rm) <= 1e-2


def test_device_resident_io_matches_host(api, orc):
    import torch
    spec, w, b = _base_setup(orc, 20, 8, 64, seed=2, ragged=True)
    ft = FinetuneSpec(max_events=64)
    m = api.DcatModel(w)
    lh, mh, hh = m.rank_forward_batch(b, ft, want_h=True)
    bd = b.to(lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64) if a.dtype == np.uint64 else a).cuda())
    ld, md, hd = m.rank_forward_batch(bd, ft, want_h=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(ld.cpu().numpy(), lh)
    np.testing.assert_array_equal(md.cpu().numpy(), mh)
    np.testing.assert_array_equal(hd.cpu().numpy(), hh)


# ------------------------------------------------------------------ errors (reference SEQFM_CHECKs)

def test_scoring_graph_replay(api, orc):
    """Repeated calls with the same sizes and buffers replay a captured CUDA graph of the scoring
    pass (third call on): results must equal the stream-launched pass, also when the data in the
    same device buffers changes between calls."""
    import torch
    spec, w, b = _base_setup(orc, 24, 6, 48, seed=9, ragged=True)
    ft = FinetuneSpec(max_events=48)
    m = api.DcatModel(w)
    bd = b.to(lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64) if a.dtype == np.uint64 else a).cuda())
    out = (torch.empty((b.n_rows, 3), device="cuda"), torch.empty((b.n_rows, 3), device="cuda"), None)
    runs = []
    for _ in range(4):  # stream, capture + launch, replay, replay
        lg, ml, _ = m.rank_forward_batch(bd, ft, out=out)
        torch.cuda.synchronize()
        runs.append((lg.cpu().numpy().copy(), ml.cpu().numpy().copy()))
    for lg, ml in runs[1:]:
        np.testing.assert_array_equal(lg, runs[0][0])
        np.testing.assert_array_equal(ml, runs[0][1])
    # new candidates in the same buffers (same plan, same sizes): the replay sees the new data
    new_c = np.random.default_rng(3).integers(0, 1_000_000, b.n_rows).astype(np.uint64)
    bd.candidate.copy_(torch.from_numpy(new_c.view(np.int64)))
    lg, ml, _ = m.rank_forward_batch(bd, ft, out=out)
    torch.cuda.synchronize()
    b2 = b.take(np.arange(b.n_rows))
    b2.candidate = new_c
    fresh = api.DcatModel(w)  # its first call launches on the stream (no graph yet)
    lr, mr, _ = fresh.rank_forward_batch(b2, ft)
    np.testing.assert_array_equal(lg.cpu().numpy(), lr)
    np.testing.assert_array_equal(ml.cpu().numpy(), mr)
    rl, rm, _, _ = orc.rank_forward_batch(w, ft, b2)
    assert rel_err(lr, rl) <= 3e-2


def test_errors(api, orc):
    spec = ModelSpec(d_model=64, n_layers=2, n_heads=4, mlp_ratio=4, max_len=20, d_emb=64)
    w = orc.init_weights(spec, 3, table=(8, 128, 8, 7, 0.05))
    m = api.DcatModel(w)
    ft = FinetuneSpec(max_events=16)
    b = make_batch(4, 3, 16, seed=1)
    m.rank_forward_batch(b, ft)
    bad = make_batch(4, 3, 16, seed=1)
    bad.ev_action[5] = 9
    with pytest.raises(RuntimeError, match="unknown action"):
        m.rank_forward_batch(bad, ft)
    bad = make_batch(4, 3, 16, seed=1)
    bad.ev_surface[3] = 4
    with pytest.raises(RuntimeError, match="unknown surface"):
        m.rank_forward_batch(bad, ft)
    long = make_batch(2, 2, 20, seed=1)  # valid 20 == max_len: the candidate position is out of range
    with pytest.raises(RuntimeError, match="position"):
        m.rank_forward_batch(long, ft)
    neg = make_batch(4, 3, 16, seed=1)
    neg.age_seconds[2] = -5.0
    with pytest.raises(RuntimeError, match="non-negative"):
        m.rank_forward_batch(neg, ft)
    with pytest.raises(RuntimeError, match="auxiliary"):
        m.rank_forward_batch(b, FinetuneSpec(variant="aux", max_events=16))
    # AuxLt needs a two-selector head (d_module = 2 d, finetune.cpp:251-256)
    with pytest.raises(RuntimeError, match="d_module"):
        m.rank_forward_batch(b, FinetuneSpec(variant="aux-lt", max_events=16))
    with pytest.raises(RuntimeError, match="max_len"):
        m.rank_forward_batch(b, FinetuneSpec(max_events=19))


@pytest.mark.gpu
def test_fixed_window(api, orc):
    """Fixed-window sequence module (context_forward_fixed / cross_forward_fixed,
    dcat.cpp:281-415) through the C ABI's `window` field: the reference-pinned goldens on every
    fill level (fp32, 1e-4), and a ragged d=256 batch in both precisions against the oracle —
    h_cand (sequence module) and logits (ranking head on the full row's context features)."""
    z = G.load("fixed")
    _, w = G.weights_from(z, orc)
    W = int(z["window"])
    m = api.DcatModel(w)
    for n in G.names(z):
        b = G.batch_from(z, n + ".")
        _, _, h = m.rank_forward_batch(b, FinetuneSpec(max_events=24, window=W), precision="fp32", want_h=True)
        assert float(np.abs(h - z[n + ".h"]).max()) <= 1e-4, n
    spec, w, b = _base_setup(orc, 4, 6, 120, seed=21, ragged=True, layout="grouped")
    m = api.DcatModel(w)
    for window in (1, 17, 64, 400):
        ft = FinetuneSpec(max_events=120, window=window)
        rl, rm, _, rh = orc.rank_forward_batch(w, ft, b)
        np.testing.assert_allclose(rh, orc.dcat_outputs_fixed(w, b, window), atol=1e-6)
        lf, mf, hf = m.rank_forward_batch(b, ft, precision="fp32", want_h=True)
        assert float(np.abs(hf - rh).max()) <= 1e-4 and rel_err(lf, rl) <= 1e-4, window
        lb, mb, hb = m.rank_forward_batch(b, ft, want_h=True)
        assert float(np.abs(hb - rh).max()) <= 3e-2 and cos_min(hb, rh) >= 0.999, window
        assert rel_err(lb, rl) <= 3e-2 and rel_err(mb, rm) <= 3e-2, window
        # the cache holds at most window - 1 tokens per unique (test_dcat.cpp:363-382)
        rep, first, b_u = orc.dedup(b)
        kept = np.minimum(b.row_valid[first], max(window - 1, 0)).sum()
        assert m.last_stats()["ctx_tokens"] == kept


@pytest.mark.gpu
def test_quantized_id_table(api, orc):
    """QuantizedTable id source (int4 / int8 rows, fp16 scale / bias; embed.hpp:80-125) through
    the C ABI: the gathers dequantize on the fly. Reference-pinned goldens in fp32 (1e-4) and a
    d=256 PinFM-shaped batch in both precisions against the oracle."""
    z = G.load("quant")
    _, w = G.weights_from(z, orc, "rank.")
    b = G.batch_from(z, "rank.")
    ft = FinetuneSpec(max_events=12)
    for bits in (4, 8):
        wq = w.with_quantized_table(bits, orc.quantize_table(w, bits))
        m = api.DcatModel(wq)
        lf, _, hf = m.rank_forward_batch(b, ft, precision="fp32", want_h=True)
        assert rel_err(lf, z[f"rank.b{bits}.logits"]) <= 1e-4
        assert float(np.abs(hf - z[f"rank.b{bits}.h"]).max()) <= 1e-4
    spec, w, b = _base_setup(orc, 4, 8, 96, seed=23, ragged=True)
    ft = FinetuneSpec(max_events=96)
    for bits in (4, 8):
        wq = w.with_quantized_table(bits, orc.quantize_table(w, bits))
        rl, rm, _, rh = orc.rank_forward_batch(wq, ft, b)
        m = api.DcatModel(wq)
        lf, _, hf = m.rank_forward_batch(b, ft, precision="fp32", want_h=True)
        assert float(np.abs(hf - rh).max()) <= 1e-4 and rel_err(lf, rl) <= 1e-4, bits
        lb, mb, hb = m.rank_forward_batch(b, ft, want_h=True)
        assert float(np.abs(hb - rh).max()) <= 3e-2 and cos_min(hb, rh) >= 0.999, bits
        assert rel_err(lb, rl) <= 3e-2 and rel_err(mb, rm) <= 3e-2, bits
        # the quantized source really is what scores: int4 differs from the fp32 table
        if bits == 4:
            l32, _, _ = api.DcatModel(w).rank_forward_batch(b, ft, precision="fp32")
            assert float(np.abs(l32 - lf).max()) > 1e-5


@pytest.mark.gpu
def test_checkpoint_and_sequence_files(api, orc):
    """A PFMC1 checkpoint written by the reference scores on the device like the saved model,
    and a PSEQ1 file becomes a request batch (on-disk inputs)."""
    from paper_2507_12704_b200 import ckpt, seqfile
    z = G.load("files")
    w = ckpt.loads_checkpoint(z["ckpt_learned.file"].tobytes()).weights()
    b = G.batch_from(z, "ckpt_learned.")
    m = api.DcatModel(w)
    lf, _, _ = m.rank_forward_batch(b, FinetuneSpec(max_events=10), precision="fp32")
    assert rel_err(lf, z["ckpt_learned.logits"]) <= 1e-4
    s = seqfile.loads(z["seq.file"].tobytes())
    sb = seqfile.ranking_batch(s, [0, 2, 2, 3, 4, 0], [11, 12, 13, 14, 15, 16], [3600.0] * 6, max_events=6)
    rl = orc.rank_forward_batch(w, FinetuneSpec(max_events=10), sb)[0]
    ls, _, _ = m.rank_forward_batch(sb, FinetuneSpec(max_events=10), precision="fp32")
    assert rel_err(ls, rl) <= 1e-4


@pytest.mark.gpu
def test_fusion_variants(api, orc):
    """LiteMean / LiteLast (pooled per-unique selector, no crossing pass) and AuxLt (learnable
    token appended to the cached context, selectors [H_lt | H_cand]) on the device: the
    reference-pinned goldens in fp32 (1e-4, dense and with empty sequences) and a ragged d=256
    batch in both precisions against the oracle."""
    z = G.load("variants")
    for n in G.names(z):
        _, w = G.weights_from(z, orc, n + ".")
        G.apply_overrides(z, w, n + ".")
        b = G.batch_from(z, n + ".")
        ft = G.ft_from(z, n + ".")
        lf, mf, _ = api.DcatModel(w).rank_forward_batch(b, ft, precision="fp32")
        assert rel_err(lf, z[n + ".logits"]) <= 1e-4, n
        assert rel_err(mf, z[n + ".module_logits"]) <= 1e-4, n
    spec = ModelSpec(d_model=256, n_layers=2, n_heads=8, mlp_ratio=4, max_len=98, d_emb=256)
    rng = np.random.default_rng(3)
    for variant in ("lite-mean", "lite-last", "aux-lt"):
        w = orc.init_weights(spec, 42, table=(8, 4096, 32, 7, 0.05), head_seed=11, sel=2 if variant == "aux-lt" else 1)
        w.head["aux_proj"][:] = (0.05 * rng.standard_normal(w.head["aux_proj"].shape)).astype(np.float32)
        b = make_batch(4, 6, 96, seed=29, ragged=True, d_aux=16)
        ft = FinetuneSpec(variant=variant, max_events=96)
        rl, rm, _, _ = orc.rank_forward_batch(w, ft, b)
        m = api.DcatModel(w)
        lf, mf, _ = m.rank_forward_batch(b, ft, precision="fp32")
        assert rel_err(lf, rl) <= 1e-4 and rel_err(mf, rm) <= 1e-4, variant
        lb, mb, _ = m.rank_forward_batch(b, ft)
        assert rel_err(lb, rl) <= 3e-2 and rel_err(mb, rm) <= 3e-2, variant
