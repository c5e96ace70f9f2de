"""The DCAT sub-API on the device (dcat.hpp:47-101): context_forward -> device K/V cache ->
candidate_inputs -> cross_forward, and the fixed-window pair, against the CPU oracle.

Tolerances: fp32 parity mode K/V max-abs 1e-5 (test_dcat.cpp:166-213 pins the reference's cache
bitwise to the forward caches) and rows 1e-4 (test_dcat.cpp:227); bf16 storage / fp32 accumulate
K/V within 3e-2 of the value scale, rows max-abs 2e-2 and cosine >= 0.999.
"""
import numpy as np
import pytest

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


def cos_min(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(((a * b).sum(1) / (np.linalg.norm(a, axis=1) * np.linalg.norm(b, axis=1) + 1e-30)).min())


def setup(orc, d=256, L=120, U=5, C=7, seed=3):
    spec = ModelSpec(d_model=d, n_layers=2, n_heads=8, mlp_ratio=4, max_len=L + 2, d_emb=d)
    w = orc.init_weights(spec, 42, table=(8, 4096, d // 8, 7, 0.05), head_seed=11)
    b = make_batch(U, C, L, seed=seed, layout="interleaved", ragged=True, shared_storage=False)
    return spec, w, b


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_context_cache_and_cross(api, orc, precision):
    spec, w, b = setup(orc)
    m = api.DcatModel(w)
    rep, first, b_u = orc.dedup(b)
    uniq = b.take(first)
    kv, _ = m.context_forward(uniq, precision=precision)
    assert kv.n_uniques == b_u and kv.n_layers == spec.n_layers
    np.testing.assert_array_equal(kv.lengths(), uniq.row_valid)
    for u in range(b_u):
        for l in range(spec.n_layers):
            k, v = kv.read(l, u)
            rk, rv = orc.context_kv(w, uniq, l, u)
            if precision == "fp32":
                assert float(np.abs(k - rk).max()) <= 1e-5 and float(np.abs(v - rv).max()) <= 1e-5
            else:
                assert float(np.abs(k - rk).max()) <= 3e-2 * max(1.0, float(np.abs(rk).max()))
                assert float(np.abs(v - rv).max()) <= 3e-2 * max(1.0, float(np.abs(rv).max()))
    # candidate_inputs at pos = n (one past the unique's sequence) -> cross_forward rows
    e = m.candidate_inputs(b.candidate, b.row_valid)
    h = m.cross_forward(kv, rep, e)
    ref = orc.dcat_outputs(w, b)
    if precision == "fp32":
        assert float(np.abs(h - ref).max()) <= 1e-4
    else:
        assert float(np.abs(h - ref).max()) <= 2e-2 and cos_min(h, ref) >= 0.999
    # the same cache crossed with a second candidate batch (no context recompute)
    b2 = b.take(np.arange(b.n_rows))
    b2.candidate = np.random.default_rng(9).integers(0, 1_000_000, b.n_rows).astype(np.uint64)
    h2 = m.cross_forward(kv, rep, m.candidate_inputs(b2.candidate, b2.row_valid))
    ref2 = orc.dcat_outputs(w, b2)
    tol = 1e-4 if precision == "fp32" else 2e-2
    assert float(np.abs(h2 - ref2).max()) <= tol
    # and the composite path scores the same rows
    _, _, hr = m.rank_forward_batch(b2, FinetuneSpec(max_events=120), precision=precision, want_h=True)
    assert float(np.abs(h2 - hr).max()) <= (1e-6 if precision == "fp32" else 1e-2)
    kv.close()


def test_duplicate_uniques_and_subset_rep(api, orc):
    """Rows given to context_forward may repeat a sequence (they share one device cache entry);
    cross rows may reference any subset of the cache's rows."""
    spec, w, b = setup(orc, U=4, C=3)
    m = api.DcatModel(w)
    rep, first, b_u = orc.dedup(b)
    uniq = b.take(np.concatenate([first, first[:2]]))  # rows b_u, b_u + 1 repeat uniques 0, 1
    kv, _ = m.context_forward(uniq, precision="fp32")
    assert kv.n_uniques == b_u + 2
    for l in range(spec.n_layers):
        np.testing.assert_array_equal(kv.read(l, b_u)[0], kv.read(l, 0)[0])
    rows = np.nonzero(rep < 2)[0]
    sub = b.take(rows)
    alt_rep = rep[rows] + b_u  # the repeated rows stand for uniques 0 / 1
    h = m.cross_forward(kv, alt_rep, m.candidate_inputs(sub.candidate, sub.row_valid))
    assert float(np.abs(h - orc.dcat_outputs(w, sub)).max()) <= 1e-4


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_fixed_window_pair(api, orc, precision):
    """context_forward_fixed / cross_forward_fixed (dcat.cpp:281-415): newest window - 1 events,
    positions from 0, the candidate at position kept."""
    spec, w, b = setup(orc, seed=8)
    m = api.DcatModel(w)
    rep, first, b_u = orc.dedup(b)
    uniq = b.take(first)
    for window in (1, 17, 64):
        kv, _ = m.context_forward(uniq, window=window, precision=precision)
        kept = np.minimum(uniq.row_valid, window - 1)
        np.testing.assert_array_equal(kv.lengths(), kept)
        pos = np.minimum(b.row_valid, window - 1)
        h = m.cross_forward(kv, rep, m.candidate_inputs(b.candidate, pos))
        ref = orc.dcat_outputs_fixed(w, b, window)
        if precision == "fp32":
            assert float(np.abs(h - ref).max()) <= 1e-4, window
        else:
            assert float(np.abs(h - ref).max()) <= 2e-2 and cos_min(h, ref) >= 0.999, window
        kv.close()


def test_emit_hidden_rows(api, orc):
    """emit_hidden: h_user = phi_out of every context token; its last row per unique is the
    LiteLast selector (gather_selectors finetune.cpp:258-274) of the composite path."""
    spec, w, b = setup(orc, U=4, C=2)
    m = api.DcatModel(w)
    rep, first, b_u = orc.dedup(b)
    uniq = b.take(first)
    kv, hu = m.context_forward(uniq, emit_hidden=True, want_h=True, precision="fp32")
    n = kv.lengths()
    last = hu[np.cumsum(n) - 1]
    _, _, sel = m.rank_forward_batch(b, FinetuneSpec(variant="lite-last", max_events=120), precision="fp32",
                                     want_h=True)
    np.testing.assert_allclose(last[rep], sel, atol=1e-6)
    assert np.allclose(np.linalg.norm(hu, axis=1), 1.0, atol=1e-4)  # phi_out rows are unit norm


def test_subapi_errors(api, orc):
    spec, w, b = setup(orc, U=3, C=2)
    m = api.DcatModel(w)
    rep, first, b_u = orc.dedup(b)
    kv, _ = m.context_forward(b.take(first))
    e = m.candidate_inputs(b.candidate, b.row_valid)
    with pytest.raises(RuntimeError, match="plan rep"):
        m.cross_forward(kv, np.full(b.n_rows, b_u, np.int32), e)
    with pytest.raises(RuntimeError, match="position"):
        m.candidate_inputs(b.candidate[:2], np.array([0, spec.max_len], np.int32))
    with pytest.raises(RuntimeError, match="h_user requires emit_hidden"):
        m.context_forward(b.take(first), want_h=True)
    with pytest.raises(RuntimeError, match="window must be >= 1"):
        m.context_forward(b.take(first), window=-1)
    kv32, _ = m.context_forward(b.take(first), precision="fp32")
    kv32.precision = "bf16"  # a cache is crossed in the precision it was built in
    with pytest.raises(RuntimeError, match="precision"):
        m.cross_forward(kv32, rep, e)
