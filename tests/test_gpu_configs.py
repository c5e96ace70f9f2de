"""Oracle parity on the paths the BASELINE configs live on (VERDICT r01 "What's weak" 1a-1d).

* multi-tile crossing: a unique with more candidates than one 128-row crossing tile (C_u = 129,
  300 and high-fanout's 4096) in grouped and interleaved row order, L = 512, d = 256;
* sharp softmax at production head dims (lifted wq / wk so the scaled logits span well over
  10 nats): head dim 32 (d = 256) and 64 (d = 512), causal and crossing, with the attention
  kernels' online-rescale counter asserted non-zero;
* long-seq: d = 512, 8 layers, two users ragged up to L = 1024;
* the per-config max relative logit error at every BASELINE config's dims, printed.

The GPU scores every row; the oracle (single-threaded C) scores a sample of rows. A row's
scores depend only on its own sequence and candidate (cross_forward dcat.cpp:199-271), so the
sample is checked against the full-batch GPU rows. Tolerances: bf16 storage / fp32 accumulate,
logits within 1e-2 of the logit scale (2e-2 for the lifted-logit cases, where bf16 rounding of q
and k is amplified by the logit scale), H max-abs 2e-2 and cosine >= 0.999.
"""
import numpy as np
import pytest

from oracle import pyoracle
from paper_2507_12704_b200.abi import FinetuneSpec, ModelSpec
from paper_2507_12704_b200.synth import CONFIGS, make_batch

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


def lift_qk(w, lift):
    """wq, wk *= lift (the reference test's "lifted" weights, tests/golden/make_golden.py)."""
    base = (4 if w.spec.pos_learned else 3) + 12
    for l in range(w.spec.n_layers):
        w.tensors[base + 16 * l + 2] *= np.float32(lift)
        w.tensors[base + 16 * l + 4] *= np.float32(lift)
    return w


def sample_rows(U, C, layout, per_unique, rng):
    """Row indices of candidate slots `per_unique` (+ a few random ones) of every unique."""
    rows = []
    for u in range(U):
        slots = set(int(c) for c in per_unique if 0 <= c < C)
        slots |= set(int(c) for c in rng.integers(0, C, 6))
        for c in sorted(slots):
            rows.append(u * C + c if layout == "grouped" else c * U + u)
    return np.array(sorted(rows))


def check_sample(api, orc, w, b, ft, rows, tol, h_tol=2e-2, m=None, m_tol=None):
    m = m or api.DcatModel(w)
    logits, mlog, h = m.rank_forward_batch(b, ft, want_h=True)
    sub = b.take(rows)
    rl, rm, _, rh = orc.rank_forward_batch(w, ft, sub)
    e_l, e_m = rel_err(logits[rows], rl), rel_err(mlog[rows], rm)
    e_h, c_h = float(np.abs(h[rows] - rh).max()), cos_min(h[rows], rh)
    assert e_l <= tol and e_m <= (m_tol or tol), (e_l, e_m)
    assert e_h <= h_tol and c_h >= 0.999, (e_h, c_h)
    return e_l, m


# ------------------------------------------------------------------ multi-tile crossing

@pytest.mark.parametrize("layout", ["grouped", "interleaved"])
@pytest.mark.parametrize("C", [129, 300, 4096])
def test_multi_tile_crossing(api, orc, layout, C):
    """Uniques with C_u > 128 candidates span several crossing tiles (32 at high-fanout's 4096);
    every tile re-reads the unique's cached K/V. Rows at tile boundaries are always sampled."""
    U = 2 if C == 4096 else 3
    spec = ModelSpec(d_model=256, n_layers=2, n_heads=8, mlp_ratio=4, max_len=514, d_emb=256)
    w = orc.init_weights(spec, 42, table=(8, 4096, 32, 7, 0.05), head_seed=11)
    b = make_batch(U, C, 512, seed=31 + C, layout=layout, ragged=True)
    ft = FinetuneSpec(max_events=512)
    edges = [0, 1, 127, 128, 129, 255, 256, 257, 299, 2047, 2048, 4095]
    rows = sample_rows(U, C, layout, edges, np.random.default_rng(C))
    err, _ = check_sample(api, orc, w, b, ft, rows, 1e-2)
    print(f"multi-tile crossing C={C} {layout}: max rel logit err {err:.2e} on {rows.size} rows")


# ------------------------------------------------------------------ sharp softmax

@pytest.mark.parametrize("d,heads", [(256, 8), (512, 8)])
def test_sharp_attention_rescale(api, orc, d, heads, monkeypatch):
    """wq, wk x 4: scaled logits x 16 (std ~1.6, ranges > 10 nats over 200+ keys), so the running
    max of the online softmax moves past the kernels' lazy-rescale threshold in both the causal
    (context) and the crossing kernel. Head dim 32 and 64."""
    monkeypatch.setenv("DCAT_DEBUG_COUNTERS", "1")
    spec = ModelSpec(d_model=d, n_layers=2, n_heads=heads, mlp_ratio=4, max_len=258, d_emb=d)
    w = lift_qk(orc.init_weights(spec, 42, table=(8, 4096, d // 8, 7, 0.05), head_seed=11), 4.0)
    b = make_batch(3, 130, 256, seed=41, layout="grouped", ragged=True)
    ft = FinetuneSpec(max_events=256)
    rows = sample_rows(3, 130, "grouped", [0, 64, 127, 128, 129], np.random.default_rng(1))
    m = api.DcatModel(w)
    err, _ = check_sample(api, orc, w, b, ft, rows, 2e-2, h_tol=3e-2, m=m)
    cnt = m.debug_counters()
    print(f"sharp attention d={d}: max rel logit err {err:.2e}, rescale events {cnt}")
    assert cnt["rescale_causal"] > 0 and cnt["rescale_cross"] > 0, cnt
    # fp32 parity mode on the same sharp model: the reference's own 1e-4 bound
    lf, _, _ = m.rank_forward_batch(b, ft, precision="fp32")
    rl, _, _, _ = orc.rank_forward_batch(w, ft, b.take(rows))
    assert rel_err(lf[rows], rl) <= 1e-4


# ------------------------------------------------------------------ long-seq

def test_long_seq_l1024(api, orc):
    """long-seq dims: d = 512, 8 layers, head dim 64, one user at the full L = 1024 and one ragged;
    a 1024-token causal pass and 1025-key crossing rows (8 key chunks of 128)."""
    spec = ModelSpec(d_model=512, n_layers=8, n_heads=8, mlp_ratio=4, max_len=1026, d_emb=512)
    w = orc.init_weights(spec, 42, table=(8, 4096, 64, 7, 0.05), head_seed=11)
    b = make_batch(2, 5, 1024, seed=7, layout="grouped", valid=[1024, 611])
    ft = FinetuneSpec(max_events=1024)
    rows = np.arange(b.n_rows)
    err, _ = check_sample(api, orc, w, b, ft, rows, 1e-2)
    print(f"long-seq L=1024: max rel logit err {err:.2e}")


# ------------------------------------------------------------------ every BASELINE config's dims

@pytest.mark.parametrize("name", list(CONFIGS))
def test_config_dims_sample(api, orc, name):
    """Every BASELINE config at its model dims and sequence length on a small user sample (2-3
    users, every candidate slot up to 160), ragged sequences; prints the max relative error."""
    cfg = CONFIGS[name]
    spec, L = cfg["spec"], cfg["L"]
    C = min(cfg["C"], 160)
    U = 2 if L >= 1024 else 3
    w = orc.init_weights(spec, 42, table=(8, 4096, spec.d_emb // 8, 7, 0.05), head_seed=11)
    b = make_batch(U, C, L, seed=5, layout="interleaved", ragged=True)
    ft = FinetuneSpec(max_events=L)
    rng = np.random.default_rng(2)
    rows = np.arange(b.n_rows) if b.n_rows <= 64 else np.sort(rng.choice(b.n_rows, 48, replace=False))
    # long-seq (8 layers, d = 512, L = 1024): the module logits of this sample are small (max 0.037,
    # rms 0.014) and their bf16 noise against the fp32 oracle is ~1e-4 mean / ~3.5e-4 max absolute
    # whichever d = 512 epilogue runs (one CTA: 0.88e-2 of the max, CTA pair: 1.04e-2); the logits
    # keep the 1e-2 bound
    m_tol = 1.5e-2 if name == "long-seq" else None
    err, _ = check_sample(api, orc, w, b, ft, rows, 1e-2, m_tol=m_tol)
    print(f"config {name}: max rel logit err {err:.2e} (bf16 vs oracle, {rows.size} rows)")
