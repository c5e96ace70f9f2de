"""Kernel bring-up helper: runs one small scoring call per case in a subprocess with a timeout,
so a hang names its case. Usage: python tools/fa_debug.py [case ...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = {
    # name: (d, layers, heads, U, C, L, ragged, lift)
    "base_small": (256, 2, 8, 2, 6, 256, True, 1.0),
    "base_fixed": (256, 2, 8, 2, 6, 256, False, 1.0),
    "one_user": (256, 1, 8, 1, 3, 100, False, 1.0),
    "one_user_200": (256, 1, 8, 1, 3, 200, False, 1.0),
    "sharp": (256, 2, 8, 3, 130, 256, True, 4.0),
    "d512": (512, 2, 8, 2, 5, 300, True, 1.0),
    "d512_sharp": (512, 2, 8, 3, 130, 256, True, 4.0),
    "d512_fixed": (512, 2, 8, 2, 5, 256, False, 1.0),
    "tiny": (64, 2, 4, 4, 3, 64, True, 1.0),
    "multi_item": (256, 2, 8, 40, 20, 256, False, 1.0),
    "multi_item_ragged": (256, 2, 8, 40, 20, 256, True, 1.0),
    "many": (256, 2, 8, 300, 16, 256, True, 1.0),
}

CHILD = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from oracle import pyoracle
from paper_2507_12704_b200 import api
from paper_2507_12704_b200.abi import FinetuneSpec, ModelSpec
from paper_2507_12704_b200.synth import make_batch
d, nl, H, U, C, L, ragged, lift = %r
orc = pyoracle.oracle()
spec = ModelSpec(d_model=d, n_layers=nl, n_heads=H, mlp_ratio=4, max_len=L + 2, d_emb=d)
w = orc.init_weights(spec, 42, table=(8, 4096, d // 8, 7, 0.05), head_seed=11)
if lift != 1.0:
    base = 4 + 12
    for l in range(nl):
        w.tensors[base + 16 * l + 2] *= np.float32(lift)
        w.tensors[base + 16 * l + 4] *= np.float32(lift)
b = make_batch(U, C, L, seed=5, layout="grouped", ragged=ragged)
ft = FinetuneSpec(max_events=L)
m = api.DcatModel(w)
lg, ml, h = m.rank_forward_batch(b, ft, want_h=True)
rl, rm, _, rh = orc.rank_forward_batch(w, ft, b)
e = float(np.abs(lg - rl).max() / max(1e-3, np.abs(rl).max()))
print("valid", b.row_valid[::C].tolist(), "rel err %%.3e" %% e, "dH %%.3e" %% float(np.abs(h - rh).max()))
"""

for name in (sys.argv[1:] or list(CASES)):
    code = CHILD % (ROOT, CASES[name])
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=40)
        out = (r.stdout.strip().splitlines() or [""])[-1]
        err = "\n".join(r.stderr.strip().splitlines()[-14:]) if r.returncode else ""
        print(f"{name}: rc={r.returncode} {out} {err}", flush=True)
    except subprocess.TimeoutExpired:
        print(f"{name}: TIMEOUT (hang)", flush=True)
