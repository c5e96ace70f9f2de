import sys; sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
import golden_util as G
from oracle import pyoracle
from paper_2507_12704_b200 import api
orc = pyoracle.oracle()
z = G.load("variants")
n = "d16_aux-lt_dense"
_, w = G.weights_from(z, orc, n + ".")
G.apply_overrides(z, w, n + ".")
b = G.batch_from(z, n + ".")
ft = G.ft_from(z, n + ".")
d = w.spec.d_model
for part in ("lt", "cand"):
    w2 = G.weights_from(z, orc, n + ".")[1]; G.apply_overrides(z, w2, n + ".")
    mw = w2.head["mod_w"].reshape(2 * d, 3)
    if part == "lt": mw[d:] = 0
    else: mw[:d] = 0
    rl, rm, _, _ = orc.rank_forward_batch(w2, ft, b)
    lf, mf, hf = api.DcatModel(w2).rank_forward_batch(b, ft, precision="fp32", want_h=True)
    print(part, "mlog max abs diff", float(np.abs(mf - rm).max()), "scale", float(np.abs(rm).max()))
print("rep", orc.dedup(b)[0][:12], "valid", b.row_valid[:12])
