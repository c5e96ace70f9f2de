"""Debug aid: d=512 (long-seq dims) small case with blocking launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import pyoracle
from paper_2507_12704_b200 import api
from paper_2507_12704_b200.abi import FinetuneSpec, ModelSpec
from paper_2507_12704_b200.synth import make_batch
layers, L, prec = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
spec = ModelSpec(512, layers, 8, 4, L + 2, 512)
w = pyoracle.oracle().init_weights(spec, 42, table=(8, 4096, 64, 7, 0.05))
b = make_batch(2, 4, L, seed=3)
m = api.DcatModel(w)
lg, ml, h = m.rank_forward_batch(b, FinetuneSpec(max_events=L), precision=prec, want_h=True)
rl, rm, _, rh = pyoracle.oracle().rank_forward_batch(w, FinetuneSpec(max_events=L), b)
print("ok", float(np.abs(h - rh).max()), float(np.abs(lg - rl).max()))
