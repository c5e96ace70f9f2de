"""Runs each rank golden in bf16 in its own process; prints which ones fail (debug aid)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
if len(sys.argv) > 1:
    import numpy as np
    import golden_util as G
    from oracle import pyoracle
    from paper_2507_12704_b200 import api
    z = G.load("rank"); n = sys.argv[1]
    spec, w = G.weights_from(z, pyoracle.oracle(), n + ".")
    G.apply_overrides(z, w, n + ".")
    b = G.batch_from(z, n + "."); ft = G.ft_from(z, n + ".")
    m = api.DcatModel(w)
    lg, ml, h = m.rank_forward_batch(b, ft, precision=sys.argv[2] if len(sys.argv) > 2 else "bf16")
    print(n, "ok", float(np.abs(lg - z[n + ".logits"]).max()))
else:
    import golden_util as G
    for n in G.names(G.load("rank")):
        r = subprocess.run([sys.executable, __file__, n], capture_output=True, text=True)
        print(n, "rc", r.returncode, (r.stdout.strip().splitlines() or [""])[-1], (r.stderr.strip().splitlines() or [""])[-1][:200])
