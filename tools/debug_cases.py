"""Debug aid: run small PinFM-dims cases in separate processes, report which fail."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1:
    import numpy as np
    from oracle import pyoracle
    from paper_2507_12704_b200 import api
    from paper_2507_12704_b200.abi import FinetuneSpec, ModelSpec
    from paper_2507_12704_b200.synth import make_batch
    U, C, L, ragged, grouped = [int(x) for x in sys.argv[1:6]]
    spec = ModelSpec(256, 1, 8, 4, L + 2, 256)
    w = pyoracle.oracle().init_weights(spec, 42, table=(8, 4096, 32, 7, 0.05))
    b = make_batch(U, C, L, seed=4, ragged=bool(ragged), layout="grouped" if grouped else "interleaved")
    m = api.DcatModel(w)
    lg, ml, h = m.rank_forward_batch(b, FinetuneSpec(max_events=L))
    print("ok", b.row_valid[:: C if grouped else 1][:U].tolist()[:8])
else:
    cases = [(2, 4, 256, 0, 0), (3, 16, 256, 1, 1), (3, 16, 256, 0, 1), (1, 4, 200, 0, 0), (1, 4, 100, 0, 0),
             (1, 4, 64, 0, 0), (1, 4, 130, 0, 0), (1, 200, 256, 0, 0), (1, 4, 255, 0, 0)]
    for cs in cases:
        for env in ({}, {"DCAT_TC_ATTENTION": "1"}):
            r = subprocess.run([sys.executable, __file__] + [str(x) for x in cs], capture_output=True, text=True,
                               env={**os.environ, **env, "CUDA_LAUNCH_BLOCKING": "1"})
            print(cs, "tc   " if env else "flash", "rc", r.returncode, (r.stdout.strip().splitlines() or [""])[-1][:60],
                  (r.stderr.strip().splitlines() or [""])[-1][:150])
