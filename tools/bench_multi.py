"""Throughput of the C++ multi-device path (dcat_multi_rank_forward_batch, csrc/multi.cu) on one
box: host batch in, host scores out (sharding, per-device H2D, scoring, NCCL gather and D2H all
inside the timed call), wall clock, median of the timed calls. One JSON line per run.
Usage: python tools/bench_multi.py --config high-fanout --devices 4 [--users-per-gpu U]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_12704_b200 import api  # noqa: E402
from paper_2507_12704_b200.abi import FinetuneSpec  # noqa: E402
from paper_2507_12704_b200.synth import CONFIGS, init_weights, make_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="pinfm-base", choices=sorted(CONFIGS))
ap.add_argument("--devices", type=int, default=1)
ap.add_argument("--users-per-gpu", type=int, default=0)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=2)
a = ap.parse_args()
cfg = CONFIGS[a.config]
U = (a.users_per_gpu or cfg["U"]) * a.devices
w = init_weights(cfg["spec"], 42)
b = make_batch(U, cfg["C"], cfg["L"], seed=1, layout="interleaved")
ft = FinetuneSpec(max_events=cfg["L"])
mm = api.MultiDcatModel(w, list(range(a.devices)))
out = (np.zeros((b.n_rows, 3), np.float32), np.zeros((b.n_rows, 3), np.float32))
for _ in range(a.warmup):
    mm.rank_forward_batch(b, ft, out=out)
ts = []
for _ in range(a.steps):
    t0 = time.perf_counter()
    mm.rank_forward_batch(b, ft, out=out)
    ts.append(time.perf_counter() - t0)
owner = mm.shard(b)
med = float(np.median(ts))
print(json.dumps({"config": a.config, "devices": a.devices, "users": U, "rows": b.n_rows,
                  "cand_per_s": round(b.n_rows / med, 1), "ms_per_call": round(med * 1e3, 3),
                  "rows_per_device": np.bincount(owner, minlength=a.devices).tolist(),
                  "path": "dcat_multi_rank_forward_batch (C++ host path, host in / host out, NCCL gather)"}),
      flush=True)
