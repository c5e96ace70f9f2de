"""Runs the PinFM-base scoring step `--calls` times on cuda:0 (device-resident
inputs) so ncu can capture the kernels of one steady-state call.
Kernel order of one call: 23 dedup/plan kernels, 2 tile builders, gather,
then the context GEMMs (phi_in1, phi_in2, qkv0, attn, o0, ffn1_0, ffn2_0, ...)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_12704_b200 import api  # noqa: E402
from paper_2507_12704_b200.abi import FinetuneSpec  # noqa: E402
from paper_2507_12704_b200.synth import CONFIGS, init_weights, make_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="pinfm-base")
ap.add_argument("--calls", type=int, default=2)
ap.add_argument("--users", type=int, default=0)
ap.add_argument("--stages", action="store_true", help="print per-stage device times of the last call")
a = ap.parse_args()
cfg = CONFIGS[a.config]
U = a.users or cfg["U"]
w = init_weights(cfg["spec"], 42)
host = make_batch(U, cfg["C"], cfg["L"], seed=1)
dev = host.to(lambda x: torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x).cuda())
m = api.DcatModel(w)
ft = FinetuneSpec(max_events=cfg["L"])
for _ in range(a.calls):
    lg, ml, _ = m.rank_forward_batch(dev, ft, profile=a.stages)
torch.cuda.synchronize()
print("ok", float(lg.float().abs().mean()))
if a.stages:  # per-stage device times (ms) of the last call
    for n, v in sorted(m.stage_times().items(), key=lambda kv: -kv[1]):
        print(f"{n:28s} {v:8.4f}")
