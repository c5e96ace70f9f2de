"""Where the bench step's time goes outside the kernels (tool, not part of the product):
device time of one call with and without an L2 flush before it, and the host time of the
Python wrapper + C call. PinFM-base, device-resident inputs."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_12704_b200 import api  # noqa: E402
from paper_2507_12704_b200.abi import FinetuneSpec  # noqa: E402
from paper_2507_12704_b200.synth import CONFIGS, init_weights, make_batch  # noqa: E402

cfg = CONFIGS["pinfm-base"]
w = init_weights(cfg["spec"], 42)
host = make_batch(cfg["U"], cfg["C"], cfg["L"], seed=1)
dev = host.to(lambda x: torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x).cuda())
m = api.DcatModel(w)
ft = FinetuneSpec(max_events=cfg["L"])
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
for _ in range(3):
    m.rank_forward_batch(dev, ft)
torch.cuda.synchronize()
for mode in ("warm", "flushed", "flushed+idle"):
    dev_ms, host_ms = [], []
    for _ in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if mode != "warm":
            flush.zero_()
        if mode == "flushed+idle":
            torch.cuda.synchronize()  # GPU idle when the call starts: host prep is fully exposed
        a.record(s)
        t0 = time.perf_counter()
        m.rank_forward_batch(dev, ft, profile=True)
        t1 = time.perf_counter()
        b.record(s)
        torch.cuda.synchronize()
        dev_ms.append(a.elapsed_time(b))
        host_ms.append((t1 - t0) * 1e3)
    st = m.stage_times()
    print(f"{mode:14s} event ms {np.median(dev_ms):.3f}  host ms {np.median(host_ms):.3f}  "
          f"device_total {st.get('device_total', 0):.3f} h2d {st.get('h2d', 0):.3f} dedup {st.get('dedup', 0):.3f} "
          f"d2h {st.get('d2h', 0):.3f}")
