"""Host-side cost of the Python wrapper around dcat_rank_forward_batch (tool, not the product):
per-piece perf_counter times on a device-resident PinFM-base batch."""
import ctypes as C
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
for _ in range(3):
    m.rank_forward_batch(dev, ft)
torch.cuda.synchronize()


def t(fn, n=50):
    a = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - a) / n * 1e6


print(f"batch.c()        {t(lambda: dev.c()):8.1f} us")
print(f"ft.c()           {t(lambda: ft.c()):8.1f} us")
print(f"torch.empty x2   {t(lambda: (torch.empty((128000, 3), device='cuda'), torch.empty((128000, 3), device='cuda'))):8.1f} us")
s = torch.cuda.current_stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for k in range(5):
    ev[0].record(s)
    a = time.perf_counter()
    m.rank_forward_batch(dev, ft)
    b = time.perf_counter()
    ev[1].record(s)
    torch.cuda.synchronize()
    print(f"call host {1e3 * (b - a):.3f} ms  events {ev[0].elapsed_time(ev[1]):.3f} ms")
