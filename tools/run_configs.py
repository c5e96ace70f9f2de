"""Runs every BASELINE.json config on one B200: throughput (device-resident, a few
steps) and parity against the CPU oracle on a small user sample of the same dims.
Usage: python tools/run_configs.py [--stages] [config ...]
--stages adds one profiled call per config (stage times in ms, top 12 by time)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle  # noqa: E402
from paper_2507_12704_b200 import api  # noqa: E402
from paper_2507_12704_b200.abi import FinetuneSpec  # noqa: E402
from paper_2507_12704_b200.synth import CONFIGS, make_batch  # noqa: E402

# per-GPU share of the 8-GPU long-seq config
PER_GPU_USERS = {"long-seq": 256}


def main(names, stages=False):
    orc = pyoracle.oracle()
    out = {}
    for name in names:
        cfg = CONFIGS[name]
        spec, C, L = cfg["spec"], cfg["C"], cfg["L"]
        U = PER_GPU_USERS.get(name, cfg["U"])
        w = orc.init_weights(spec, 42, table=(8, 4096, spec.d_emb // 8, 7, 0.05), head_seed=11)
        ft = FinetuneSpec(max_events=L)
        m = api.DcatModel(w)
        # parity on a small sample with the same dims (2 users, <= 6 candidates, ragged)
        sample = make_batch(2, min(C, 6), L, seed=11, ragged=True, layout="grouped")
        t0 = time.time()
        rl, rm, _, rh = orc.rank_forward_batch(w, ft, sample)
        t_cpu = time.time() - t0
        lg, ml, h = m.rank_forward_batch(sample, ft, want_h=True)
        scale = max(1e-3, float(np.abs(rl).max()))
        par = {"max_abs_dH": float(np.abs(h - rh).max()), "max_rel_logits": float(np.abs(lg - rl).max() / scale),
               "oracle_s": round(t_cpu, 1)}
        # throughput on the full per-GPU batch
        host = make_batch(U, C, L, seed=1)
        dev = host.to(lambda a: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).cuda())
        for _ in range(2):
            m.rank_forward_batch(dev, ft)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        K = 5
        ev[0].record()
        for _ in range(K):
            m.rank_forward_batch(dev, ft)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / K
        out[name] = {"users": U, "cands": C, "L": L, "rows": host.n_rows, "ms_per_step": round(ms, 3),
                     "cand_per_s": round(host.n_rows / ms * 1e3, 1), "parity": par}
        if stages:
            m.rank_forward_batch(dev, ft, profile=True)
            torch.cuda.synchronize()
            st = sorted(m.stage_times().items(), key=lambda kv: -kv[1])[:12]
            out[name]["stages_ms"] = {k: round(v, 3) for k, v in st}
        print(name, json.dumps(out[name]), flush=True)
        del m, dev
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if a != "--stages"]
    main(args or ["tiny", "pinfm-base", "low-dedup", "high-fanout", "long-seq"], stages="--stages" in sys.argv)
